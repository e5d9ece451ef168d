"""Exactness of the culled on-the-fly sweeps (sweep.cu: k_row_otf_cull,
k_col_otf_cull).  A skipped block is one whose every
exponent is provably below -127, where ex2.approx.ftz returns +0, so the
culled solve must equal, BITWISE, the same Morton-ordered sweeps visiting
every block (otg_debug_cull(0)); against the dense sweeps in the caller's
order (otg_debug_cull(-1): a different summation order) the potentials agree
to fp32-accumulation rounding (2e-6 of max |v|), the iteration counts
exactly."""
import numpy as np
import pytest

from paper_2605_30267_b200 import _capi, ot

pytestmark = pytest.mark.gpu


def _solve(n, iters, mode, seed=5):
    lib = _capi.load()
    prev = lib.otg_debug_cull(mode)
    try:
        x, y = ot.gen_config(5, n, n, seed)
        a = np.full(n, 1 / n)
        p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
        fixed = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters))
        tol = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-3, max_total_inner=3000))
        p.close()
    finally:
        lib.otg_debug_cull(prev)
    return fixed, tol


@pytest.mark.parametrize("n", [8192, 20000])
def test_cull_is_bitwise_invisible(n):
    culled, ct = _solve(n, 40, 1)
    visited, vt = _solve(n, 40, 0)
    assert np.array_equal(culled.potentials.v, visited.potentials.v)
    assert np.array_equal(culled.potentials.u, visited.potentials.u)
    assert ct.iterations == vt.iterations
    assert np.array_equal(ct.potentials.v, vt.potentials.v)


def test_cull_matches_dense_order():
    n = 20000
    culled, ct = _solve(n, 40, 1)
    dense, dt = _solve(n, 40, -1)
    scale = max(1.0, float(np.max(np.abs(dense.potentials.v))))
    # (fp32 block partials summed in another column order, over 40 iterations)
    assert float(np.max(np.abs(culled.potentials.v - dense.potentials.v))) / scale < 2e-6
    assert ct.iterations == dt.iterations and ct.converged and dt.converged
    assert abs(ct.final_violation - dt.final_violation) <= 1e-6 * dt.final_violation + 1e-12


@pytest.mark.gpu
def test_cull_stats_on_a_fresh_handle():
    """The culling bound reads each row's last argmax column: on a handle that
    was never evaluated otg_cull_stats once indexed with uninitialised memory
    (an illegal address that killed the context).  Device state now starts
    zeroed: the call is harmless and the context stays usable."""
    n = m = 4096
    x, y = ot.gen_config(5, n, m, 5)
    p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3,
                                        norm="none", storage="on_the_fly")
    r0, c0 = ot.cull_stats(p)
    assert 0.0 <= r0 <= 1.0 and 0.0 <= c0 <= 1.0
    ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
    rows, cols = ot.cull_stats(p)
    assert 0.0 < rows <= 1.0 and 0.0 < cols <= 1.0
    p.close()
