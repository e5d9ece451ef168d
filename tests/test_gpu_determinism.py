"""Repeatability: every solver path gives bitwise the same potentials when a
solve is repeated on the same handle (integer / fixed-order reductions
throughout; atomics only for counters and lists whose consumers are
order-independent)."""
import numpy as np
import pytest

from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu


def _twice(p, cfg):
    r1 = ot.homotopy_solve(p, cfg)
    r2 = ot.homotopy_solve(p, cfg)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.potentials.v, r2.potentials.v)
    assert np.array_equal(r1.potentials.u, r2.potentials.u)
    return r1


@pytest.mark.parametrize("sweep", ["two_pass", "single_pass"])
@pytest.mark.parametrize("eps", [2e-3, 4e-4])  # 4e-4: columns underflow early (exact fallback)
def test_fp32_stored_repeatable(sweep, eps):
    n, m = 1024, 3000
    x, y = ot.gen_config(3, n, m, 21)
    p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, eps,
                                        sweep=sweep)
    r = _twice(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=60))
    if eps < 1e-3:
        assert r.fallback_columns > 0  # the flagged-column path ran


def test_fp64_dense_repeatable():
    a, b, C = ot.gen_config(1, 300, 280, 1)
    p = ot.rescale_problem(ot.make_problem(a, b, C, 0.01))
    _twice(p, ot.HomotopyConfig(tol_l1=1e-9))


def test_on_the_fly_culled_repeatable():
    n = m = 6000
    x, y = ot.gen_config(5, n, m, 5)
    p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3,
                                        norm="none", storage="on_the_fly")
    assert ot.cull_stats(p)[0] >= 0.0
    _twice(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=40))


def test_batched_repeatable():
    n, m, x, y = ot.gen_config4(64, 4, 64)
    bp = ot.BatchProblem.cosine(n, m, x, y, 5e-3, norm="none")
    cfg = ot.HomotopyConfig(tol_l1=1e-6)
    r1, r2 = bp.homotopy_solve(cfg), bp.homotopy_solve(cfg)
    assert np.array_equal(r1.iterations, r2.iterations)
    for k in range(len(n)):
        assert np.array_equal(r1.v[k], r2.v[k])
    bp.close()
