"""Energy / radius instrumentation on the device (fused into the vector-update
epilogue, csrc/sweep.cu apply_cols / apply_tail) against the oracle
(accel.cpp:38-114, diag.cpp:76-88, 206-215): per-row trace columns, stage
boundary energies, r_hat / c_star, the rejected reference, and the
reference's own properties (test_accel.cpp:272-348)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu


def close(a, b, tol):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    assert a.shape == b.shape
    both_nan = np.isnan(a) & np.isnan(b)
    assert np.array_equal(np.isnan(a), np.isnan(b))
    d = np.abs(np.where(both_nan, 0, a) - np.where(both_nan, 0, b))
    assert np.all(d <= tol * np.maximum(1.0, np.abs(np.where(both_nan, 0, b)))), float(d.max())


@pytest.mark.parametrize("n,m,seed,eps,rescale", [(8, 8, 27, 0.2, False), (200, 150, 3, 0.05, True)])
def test_instrumented_homotopy_matches_oracle(n, m, seed, eps, rescale):
    q = O.synthetic_rescaled(n, m, seed, eps)
    vs, fs = O.reference_solve(q, 1e-12)
    p = ot.synthetic_rescaled(n, m, seed, eps)
    instr = ot.AccelInstrumentation(reference=ot.ReferenceSolution(vs, fs), stability=True)
    cfg = ot.HomotopyConfig(tol_l1=1e-9, record_trace=True, rescale_w_across_stages=rescale)
    h = ot.homotopy_solve_instrumented(p, cfg, instr)
    o = O.homotopy_solve(q, tol_l1=1e-9, record_trace=True, stability=True,
                         rescale_w_across_stages=rescale, reference=(vs, fs))
    assert h.result.converged and o.converged
    assert h.result.iterations == o.iterations
    close(h.result.trace.as_array(), o.trace, 1e-9)
    close([b.energy for b in h.boundaries], o.boundaries[:, 4], 1e-9)
    assert h.r_hat == pytest.approx(o.r_hat, rel=1e-9)
    assert h.c_star == pytest.approx(O.homotopy_rate_constant(0.5, o.r_hat), rel=1e-9)
    # the reference's properties (test_accel.cpp:286-312)
    e = np.array([r.energy for r in h.result.trace.records])
    assert np.all(np.isfinite(e)) and np.all(e >= -1e-9)
    rx = np.array([r.radius_x_d for r in h.result.trace.records])
    ry = np.array([r.radius_y for r in h.result.trace.records])
    assert np.all(rx <= h.r_hat + 1e-15) and np.all(ry <= h.r_hat + 1e-15)
    assert max(rx.max(), ry.max()) == pytest.approx(h.r_hat, rel=1e-12)
    assert all(b.energy is not None and b.energy >= -1e-9 for b in h.boundaries)


def test_single_stage_energy_decay_and_parity():  # test_accel.cpp:326-348
    q = O.synthetic_rescaled(5, 5, 66, 0.005)
    vs, fs = O.reference_solve(q, 1e-13)
    p = ot.synthetic_rescaled(5, 5, 66, 0.005)
    mu, alpha = 0.2, math.sqrt(0.4)
    run = ot.acc_run(p, np.zeros(5), np.zeros(5), mu, 60, record_trace=True,
                     instr=ot.AccelInstrumentation(reference=ot.ReferenceSolution(vs, fs)))
    o = O.acc_run(q, np.zeros(5), np.zeros(5), mu, 60, record_trace=True, reference=(vs, fs))
    close(run.trace.as_array(), o.trace, 1e-9)
    assert run.max_radius_x_d == pytest.approx(o.r_max_x, rel=1e-9)
    e = np.array([r.energy for r in run.trace.records])
    floor = e.min()
    d0 = e[0] - floor
    ks, ls = [], []
    for k, ek in enumerate(e):
        if ek - floor <= 1e-3 * d0:
            break
        ks.append(k)
        ls.append(math.log(ek - floor))
    assert len(ks) >= 8
    assert math.exp(np.polyfit(ks, ls, 1)[0]) <= 1.0 / (1.0 + alpha) + 0.05


def test_acc_solve_reference_columns():  # accel.cpp:211-213
    q = O.synthetic_rescaled(40, 30, 5, 0.1)
    vs, fs = O.reference_solve(q, 1e-12)
    p = ot.synthetic_rescaled(40, 30, 5, 0.1)
    cfg = ot.SolveConfig(tol_l1=1e-8, record_trace=True, reference=ot.ReferenceSolution(vs, fs))
    g = ot.acc_solve(p, None, 0.3, cfg)
    o = O.acc_solve(q, np.zeros(30), mu=0.3, tol_l1=1e-8, record_trace=True, reference=(vs, fs))
    assert g.iterations == o.iterations
    close(g.trace.as_array(), o.trace, 1e-9)


def test_bogus_reference_is_rejected():  # test_diag.cpp:114-117
    q = O.skewed_2x2()
    vs, fs = O.reference_solve(q, 1e-13)
    p = ot.rescale_problem(ot.make_problem([0.7, 0.3], [0.5, 0.5], [[0.0, 1.0], [1.0, 0.0]], 1.0))
    f0 = O.eval_normalized_step(q, np.zeros(2))["f_value"]
    bogus = ot.AccelInstrumentation(reference=ot.ReferenceSolution(vs, f0 + 1.0))
    with pytest.raises(ot.OtError):
        ot.homotopy_solve_instrumented(p, ot.HomotopyConfig(tol_l1=1e-9), bogus)


def test_fp32_points_energy_columns():
    n, m, eps = 256, 200, 2e-2
    x, y = ot.gen_config(3, n, m, 4)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p = ot.TransportProblem.from_points(a, b, x, y, eps)
    q = O.Problem(a, b, p.stored_cost(), cost_div=eps)
    vs, fs = O.reference_solve(q, 1e-11)
    # a short run: f(x) stays far above f*, where fp32 evaluation error (~1e-7
    # relative) cannot trip the f* <= f(x) + 1e-9 check of diag.cpp:78-81
    instr = ot.AccelInstrumentation(reference=ot.ReferenceSolution(vs, fs))
    cfg = ot.HomotopyConfig(tol_l1=1e-6, record_trace=True, max_total_inner=12)
    h = ot.homotopy_solve_instrumented(p, cfg, instr)
    o = O.homotopy_solve(q, tol_l1=1e-6, record_trace=True, reference=(vs, fs), max_total_inner=12)
    assert h.result.iterations == o.iterations
    k = min(len(h.result.trace.records), len(o.trace))
    ge = np.array([r.energy for r in h.result.trace.records[:k]])
    assert np.all(np.abs(ge - o.trace[:k, 12]) <= 1e-5 * np.maximum(1.0, np.abs(o.trace[:k, 12])))


def test_reference_solve_after_a_plain_solve_on_the_same_handle():
    """The chunk graph is cached per handle: a reference-instrumented solve
    after a plain one must find v* where the graph looks for it (round 2
    fix: v* allocated with the handle, not at the first reference solve)."""
    q = O.synthetic_rescaled(40, 30, 9, 0.05)
    vs, fs = O.reference_solve(q, 1e-12)
    p = ot.synthetic_rescaled(40, 30, 9, 0.05)
    cfg = ot.HomotopyConfig(tol_l1=1e-9, record_trace=True)
    plain = ot.homotopy_solve_instrumented(p, cfg, None)
    instr = ot.AccelInstrumentation(reference=ot.ReferenceSolution(vs, fs), stability=True)
    h = ot.homotopy_solve_instrumented(p, cfg, instr)
    o = O.homotopy_solve(q, tol_l1=1e-9, record_trace=True, stability=True, reference=(vs, fs))
    assert plain.result.iterations == h.result.iterations == o.iterations
    close(h.result.trace.as_array(), o.trace, 1e-9)
