"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

fp64 storage: per-iterate dual variables to relative 1e-9 and iteration
counts exact (north_star).  fp32 storage: final transport cost to relative
1e-6 and iteration count within +-1%.  Known-answer tests replay the
reference's own values (tests/golden/kat.json) through the C-ABI.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from otg_testutil import approx
from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu

REL64 = 1e-9   # fp64 path, per-iterate (north_star)
REL32 = 1e-6   # fp32 path, final transport cost (north_star)


def skewed():
    return ot.make_problem([0.7, 0.3], [0.5, 0.5], [[0.0, 1.0], [1.0, 0.0]], 1.0)


def flat():
    return ot.make_problem([0.5, 0.5], [0.5, 0.5], np.zeros((2, 2)), 1.0)


def gpu_rescaled(n, m, seed, eps):
    return ot.synthetic_rescaled(n, m, seed, eps)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


# ------------------------------------------------------------- KATs ----

def test_kat_row_solve_and_columns(kat):
    p = skewed()
    u, col = ot.row_solve_marginals(p, np.zeros(2))
    for x, y in zip(u, kat["row_solve_skewed_v0"]["value"]):
        assert approx(x, y, 1e-14)
    for x, y in zip(col, kat["col_sums_skewed_v0"]["value"]):
        assert approx(x, y, 1e-14)
    for x, y in zip(ot.grad_f(p, np.zeros(2)), kat["grad_f_skewed_v0"]["value"]):
        assert approx(x, y, 1e-13)
    assert approx(ot.reduced_f(p, np.zeros(2)), kat["reduced_f_skewed_v0"]["value"], 1e-14)
    uf = ot.row_solve(flat(), np.zeros(2))
    assert all(approx(x, math.log(0.25), 1e-15) for x in uf)


def test_kat_sinkhorn_step(kat):
    p = skewed()
    s = ot.sinkhorn_v_step(p, np.zeros(2))
    for x, y in zip(s, kat["sinkhorn_v_step_skewed_v0"]["value"]):
        assert approx(x, y, 1e-13)
    z = ot.normalized_sinkhorn_map(p, np.zeros(2))
    for x, y in zip(z, kat["normalized_map_skewed_v0"]["value"]):
        assert approx(x, y, 1e-13)
    assert abs(z.sum()) <= 1e-12
    with pytest.raises(ot.GaugeViolation):
        ot.normalized_sinkhorn_map(p, np.array([0.5, 0.4]))


def test_kat_acc_step(kat):
    p = skewed()
    r = ot.acc_run(p, np.zeros(2), np.zeros(2), 0.5, 1)
    assert r.evaluations == 2
    for x, y in zip(r.state.x, kat["acc_step_skewed_x"]["value"]):
        assert approx(x, y, 1e-13)
    for x, y in zip(r.state.w, kat["acc_step_skewed_w"]["value"]):
        assert approx(x, y, 1e-13)


def test_kat_extreme_potentials_fallback(kat):  # test_sinkhorn.cpp:251-272
    k = kat["extreme_potentials"]
    p = skewed()
    v = np.array(k["v"])
    g = ot.grad_f(p, v)
    assert g[0] == k["grad0"]
    nxt = ot.sinkhorn_v_step(p, v)
    assert np.all(np.isfinite(nxt)) and nxt[0] > k["next0_gt"]
    ref = O.sinkhorn_v_step(O.skewed_2x2(), v)
    assert approx(nxt[0], ref[0], 1e-15)


def test_kat_plan_stats(kat):
    p = skewed()
    u = ot.row_solve(p, np.zeros(2))
    st = ot.plan_stats(p, u, np.zeros(2))
    assert approx(st.marginal_violation_l1, kat["marginal_violation_skewed_v0"]["value"], 1e-13)
    assert approx(st.primal_cost, kat["primal_cost_skewed_v0"]["value"], 1e-13)
    with pytest.raises(ot.PotentialOverflow):
        ot.plan_stats(p, np.full(2, 800.0), np.zeros(2))


def test_kat_homotopy_schedule(kat):
    k = kat["homotopy_schedule"]
    inst = k["instance"]
    p = gpu_rescaled(inst["n"], inst["m"], inst["seed"], inst["eps"])
    h = ot.homotopy_solve_instrumented(p, ot.HomotopyConfig(max_outer=3, tol_l1=1e-15))
    assert not h.result.converged
    assert h.result.iterations == k["iterations"] and h.result.outer_stages == k["outer_stages"]
    assert [b.stage for b in h.boundaries] == [0, 1, 2]
    assert [b.mu for b in h.boundaries] == k["mu"]
    assert all(approx(b.alpha, a, 1e-15) for b, a in zip(h.boundaries, k["alpha"]))
    assert [b.inner_before for b in h.boundaries] == k["inner_before"]


# ------------------------------------------- fp64 per-iterate parity ----

@pytest.mark.parametrize("n,m,seed,eps", [(5, 5, 33, 0.6), (37, 23, 5, 0.3), (64, 130, 9, 0.05),
                                          (300, 257, 2, 0.02), (3, 3000, 4, 0.5)])
def test_eval_step_fp64_parity(n, m, seed, eps):
    p = gpu_rescaled(n, m, seed, eps)
    q = O.synthetic_rescaled(n, m, seed, eps)
    rng = O.Rng(seed + 1)
    for _ in range(3):
        v = O.random_zero_sum(rng, m, 2.0)
        e = ot.eval_normalized_step(p, v)
        r = O.eval_normalized_step(q, v)
        assert rel(e.v_next, r["v_next"]) <= 1e-12
        assert rel(e.u, r["u"]) <= 1e-12
        assert rel(e.grad, r["grad"]) <= 1e-12
        assert approx(e.grad_l1, r["grad_l1"], 1e-12)
        assert approx(e.f_value, r["f_value"], 1e-12)


def test_sinkhorn_fp64_per_iterate_parity():
    q = O.synthetic_rescaled(40, 30, 77, 0.05)
    p = gpu_rescaled(40, 30, 77, 0.05)
    r = ot.sinkhorn_solve(p, np.zeros(30), ot.SolveConfig(tol_l1=1e-10, record_trace=True))
    ro = O.sinkhorn_solve(q, np.zeros(30), tol_l1=1e-10, record_trace=True)
    assert r.converged == ro.converged and r.iterations == ro.iterations
    assert r.evaluations == ro.evaluations == r.iterations + 1
    tr = r.trace.as_array()
    assert tr.shape == ro.trace.shape
    assert np.array_equal(tr[:, 0], ro.trace[:, 0])
    # the violation is a cancellation sum |c - b|: compare it on the scale of
    # sum(b) = 1 (1e-14 absolute) plus relative 1e-9
    assert np.all(np.abs(tr[:, 2] - ro.trace[:, 2]) <= 1e-14 + REL64 * ro.trace[:, 2])
    assert rel(tr[:, 4], ro.trace[:, 4]) <= REL64
    assert rel(r.potentials.v, ro.v) <= REL64 and rel(r.potentials.u, ro.u) <= REL64
    assert approx(r.max_v_inf, ro.max_v_inf, REL64)


@pytest.mark.parametrize("steps", [0, 1, 7, 40])
def test_acc_run_fp64_per_iterate_parity(steps):
    q = O.synthetic_rescaled(33, 21, 15, 0.1)
    p = gpu_rescaled(33, 21, 15, 0.1)
    z = np.zeros(21)
    # per-iterate: compare after every prefix length
    for k in sorted({0, 1, steps // 2, steps}):
        g = ot.acc_run(p, z, z, 0.5, k)
        o = O.acc_run(q, z, z, 0.5, k)
        assert g.evaluations == o.evaluations == k + 1
        assert rel(g.state.x, o.v) <= REL64 and rel(g.state.w, o.w) <= REL64
        assert approx(g.final_violation, o.final_violation, REL64)


def test_acc_solve_fp64_parity():
    q = O.synthetic_rescaled(50, 40, 3, 0.05)
    p = gpu_rescaled(50, 40, 3, 0.05)
    g = ot.acc_solve(p, None, 0.5, ot.SolveConfig(tol_l1=1e-9, record_trace=True, trace_stride=3))
    o = O.acc_solve(q, np.zeros(40), 0.5, tol_l1=1e-9, record_trace=True, trace_stride=3)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert rel(g.potentials.v, o.v) <= REL64 and rel(g.potentials.u, o.u) <= REL64
    assert np.array_equal(g.trace.as_array()[:, 0], o.trace[:, 0])


def cfg1_pair(n, m, seed, eps, dtype=np.float64):
    """BASELINE config 1 inputs: a, b ~ U(0.1,1] normalised, C ~ U[0,1) raw."""
    a, b, Cm = ot.gen_config(1, n, m, seed)
    Cs = Cm.astype(dtype)
    p = ot.rescale_problem(ot.make_problem(a, b, Cs, eps))
    q = O.Problem(a, b, Cs, cost_div=eps)
    return p, q


@pytest.mark.parametrize("n,m,seed,eps,tol", [(6, 6, 18, 0.5, 1e-12), (60, 45, 8, 0.02, 1e-9),
                                              (200, 300, 1, 0.01, 1e-8)])
def test_homotopy_fp64_parity(n, m, seed, eps, tol):
    p, q = cfg1_pair(n, m, seed, eps)
    cfg = ot.HomotopyConfig(tol_l1=tol, record_trace=True)
    g = ot.homotopy_solve_instrumented(p, cfg, ot.AccelInstrumentation(stability=True))
    o = O.homotopy_solve(q, tol_l1=tol, record_trace=True, stability=True)
    assert g.result.iterations == o.iterations and g.result.converged == o.converged
    assert g.result.outer_stages == o.outer_stages
    assert rel(g.result.potentials.v, o.v) <= REL64 and rel(g.result.potentials.u, o.u) <= REL64
    assert g.conditions_checked == o.conditions_checked
    assert g.conditions_held == o.conditions_held
    tr = g.result.trace.as_array()
    assert tr.shape == o.trace.shape
    assert rel(tr[:, 4], o.trace[:, 4]) <= REL64
    c = ~np.isnan(o.trace[:, 7])
    assert np.array_equal(c, ~np.isnan(tr[:, 7]))
    if c.any():
        assert rel(tr[c, 7:12], o.trace[c, 7:12]) <= 1e-7


def test_homotopy_state_carry_over_and_rescale():  # test_accel.cpp:193-219
    p = gpu_rescaled(5, 7, 19, 0.4)
    two = ot.homotopy_solve(p, ot.HomotopyConfig(max_outer=2, tol_l1=1e-15))
    assert two.iterations == 10
    z = np.zeros(7)
    st1 = ot.acc_run(p, z, z, 0.5, 4)
    st2 = ot.acc_run(p, st1.state.x, st1.state.w, 0.25, 6)
    assert np.max(np.abs(two.potentials.v - st2.state.x)) <= 1e-15
    resc = ot.homotopy_solve(p, ot.HomotopyConfig(max_outer=2, tol_l1=1e-15,
                                                  rescale_w_across_stages=True))
    st2r = ot.acc_run(p, st1.state.x, st1.state.w * math.sqrt(0.5), 0.25, 6)
    assert np.max(np.abs(resc.potentials.v - st2r.state.x)) <= 1e-15
    assert np.max(np.abs(resc.potentials.v - two.potentials.v)) > 1e-12


def test_solver_bookkeeping_and_caps():  # test_sinkhorn.cpp:160-203, test_accel.cpp:221-249
    r = ot.sinkhorn_solve(flat(), np.zeros(2), ot.SolveConfig(tol_l1=1e-8))
    assert r.converged and r.iterations == 0 and r.evaluations == 1
    r = ot.sinkhorn_solve(skewed(), np.zeros(2), ot.SolveConfig(tol_l1=1e-14, max_iters=1))
    assert not r.converged and r.iterations == 1 and r.final_violation > 1e-14
    a = ot.sinkhorn_solve(skewed(), np.array([1.0, 2.0]), ot.SolveConfig(tol_l1=1e-8))
    b = ot.sinkhorn_solve(skewed(), np.array([-0.5, 0.5]), ot.SolveConfig(tol_l1=1e-8))
    assert np.array_equal(a.potentials.v, b.potentials.v) and a.iterations == b.iterations
    h = ot.homotopy_solve(gpu_rescaled(5, 5, 23, 0.5),
                          ot.HomotopyConfig(tol_l1=1e-15, max_total_inner=5))
    assert not h.converged and h.iterations == 5
    assert ot.homotopy_solve(flat(), ot.HomotopyConfig(tol_l1=1e-8)).iterations == 0
    with pytest.raises(ot.OtError):
        ot.homotopy_solve(skewed(), ot.HomotopyConfig(mu0=1.0))
    with pytest.raises(ot.OtError):
        ot.acc_run(skewed(), np.zeros(2), np.zeros(2), 0.5, -1)
    with pytest.raises(ot.GaugeViolation):
        ot.acc_run(skewed(), np.array([0.5, 0.4]), np.zeros(2), 0.5, 1)


def test_bitwise_determinism():
    p = gpu_rescaled(200, 150, 99, 0.05)
    cfg = ot.SolveConfig(tol_l1=1e-9, record_trace=True)
    r1 = ot.sinkhorn_solve(p, None, cfg)
    r2 = ot.sinkhorn_solve(p, None, cfg)
    assert np.array_equal(r1.potentials.v, r2.potentials.v)
    assert np.array_equal(r1.potentials.u, r2.potentials.u)
    assert r1.trace.to_csv() == r2.trace.to_csv()
    assert r1.trace.to_csv().startswith(ot.SolverTrace.csv_header())


def test_virtual_shards_match_unsharded():
    a, b, Cm = ot.synthetic_instance(97, 64, 5)
    p1 = ot.rescale_problem(ot.make_problem(a, b, Cm, 0.03))
    p4 = ot.rescale_problem(ot.make_problem(a, b, Cm, 0.03)).to_device(virtual_shards=4)
    cfg = ot.HomotopyConfig(tol_l1=1e-9)
    r1 = ot.homotopy_solve(p1, cfg)
    r4 = ot.homotopy_solve(p4, cfg)
    assert r1.iterations == r4.iterations
    assert rel(r1.potentials.v, r4.potentials.v) <= 1e-12


# --------------------------------------------------------- fp32 path ----

def _fp32_pair(n, m, seed, eps):
    return cfg1_pair(n, m, seed, eps, np.float32)


@pytest.mark.parametrize("n,m,seed,eps", [(64, 64, 1, 0.05), (257, 131, 2, 0.02),
                                          (1024, 2048, 3, 0.01), (100, 4099, 4, 0.05)])
def test_fp32_eval_parity(n, m, seed, eps):
    p, q = _fp32_pair(n, m, seed, eps)
    rng = O.Rng(seed)
    v = O.random_zero_sum(rng, m, 3.0)
    e = ot.eval_normalized_step(p, v)
    r = O.eval_normalized_step(q, v)
    assert rel(e.u, r["u"]) <= 1e-6
    assert np.max(np.abs(e.grad - r["grad"])) <= 1e-6 * np.max(np.abs(r["grad"]) + q.b)
    assert abs(e.grad_l1 - r["grad_l1"]) <= 2e-6 * max(r["grad_l1"], 1e-3)


@pytest.mark.parametrize("n,m,seed,eps,tol", [(128, 96, 7, 0.05, 1e-6), (512, 512, 8, 0.02, 1e-6)])
def test_fp32_homotopy_cost_and_iterations(n, m, seed, eps, tol):
    p, q = _fp32_pair(n, m, seed, eps)
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=tol))
    o = O.homotopy_solve(q, tol_l1=tol)
    assert g.converged and o.converged
    assert abs(g.iterations - o.iterations) <= max(1, int(0.01 * o.iterations))
    cg = ot.plan_stats(p, g.potentials.u, g.potentials.v).primal_cost
    co = O.plan_stats(q, o.u, o.v, eps)["primal_cost"]
    assert abs(cg - co) <= REL32 * abs(co)


def test_fp32_sqeuclid_points_cost_bitwise():
    x, y = ot.gen_config(3, 200, 150, 3)
    n, m = 200, 150
    p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
    Cg = p.stored_cost()
    Co, lo, hi = O.cost_sqeuclidean(x, y)
    assert np.array_equal(Cg, Co.astype(np.float32))
    assert p.handle.info.cost_raw_max == hi


def test_fp32_fallback_columns_exact():
    # far-away target points: their columns underflow in fp32 at v = 0
    x = np.array([[0.0], [0.1], [0.2], [0.3]])
    y = np.array([[0.0], [0.15], [1.0], [0.25]])
    a = np.full(4, 0.25)
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none")
    C32 = p.stored_cost()
    q = O.Problem(a, a, C32, cost_div=1e-3)
    e = ot.eval_normalized_step(p, np.zeros(4))
    r = O.eval_normalized_step(q, np.zeros(4))
    assert np.all(np.isfinite(e.v_next))
    assert rel(e.v_next, r["v_next"]) <= 1e-6


def test_config1_full_size_fp64_both_solvers():
    """BASELINE config 1 at its full size: n = m = 1000, fp64, eps = 1e-2,
    tol 1e-8: Sinkhorn and acc-homotopy, iteration counts exact."""
    p, q = cfg1_pair(1000, 1000, 1, 1e-2)
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-8, max_total_inner=10000))
    o = O.homotopy_solve(q, tol_l1=1e-8, max_total_inner=10000)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert rel(g.potentials.v, o.v) <= REL64
    gs = ot.sinkhorn_solve(p, None, ot.SolveConfig(tol_l1=1e-8, max_iters=10000))
    os_ = O.sinkhorn_solve(q, np.zeros(1000), tol_l1=1e-8, max_iters=10000)
    assert gs.iterations == os_.iterations and gs.converged == os_.converged
    assert rel(gs.potentials.v, os_.v) <= REL64


# ------------------------------------------- fused single-pass sweep ----

def _points_problem(n, m, seed, eps, fused):
    x, y = ot.gen_config(3, n, m, seed)
    return ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, eps,
                                           sweep="single_pass" if fused else "two_pass")


@pytest.mark.parametrize("n,m", [(512, 8192), (300, 4100), (1000, 1024), (257, 65536)])
def test_fused_eval_matches_oracle_and_two_pass(n, m):
    pf = _points_problem(n, m, 5, 1e-3, True)
    p2 = _points_problem(n, m, 5, 1e-3, False)
    assert np.array_equal(pf.stored_cost(), p2.stored_cost())
    q = O.Problem(np.full(n, 1 / n), np.full(m, 1 / m), pf.stored_cost(), cost_div=1e-3)
    rng = O.Rng(7)
    v = O.random_zero_sum(rng, m, 30.0)
    ef = ot.eval_normalized_step(pf, v)
    e2 = ot.eval_normalized_step(p2, v)
    r = O.eval_normalized_step(q, v)
    for e in (ef, e2):
        assert rel(e.u, r["u"]) <= 2e-6
        assert rel(e.v_next, r["v_next"]) <= 2e-6
        assert abs(e.grad_l1 - r["grad_l1"]) <= 2e-6 * max(r["grad_l1"], 1e-3)
        assert abs(e.f_value - r["f_value"]) <= 1e-6 * max(1.0, abs(r["f_value"]))


@pytest.mark.parametrize("n,m,eps", [
    (300, 4100, 2e-3), (257, 65536, 1e-3), (2048, 2048, 5e-4),
    (150, 8192, 1e-3), (1000, 1001, 2e-3), (4099, 5003, 1e-3), (37, 777, 5e-3)])
def test_fused_single_pass_matches_two_pass_solve(n, m, eps):
    """Steady-state single-pass kernel (grid-wide band pipeline, tensor-memory
    staging, shift estimates, loose-row redo + column patch) against the
    two-pass kernels, including ragged slices (m not a multiple of the slice
    width) and partial last bands."""
    pf = _points_problem(n, m, 11, eps, True)
    p2 = _points_problem(n, m, 11, eps, False)
    assert pf.handle.info.sweep_mode == 2 and p2.handle.info.sweep_mode == 1
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=40)
    gf = ot.homotopy_solve(pf, cfg)
    g2 = ot.homotopy_solve(p2, cfg)
    assert gf.iterations == g2.iterations
    assert rel(gf.potentials.v, g2.potentials.v) <= 2e-6
    assert rel(gf.potentials.u, g2.potentials.u) <= 2e-6
    assert abs(gf.final_violation - g2.final_violation) <= 1e-5 * max(g2.final_violation, 1e-3)


def test_fused_homotopy_cost_and_iterations():
    n, m, eps, tol = 512, 2048, 5e-3, 1e-6
    pf = _points_problem(n, m, 9, eps, True)
    q = O.Problem(np.full(n, 1 / n), np.full(m, 1 / m), pf.stored_cost(), cost_div=eps)
    g = ot.homotopy_solve(pf, ot.HomotopyConfig(tol_l1=tol))
    o = O.homotopy_solve(q, tol_l1=tol)
    assert g.converged and o.converged
    assert abs(g.iterations - o.iterations) <= max(1, int(0.01 * o.iterations))
    cg = ot.plan_stats(pf, g.potentials.u, g.potentials.v).primal_cost
    co = O.plan_stats(q, o.u, o.v, eps)["primal_cost"]
    assert abs(cg - co) <= REL32 * abs(co)


@pytest.mark.parametrize("solver", ["sinkhorn", "acc", "acc_warm"])
def test_single_pass_zero_point_seed(solver):
    """Solves on a single-pass handle that start at the zero point skip the
    exact two-pass seed evaluation (the row statistics of p = 0 come from the
    cost's row minima); a warm start (acc_warm: nonzero v0) takes the exact
    seed.  Both agree with the two-pass handle to the fp32 bar."""
    n, m, eps = 300, 4100, 2e-3
    pf = _points_problem(n, m, 13, eps, True)
    p2 = _points_problem(n, m, 13, eps, False)
    assert pf.handle.info.sweep_mode == 2 and p2.handle.info.sweep_mode == 1
    cfg = ot.SolveConfig(tol_l1=1e-300, max_iters=40)
    v0 = None
    if solver == "acc_warm":
        v0 = O.random_zero_sum(O.Rng(3), m, 5.0)
    if solver == "sinkhorn":
        gf, g2 = ot.sinkhorn_solve(pf, v0, cfg), ot.sinkhorn_solve(p2, v0, cfg)
    else:
        gf, g2 = ot.acc_solve(pf, v0, 0.5, cfg), ot.acc_solve(p2, v0, 0.5, cfg)
    assert gf.iterations == g2.iterations == 40
    assert rel(gf.potentials.v, g2.potentials.v) <= 2e-6
    assert rel(gf.potentials.u, g2.potentials.u) <= 2e-6


def test_single_pass_instrumented_trace_matches_two_pass():
    """The steady single-pass graph runs the solver's control step inside the
    patch/merge kernel: an instrumented homotopy solve (trace rows, stability
    conditions, energy / radii against a reference solution) on a single-pass
    handle matches the two-pass handle's trace to the fp32 bar, with the same
    iteration count and condition counters."""
    n, m, eps = 300, 4100, 2e-3
    pf = _points_problem(n, m, 17, eps, True)
    p2 = _points_problem(n, m, 17, eps, False)
    assert pf.handle.info.sweep_mode == 2 and p2.handle.info.sweep_mode == 1
    ref = ot.homotopy_solve(p2, ot.HomotopyConfig(tol_l1=1e-5, max_total_inner=3000))
    instr = ot.AccelInstrumentation(
        reference=ot.ReferenceSolution(ref.potentials.v, ref.final_reduced_f), stability=True)
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=40, record_trace=True)
    hf = ot.homotopy_solve_instrumented(pf, cfg, instr)
    h2 = ot.homotopy_solve_instrumented(p2, cfg, instr)
    assert hf.result.iterations == h2.result.iterations == 40
    assert hf.conditions_checked == h2.conditions_checked
    tf, t2 = hf.result.trace.as_array(), h2.result.trace.as_array()
    assert tf.shape == t2.shape and tf.shape[0] > 0
    fin = np.isfinite(t2)
    assert np.array_equal(np.isfinite(tf), fin)
    d = np.abs(tf[fin] - t2[fin]) / np.maximum(1.0, np.abs(t2[fin]))
    assert d.max() <= 1e-5, float(d.max())
