"""Pin the CPU oracle to the reference's known-answer tests and contracts.

Each check names the reference test it restates (paths under
/root/reference/proj/tests).  These run on CPU only; they are what makes the
oracle trustworthy as the checker for the GPU parity tests.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from otg_testutil import approx


def close(vec, ref, eps):
    return all(approx(a, b, eps) for a, b in zip(np.ravel(vec), np.ravel(ref)))


def test_rng_golden_sequence(kat):  # test_data.cpp:47-70
    r = O.Rng(42)
    assert [r.next_u64() for _ in range(4)] == [int(x) for x in kat["rng42_u64"]["value"]]
    r = O.Rng(42)
    assert [r.next_double() for _ in range(4)] == kat["rng42_double"]["value"]
    r = O.Rng(7)
    for _ in range(200):
        assert r.next_below(10) < 10
        assert r.next_below(1) == 0
    assert O.Rng(1).next_u64() != O.Rng(2).next_u64()


def test_synthetic_instance(kat):  # test_data.cpp:72-105
    k = kat["synthetic_2_3_7"]
    a, b, C = O.synthetic_instance(2, 3, 7)
    assert close(a, k["a"], k["eps"]) and close(b, k["b"], k["eps"])
    assert close(C.ravel(), k["C"], k["eps"])
    assert abs(C.sum() - 1.0) <= 1e-12
    a2, b2, C2 = O.synthetic_instance(2, 3, 7)
    assert np.array_equal(C, C2) and np.array_equal(a, a2)
    assert not np.array_equal(C, O.synthetic_instance(2, 3, 8)[2])
    with pytest.raises(O.OracleError) as e:
        O.synthetic_instance(0, 3, 7)
    assert e.value.kind == "DimensionMismatch"


def test_row_solve_and_column_sums(kat):  # test_dual.cpp:68-90, 223-253
    p = O.skewed_2x2()
    u, col = O.row_solve_marginals(p, np.zeros(2))
    assert close(u, kat["row_solve_skewed_v0"]["value"], 1e-14)
    assert close(col, kat["col_sums_skewed_v0"]["value"], 1e-14)
    uf = O.row_solve(O.flat_2x2(), np.zeros(2))
    assert close(uf, [math.log(0.25)] * 2, 1e-15)
    # u(v + c 1) = u(v) - c 1
    rng = O.Rng(41)
    q = O.synthetic_rescaled(5, 4, 3, 0.7)
    for _ in range(10):
        v = O.random_zero_sum(rng, q.m, 2.0)
        c = 3.0 * rng.next_double() - 1.5
        assert np.max(np.abs(O.row_solve(q, v + c) - (O.row_solve(q, v) - c))) <= 1e-12


def test_grad_and_reduced_f(kat):  # test_dual.cpp:40-62, 95-144
    p = O.skewed_2x2()
    assert close(O.grad_f(p, np.zeros(2)), kat["grad_f_skewed_v0"]["value"], 1e-13)
    assert approx(O.reduced_f(p, np.zeros(2)), kat["reduced_f_skewed_v0"]["value"], 1e-14)
    u0 = O.row_solve(p, np.zeros(2))
    assert approx(O.dual_F(p, u0, np.zeros(2)), kat["dual_F_skewed_u0_v0"]["value"], 1e-14)
    assert np.max(np.abs(O.grad_f(O.flat_2x2(), np.zeros(2)))) <= 1e-15
    rng = O.Rng(59)
    q = O.synthetic_rescaled(7, 5, 2, 0.5)
    for _ in range(10):
        v = O.random_zero_sum(rng, q.m, 2.5)
        assert abs(O.grad_f(q, v).sum()) <= 1e-12
    # central differences (test_dual.cpp:115-127)
    rng = O.Rng(61)
    for t in range(5):
        n, m = 2 + rng.next_below(7), 2 + rng.next_below(7)
        q = O.synthetic_rescaled(n, m, 100 + t, 0.5)
        v = O.random_zero_sum(rng, m, 1.0)
        g = O.grad_f(q, v)
        fd = np.empty(m)
        for j in range(m):
            hi, lo = v.copy(), v.copy()
            hi[j] += 1e-5
            lo[j] -= 1e-5
            fd[j] = (O.reduced_f(q, hi) - O.reduced_f(q, lo)) / 2e-5
        assert np.linalg.norm(g - fd) <= 1e-6 * max(1.0, np.linalg.norm(g))


def test_hessian_cap():  # test_dual.cpp:168-175
    m = 2001
    p = O.Problem(np.ones(1), np.full(m, 1.0 / m), np.zeros((1, m)))
    with pytest.raises(O.OracleError) as e:
        O.hessian_f(p, np.zeros(m))
    assert e.value.kind == "DimensionTooLarge"


def test_sinkhorn_step_closed_forms(kat):  # test_sinkhorn.cpp:15-58
    p = O.skewed_2x2()
    assert close(O.sinkhorn_v_step(p, np.zeros(2)), kat["sinkhorn_v_step_skewed_v0"]["value"], 1e-13)
    z = O.normalized_sinkhorn_map(p, np.zeros(2))
    assert close(z, kat["normalized_map_skewed_v0"]["value"], 1e-13)
    assert abs(z.sum()) <= 1e-12
    with pytest.raises(O.OracleError):
        O.normalized_sinkhorn_map(p, np.array([0.5, 0.4]))
    # mirror-descent identity (test_sinkhorn.cpp:39-51)
    rng = O.Rng(83)
    for q in (p, O.synthetic_rescaled(6, 4, 21, 0.4), O.synthetic_rescaled(3, 8, 22, 1.5)):
        for _ in range(6):
            v = O.random_zero_sum(rng, q.m, 2.0)
            lhs = O.sinkhorn_v_step(q, v)
            rhs = v - O.grad_phi_star(q.b, O.grad_f(q, v))
            assert np.max(np.abs(lhs - rhs)) <= 1e-12


def test_eval_bundle():  # test_sinkhorn.cpp:72-87
    p = O.synthetic_rescaled(5, 5, 33, 0.6)
    rng = O.Rng(89)
    for _ in range(6):
        v = O.random_zero_sum(rng, p.m, 1.5)
        e = O.eval_normalized_step(p, v)
        assert np.max(np.abs(e["v_next"] - O.normalized_sinkhorn_map(p, v))) <= 1e-13
        assert np.max(np.abs(e["u"] - O.row_solve(p, v))) <= 1e-13
        assert np.max(np.abs(e["grad"] - O.grad_f(p, v))) <= 1e-13
        assert approx(e["grad_l1"], np.abs(e["grad"]).sum(), 1e-14)
        assert approx(e["f_value"], O.reduced_f(p, v), 1e-13)
        assert abs(e["v_next"].sum()) <= 1e-12


def test_sinkhorn_bookkeeping():  # test_sinkhorn.cpp:160-203
    r = O.sinkhorn_solve(O.flat_2x2(), np.zeros(2), tol_l1=1e-8)
    assert r.converged and r.iterations == 0 and r.evaluations == 1 and r.final_violation <= 1e-15
    p = O.skewed_2x2()
    r = O.sinkhorn_solve(p, np.zeros(2), tol_l1=1e-8)
    assert r.converged and r.iterations >= 1 and r.evaluations == r.iterations + 1
    assert r.final_violation < 1e-8
    assert approx(r.final_violation, np.abs(O.grad_f(p, r.v)).sum(), 1e-12)
    assert approx(r.final_reduced_f, O.reduced_f(p, r.v), 1e-13)
    assert abs(r.v.sum()) <= 1e-10
    assert np.max(np.abs(r.u - O.row_solve(p, r.v))) <= 1e-12
    r = O.sinkhorn_solve(p, np.zeros(2), tol_l1=1e-14, max_iters=1)
    assert not r.converged and r.iterations == 1 and r.final_violation > 1e-14
    a = O.sinkhorn_solve(p, np.array([1.0, 2.0]), tol_l1=1e-8)
    b = O.sinkhorn_solve(p, O.project_zero_sum([1.0, 2.0]), tol_l1=1e-8)
    assert np.array_equal(a.v, b.v) and a.iterations == b.iterations


def test_sinkhorn_determinism_and_trace():  # test_sinkhorn.cpp:219-249
    p = O.synthetic_rescaled(8, 5, 99, 0.4)
    r1 = O.sinkhorn_solve(p, np.zeros(5), tol_l1=1e-9, record_trace=True)
    r2 = O.sinkhorn_solve(p, np.zeros(5), tol_l1=1e-9, record_trace=True)
    assert np.array_equal(r1.v, r2.v) and np.array_equal(r1.u, r2.u)
    assert np.array_equal(np.nan_to_num(r1.trace), np.nan_to_num(r2.trace))
    q = O.synthetic_rescaled(10, 10, 77, 0.3)
    r = O.sinkhorn_solve(q, np.zeros(10), tol_l1=1e-10, record_trace=True)
    f = r.trace[:, 4]
    assert r.converged and np.all(np.diff(f) <= 1e-12)


def test_extreme_potentials_fallback(kat):  # test_sinkhorn.cpp:251-272
    k = kat["extreme_potentials"]
    p = O.skewed_2x2()
    v = np.array(k["v"])
    u = O.row_solve(p, v)
    g = O.grad_f(p, v)
    assert g[0] == k["grad0"]
    nxt = O.sinkhorn_v_step(p, v)
    assert np.all(np.isfinite(nxt))
    e0 = u[0] + v[0] - p.C[0, 0]
    e1 = u[1] + v[0] - p.C[1, 0]
    top = max(e0, e1)
    cl = top + math.log(math.exp(e0 - top) + math.exp(e1 - top))
    assert approx(nxt[0], v[0] + math.log(p.b[0]) - cl, 1e-15)
    assert nxt[0] > k["next0_gt"]


def test_acc_step_hand_values(kat):  # test_accel.cpp:36-61
    p = O.skewed_2x2()
    x, w, Sx, ev = O.acc_step(p, np.zeros(2), np.zeros(2), 0.5)
    assert ev == kat["acc_step_evals_uncached"]["value"]
    assert close(x, kat["acc_step_skewed_x"]["value"], 1e-13)
    assert close(w, kat["acc_step_skewed_w"]["value"], 1e-13)
    assert np.max(np.abs(Sx - O.normalized_sinkhorn_map(p, x))) <= 1e-12
    _, _, _, ev2 = O.acc_step(p, x, w, 0.5, Sx)
    assert ev2 == kat["acc_step_evals_cached"]["value"]


def test_acc_fixed_point():  # test_accel.cpp:63-75
    p = O.skewed_2x2()
    ref = O.sinkhorn_solve(p, np.zeros(2), tol_l1=1e-12, max_iters=4000000)
    for mu in (0.5, 0.32, 0.05):
        x, w, _, _ = O.acc_step(p, ref.v, math.sqrt(2 * mu) * ref.v, mu)
        assert np.max(np.abs(x - ref.v)) <= 1e-10
        assert np.max(np.abs(w - math.sqrt(2 * mu) * ref.v)) <= 1e-10


def test_acc_run_counting():  # test_accel.cpp:77-118
    p = O.synthetic_rescaled(5, 5, 12, 0.5)
    z = np.zeros(5)
    r = O.acc_run(p, z, z, 0.5, 0)
    assert r.evaluations == 1 and np.array_equal(r.v, z) and np.array_equal(r.w, z)
    assert approx(r.final_violation, np.abs(O.grad_f(p, z)).sum(), 1e-13)
    with pytest.raises(O.OracleError):
        O.acc_run(p, z, z, 0.5, -1)
    for m in (1, 5, 20):
        assert O.acc_run(p, z, z, 0.5, m).evaluations == m + 1
    r1 = O.acc_run(p, z, z, 0.5, 5, record_trace=True, trace_stride=1)
    assert [int(t) for t in r1.trace[:, 0]] == list(range(6))
    assert np.all(r1.trace[:, 5] == 0.5)
    r2 = O.acc_run(p, z, z, 0.5, 5, record_trace=True, trace_stride=2)
    assert [int(t) for t in r2.trace[:, 0]] == [0, 2, 4, 5]


def test_acc_solve():  # test_accel.cpp:136-162
    r = O.acc_solve(O.flat_2x2(), np.zeros(2), 0.5, tol_l1=1e-8)
    assert r.converged and r.iterations == 0 and r.evaluations == 1
    p = O.skewed_2x2()
    r = O.acc_solve(p, np.zeros(2), 0.5, tol_l1=1e-8)
    assert r.converged and r.iterations >= 1 and r.evaluations == r.iterations + 1
    assert r.final_violation < 1e-8
    assert np.max(np.abs(r.u - O.row_solve(p, r.v))) <= 1e-12
    with pytest.raises(O.OracleError):
        O.acc_solve(p, np.zeros(2), 0.5, tol_l1=-1.0)


def test_homotopy_schedule(kat):  # test_accel.cpp:164-191
    k = kat["homotopy_schedule"]
    inst = k["instance"]
    p = O.synthetic_rescaled(inst["n"], inst["m"], inst["seed"], inst["eps"])
    h = O.homotopy_solve(p, mu0=0.5, m0=4, max_outer=3, tol_l1=1e-15)
    assert not h.converged and h.iterations == k["iterations"] and h.outer_stages == k["outer_stages"]
    assert list(h.boundaries[:, 0]) == [0, 1, 2]
    assert list(h.boundaries[:, 1]) == k["mu"]
    assert close(h.boundaries[:, 2], k["alpha"], 1e-15)
    assert list(h.boundaries[:, 3]) == k["inner_before"]


def test_homotopy_state_carry_over(kat):  # test_accel.cpp:193-219
    inst = kat["homotopy_two_stage_iterations"]["instance"]
    p = O.synthetic_rescaled(inst["n"], inst["m"], inst["seed"], inst["eps"])
    two = O.homotopy_solve(p, max_outer=2, tol_l1=1e-15)
    assert two.iterations == kat["homotopy_two_stage_iterations"]["value"]
    z = np.zeros(7)
    st1 = O.acc_run(p, z, z, 0.5, 4)
    st2 = O.acc_run(p, st1.v, st1.w, 0.25, 6)
    assert np.max(np.abs(two.v - st2.v)) <= 1e-15
    resc = O.homotopy_solve(p, max_outer=2, tol_l1=1e-15, rescale_w_across_stages=True)
    st2r = O.acc_run(p, st1.v, st1.w * (math.sqrt(0.5) / 1.0), 0.25, 6)
    assert np.max(np.abs(resc.v - st2r.v)) <= 1e-15
    assert np.max(np.abs(resc.v - two.v)) > 1e-12


def test_homotopy_convergence_and_caps():  # test_accel.cpp:221-270
    r = O.homotopy_solve(O.flat_2x2(), tol_l1=1e-8)
    assert r.converged and r.iterations == 0
    p = O.skewed_2x2()
    r = O.homotopy_solve(p, tol_l1=1e-8)
    assert r.converged and r.final_violation < 1e-8 and r.evaluations == r.iterations + 1
    assert np.max(np.abs(r.u - O.row_solve(p, r.v))) <= 1e-12
    r = O.homotopy_solve(O.synthetic_rescaled(5, 5, 23, 0.5), tol_l1=1e-15, max_total_inner=5)
    assert not r.converged and r.iterations == 5
    for kw in (dict(mu0=0.0), dict(mu0=1.0), dict(m0=0), dict(tol_l1=0.0), dict(trace_stride=0),
               dict(max_total_inner=0)):
        with pytest.raises(O.OracleError):
            O.homotopy_solve(p, **kw)


def test_homotopy_stability_counters():  # test_accel.cpp:272-324
    p = O.synthetic_rescaled(8, 8, 27, 0.2)
    h = O.homotopy_solve(p, tol_l1=1e-9, record_trace=True, stability=True)
    assert h.converged and h.conditions_checked > 0 and h.conditions_held <= h.conditions_checked
    q = O.skewed_2x2()
    ref = O.sinkhorn_solve(q, np.zeros(2), tol_l1=1e-13, max_iters=4000000)
    r = O.acc_run(q, ref.v, ref.v, 0.5, 3, stability=True)
    assert r.conditions_checked == 0 and r.conditions_held == 0


def test_plan_statistics(kat):  # test_core.cpp:131-190
    p = O.skewed_2x2()
    u = O.row_solve(p, np.zeros(2))
    st = O.plan_stats(p, u, np.zeros(2))
    P = np.exp(-p.C + u[:, None])
    assert close(P.ravel(), kat["plan_skewed_u0_v0"]["value"], 1e-14)
    assert close(st["col_sums"], kat["col_sums_skewed_v0"]["value"], 1e-14)
    assert np.max(np.abs(st["row_sums"] - p.a)) <= 1e-14
    assert approx(st["marginal_violation_l1"], kat["marginal_violation_skewed_v0"]["value"], 1e-13)
    assert approx(st["primal_cost"], kat["primal_cost_skewed_v0"]["value"], 1e-13)
    with pytest.raises(O.OracleError) as e:
        O.plan_stats(p, np.full(2, 800.0), np.zeros(2))
    assert e.value.kind == "PotentialOverflow"
    f = O.flat_2x2()
    uf = np.full(2, math.log(0.25))
    assert approx(O.entropic_objective(f, uf, np.zeros(2)),
                  kat["entropic_objective_flat_uniform"]["value"], 1e-14)
    assert approx(O.entropic_objective(p, u, np.zeros(2)),
                  kat["entropic_objective_skewed_rowsolved"]["value"], 1e-13)


def test_mirror_helpers(kat):  # test_mirror.cpp
    hh = np.array([0.5, 0.5])
    assert close(O.grad_phi(hh, [1.0, -1.0]), kat["grad_phi_half_half_1_m1"]["value"], 1e-15)
    assert approx(O.phi_star(hh, [0.5, 0.0]), kat["phi_star_half_half_05_0"]["value"], 1e-15)
    assert approx(O.bregman_phi_star_from_zero(hh, [0.5, 0.0]),
                  kat["bregman_from_zero_half_half_05_0"]["value"], 1e-15)
    assert approx(O.metric_D(np.ones(1), [math.log(2.0)])[0], kat["metric_D_one_ln2"]["value"], 1e-15)
    assert close(O.metric_D(hh, [1.0, -1.0]), kat["metric_D_half_half_1_m1"]["value"], 1e-15)
    tiny = O.metric_D(hh, [1e-10, -1e-10])
    assert abs(tiny[0] - 0.5 * (1 + 0.5e-10)) <= 5e-16 and abs(tiny[1] - 0.5 * (1 - 0.5e-10)) <= 5e-16
    with pytest.raises(O.OracleError) as e:
        O.grad_phi_star(hh, [-0.5, 0.0])
    assert e.value.kind == "DomainViolation"


def test_stability_coefficient(kat):  # test_diag.cpp:157-199
    k = kat["stability_c1_coef"]
    p = O.skewed_2x2()
    xk = np.zeros(2)
    xk1 = O.normalized_sinkhorn_map(p, xk)
    yk, yk1 = np.array([0.05, -0.05]), np.array([-0.02, 0.02])
    g, g1 = O.grad_f(p, xk), O.grad_f(p, xk1)
    breg = O.bregman_phi_star_from_zero(p.b, g)
    for alpha, coef in zip(k["alpha"], k["coef"]):
        r = O.stability_conditions_from_grads(p.b, g, g1, xk, xk1, yk, yk1, alpha)
        assert approx(r["c1_rhs"], coef * breg, k["eps"])
    with pytest.raises(O.OracleError):
        O.stability_conditions_from_grads(p.b, g, g1, xk, xk1, yk, yk1, 2.0)


def test_streaming_mt_sweep_matches_single_thread():
    p = O.synthetic_rescaled(37, 23, 5, 0.3)
    rng = O.Rng(3)
    v = O.random_zero_sum(rng, p.m, 1.0)
    u, col = O.row_solve_marginals(p, v)
    u2, col2 = O.sweep_rows_mt(p, v, 0, p.n, 4)
    assert np.max(np.abs(u - u2)) == 0.0
    assert np.max(np.abs(col - col2)) <= 1e-15


def test_fp32_cost_upcast_matches_fp64():
    """The fp32 path's oracle input: C32 up-cast exactly, divided by eps on load."""
    a, b, C = O.synthetic_instance(6, 9, 4)
    C32 = C.astype(np.float32)
    p32 = O.Problem(a, b, C32, cost_div=0.05)
    p64 = O.Problem(a, b, C32.astype(np.float64) / 0.05)
    v = np.linspace(-1, 1, 9)
    v -= v.mean()
    assert np.array_equal(O.row_solve_marginals(p32, v)[1], O.row_solve_marginals(p64, v)[1])
