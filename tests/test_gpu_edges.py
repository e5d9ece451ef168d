"""Edge cases of the device path (the reference's tests cover 1 x k, k x 1,
ragged sizes, degenerate costs, tiny epsilon) and full-size properties of
BASELINE config 3 (65536^2 fp32) that do not need the CPU oracle: the solve
converges, the plan it implies has the reported marginal error, repeated
solves are bitwise identical, and the barycentric projection stays in the
hull of the source points."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


@pytest.mark.parametrize("n,m", [(1, 1), (1, 7), (7, 1), (2, 3), (3, 2), (1, 4096), (4096, 1)])
def test_degenerate_shapes_fp64(n, m):
    a, b, Cm = ot.synthetic_instance(n, m, 4)
    p = ot.rescale_problem(ot.make_problem(a, b, Cm, 0.1))
    q = O.Problem(a, b, Cm / 0.1)
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-10, max_total_inner=2000))
    o = O.homotopy_solve(q, tol_l1=1e-10, max_total_inner=2000)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert rel(g.potentials.v, o.v) <= 1e-9


@pytest.mark.parametrize("n,m", [(1, 5), (5, 1), (3, 3), (129, 5), (5, 129), (1000, 1003)])
@pytest.mark.parametrize("storage", ["f32", "on_the_fly"])
def test_ragged_shapes_fp32(n, m, storage):
    x, y = ot.gen_config(5, n, m, 6)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p = ot.TransportProblem.from_points(a, b, x, y, 2e-2, norm="none", storage=storage)
    C32 = O.cost_sqeuclid_f32(x.astype(np.float32), y.astype(np.float32))
    q = O.Problem(a, b, C32, cost_div=2e-2)  # the TRUE epsilon for both storages
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-6, max_total_inner=3000))
    o = O.homotopy_solve(q, tol_l1=1e-6, max_total_inner=3000)
    assert g.converged == o.converged
    assert abs(g.iterations - o.iterations) <= max(1, int(0.01 * o.iterations))
    cg = ot.plan_stats(p, g.potentials.u, g.potentials.v).primal_cost
    co = O.plan_stats(q, o.u, o.v, 2e-2)["primal_cost"]
    assert abs(cg - co) <= 1e-6 * abs(co) + 1e-12


def test_constant_cost_is_one_sinkhorn_step():
    """C = const: the plan a b^T is reached in one evaluation (any eps)."""
    n, m = 300, 200
    a = np.linspace(1, 2, n); a /= a.sum()
    b = np.linspace(2, 1, m); b /= b.sum()
    p = ot.rescale_problem(ot.make_problem(a, b, np.full((n, m), 0.7), 1e-3))
    r = ot.sinkhorn_solve(p, None, ot.SolveConfig(tol_l1=1e-12))
    assert r.converged and r.iterations <= 1


def test_tiny_epsilon_fp32_fallback_heavy():
    """eps small enough that many columns underflow in fp32 and take the exact
    fallback: still converges to the oracle's cost."""
    n, m, eps, tol = 128, 192, 5e-4, 1e-5
    x, y = ot.gen_config(3, n, m, 8)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p = ot.TransportProblem.from_points(a, b, x, y, eps)
    q = O.Problem(a, b, p.stored_cost(), cost_div=eps)
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=tol, max_total_inner=20000))
    o = O.homotopy_solve(q, tol_l1=tol, max_total_inner=20000)
    assert g.converged and o.converged
    assert g.fallback_columns > 0  # the exact column LSE was exercised
    assert abs(g.iterations - o.iterations) <= max(1, int(0.01 * o.iterations))
    cg = ot.plan_stats(p, g.potentials.u, g.potentials.v).primal_cost
    co = O.plan_stats(q, o.u, o.v, eps)["primal_cost"]
    assert abs(cg - co) <= 1e-6 * abs(co)


def test_config3_full_size_properties():
    N = 65536
    x, y = ot.gen_config(3, N, N, 3)
    a = np.full(N, 1.0 / N)
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3)
    cfg = ot.HomotopyConfig(tol_l1=1e-6, max_total_inner=5000)
    r1 = ot.homotopy_solve(p, cfg)
    assert r1.converged and r1.final_violation < 1e-6
    st = ot.plan_stats(p, r1.potentials.u, r1.potentials.v)
    # the plan of the returned potentials, evaluated in fp64 on the same fp32
    # cost, meets the tolerance up to the fp32 evaluation error of the solver
    # (~1e-6 relative per column, summed over 65536 columns)
    assert st.marginal_violation_l1 <= 2e-6
    assert abs(st.marginal_violation_l1 - r1.final_violation) <= 0.2 * r1.final_violation
    r2 = ot.homotopy_solve(p, cfg)
    assert r2.iterations == r1.iterations
    assert np.array_equal(r1.potentials.v, r2.potentials.v)
    bary = ot.barycentric_projection(p, r1.potentials.u, r1.potentials.v, x)
    for ch in range(3):
        assert bary[:, ch].min() >= x[:, ch].min() - 1e-9
        assert bary[:, ch].max() <= x[:, ch].max() + 1e-9


def test_config5_full_size_properties():
    """BASELINE config 5 at its full size (200000^2, cost never stored): a
    short homotopy run is deterministic, drives the violation down, and the
    plan of its potentials (one more streaming pass) has the marginal error
    the solver reported."""
    N = 200_000
    x, y = ot.gen_config(5, N, N, 5)
    a = np.full(N, 1.0 / N)
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=12)
    r1 = ot.homotopy_solve(p, cfg)
    r2 = ot.homotopy_solve(p, cfg)
    assert r1.iterations == r2.iterations == 12
    assert np.array_equal(r1.potentials.v, r2.potentials.v)
    assert np.array_equal(r1.potentials.u, r2.potentials.u)
    assert np.isfinite(r1.potentials.v).all() and abs(r1.potentials.v.mean()) < 1e-9
    st = ot.plan_stats(p, r1.potentials.u, r1.potentials.v)
    assert abs(st.marginal_violation_l1 - r1.final_violation) <= 0.05 * r1.final_violation
    r0 = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=1))
    assert r1.final_violation < r0.final_violation


def test_config2_full_size_properties():
    """BASELINE config 2 (8192^2, stored fp32, both eps): converges to 1e-6,
    bitwise reproducible, and the plan's marginal error matches."""
    x, y = ot.gen_config(2, 8192, 8192, 2)
    a = np.full(8192, 1.0 / 8192)
    for eps in (1e-2, 1e-3):
        p = ot.TransportProblem.from_points(a, a, x, y, eps)
        for kind in ("sinkhorn", "acc-homotopy"):
            r = ot.run_solver(p, ot.SolverSpec(kind=kind, max_iters=200000), 1e-6)
            r2 = ot.run_solver(p, ot.SolverSpec(kind=kind, max_iters=200000), 1e-6)
            assert r.converged and r.iterations == r2.iterations
            assert np.array_equal(r.potentials.v, r2.potentials.v)
            st = ot.plan_stats(p, r.potentials.u, r.potentials.v)
            assert st.marginal_violation_l1 <= 1.2e-6
        p.close()


def test_many_flagged_columns_sorted_fallback():
    """> 512 columns whose linear-domain mass underflows (the sorted, thread-per-
    column fallback of k_fallback): one evaluation at v = 0 against the oracle."""
    rng = np.random.default_rng(5)
    n, m = 384, 3000
    x = rng.uniform(0.0, 0.1, size=(n, 3))
    y = np.concatenate([rng.uniform(0.0, 0.1, size=(m // 3, 3)),
                        rng.uniform(0.9, 1.0, size=(m - m // 3, 3))])
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p = ot.TransportProblem.from_points(a, b, x, y, 5e-4)
    q = O.Problem(a, b, p.stored_cost(), cost_div=5e-4)
    e = ot.eval_normalized_step(p, np.zeros(m))
    r = O.eval_normalized_step(q, np.zeros(m))
    assert rel(e.v_next, r["v_next"]) <= 2e-6
    assert rel(e.u, r["u"]) <= 2e-6
    assert abs(e.grad_l1 - r["grad_l1"]) <= 2e-6 * max(r["grad_l1"], 1e-3)
    # the exact column LSE ran for (at least) the far columns
    s = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=1))
    assert s.fallback_columns >= m - m // 3


@pytest.mark.parametrize("sweep", ["single_pass"])
def test_flagged_columns_in_the_steady_single_pass_graph(sweep):
    """Underflowed columns on a single-pass handle: the solve starts at the
    zero point, so its first evaluations already run the steady chunk graph
    (no exact-path kernels, finalize folded into the patch/merge kernel);
    evaluations with flagged columns must fall through to k_finalize's exact
    column LSE.  Against the two-pass handle and the oracle."""
    rng = np.random.default_rng(5)
    n, m = 384, 3000
    x = rng.uniform(0.0, 0.1, size=(n, 3))
    y = np.concatenate([rng.uniform(0.0, 0.1, size=(m // 3, 3)),
                        rng.uniform(0.9, 1.0, size=(m - m // 3, 3))])
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    ps = ot.TransportProblem.from_points(a, b, x, y, 5e-4, sweep=sweep)
    p2 = ot.TransportProblem.from_points(a, b, x, y, 5e-4, sweep="two_pass")
    assert ps.handle.info.sweep_mode == 2 and p2.handle.info.sweep_mode == 1
    s1 = ot.homotopy_solve(ps, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=1))
    assert s1.fallback_columns >= m - m // 3
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=30)
    gs, g2 = ot.homotopy_solve(ps, cfg), ot.homotopy_solve(p2, cfg)
    assert gs.fallback_columns == g2.fallback_columns > 0
    # deterministic although the flagged-column list is filled by atomics (the
    # finalize sums the flagged columns in column order)
    for p_, g_ in ((ps, gs), (p2, g2)):
        again = ot.homotopy_solve(p_, cfg)
        assert np.array_equal(again.potentials.v, g_.potentials.v)
        assert np.array_equal(again.potentials.u, g_.potentials.u)
    assert gs.iterations == g2.iterations == 30
    assert rel(gs.potentials.v, g2.potentials.v) <= 2e-6
    q = O.Problem(a, b, ps.stored_cost(), cost_div=5e-4)
    o = O.homotopy_solve(q, tol_l1=1e-300, max_total_inner=30)
    assert rel(gs.potentials.v, o.v) <= 2e-6
