"""On-the-fly squared-Euclidean path (BASELINE config 5): the cost is
recomputed per tile from fp32 points and never stored; parity against the
oracle on the identical fp32 cost (oracle.cost_sqeuclid_f32) at the caller's
TRUE epsilon (the device's internal scale is log2(e)/eps rounded to fp32,
within 2^-25 relative: ot.otf_epsilon)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot

REL32 = 1e-6


def _pair(n, m, seed, eps):
    x, y = ot.gen_config(5, n, m, seed)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p = ot.TransportProblem.from_points(a, b, x, y, eps, norm="none", storage="on_the_fly")
    C32 = O.cost_sqeuclid_f32(x.astype(np.float32), y.astype(np.float32))
    return p, O.Problem(a, b, C32, cost_div=eps), C32


def test_otf_epsilon():
    """The on-the-fly sweeps' internal epsilon: log2(e)/eps rounded to fp32
    exactly (the instance itself keeps eps)."""
    for eps in (1e-3, 2e-3, 5e-3, 2e-2, 0.05, 1.0, 3e-7):
        e = ot.otf_epsilon(eps)
        assert abs(e - eps) <= 2.0 ** -24 * eps
        kh = np.float32(ot.LOG2E / eps)
        assert np.float32(ot.LOG2E / e) == kh
        assert np.float32((1.0 / e) * ot.LOG2E) == kh  # the sweeps' kh from kappa = 1/e


def test_otf_rejects_unsupported_on_cpu():
    x = np.random.rand(4, 5)
    with pytest.raises(ot.Unsupported):
        ot.TransportProblem.from_points(np.full(4, .25), np.full(4, .25), x, x, 1e-3,
                                        norm="none", storage="on_the_fly")


@pytest.mark.gpu
def test_otf_cost_matches_oracle_bitwise():
    p, _, C32 = _pair(300, 257, 5, 1e-3)
    assert p.handle.info.storage == 2
    assert p.handle.info.epsilon == 1e-3  # the caller's epsilon, not the internal scale
    assert np.array_equal(p.stored_cost(), C32)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(256, 1024), (300, 1031), (1000, 4096)])
def test_otf_eval_parity(n, m):
    p, q, _ = _pair(n, m, 7, 1e-3)
    rng = O.Rng(3)
    v = O.random_zero_sum(rng, m, 50.0)
    e = ot.eval_normalized_step(p, v)
    r = O.eval_normalized_step(q, v)
    assert np.max(np.abs(e.u - r["u"])) <= 2e-6 * max(1.0, np.max(np.abs(r["u"])))
    assert np.max(np.abs(e.v_next - r["v_next"])) <= 2e-6 * max(1.0, np.max(np.abs(r["v_next"])))
    assert abs(e.grad_l1 - r["grad_l1"]) <= 2e-6 * max(r["grad_l1"], 1e-3)


@pytest.mark.gpu
def test_otf_homotopy_cost_and_iterations():
    n, m, eps, tol = 512, 768, 5e-3, 1e-5
    p, q, _ = _pair(n, m, 11, eps)
    g = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=tol))
    o = O.homotopy_solve(q, tol_l1=tol)
    assert g.converged and o.converged
    assert abs(g.iterations - o.iterations) <= max(1, int(0.01 * o.iterations))
    cg = ot.plan_stats(p, g.potentials.u, g.potentials.v).primal_cost
    co = O.plan_stats(q, o.u, o.v, eps)["primal_cost"]
    assert abs(cg - co) <= REL32 * abs(co)


@pytest.mark.gpu
def test_otf_matches_stored_fp32_path():
    """Same fp32 cost stored vs recomputed: the same solver trajectory up to
    fp32 exponent rounding (the on-the-fly kernels form the exponent with
    three FP32 ops and apply the column's low part as a factor 2^F, the
    stored-cost kernels add it: relative 1e-7 on the potentials)."""
    n, m, eps = 400, 1200, 2e-3
    p, _, C32 = _pair(n, m, 13, eps)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    ps = ot.rescale_problem(ot.make_problem(a, b, C32, ot.otf_epsilon(eps)))
    cfg = ot.HomotopyConfig(tol_l1=1e-6, max_total_inner=300)
    g1 = ot.homotopy_solve(p, cfg)
    g2 = ot.homotopy_solve(ps, cfg)
    assert g1.iterations == g2.iterations
    assert np.max(np.abs(g1.potentials.v - g2.potentials.v)) <= 1e-7 * max(1.0, np.max(np.abs(g2.potentials.v)))
