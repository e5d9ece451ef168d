"""Device diagnostics of dual.hpp: dual_F (dual.cpp:88-101) and hessian_f
(dual.cpp:118-136) through the C-ABI, against the oracle and the reference
test_dual.cpp properties (KAT value, symmetry, H 1 = 0, central differences
of grad_f, the m = 2000 cap)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu


def test_dual_F_kat(kat):
    p = ot.make_problem([0.7, 0.3], [0.5, 0.5], [[0.0, 1.0], [1.0, 0.0]], 1.0)
    u0 = ot.row_solve(p, np.zeros(2))
    got = ot.dual_F(p, u0, np.zeros(2))
    want = kat["dual_F_skewed_u0_v0"]["value"]
    assert abs(got - want) <= 1e-14 * max(1.0, abs(want))


@pytest.mark.parametrize("n,m,seed", [(7, 5, 2), (64, 48, 3), (300, 257, 4), (1000, 700, 5)])
def test_dual_F_matches_oracle(n, m, seed):
    q = O.synthetic_rescaled(n, m, seed, 0.1)
    p = ot.make_problem(q.a, q.b, q.C, 1.0)
    rng = O.Rng(seed + 10)
    for _ in range(3):
        u = O.random_zero_sum(rng, n, 2.0)
        v = O.random_zero_sum(rng, m, 2.0)
        got, want = ot.dual_F(p, u, v), O.dual_F(q, u, v)
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    # at the row solve the dual equals the reduced objective (dual.cpp:103-108)
    v = O.random_zero_sum(rng, m, 1.0)
    u = ot.row_solve(p, v)
    assert abs(ot.dual_F(p, u, v) - ot.reduced_f(p, v)) <= 1e-12


def test_dual_F_overflow():
    p = ot.make_problem([0.5, 0.5], [0.5, 0.5], np.zeros((2, 2)), 1.0)
    with pytest.raises(ot.PotentialOverflow):
        ot.dual_F(p, np.full(2, 400.0), np.full(2, 400.0))
    with pytest.raises(ot.DimensionMismatch):
        ot.dual_F(p, np.zeros(3), np.zeros(2))


@pytest.mark.parametrize("n,m,seed", [(7, 5, 2), (40, 33, 3), (500, 129, 4), (2000, 1000, 6)])
def test_hessian_matches_oracle(n, m, seed):
    q = O.synthetic_rescaled(n, m, seed, 0.1)
    p = ot.make_problem(q.a, q.b, q.C, 1.0)
    v = O.random_zero_sum(O.Rng(seed), m, 1.5)
    H = ot.hessian_f(p, v)
    R = O.hessian_f(q, v)
    scale = np.max(np.abs(R))
    assert np.max(np.abs(H - R)) <= 1e-12 * scale
    assert np.array_equal(H, H.T) or np.max(np.abs(H - H.T)) <= 1e-15 * scale


def test_hessian_properties():  # test_dual.cpp:146-166
    rng = O.Rng(71)
    for t in range(4):
        n, m = 2 + rng.next_below(9), 2 + rng.next_below(9)
        q = O.synthetic_rescaled(n, m, 200 + t, 0.5)
        p = ot.make_problem(q.a, q.b, q.C, 1.0)
        v = O.random_zero_sum(rng, m, 1.0)
        H = ot.hessian_f(p, v)
        assert np.max(np.abs(H - H.T)) <= 1e-14
        assert np.max(np.abs(H @ np.ones(m))) <= 1e-13  # constant shifts are flat
        assert np.min(np.linalg.eigvalsh(H)) >= -1e-13  # f is convex
        fd = np.empty((m, m))
        for j in range(m):
            hi, lo = v.copy(), v.copy()
            hi[j] += 1e-5
            lo[j] -= 1e-5
            fd[:, j] = (ot.grad_f(p, hi) - ot.grad_f(p, lo)) / 2e-5
        assert np.linalg.norm(H - fd) <= 1e-6 * max(1.0, np.linalg.norm(H))


def test_hessian_on_the_fly_and_f32():
    n, m = 400, 300
    x, y = ot.gen_config(3, n, m, 9)
    pts = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 0.05)
    q = O.Problem(np.full(n, 1 / n), np.full(m, 1 / m), pts.stored_cost(), cost_div=0.05)
    v = O.random_zero_sum(O.Rng(3), m, 1.0)
    H, R = ot.hessian_f(pts, v), O.hessian_f(q, v)
    # the row statistics come from the fp32 sweep: the fp32 bar (1e-6 relative)
    assert np.max(np.abs(H - R) / (np.abs(R) + 1e-300)) <= 1e-6
    assert np.max(np.abs(H @ np.ones(m))) <= 1e-6 * np.max(np.abs(R))


def test_hessian_cap():  # test_dual.cpp:168-175
    m = 2001
    p = ot.make_problem(np.ones(1), np.full(m, 1.0 / m), np.zeros((1, m)), 1.0)
    with pytest.raises(ot.DimensionTooLarge):
        ot.hessian_f(p, np.zeros(m))
    p = ot.make_problem(np.ones(1), np.full(2000, 1.0 / 2000), np.zeros((1, 2000)), 1.0)
    H = ot.hessian_f(p, np.zeros(2000))
    assert H.shape == (2000, 2000)
