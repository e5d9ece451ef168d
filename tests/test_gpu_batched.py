"""Batched path (BASELINE config 4): many small problems, one CTA each,
against the CPU oracle problem by problem."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot


def _random_batch(count, seed, lo=2, hi=64):
    rng = O.Rng(seed)
    a_list, b_list, C_list = [], [], []
    for _ in range(count):
        n = lo + rng.next_below(hi - lo + 1)
        m = lo + rng.next_below(hi - lo + 1)
        a = np.array([1.0 - 0.9 * rng.next_double() for _ in range(n)])
        b = np.array([1.0 - 0.9 * rng.next_double() for _ in range(m)])
        C = np.array([rng.next_double() for _ in range(n * m)], dtype=np.float32).reshape(n, m)
        a_list.append(a / a.sum())
        b_list.append(b / b.sum())
        C_list.append(C)
    return a_list, b_list, C_list


def test_batched_validation_on_cpu():
    a, b = [np.full(65, 1 / 65)], [np.full(3, 1 / 3)]
    with pytest.raises(ot.DimensionMismatch):
        ot.BatchProblem.dense(a, b, [np.zeros((65, 3), np.float32)], 0.1)
    with pytest.raises(ot.InvalidMarginals):
        ot.BatchProblem.dense([np.array([0.5, 0.6])], [np.array([0.5, 0.5])],
                              [np.zeros((2, 2), np.float32)], 0.1)


@pytest.mark.gpu
def test_batched_dense_matches_oracle():
    a_list, b_list, C_list = _random_batch(40, 11)
    eps, tol = 0.05, 1e-9
    bp = ot.BatchProblem.dense(a_list, b_list, C_list, eps)
    r = bp.homotopy_solve(ot.HomotopyConfig(tol_l1=tol))
    for k in range(len(a_list)):
        q = O.Problem(a_list[k], b_list[k], C_list[k], cost_div=eps)
        o = O.homotopy_solve(q, tol_l1=tol)
        assert r.iterations[k] == o.iterations, k
        assert bool(r.converged[k]) == o.converged
        assert np.max(np.abs(r.v[k] - o.v)) <= 1e-9 * max(1.0, np.max(np.abs(o.v)))
        assert np.max(np.abs(r.u[k] - o.u)) <= 1e-9 * max(1.0, np.max(np.abs(o.u)))
        assert abs(r.final_violation[k] - o.final_violation) <= 1e-14 + 1e-9 * o.final_violation


@pytest.mark.gpu
@pytest.mark.parametrize("norm,onorm", [("none", 2), ("minmax", 0), ("halfrange", 1)])
def test_batched_cosine_cost_bitwise(norm, onorm):
    n, m, x, y = ot.gen_config4(12, 4, 64)
    bp = ot.BatchProblem.cosine(n, m, x, y, 5e-3, norm=norm)
    costs = bp.stored_cost()
    ox, oy = 0, 0
    for k in range(len(n)):
        xs = x[ox:ox + n[k]].astype(np.float64)
        ys = y[oy:oy + m[k]].astype(np.float64)
        Co, _, _ = O.cost_cosine(xs, ys, onorm)
        assert np.array_equal(costs[k], Co.astype(np.float32)), k
        ox += n[k]
        oy += m[k]


@pytest.mark.gpu
def test_batched_config4_subset_matches_oracle():
    """BASELINE config 4 shapes (768-dim embeddings, raw 1 - cos, eps 5e-3,
    tol 1e-6) on the first problems of the seeded stream."""
    n, m, x, y = ot.gen_config4(24, 4, 768)
    bp = ot.BatchProblem.cosine(n, m, x, y, 5e-3, norm="none")
    r = bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))
    costs = bp.stored_cost()
    for k in range(len(n)):
        q = O.Problem(np.full(n[k], 1 / n[k]), np.full(m[k], 1 / m[k]), costs[k], cost_div=5e-3)
        o = O.homotopy_solve(q, tol_l1=1e-6)
        assert r.iterations[k] == o.iterations, (k, r.iterations[k], o.iterations)
        assert np.max(np.abs(r.v[k] - o.v)) <= 1e-9 * max(1.0, np.max(np.abs(o.v)))
