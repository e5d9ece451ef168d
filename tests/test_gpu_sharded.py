"""Row-sharded device path over NCCL on one GPU: a world_size-1 communicator
drives the sharded code path (post-all-reduce flagging, cross-rank exact
column fallback, sharded plan_stats) and must reproduce the unsharded solve
bit for bit (the all-reduce of one rank is the identity).  Multi-rank
decomposition is covered on CPU by tests/test_sharded_gloo.py."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import dist as D
from paper_2605_30267_b200 import ot

pytestmark = pytest.mark.gpu


def _pair_dense(n, m, seed, eps):
    a, b, Cm = ot.synthetic_instance(n, m, seed)
    mk = lambda: ot.rescale_problem(ot.make_problem(a, b, Cm, eps))
    p1 = mk()
    ps = mk().to_device(world_size=1, rank=0, row_begin=0, row_end=n,
                        nccl_unique_id=ot.nccl_unique_id())
    return p1, ps


def test_nccl_one_rank_is_sharded():
    p1, ps = _pair_dense(40, 30, 1, 0.05)
    assert ps.handle.info.world_size == 1
    assert ps.handle.info.n_local == 40


def test_nccl_one_rank_homotopy_bitwise():
    p1, ps = _pair_dense(300, 200, 2, 0.02)
    cfg = ot.HomotopyConfig(tol_l1=1e-9)
    r1, rs = ot.homotopy_solve(p1, cfg), ot.homotopy_solve(ps, cfg)
    assert r1.iterations == rs.iterations and rs.converged
    assert np.array_equal(r1.potentials.v, rs.potentials.v)
    assert np.array_equal(r1.potentials.u, rs.potentials.u)
    s1 = ot.plan_stats(p1, r1.potentials.u, r1.potentials.v)
    ss = ot.plan_stats(ps, rs.potentials.u, rs.potentials.v)
    assert ss.primal_cost == s1.primal_cost
    assert ss.marginal_violation_l1 == s1.marginal_violation_l1


def test_nccl_one_rank_sinkhorn_matches_oracle():
    n, m, eps = 257, 131, 0.05
    a, b, Cm = ot.synthetic_instance(n, m, 3)
    ps = ot.rescale_problem(ot.make_problem(a, b, Cm, eps)).to_device(
        world_size=1, rank=0, row_begin=0, row_end=n, nccl_unique_id=ot.nccl_unique_id())
    q = O.synthetic_rescaled(n, m, 3, eps)
    g = ot.sinkhorn_solve(ps, None, ot.SolveConfig(tol_l1=1e-9))
    o = O.sinkhorn_solve(q, np.zeros(m), tol_l1=1e-9)
    assert g.iterations == o.iterations
    assert np.max(np.abs(g.potentials.v - o.v)) <= 1e-9 * max(1.0, np.max(np.abs(o.v)))


def test_nccl_one_rank_fp32_fallback_columns():
    """Underflowed fp32 columns take the cross-rank exact LSE path."""
    x = np.array([[0.0], [0.1], [0.2], [0.3]])
    y = np.array([[0.0], [0.15], [1.0], [0.25]])
    a = np.full(4, 0.25)
    p1 = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none")
    ps = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", world_size=1, rank=0,
                                         row_begin=0, row_end=4,
                                         nccl_unique_id=ot.nccl_unique_id())
    e1 = ot.eval_normalized_step(p1, np.zeros(4))
    es = ot.eval_normalized_step(ps, np.zeros(4))
    assert np.all(np.isfinite(es.v_next))
    assert np.array_equal(e1.v_next, es.v_next)


def test_nccl_one_rank_otf_points():
    n, m = 512, 777
    x, y = ot.gen_config(5, n, m, 4)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    p1 = ot.TransportProblem.from_points(a, b, x, y, 5e-3, norm="none", storage="on_the_fly")
    ps = D.sharded_points_problem(a, b, x, y, 5e-3, 1, 0, ot.nccl_unique_id(), device=0,
                                  norm="none", storage="on_the_fly")
    cfg = ot.HomotopyConfig(tol_l1=1e-5, max_total_inner=400)
    r1, rs = ot.homotopy_solve(p1, cfg), ot.homotopy_solve(ps, cfg)
    assert r1.iterations == rs.iterations
    assert np.array_equal(r1.potentials.v, rs.potentials.v)

