"""Row sharding on CPU: world_size-2 gloo groups run the
sharded decomposition the device path uses (oracle/sharded.py: local row
sweep, SUM all-reduce of the m column partials + <u, a>, cross-rank exact
column LSE for underflowed columns, replicated epilogue) and must reproduce
the unsharded oracle; plus the host-side helpers of paper_2605_30267_b200.dist."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from oracle import sharded as S
from paper_2605_30267_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ar(op):
    def f(arr):
        t = torch.from_numpy(arr)
        dist.all_reduce(t, op=op)
    return f


def _problem(kind):
    if kind == "synthetic":
        return O.synthetic_rescaled(61, 47, 3, 0.05)
    if kind == "extreme":
        return O.skewed_2x2()
    raise ValueError(kind)


def _worker(rank, world, port, kind, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = _problem(kind)
        r0, r1 = D.shard_rows(p.n, world, rank)
        asum, amax = _ar(dist.ReduceOp.SUM), _ar(dist.ReduceOp.MAX)
        res = {}
        if kind == "synthetic":
            v = O.random_zero_sum(O.Rng(5), p.m, 2.0)
            res["eval"] = S.sharded_eval(p, v, r0, r1, asum, amax)
            res["solve"] = S.sharded_sinkhorn(p, r0, r1, asum, amax, tol_l1=1e-9)
            res["u_all"] = D.gather_u(res["solve"]["u"])
        else:
            v = np.array([-750.0, 750.0])  # test_sinkhorn.cpp:251-272 extreme potentials
            res["eval"] = S.sharded_eval(p, v, r0, r1, asum, amax)
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(kind, world=2):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), kind, out), nprocs=world,
                       start_method="spawn", join=True)
    return dict(out)


def test_shard_rows_partition():
    for n in (1, 2, 7, 1000, 65537):
        for w in (1, 2, 3, 8):
            spans = [D.shard_rows(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_gloo2_sharded_eval_and_sinkhorn_match_oracle():
    res = _run("synthetic")
    p = _problem("synthetic")
    v = O.random_zero_sum(O.Rng(5), p.m, 2.0)
    ref = O.eval_normalized_step(p, v)
    for r in (0, 1):
        e = res[r]["eval"]
        np.testing.assert_allclose(e["v_next"], ref["v_next"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(e["grad"], ref["grad"], rtol=0, atol=1e-14)
        assert abs(e["f_value"] - ref["f_value"]) <= 1e-13
    r0, r1 = D.shard_rows(p.n, 2, 0)
    np.testing.assert_allclose(res[0]["eval"]["u"], ref["u"][r0:r1], rtol=0, atol=1e-13)
    # replicated epilogue: both ranks hold bit-identical m-vectors
    assert np.array_equal(res[0]["eval"]["v_next"], res[1]["eval"]["v_next"])
    o = O.sinkhorn_solve(p, np.zeros(p.m), tol_l1=1e-9)
    for r in (0, 1):
        s = res[r]["solve"]
        assert s["iterations"] == o.iterations and s["converged"] == o.converged
        np.testing.assert_allclose(s["v"], o.v, rtol=0, atol=1e-10)
    np.testing.assert_allclose(res[0]["u_all"], o.u, rtol=0, atol=1e-10)


def test_gloo2_sharded_cross_rank_column_fallback():
    """Column 0 underflows (c_0 < 1e-280); its exact LSE spans rows held by
    both ranks: MAX then SUM all-reduce must equal the oracle."""
    res = _run("extreme")
    p = _problem("extreme")
    ref = O.eval_normalized_step(p, np.array([-750.0, 750.0]))
    for r in (0, 1):
        e = res[r]["eval"]
        assert np.all(np.isfinite(e["v_next"]))
        np.testing.assert_allclose(e["v_next"], ref["v_next"], rtol=1e-15, atol=0)
