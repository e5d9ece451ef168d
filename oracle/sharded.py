"""TEST INFRASTRUCTURE — row-sharded restatement of the oracle's evaluation.

Only tests/ may import this.  It states, on the CPU, the decomposition the
device path uses when the rows are split across ranks (SURVEY §8e,
sweep.cu launch_eval): every rank sweeps its own contiguous row block
(dual.cpp:29-42 restricted to rows [r0, r1)), the column partial sums plus
the local <u, a> are SUM-all-reduced, the columns whose mass fell below
1e-280 take the exact log-sum-exp of dual.cpp:44-70 as a cross-rank MAX
then SUM all-reduce, and the m-vector epilogue of sinkhorn.cpp:51-63 runs
replicated.  `allreduce_sum` / `allreduce_max` are callables over float64
numpy arrays (in place), so the same function runs under gloo in the tests.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

TINY = 1e-280  # dual.cpp:53


def shard_rows(n: int, world: int, rank: int):
    return n * rank // world, n * (rank + 1) // world


def sharded_eval(p: O.Problem, v, r0: int, r1: int, allreduce_sum, allreduce_max):
    v = np.ascontiguousarray(v, dtype=np.float64)
    m = p.m
    u, col = O.sweep_rows_mt(p, v, r0, r1, 1)
    a = p.a[r0:r1]
    buf = np.empty(m + 1)
    buf[:m] = col
    buf[m] = float(np.dot(u, a)) if r1 > r0 else 0.0
    allreduce_sum(buf)
    col, ua = buf[:m].copy(), buf[m]
    col_log = np.empty(m)
    ok = col >= TINY
    col_log[ok] = np.log(col[ok])
    flagged = np.flatnonzero(~ok)
    if flagged.size:  # flagged set is identical on every rank (post-reduce)
        Cl = p.C[r0:r1][:, flagged]
        z = u[:, None] + v[flagged][None, :] - Cl
        top = z.max(axis=0) if r1 > r0 else np.full(flagged.size, -np.inf)
        allreduce_max(top)
        s = np.exp(z - top[None, :]).sum(axis=0) if r1 > r0 else np.zeros(flagged.size)
        allreduce_sum(s)
        col_log[flagged] = top + np.log(s)
        col[flagged] = np.exp(col_log[flagged])
    if not np.all(np.isfinite(col_log)):
        raise O.OracleError(3, "column log-mass degenerated")
    grad = col - p.b
    y = v + (np.log(p.b) - col_log)
    return dict(u=u, grad=grad, grad_l1=float(np.abs(grad).sum()),
                f_value=1.0 - ua - float(np.dot(v, p.b)), v_next=y - y.mean())


def sharded_sinkhorn(p: O.Problem, r0, r1, allreduce_sum, allreduce_max, tol_l1=1e-6,
                     max_iters=200000):
    """sinkhorn.cpp:65-115 with the sharded evaluation; every rank takes the
    same stop decision because grad_l1 is computed from reduced columns."""
    v = np.zeros(p.m)
    for k in range(max_iters + 1):
        e = sharded_eval(p, v, r0, r1, allreduce_sum, allreduce_max)
        if e["grad_l1"] < tol_l1 or k >= max_iters:
            return dict(iterations=k, converged=e["grad_l1"] < tol_l1, u=e["u"], v=v,
                        final_violation=e["grad_l1"])
        v = e["v_next"]
