"""Secondary measurements for the other BASELINE configs (not the driver's
headline line): config 1 (fp64 1000^2, both solvers), config 2 (8192^2 fp32,
eps 1e-2 / 1e-3, both solvers), config 4 (4096 small cosine problems), config
5 (200000^2 on the fly, fixed 2000 iterations + time to 1e-5; --cfg5-iters).
One JSON line per measurement."""
import argparse
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot


def line(**kw):
    print(json.dumps(kw), flush=True)


def cfg1():
    a, b, C = ot.gen_config(1, 1000, 1000, 1)
    p = ot.rescale_problem(ot.make_problem(a, b, C, 1e-2))
    for kind in ("sinkhorn", "acc-homotopy"):
        ot.run_solver(p, ot.SolverSpec(kind=kind, max_iters=10000), 1e-8)  # warm
        r = ot.run_solver(p, ot.SolverSpec(kind=kind, max_iters=10000), 1e-8)
        line(config=1, solver=kind, iterations=r.iterations, converged=r.converged,
             seconds=r.device_seconds, us_per_iter=1e6 * r.device_seconds / max(r.evaluations, 1),
             final_violation=r.final_violation)


def cfg2():
    x, y = ot.gen_config(2, 8192, 8192, 2)
    a = np.full(8192, 1 / 8192)
    for eps in (1e-2, 1e-3):
        p = ot.TransportProblem.from_points(a, a, x, y, eps)
        for kind in ("sinkhorn", "acc-homotopy"):
            spec = ot.SolverSpec(kind=kind, max_iters=200000)
            ot.run_solver(p, spec, 1e-6)  # warm
            r = ot.run_solver(p, spec, 1e-6)  # timed without per-launch events
            t = ot.run_solver(p, spec, 1e-6, time_sweeps=True)  # the kernel split
            line(config=2, eps=eps, solver=kind, iterations=r.iterations, converged=r.converged,
                 seconds=r.device_seconds, iters_per_s=r.iterations / r.device_seconds,
                 row_ms=1e3 * t.row_pass_seconds / t.evaluations,
                 col_ms=1e3 * t.col_pass_seconds / t.evaluations,
                 row_frac=(8192 * 8192 * 4) / (t.row_pass_seconds / t.evaluations) / 1e9 / 6542.4,
                 col_frac=(8192 * 8192 * 4) / (t.col_pass_seconds / t.evaluations) / 1e9 / 6542.4)
        p.close()


def cfg4():
    n, m, x, y = ot.gen_config4(4096, 4, 768)
    bp = ot.BatchProblem.cosine(n, m, x, y, 5e-3, norm="none")
    bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))  # warm
    r = bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))
    pairs = float((r.iterations + 1) @ (2.0 * n.astype(np.float64) * m))
    line(config=4, problems=len(n), converged=int(r.converged.sum()),
         total_iterations=int(r.total_iterations), seconds=r.device_seconds,
         problems_per_s=len(n) / r.device_seconds,
         pair_evals_per_s=pairs / r.device_seconds)


def cfg5(iters, n):
    x, y = ot.gen_config(5, n, n, 5)
    a = np.full(n, 1 / n)
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters)
    r = ot.homotopy_solve(p, cfg)  # timed without per-launch events
    t = ot.homotopy_solve(p, cfg, time_sweeps=True)  # the kernel split
    pairs = 2.0 * n * n * r.evaluations
    mufu = 16 * 148 * 1.965e9  # ex2 / s at the max SM clock (one ex2 per pair)
    line(config=5, n=n, iterations=r.iterations, seconds=r.device_seconds,
         iters_per_s=r.iterations / r.device_seconds, pair_evals_per_s=pairs / r.device_seconds,
         mufu_frac=pairs / r.device_seconds / mufu,
         row_ms=1e3 * t.row_pass_seconds / t.evaluations,
         col_ms=1e3 * t.col_pass_seconds / t.evaluations)
    t = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-5, max_total_inner=20000))
    line(config=5, n=n, tol=1e-5, iterations=t.iterations, converged=t.converged,
         seconds=t.device_seconds)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--cfg5-iters", type=int, default=200)
    ap.add_argument("--cfg5-n", type=int, default=200000)
    args = ap.parse_args()
    todo = [int(c) for c in args.configs.split(",")]
    if 1 in todo: cfg1()
    if 2 in todo: cfg2()
    if 4 in todo: cfg4()
    if 5 in todo: cfg5(args.cfg5_iters, args.cfg5_n)
