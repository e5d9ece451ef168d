"""Secondary measurements for the other BASELINE configs (the driver's headline
line is bench.py, config 3).  One JSON line per measurement, each with the SM
clocks sampled during its timed region (bench.ClockSampler), a roofline
fraction where one applies, and the single-threaded CPU oracle on the same
inputs (the reference is single-threaded):

  cfg1  1000^2 fp64 C ~ U[0,1), eps 1e-2, Sinkhorn and Acc-Sinkhorn (homotopy)
        to 1e-8: device time and us / iteration (latency-bound, C in L2);
        CPU: both full solves
  cfg2  8192^2 fp32 sqeuclid/max, eps 1e-2 and 1e-3, both solvers to 1e-6:
        iterations/s, sweep times, HBM fraction; CPU: a fixed number of
        evaluations -> iterations/s
  cfg4  4096 cosine problems (n, m in 8..64, d 768), eps 5e-3, homotopy to
        1e-6, one CTA per problem: problems/s; CPU: every problem in turn
  cfg5  200000^2 cost on the fly, eps 1e-3: a fixed 2000-iteration run and
        the time to 1e-5; pair evaluations/s against the MUFU ex2 rate and the
        combined MUFU + FMA bound; CPU: one evaluation over a row subset,
        extrapolated

    python tools/bench_configs.py [--configs 1,2,4,5] [--cfg5-iters 2000] [--no-cpu]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from bench import ClockSampler, peaks  # noqa: E402
from paper_2605_30267_b200 import ot  # noqa: E402

SMS, FMAX = 148, 1.965e9
R_MUFU = 16 * SMS * FMAX
R_FMA = 128 * SMS * FMAX
COMBINED = 1.0 / min(max((1 - x / 100) / R_MUFU, (5 + 8 * x / 100) / R_FMA) for x in range(101))


def line(**kw):
    print(json.dumps(kw), flush=True)


def cpu_time(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def cfg1(cpu):
    from oracle import oracle as O
    a, b, C = ot.gen_config(1, 1000, 1000, 1)
    p = ot.rescale_problem(ot.make_problem(a, b, C, 1e-2))
    q = O.Problem(a, b, C, cost_div=1e-2)
    for kind in ("sinkhorn", "acc-homotopy"):
        spec = ot.SolverSpec(kind=kind, max_iters=10000)
        ot.run_solver(p, spec, 1e-8)  # warm
        with ClockSampler(0) as clk:
            r = ot.run_solver(p, spec, 1e-8)
        rec = dict(config=1, solver=kind, iterations=r.iterations, converged=r.converged,
                   seconds=r.device_seconds, iters_per_s=r.iterations / r.device_seconds,
                   us_per_evaluation=1e6 * r.device_seconds / max(r.evaluations, 1),
                   final_violation=r.final_violation, clocks=clk.summary(),
                   roofline="latency-bound (8 MB cost in L2): us / evaluation")
        if cpu:
            s, o = cpu_time(lambda: O.sinkhorn_solve(q, np.zeros(1000), tol_l1=1e-8, max_iters=10000)
                            if kind == "sinkhorn" else O.homotopy_solve(q, tol_l1=1e-8))
            rec["cpu_baseline"] = dict(seconds=s, iterations=o.iterations, cores=1,
                                       iters_per_s=o.iterations / s, kind="port",
                                       sample="full solve")
            rec["speedup_vs_cpu"] = s / r.device_seconds
        line(**rec)


def cfg2(cpu):
    from oracle import oracle as O
    n = m = 8192
    x, y = ot.gen_config(2, n, m, 2)
    a = np.full(n, 1 / n)
    peak, _ = peaks()
    C32 = None
    for eps in (1e-2, 1e-3):
        p = ot.TransportProblem.from_points(a, a, x, y, eps)
        if C32 is None:
            C32 = p.stored_cost()
        for kind in ("sinkhorn", "acc-homotopy"):
            spec = ot.SolverSpec(kind=kind, max_iters=200000)
            ot.run_solver(p, spec, 1e-6)  # warm
            with ClockSampler(0) as clk:
                r = ot.run_solver(p, spec, 1e-6)
            t = ot.run_solver(p, spec, 1e-6, time_sweeps=True)
            row = t.row_pass_seconds / t.evaluations
            col = t.col_pass_seconds / t.evaluations
            bytes_pass = n * m * 4.0
            rec = dict(config=2, eps=eps, solver=kind, iterations=r.iterations,
                       converged=r.converged, seconds=r.device_seconds,
                       iters_per_s=r.iterations / r.device_seconds,
                       sweep_mode=int(p.handle.info.sweep_mode),
                       row_ms=1e3 * row, col_ms=1e3 * col,
                       # two-pass: each pass reads the cost once; single pass
                       # (mode 2): ONE read for the whole evaluation sweep
                       row_frac=(bytes_pass / row / 1e9 / peak
                                 if row > 0 and p.handle.info.sweep_mode != 2 else None),
                       col_frac=(bytes_pass / col / 1e9 / peak
                                 if col > 0 and p.handle.info.sweep_mode != 2 else None),
                       sweep_frac=(bytes_pass / (row + col) / 1e9 / peak
                                   if p.handle.info.sweep_mode == 2 and row + col > 0 else None),
                       clocks=clk.summary())
            if cpu:
                q = O.Problem(a, a, C32, cost_div=eps)
                v = np.zeros(m)
                s, _ = cpu_time(lambda: [O.eval_normalized_step(q, v) for _ in range(3)])
                rec["cpu_baseline"] = dict(iters_per_s=3 / s, cores=1, kind="port",
                                           sample="3 evaluations of the full 8192^2 instance")
                rec["speedup_vs_cpu"] = rec["iters_per_s"] / (3 / s)
            line(**rec)
        p.close()


def cfg4(cpu):
    from oracle import oracle as O
    n, m, x, y = ot.gen_config4(4096, 4, 768)
    bp = ot.BatchProblem.cosine(n, m, x, y, 5e-3, norm="none")
    bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))  # warm
    with ClockSampler(0) as clk:
        r = bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))
    pairs = float((r.iterations + 1) @ (2.0 * n.astype(np.float64) * m))
    rec = dict(config=4, problems=len(n), converged=int(r.converged.sum()),
               total_iterations=int(r.total_iterations), seconds=r.device_seconds,
               problems_per_s=len(n) / r.device_seconds,
               pair_evals_per_s=pairs / r.device_seconds,
               mufu_frac=pairs / r.device_seconds / R_MUFU, clocks=clk.summary(),
               roofline="one CTA per problem, cost in smem: pair evaluations vs the ex2 rate")
    if cpu:
        costs = bp.stored_cost()
        def run_all():
            its = 0
            for k in range(len(n)):
                q = O.Problem(np.full(n[k], 1 / n[k]), np.full(m[k], 1 / m[k]),
                              costs[k].astype(np.float32), cost_div=5e-3)
                its += O.homotopy_solve(q, tol_l1=1e-6).iterations
            return its
        s, its = cpu_time(run_all)
        rec["cpu_baseline"] = dict(seconds=s, problems_per_s=len(n) / s, iterations=its, cores=1,
                                   kind="port", sample="all 4096 problems, one after another")
        rec["speedup_vs_cpu"] = s / r.device_seconds
    line(**rec)


def cfg5(iters, n, cpu):
    from oracle import oracle as O
    x, y = ot.gen_config(5, n, n, 5)
    a = np.full(n, 1 / n)
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
    cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters)
    ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))  # warm
    with ClockSampler(0, period_s=0.02) as clk:
        r = ot.homotopy_solve(p, cfg)
    t = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=min(iters, 50)),
                          time_sweeps=True)
    pairs = 2.0 * n * n * r.evaluations
    rate = pairs / r.device_seconds
    rec = dict(config=5, n=n, iterations=r.iterations, seconds=r.device_seconds,
               iters_per_s=r.iterations / r.device_seconds, pair_evals_per_s=rate,
               mufu_frac=rate / R_MUFU, combined_bound_frac=rate / COMBINED,
               row_ms=1e3 * t.row_pass_seconds / t.evaluations,
               col_ms=1e3 * t.col_pass_seconds / t.evaluations, clocks=clk.summary())
    if cpu:
        rows = 64
        Cr = O.cost_sqeuclid_f32(x[:rows].astype(np.float32), y.astype(np.float32))
        q = O.Problem(np.full(rows, 1 / rows), np.full(n, 1 / n), Cr, cost_div=1e-3)
        v = np.zeros(n)
        s, _ = cpu_time(lambda: O.sweep_rows_mt(q, v, 0, rows, 1))
        per_iter = s * n / rows
        rec["cpu_baseline"] = dict(iters_per_s=1 / per_iter, cores=1, kind="port",
                                   sample=f"one sweep of {rows} rows x {n} columns, extrapolated "
                                          f"to one full evaluation ({per_iter:.0f} s)")
        rec["speedup_vs_cpu"] = rec["iters_per_s"] * per_iter
    line(**rec)
    with ClockSampler(0, period_s=0.02) as clk:
        tt = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-5, max_total_inner=20000))
    st = ot.plan_stats(p, tt.potentials.u, tt.potentials.v)
    line(config=5, n=n, tol=1e-5, iterations=tt.iterations, converged=tt.converged,
         seconds=tt.device_seconds, plan_violation_l1_fp64=st.marginal_violation_l1,
         clocks=clk.summary())


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--cfg5-iters", type=int, default=2000)
    ap.add_argument("--cfg5-n", type=int, default=200000)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    todo = [int(c) for c in args.configs.split(",")]
    cpu = not args.no_cpu
    if 1 in todo:
        cfg1(cpu)
    if 2 in todo:
        cfg2(cpu)
    if 4 in todo:
        cfg4(cpu)
    if 5 in todo:
        cfg5(args.cfg5_iters, args.cfg5_n, cpu)
