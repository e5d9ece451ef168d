"""Generate the config-scale parity fixtures (tests/golden/config_fixtures.json).

Runs the CPU oracle (oracle/otoracle.cpp: the reference's fp64 algorithm,
sinkhorn.cpp:65-115 / accel.cpp:234-305, stop rule accel.cpp:272, primal
cost core.cpp:77-79) on the BASELINE configs at their full sizes, with the
oracle's own input generators (no libotg), and records what the GPU parity
tests assert against (tests/test_gpu_configs.py):

  iterations, evaluations, converged, final_violation, the fp64 plan statistics
  of the returned potentials (marginal violation, primal cost in the original
  units), quantiles and a strided sample of v, and a digest of v (oracle
  reproducibility only).

Instances (the same arrays the GPU solves: the GPU stores the identical fp32
cost, tests/test_oracle_gen.py):
  cfg2   8192^2, seed 2, fp32 C = fl32(sqeuclid / max), eps 1e-2 and 1e-3,
         Sinkhorn and Acc-Sinkhorn (homotopy mu0 0.5, m0 4), tol 1e-6
  cfg3   65536^2, seed 3, same cost (17.2 GB fp32), eps 1e-3, homotopy, tol 1e-6
  cfg5s  20000^2 cfg5-shaped (seed 5), raw fp32 on-the-fly cost
         fl32((x - y)^2) at the TRUE eps 1e-3, homotopy, tol 1e-5

Run in the CPU container (the oracle is threaded: deterministic for a given
thread count, equal to the single-threaded order to rounding):

    python tests/golden/make_config_fixtures.py --only cfg2 --threads 8
    python tests/golden/make_config_fixtures.py --only cfg3 --threads 8   # ~1 h
"""
import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "config_fixtures.json")
SAMPLE_STRIDE = 257


def summarise(p, res, eps, threads, seconds, extra):
    with O.threads(threads):
        st = O.plan_stats(p, res.u, res.v, eps)
    v = res.v
    q = np.quantile(v, [0.0, 0.01, 0.1, 0.25, 0.5, 0.75, 0.9, 0.99, 1.0]).tolist()
    d = dict(iterations=int(res.iterations), evaluations=int(res.evaluations),
             converged=bool(res.converged), final_violation=float(res.final_violation),
             final_reduced_f=float(res.final_reduced_f),
             plan_violation_l1=float(st["marginal_violation_l1"]),
             primal_cost=float(st["primal_cost"]),
             v_quantiles=q, v_sample_stride=SAMPLE_STRIDE,
             v_sample=v[::SAMPLE_STRIDE].tolist(),
             u_sample=res.u[::SAMPLE_STRIDE].tolist(),
             v_digest=hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16],
             oracle_threads=threads, oracle_seconds=round(seconds, 1),
             host=platform.processor() or platform.machine())
    d.update(extra)
    return d


def solve(p, solver, tol, threads):
    t0 = time.time()
    with O.threads(threads):
        if solver == "sinkhorn":
            r = O.sinkhorn_solve(p, tol_l1=tol, max_iters=200000)
        else:
            r = O.homotopy_solve(p, tol_l1=tol)
    return r, time.time() - t0


def cfg2(threads):
    n = m = 8192
    x, y = O.gen_config(2, n, m, 2)
    Cm, mx = O.cost_sqeuclid_max_f32(x, y, threads=threads)
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    out = {}
    for eps in (1e-2, 1e-3):
        p = O.Problem(a, b, Cm, cost_div=eps)
        for solver in ("sinkhorn", "homotopy"):
            r, s = solve(p, solver, 1e-6, threads)
            key = f"cfg2_eps{eps:g}_{solver}"
            out[key] = summarise(p, r, eps, threads, s, dict(
                config=2, n=n, m=m, seed=2, eps=eps, solver=solver, tol_l1=1e-6,
                cost="fl32(sqeuclid / max), stored fp32", raw_max=mx))
            print(key, out[key]["iterations"], out[key]["primal_cost"], f"{s:.0f}s", flush=True)
    return out


def cfg3(threads):
    n = m = 65536
    x, y = O.gen_config(3, n, m, 3)
    t0 = time.time()
    Cm, mx = O.cost_sqeuclid_max_f32(x, y, threads=threads)
    print(f"cfg3 cost built in {time.time() - t0:.0f}s", flush=True)
    a = np.full(n, 1.0 / n)
    p = O.Problem(a, a.copy(), Cm, cost_div=1e-3)
    r, s = solve(p, "homotopy", 1e-6, threads)
    d = summarise(p, r, 1e-3, threads, s, dict(
        config=3, n=n, m=m, seed=3, eps=1e-3, solver="homotopy", tol_l1=1e-6,
        cost="fl32(sqeuclid / max), stored fp32", raw_max=mx))
    print("cfg3", d["iterations"], d["primal_cost"], f"{s:.0f}s", flush=True)
    return {"cfg3_eps0.001_homotopy": d}


def cfg5s(threads):
    n = m = 20000
    x, y = O.gen_config(5, n, m, 5)
    Cm = O.cost_sqeuclid_f32(x, y)
    a = np.full(n, 1.0 / n)
    p = O.Problem(a, a.copy(), Cm, cost_div=1e-3)
    r, s = solve(p, "homotopy", 1e-5, threads)
    d = summarise(p, r, 1e-3, threads, s, dict(
        config=5, n=n, m=m, seed=5, eps=1e-3, solver="homotopy", tol_l1=1e-5,
        cost="fl32((x-y)^2) of fp32 points, raw (on the fly)"))
    print("cfg5s", d["iterations"], d["primal_cost"], f"{s:.0f}s", flush=True)
    return {"cfg5s_eps0.001_homotopy": d}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["cfg2", "cfg3", "cfg5s"], action="append")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    todo = args.only or ["cfg2", "cfg5s", "cfg3"]
    for name in todo:
        got = {"cfg2": cfg2, "cfg3": cfg3, "cfg5s": cfg5s}[name](args.threads)
        cur = json.load(open(OUT)) if os.path.exists(OUT) else {}
        cur.update(got)
        with open(OUT, "w") as f:
            json.dump(cur, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main()
