"""cfg2 (8192^2 fp32) iterations/s and the in-solve kernel split under the
current OTG_* knobs: python tools/cfg2_probe.py [eps]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
sweep = sys.argv[2] if len(sys.argv) > 2 else "auto"
x, y = ot.gen_config(2, 8192, 8192, 2)
a = np.full(8192, 1 / 8192)
p = ot.TransportProblem.from_points(a, a, x, y, eps, sweep=sweep)
spec = ot.SolverSpec(kind="acc-homotopy", max_iters=200000)
ot.run_solver(p, spec, 1e-6)
runs = [ot.run_solver(p, spec, 1e-6) for _ in range(5)]
r = min(runs, key=lambda q: q.device_seconds)
t = ot.run_solver(p, spec, 1e-6, time_sweeps=True)
ev = t.evaluations
print(f"[{sweep} mode {p.handle.info.sweep_mode}] it/s {r.iterations / r.device_seconds:8.1f}  us/eval {1e6 * r.device_seconds / r.evaluations:7.1f}"
      f"  row {1e6 * t.row_pass_seconds / ev:6.1f}  col {1e6 * t.col_pass_seconds / ev:6.1f}"
      f"  iters {r.iterations}  launches/eval {r.kernel_launches / max(r.evaluations, 1):.1f}")
