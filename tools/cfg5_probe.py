"""cfg5 (200000^2 on the fly, eps 1e-3): iterations/s over a fixed run and
the per-pass split (CUDA events): python tools/cfg5_probe.py [n] [iters]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x, y = ot.gen_config(5, n, n, 5)
a = np.full(n, 1 / n)
p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters)
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
r = ot.homotopy_solve(p, cfg)
t = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=min(iters, 50)),
                      time_sweeps=True)
print(f"n={n} iters={r.iterations} it/s {r.iterations / r.device_seconds:.2f} "
      f"row {1e3 * t.row_pass_seconds / t.evaluations:.2f} ms col {1e3 * t.col_pass_seconds / t.evaluations:.2f} ms "
      f"| v[0:3] {r.potentials.v[:3]} viol {r.final_violation:.3e} blocks visited (row, col) {ot.cull_stats(p)}")
