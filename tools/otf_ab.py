"""cfg5-shaped A/B timing (steady state): python tools/otf_ab.py N ITERS -> row/col ms per evaluation"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
it = int(sys.argv[2]) if len(sys.argv) > 2 else 60
x, y = ot.gen_config(5, n, n, 5)
a = np.full(n, 1 / n)
p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=it)
r = ot.homotopy_solve(p, cfg)
t = ot.homotopy_solve(p, cfg, time_sweeps=True)
print(f"it/s {r.iterations / r.device_seconds:.2f} row ms {1e3 * t.row_pass_seconds / t.evaluations:.3f} "
      f"col ms {1e3 * t.col_pass_seconds / t.evaluations:.3f}")
