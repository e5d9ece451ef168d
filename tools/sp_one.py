"""One cfg3-shaped fp32 solve of a few iterations (for ncu captures of k_sweep1)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
it = int(sys.argv[3]) if len(sys.argv) > 3 else 3
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=it))
print("ok", r.iterations, p.handle.info.sweep_mode)
