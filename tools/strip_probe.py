"""cfg2-shaped whole-row single pass: a short solve for ncu / timing probes.
python tools/strip_probe.py [n] [m] [iters] [eps]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
it = int(sys.argv[3]) if len(sys.argv) > 3 else 12
eps = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-3
x, y = ot.gen_config(2, n, m, 2)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, eps)
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=it))
print("ok", r.iterations, p.handle.info.sweep_mode)
