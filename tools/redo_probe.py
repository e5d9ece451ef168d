"""How many rows does the fp32 row pass redo exactly, per iteration window?"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
x, y = ot.gen_config(3, n, n, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(n, 1 / n), x, y, 1e-3)
prev = 0
for K in (1, 2, 5, 10, 20, 50, 100, 200, 400, 732):
    r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=K), time_sweeps=True)
    print(f"iters {K:4d} redos {r.row_redos:8d} ({r.row_redos / (n * (K + 1)):.3f} of rows) "
          f"row ms/eval {1e3 * r.row_pass_seconds / r.evaluations:.3f} "
          f"col ms/eval {1e3 * r.col_pass_seconds / r.evaluations:.3f}")
