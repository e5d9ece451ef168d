"""cfg5-shaped on-the-fly problem for ncu: python tools/profile_otf.py N"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
x, y = ot.gen_config(5, n, n, 5)
a = np.full(n, 1 / n)
p = ot.TransportProblem.from_points(a, a, x, y, 1e-3, norm="none", storage="on_the_fly")
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4), time_sweeps=True)
print("row ms", 1e3 * r.row_pass_seconds / r.evaluations, "col ms", 1e3 * r.col_pass_seconds / r.evaluations)
