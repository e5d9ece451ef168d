import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = 65536
x, y = ot.gen_config(3, n, n, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(n, 1 / n), x, y, 1e-3)
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
print("fallback columns", r.fallback_columns if hasattr(r, 'fallback_columns') else None)
print([k for k in dir(r) if 'fall' in k or 'redo' in k])
