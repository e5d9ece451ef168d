"""Seed-evaluation cost (exact first row pass + flagged-column fallback) at
65536^2 for A/B builds (OTG_LIB): device time of a 1-iteration solve."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = 65536
x, y = ot.gen_config(3, n, n, 3)
p = ot.TransportProblem.from_points(np.full(n, 1.0 / n), np.full(n, 1.0 / n), x, y, 1e-3)
cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=1)
ot.homotopy_solve(p, cfg)
ts = [ot.homotopy_solve(p, cfg) for _ in range(3)]
print("seed+1 ms", [round(1e3 * r.device_seconds, 3) for r in ts], "fallback cols", ts[-1].fallback_columns)
r20 = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=20))
r40 = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=40))
print("20-step", round(1e3 * r20.device_seconds, 2), "40-step", round(1e3 * r40.device_seconds, 2),
      "v0", r20.potentials.v[:3], r40.final_violation)
