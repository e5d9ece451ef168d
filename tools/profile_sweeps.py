"""Profiling driver: one cfg3-shaped problem (rows x 65536, fp32), a few evaluations,
then one isolated row pass + column pass (for ncu -k regex:k_row|k_col)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = 65536
x, y = ot.gen_config(3, rows, m, 3)
p = ot.TransportProblem.from_points(np.full(rows, 1.0 / rows), np.full(m, 1.0 / m), x, y, 1e-3)
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
ms, by = ot.time_sweeps(p, r.potentials.v, reps=6)
info = p.handle.info
print("rows", rows, "mode", info.sweep_mode, "clusters", info.sweep_clusters, "splits",
      info.col_splits, "ms", [round(x, 4) for x in ms], "GB/s pass1",
      round(by[0] / ms[0] / 1e6, 1), "pass2", round(by[1] / max(ms[1], 1e-9) / 1e6, 1))
