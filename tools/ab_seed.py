"""Seed (first-evaluation) row pass time at 65536^2 for A/B builds (OTG_LIB)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
x, y = ot.gen_config(3, n, 65536, 3)
p = ot.TransportProblem.from_points(np.full(n, 1.0 / n), np.full(65536, 1.0 / 65536), x, y, 1e-3)
ms, by = ot.time_sweeps(p, np.zeros(65536), reps=4)
print("first-eval row ms", round(ms[0], 3), "col ms", round(ms[1], 3))
