"""Device handle creation time for cfg3 (points -> 17.2 GB fp32 cost on the
device, normaliser, zero-point row statistics): python tools/build_time.py"""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
x, y = ot.gen_config(3, n, n, 3)
a = np.full(n, 1 / n)
for k in range(3):
    t = time.perf_counter()
    p = ot.TransportProblem.from_points(a, a, x, y, 1e-3)
    print(f"from_points {n}^2: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
    p.close()
