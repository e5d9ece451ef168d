"""Timeline of the single-pass kernel (CTA 0, thread 0): OTG_SP_TRACE=1 python tools/sp_trace.py N"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_30267_b200 import ot, _capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else n
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
lib = ctypes.CDLL(os.path.join(os.path.dirname(_capi.__file__), "libotg.so"))
buf = (ctypes.c_longlong * (256 * 8))()
print("rc", lib.otg_debug_sp_trace(buf, 256 * 8))
a = np.array(buf, dtype=np.int64).reshape(256, 8)
t0 = a[0, 0]
names = ["S:start", "S:full", "S:done", "C:sdone", "C:pub", "C:xwait", "C:col", "L:issue"]
t0 = a[0, 0]
for k in range(0, 40):
    row = a[k, :8] - t0
    print(k, " ".join(f"{nm}={v:9d}" for nm, v in zip(names, row)))
print("stats cycles/row (40..200):", (a[200, 1] - a[40, 1]) / 160,
      " column cycles/row:", (a[200, 6] - a[40, 6]) / 160)
