"""Per-quarter timeline of the single-pass sweep (debug stamps): for bands
t = q mod 4 of CTA 0: row start (R1), row done (Rc), publish (P), the column
warp seeing the band complete (Cw), its TMEM wait done (C0), slot released (C1)."""
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot, _capi

n, m, q = 16384, 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib = _capi.load()
lib.otg_debug_sp_trace.argtypes = [C.c_int, C.c_void_p]
lib.otg_debug_sp_trace(1, None)
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4))
buf = np.zeros(2 * 12 * 256, dtype=np.uint64)
lib.otg_debug_sp_trace(0, buf.ctypes.data)
b = buf.reshape(2, 12, 256).astype(np.int64)[0]
t0 = b[0][0]
for t in range(q + 40, q + 120, 4):
    f = lambda w: (b[w][t] - t0) / 1e3
    print(f"band {t:3d}: R1 {f(2):7.2f} Rc {f(7):7.2f} P {f(3):7.2f} Cw {f(4):7.2f} C0 {f(5):7.2f} C1 {f(6):7.2f}"
          f" | row {f(7) - f(2):5.2f} pub->seen {f(4) - f(3):5.2f} col {f(6) - f(5):5.2f}")
