"""Band cadence of the single-pass sweep from the debug timeline (last launch
of a 4-iteration solve): mean loader issue interval, row-warp band time
(full -> slot release), column-warp band time, over bands 32..223 of CTA 0."""
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot, _capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
lib = _capi.load()
lib.otg_debug_sp_trace.argtypes = [C.c_int, C.c_void_p]
lib.otg_debug_sp_trace(1, None)
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4))
buf = np.zeros(2 * 12 * 256, dtype=np.uint64)
lib.otg_debug_sp_trace(0, buf.ctypes.data)
b = buf.reshape(2, 12, 256).astype(np.int64)[0] / 1e3
sl = slice(32, 224)
L = np.diff(b[0][sl]).mean()
row = (b[7][sl] - b[2][sl]).mean()
col = (b[6][sl] - b[5][sl]).mean()
wait_data = (b[2][sl] - b[1][sl]).mean()
print(f"{n}x{m}: loader interval {L:.3f} us/band, row band {row:.3f} us, col band {col:.3f} us, "
      f"row wait for data {wait_data:.3f} us")
