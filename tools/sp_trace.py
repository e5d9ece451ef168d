"""Timeline of the single-pass sweep (fused.cu k_sweep1, debug stamps via
otg_debug_sp_trace): per band of CTA 0 and of the last CTA, globaltimer ns of
loader issue (L), row warp 1 before/after the full wait (R0/R1), row publish
(P), watcher window ready (W, per 4 bands), column start/end (C0/C1).

    python tools/sp_trace.py [n] [m]
"""
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
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4))
buf = np.zeros(2 * 12 * 256, dtype=np.uint64)
lib.otg_debug_sp_trace(0, buf.ctypes.data)
b = buf.reshape(2, 12, 256).astype(np.int64)
t0 = b[0][0][0]
names = ["L", "R0", "R1", "P", "Cw", "C0", "C1", "Rc", "-", "-", "Rt"]
for cta in range(2):
    print(f"--- CTA {'0' if cta == 0 else 'last'} (us from CTA0 first issue)")
    for t in list(range(0, 40)) + list(range(100, 116)):
        row = []
        for w, nm in enumerate(names):
            v = b[cta][w][t]
            row.append(f"{nm} {(v - t0) / 1e3:7.2f}" if v else f"{nm}    -   ")
        print(f"band {t:4d}: " + "  ".join(row))
