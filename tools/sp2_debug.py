"""k_sp2 stuck-wait records: OTG_FUSED=2 OTG_SP_TRACE=1 python tools/sp2_debug.py n m [lag]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_30267_b200 import ot, _capi
n, m = int(sys.argv[1]), int(sys.argv[2])
x, y = ot.gen_config(3, n, m, 11)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 5e-4)
lib = ctypes.CDLL(os.path.join(os.path.dirname(_capi.__file__), "libotg.so"))
try:
    r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=40))
    print("ok", r.iterations)
except Exception as e:
    print("error", e)
buf = (ctypes.c_longlong * (256 * 8))()
lib.otg_debug_sp_trace(buf, 256 * 8)
a = np.array(buf, dtype=np.int64).reshape(256, 8)
print("records", a[0, 0])
names = {1: "producer(ia,ib,lag_rows,n)", 2: "reducer(c,cnt,E,G)", 3: "column(c,ready,want,cw)",
         4: "stats fullA(row,parity)", 5: "column fullB(row,parity)"}
for r in a[1:1 + min(a[0, 0], 60)]:
    print(names.get(int(r[0]), r[0]), "cta", r[1], "tid", r[2], "|", r[3], r[4], r[5], r[6])
