"""Per-band phase breakdown of the single-pass sweep (fused.cu k_sweep1) from
the debug timeline (otg_debug_sp_trace; last launch of a 4-iteration solve),
CTA 0, bands 32..255 (us, means):

  tmem   row warp waits for its TMEM slot      R0(t) - P(t-4)
  ring   row warp waits for the band's data    R1(t) - R0(t)
  rows   exponentials + row totals             Rc(t) - R1(t)
  pub    TMEM commit + global red of the sums  P(t) - Rc(t)
  grid   sums complete after this CTA's publish Cw(t) - P(t)
  cpre   w + wait for the TMEM band            C0(t) - Cw(t)
  fold   tcgen05.ld + FMA fold                 C1(t) - C0(t)
  cycle  interval between a row warp's bands    R0(t + 4) - R0(t)
  band   loader issue interval                 L(t+1) - L(t)

    python tools/sp_phases.py [n] [m]
"""
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot, _capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
m = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
T0 = int(sys.argv[3]) if len(sys.argv) > 3 else 40   # band range of the means
T1 = int(sys.argv[4]) if len(sys.argv) > 4 else 240
lib = _capi.load()
lib.otg_debug_sp_trace.argtypes = [C.c_int, C.c_void_p]
lib.otg_debug_sp_trace(1, None)
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3,
                                    sweep="single_pass")
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4))
buf = np.zeros(2 * 12 * 256, dtype=np.uint64)
lib.otg_debug_sp_trace(0, buf.ctypes.data)
for cta, name in ((0, "CTA 0"), (1, "last CTA")):
    b = buf.reshape(2, 12, 256).astype(np.int64)[cta] / 1e3
    L, R0, R1, P, Cw, C0, C1, Rc = (b[k] for k in (0, 1, 2, 3, 4, 5, 6, 7))
    t = np.arange(T0, T1)
    ph = dict(tmem=R0[t] - P[t - 4], ring=R1[t] - R0[t], rows=Rc[t] - R1[t], pub=P[t] - Rc[t],
              grid=Cw[t] - P[t], cpre=C0[t] - Cw[t], fold=C1[t] - C0[t],
              cycle=R0[t + 4] - R0[t],
              band=L[t + 1] - L[t])
    print(f"{n}x{m} {name}: " + "  ".join(f"{k} {np.mean(v):.3f}" for k, v in ph.items()
                                         ))
B = buf.reshape(2, 12, 256).astype(np.int64) / 1e3
t = np.arange(T0, T1)
d = B[1][3][t] - B[0][3][t]
late = np.maximum(B[0][3][t], B[1][3][t])
print(f"publish skew last-CTA minus CTA0: mean {d.mean():.3f} sd {d.std():.3f} us; "
      f"CTA0 sums complete after the later of the two publishes: {np.mean(B[0][4][t] - late):.3f} us")
b0 = B[0]
nz = b0[0][b0[0] > 0]
c1 = b0[6][b0[6] > 0]
if nz.size and c1.size:
    print(f"CTA 0: first band issued -> last recorded fold end {c1.max() - nz.min():.2f} us over "
          f"{int((b0[6] > 0).sum())} bands")
