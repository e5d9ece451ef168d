"""In-solve sweep timings at the bench size for env knob settings:
python tools/row_sweep.py 'OTG_ROW_PF=0' 'OTG_ROW_PF=1' ...  (one subprocess each)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r)
import numpy as np
from paper_2605_30267_b200 import ot
n = int(__import__("os").environ.get("RS_N", "65536")); m = int(__import__("os").environ.get("RS_M", "65536"))
x, y = ot.gen_config(3, n, m, 3)
p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3)
ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=4))
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=30), time_sweeps=True)
r2 = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=30))
e = r.evaluations
print(f"row {r.row_pass_seconds / e * 1e3:.4f} ms  col {r.col_pass_seconds / e * 1e3:.4f} ms  "
      f"epi {r.epilogue_seconds / e * 1e3:.4f} ms  step(ev) {r.device_seconds / r.iterations * 1e3:.4f} "
      f"step {r2.device_seconds / r2.iterations * 1e3:.4f} ms  redos {r.row_redos}  "
      f"fallback cols {r.fallback_columns}  mode {p.handle.info.sweep_mode} "
      f"clusters {p.handle.info.sweep_clusters}")
''' % ROOT
for spec in sys.argv[1:] or [""]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(f"{spec or 'default'}: {r.stdout.strip() or r.stderr[-500:]}", flush=True)
