"""Single pass vs two-pass per shape (fp32 stored, cfg3-shaped points, eps
1e-3): device us per evaluation over a 60-iteration homotopy run.
    python tools/sp_crossover.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot

shapes = [(2048, 8192), (4096, 8192), (8192, 8192), (16384, 8192), (8192, 2048), (8192, 4096),
          (32768, 4096), (65536, 1024), (4096, 16384), (8192, 16384), (2048, 65536),
          (4096, 65536), (8192, 65536), (16384, 65536)]
for n, m in shapes:
    x, y = ot.gen_config(3, n, m, 3)
    out = []
    for sw in ("two_pass", "single_pass"):
        p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3, sweep=sw)
        cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=60)
        ot.homotopy_solve(p, cfg)
        best = min(ot.homotopy_solve(p, cfg).device_seconds for _ in range(3))
        info = p.handle.info
        out.append((sw, info.sweep_mode, info.sweep_clusters, 1e6 * best / 60))
        p.close()
    print(f"{n:6d} x {m:6d}: " + "  ".join(f"{sw}(mode {md}, H {h}) {us:8.1f} us" for sw, md, h, us in out),
          flush=True)
