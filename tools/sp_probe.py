"""Single-pass sweep probe: cfg3-shaped fp32 problems, the single-pass kernel
against the two-pass kernels (same instance, same iterations): potentials,
iteration counts, per-evaluation sweep time (CUDA events inside the solve).

    python tools/sp_probe.py [n m iters] ...
"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot

sizes = [(2048, 65536, 12), (8192, 8192, 12), (65536, 65536, 12)]
if len(sys.argv) > 1:
    a = list(map(int, sys.argv[1:]))
    sizes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
for n, m, iters in sizes:
    x, y = ot.gen_config(3, n, m, 3)
    out = {}
    for sweep in ("single_pass", "two_pass"):
        p = ot.TransportProblem.from_points(np.full(n, 1 / n), np.full(m, 1 / m), x, y, 1e-3,
                                            sweep=sweep)
        cfg = ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters)
        r = ot.homotopy_solve(p, cfg)
        t = ot.homotopy_solve(p, cfg, time_sweeps=True)
        out[sweep] = (r, t, p.handle.info.sweep_mode)
        p.close()
    (ra, ta, ma), (r2, t2, m2) = out["single_pass"], out["two_pass"]
    dv = np.max(np.abs(ra.potentials.v - r2.potentials.v)) / max(1.0, np.max(np.abs(r2.potentials.v)))
    du = np.max(np.abs(ra.potentials.u - r2.potentials.u)) / max(1.0, np.max(np.abs(r2.potentials.u)))
    ev = ta.evaluations
    print(f"{n}x{m}: modes {ma}/{m2} it {ra.iterations}/{r2.iterations} rel dv {dv:.2e} du {du:.2e} "
          f"redo {ra.row_redos}/{r2.row_redos} | single: row {1e3 * ta.row_pass_seconds / ev:.3f} "
          f"col {1e3 * ta.col_pass_seconds / ev:.3f} epi {1e3 * ta.epilogue_seconds / ev:.3f} ms | "
          f"two-pass: row {1e3 * t2.row_pass_seconds / ev:.3f} col {1e3 * t2.col_pass_seconds / ev:.3f} "
          f"epi {1e3 * t2.epilogue_seconds / ev:.3f} ms | dev s {ra.device_seconds:.4f}/{r2.device_seconds:.4f}",
          flush=True)
