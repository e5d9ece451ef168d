"""Column-pass launch-shape sweep at the bench size: python tools/col_sweep.py
(one subprocess per (OTG_COL_T, OTG_COL_SPLITS) because libotg reads them once)."""
import itertools, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [
    (256, s, pad) for pad in (0, 32, 128, 1024) for s in (16, 20, 21, 22, 24, 28)]
for shp in shapes:
    t, s, pad = (tuple(shp) + (0, 0))[:3]
    env = dict(os.environ, OTG_COL_T=str(t), OTG_COL_SPLITS=str(s), OTG_LDC_PAD=str(pad))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_sweeps.py"), "65536"],
                       env=env, capture_output=True, text=True, cwd=ROOT)
    print(f"T={t} splits={s or 'auto'} pad={pad}: {r.stdout.strip() or r.stderr[-400:]}", flush=True)
