"""ptxas register / spill report for one csrc file: python tools/regs.py sweep.cu [filter]"""
import re, subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30267_b200 import build as b
src = os.path.join(b.CSRC, sys.argv[1])
flt = sys.argv[2] if len(sys.argv) > 2 else ""
r = subprocess.run([b.NVCC, "-Xptxas", "-v", *b.ARCH, *b.FLAGS, "-c", src, "-o", "/tmp/_regs.o"],
                   capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-3000:]); sys.exit(1)
fn = None
for l in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        fn = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        fn = re.sub(r"otg::\(anonymous namespace\)::", "", fn).split("(")[0]
    if fn and flt in fn and ("registers" in l or "spill" in l):
        print(f"{fn:40s} {l.split("info    :")[-1].strip()[:110]}")
