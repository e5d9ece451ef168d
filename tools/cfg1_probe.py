"""cfg1 (1000^2 fp64) acc-homotopy to 1e-8: us per evaluation."""
import sys
sys.path.insert(0, '.')
from paper_2605_30267_b200 import ot
a, b, C = ot.gen_config(1, 1000, 1000, 1)
p = ot.rescale_problem(ot.make_problem(a, b, C, 1e-2))
spec = ot.SolverSpec(kind="acc-homotopy", max_iters=10000)
ot.run_solver(p, spec, 1e-8)
r = ot.run_solver(p, spec, 1e-8)
print("cfg1 us/eval", round(1e6 * r.device_seconds / r.evaluations, 2), "iters", r.iterations)
