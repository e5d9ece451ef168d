"""cfg1 (1000^2 fp64) acc-homotopy to 1e-8: us per evaluation (min over 7
solves), and the in-graph split (row / column / epilogue, CUDA events)."""
import sys
sys.path.insert(0, '.')
from paper_2605_30267_b200 import ot
a, b, C = ot.gen_config(1, 1000, 1000, 1)
p = ot.rescale_problem(ot.make_problem(a, b, C, 1e-2))
spec = ot.SolverSpec(kind="acc-homotopy", max_iters=10000)
ot.run_solver(p, spec, 1e-8)
us = []
for _ in range(7):
    r = ot.run_solver(p, spec, 1e-8)
    us.append(1e6 * r.device_seconds / r.evaluations)
t = ot.run_solver(p, spec, 1e-8, time_sweeps=True)
ev = t.evaluations
print("cfg1 us/eval min %.2f median %.2f" % (min(us), sorted(us)[3]), "iters", r.iterations,
      "| timed: row %.2f col %.2f epi %.2f us/eval" % (1e6 * t.row_pass_seconds / ev,
                                                   1e6 * t.col_pass_seconds / ev,
                                                   1e6 * t.epilogue_seconds / ev))
