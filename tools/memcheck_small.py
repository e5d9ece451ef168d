"""Small exercise of every kernel family for compute-sanitizer memcheck."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
for (n, m) in [(5, 5), (37, 23), (3, 3000), (300, 257), (9, 13)]:
    p = ot.synthetic_rescaled(n, m, 33, 0.6)
    ot.homotopy_solve_instrumented(p, ot.HomotopyConfig(tol_l1=1e-9, record_trace=True),
                                   ot.AccelInstrumentation(stability=True))
    ot.sinkhorn_solve(p)
    a, b, C = ot.gen_config(1, n, m, 1)
    q = ot.rescale_problem(ot.make_problem(a, b, C.astype(np.float32), 0.01))
    r = ot.homotopy_solve(q, ot.HomotopyConfig(tol_l1=1e-6))
    ot.plan_stats(q, r.potentials.u, r.potentials.v)
    q4 = ot.rescale_problem(ot.make_problem(a, b, C, 0.01)).to_device(virtual_shards=2)
    ot.homotopy_solve(q4, ot.HomotopyConfig(tol_l1=1e-6))
x = np.array([[0.0], [0.1], [0.2], [0.3]]); y = np.array([[0.0], [0.15], [1.0], [0.25]])
p = ot.TransportProblem.from_points(np.full(4, .25), np.full(4, .25), x, y, 1e-3, norm="none")
ot.eval_normalized_step(p, np.zeros(4))
print("memcheck exercise done")
# on-the-fly culled sweeps (>= 4096 rows and columns: Morton order, block skips)
x, y = ot.gen_config(5, 4096, 4100, 5)
pc = ot.TransportProblem.from_points(np.full(4096, 1 / 4096), np.full(4100, 1 / 4100), x, y, 1e-3,
                                     norm="none", storage="on_the_fly")
ot.cull_stats(pc)  # never evaluated: zeroed state, harmless
ot.homotopy_solve(pc, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=3))
assert ot.cull_stats(pc)[0] > 0.0
# batched path (one CTA per problem)
n4, m4, x4, y4 = ot.gen_config4(12, 4, 64)
bp = ot.BatchProblem.cosine(n4, m4, x4, y4, 5e-3, norm="none")
bp.homotopy_solve(ot.HomotopyConfig(tol_l1=1e-6))
bp.close()
print("memcheck exercise (culled on-the-fly, batched) done")
