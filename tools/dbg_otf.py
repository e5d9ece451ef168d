import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2605_30267_b200 import ot
from oracle import oracle as O
n, m, eps = 400, 1200, 2e-3
x, y = ot.gen_config(5, n, m, 13)
a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
p = ot.TransportProblem.from_points(a, b, x, y, eps, norm="none", storage="on_the_fly")
C32 = O.cost_sqeuclid_f32(x.astype(np.float32), y.astype(np.float32))
ps = ot.rescale_problem(ot.make_problem(a, b, C32, eps))
print("cost equal", np.array_equal(p.stored_cost(), ps.stored_cost()))
v = O.random_zero_sum(O.Rng(3), m, 30.0)
e1, e2 = ot.eval_normalized_step(p, v), ot.eval_normalized_step(ps, v)
print("eval u diff", np.abs(e1.u - e2.u).max(), "vnext diff", np.abs(e1.v_next - e2.v_next).max())
for K in (1, 2, 3, 5, 10, 50):
    g1 = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=K))
    g2 = ot.homotopy_solve(ps, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=K))
    print(K, "v diff", np.abs(g1.potentials.v - g2.potentials.v).max(), "u diff", np.abs(g1.potentials.u - g2.potentials.u).max(), g1.row_redos, g2.row_redos)
