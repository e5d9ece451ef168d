"""How much of cfg3's stored-cost work could exact (FTZ) block culling skip?

Solves cfg3 (65536^2 Beta point clouds, cost normalised to max 1, eps 1e-3)
for a few iteration counts and measures, with torch on the GPU,
  * the fraction of pairs whose base-2 exponent t_ij = V_j - S_i - kh c_ij is
    at or above -126 relative to the row max (below it ex2.approx.ftz is +0),
  * after a Morton sort of rows and columns, the fraction of (row tile x
    column block) blocks a min-cost table test keeps:
        max_{j in B} V_j - min_{i in T} S_i - kh * min_{T x B} c < -128 -> skip
    python tools/cull_probe3.py [n] [iters,iters,...]
"""
import sys

sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2605_30267_b200 import ot

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
iters_list = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "5,50,200,732").split(",")]
eps = 1e-3
x, y = ot.gen_config(3, n, n, 3)
a = np.full(n, 1 / n)
dev = torch.device("cuda")
X = torch.tensor(np.asarray(x, dtype=np.float64).reshape(n, 3), device=dev)
Y = torch.tensor(np.asarray(y, dtype=np.float64).reshape(n, 3), device=dev)
kh = float(np.float32(np.log2(np.e) / eps))


def morton(P):
    lo = P.min(0).values
    hi = P.max(0).values
    q = torch.clamp(((P - lo) / (hi - lo) * 1024).long(), 0, 1023)
    code = torch.zeros(P.shape[0], dtype=torch.long, device=dev)
    for b in range(10):
        for d in range(3):
            code |= ((q[:, d] >> b) & 1) << (3 * b + d)
    return torch.argsort(code)


pr, pc = morton(X), morton(Y)
Xs, Ys = X[pr], Y[pc]
# normalisation constant: max over all pairs (chunked)
cmax = 0.0
for k in range(0, n, 2048):
    c = torch.cdist(X[k:k + 2048], Y) ** 2
    cmax = max(cmax, float(c.max()))

p = ot.TransportProblem.from_points(a, a, x, y, eps)
for iters in iters_list:
    r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters))
    V = torch.tensor(r.potentials.v * np.log2(np.e), device=dev)[pc]
    S = torch.empty(n, device=dev, dtype=torch.float64)
    alive = 0
    tiles = {(RT, CB): 0 for RT in (16, 32, 64, 128) for CB in (32, 64, 128, 256)}
    for k in range(0, n, 1024):
        c = ((torch.cdist(Xs[k:k + 1024], Ys) ** 2) / cmax).float().double()
        t = V[None, :] - kh * c
        mx = t.max(1).values
        S[k:k + 1024] = mx
        alive += int((t - mx[:, None] >= -126).sum())
        for (RT, CB) in tiles:
            cm = c.view(1024 // RT, RT, n // CB, CB).amin(dim=(1, 3))
            Vm = V.view(n // CB, CB).amax(1)
            Sm = mx.view(1024 // RT, RT).amin(1)
            bound = Vm[None, :] - Sm[:, None] - kh * cm
            tiles[(RT, CB)] += int((bound >= -128).sum())
    print(f"n={n} iters={iters} viol={r.final_violation:.2e}: pairs alive {alive / n / n:.4f}", flush=True)
    for (RT, CB), kept in tiles.items():
        print(f"   {RT:4d} rows x {CB:4d} cols: blocks kept {kept / (n // RT) / (n // CB):.4f}")
