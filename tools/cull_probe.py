"""How much of cfg5's pair work could block culling skip exactly (FTZ)?

Solves the cfg5-shaped on-the-fly problem for a few iterations, then, with
torch on the GPU, measures
  * the fraction of pairs whose base-2 exponent t_ij = V_j - S_i - kh c_ij is
    above -126 (S_i = the row max: ex2.approx.ftz returns exactly 0 below),
  * after a Morton sort of rows and columns, the fraction of (row tile x
    column block) pairs a bounding-box test would skip:
        max_{j in B} V_j - min_{i in T} S_i - kh * mindist^2(T, B) < -128.
    python tools/cull_probe.py [n] [iters] [row_tile] [col_block]
"""
import sys

sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2605_30267_b200 import ot

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
RT = int(sys.argv[3]) if len(sys.argv) > 3 else 256
CB = int(sys.argv[4]) if len(sys.argv) > 4 else 64
x, y = ot.gen_config(5, n, n, 5)
a = np.full(n, 1 / n)
eps = 1e-3
p = ot.TransportProblem.from_points(a, a, x, y, eps, norm="none", storage="on_the_fly")
r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=iters))
v = r.potentials.v
dev = torch.device("cuda")
X = torch.tensor(np.asarray(x, dtype=np.float32).reshape(n, 3), device=dev)
Y = torch.tensor(np.asarray(y, dtype=np.float32).reshape(n, 3), device=dev)
eps_eff = ot.otf_epsilon(eps) if hasattr(ot, "otf_epsilon") else eps
kh = float(np.float32(np.log2(np.e) / eps_eff))
V = torch.tensor(v * np.log2(np.e), device=dev, dtype=torch.float64)


def exps(rows):
    c = ((X[rows, None, :] - Y[None, :, :]) ** 2).sum(-1).double()
    return V[None, :] - kh * c


# row shifts (base-2 row max) for every row, in chunks
S = torch.empty(n, device=dev, dtype=torch.float64)
alive = 0
for k in range(0, n, 512):
    rows = torch.arange(k, min(n, k + 512), device=dev)
    t = exps(rows)
    mx = t.max(1).values
    S[rows] = mx
    alive += int((t - mx[:, None] >= -126).sum())
print(f"n={n} iters={iters}: pairs with t >= -126 (ex2 nonzero): {alive / n / n:.4f}")


def morton(P):
    q = torch.clamp((P * 1024).long(), 0, 1023)
    code = torch.zeros(P.shape[0], dtype=torch.long, device=dev)
    for b in range(10):
        for d in range(3):
            code |= ((q[:, d] >> b) & 1) << (3 * b + d)
    return torch.argsort(code)


pr, pc = morton(X), morton(Y)
Xs, Ys, Ss, Vs = X[pr], Y[pc], S[pr], V[pc]
nt, nb = (n + RT - 1) // RT, (n + CB - 1) // CB


def boxes(P, T):
    k = (P.shape[0] + T - 1) // T
    pad = k * T - P.shape[0]
    Q = torch.cat([P, P[-1:].expand(pad, 3)]) if pad else P
    Q = Q.view(k, T, 3)
    return Q.min(1).values, Q.max(1).values


def tile_red(v, T, op):
    k = (v.shape[0] + T - 1) // T
    pad = k * T - v.shape[0]
    w = torch.cat([v, v[-1:].expand(pad)]) if pad else v
    w = w.view(k, T)
    return w.min(1).values if op == "min" else w.max(1).values


rlo, rhi = boxes(Xs, RT)
clo, chi = boxes(Ys, CB)
Smin = tile_red(Ss, RT, "min")
Vmax = tile_red(Vs, CB, "max")
kept = 0
for k in range(nt):
    gap = torch.clamp(torch.maximum(clo - rhi[k], rlo[k] - chi), min=0)
    d2 = (gap.double() ** 2).sum(1)
    bound = Vmax - Smin[k] - kh * d2
    kept += int((bound >= -128).sum())
print(f"Morton tiles {RT} rows x {CB} columns: blocks kept {kept / nt / nb:.4f} "
      f"(pair work kept ~{kept / nt / nb:.4f}, exact pairs alive {alive / n / n:.4f})")

# per-row point-to-box bound, skip decided per tile of RT rows (all rows culled)
for CBk in (16, 64):
    clo, chi = boxes(Ys, CBk)
    Vmax = tile_red(Vs, CBk, "max")
    nbk = clo.shape[0]
    for RTk in (32, 256):
        kept_t = 0
        kept_r = 0
        for k0 in range(0, n, 4096):
            rows = torch.arange(k0, min(n, k0 + 4096), device=dev)
            xr = Xs[rows]
            gap = torch.clamp(torch.maximum(clo[None] - xr[:, None], xr[:, None] - chi[None]), min=0)
            d2 = (gap.double() ** 2).sum(-1)
            live = (Vmax[None] - Ss[rows][:, None] - kh * d2) >= -128  # rows x blocks
            kept_r += int(live.sum())
            L = live.shape[0] // RTk * RTk
            kept_t += int(live[:L].view(-1, RTk, nbk).any(1).sum()) * RTk + int(live[L:].any(0).sum()) * (live.shape[0] - L)
        print(f"per-row box test, {CBk}-column blocks: row-level kept {kept_r / n / nbk:.4f}, "
              f"{RTk}-row tiles kept {kept_t / n / nbk:.4f}")

# column pass: per-column point-to-box test against 16/32-row sorted blocks,
# skip decided per warp of W consecutive sorted columns
for RBk in (16, 32):
    rlo, rhi = boxes(Xs, RBk)
    nmax = tile_red(-Ss, RBk, "max")
    nrb = rlo.shape[0]
    for W in (32, 64, 128):
        kept_c = 0
        kept_w = 0
        for k0 in range(0, n, 4096):
            cols = torch.arange(k0, min(n, k0 + 4096), device=dev)
            yc = Ys[cols]
            gap = torch.clamp(torch.maximum(rlo[None] - yc[:, None], yc[:, None] - rhi[None]), min=0)
            d2 = (gap.double() ** 2).sum(-1)
            live = (Vs[cols][:, None] + nmax[None] - kh * d2) >= -128  # cols x row blocks
            kept_c += int(live.sum())
            L = live.shape[0] // W * W
            kept_w += int(live[:L].view(-1, W, nrb).any(1).sum()) * W + int(live[L:].any(0).sum()) * (live.shape[0] - L)
        print(f"column pass, {RBk}-row blocks: column-level kept {kept_c / n / nrb:.4f}, "
              f"{W}-column warps kept {kept_w / n / nrb:.4f}")
