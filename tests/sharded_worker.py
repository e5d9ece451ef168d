"""One rank of a row-sharded libotg solve whose collective is a gloo host
all-reduce (otg_device_opts.allreduce), for tests/test_sharded_libotg.py.
Several ranks may share one GPU: the only cross-rank dependency is the host
all-reduce, so no kernel waits on another process.

    python tests/sharded_worker.py RANK WORLD PORT CASE OUT.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def instance(case):
    from paper_2605_30267_b200 import ot
    if case in ("f32_points", "f32_points_sp"):  # cfg3-shaped points, stored fp32
        # f32_points: the two-pass kernels (bitwise against virtual shards);
        # f32_points_sp: the single-pass sweep on each rank's rows
        n, m = 1536, 1100
        x, y = ot.gen_config(3, n, m, 3)
        return dict(kind="points", x=x, y=y, a=np.full(n, 1 / n), b=np.full(m, 1 / m),
                    eps=2e-2, storage="f32", norm="max", tol=1e-7, iters=60,
                    sweep="two_pass" if case == "f32_points" else "single_pass")
    if case == "otf_points":  # cfg5-shaped, cost on the fly
        n, m = 1200, 1500
        x, y = ot.gen_config(5, n, m, 5)
        return dict(kind="points", x=x, y=y, a=np.full(n, 1 / n), b=np.full(m, 1 / m),
                    eps=0.1, storage="on_the_fly", norm="none", tol=1e-6, iters=60)
    if case == "otf_cull":  # cfg5-shaped at eps 1e-3, large enough for the culled sweeps
        # (>= 4096 local rows and columns): each rank Morton-orders its own rows
        n, m = 9000, 6000
        x, y = ot.gen_config(5, n, m, 5)
        return dict(kind="points", x=x, y=y, a=np.full(n, 1 / n), b=np.full(m, 1 / m),
                    eps=1e-3, storage="on_the_fly", norm="none", tol=1e-5, iters=40)
    if case == "f64_dense":  # dense fp64 rows through the dense contract
        n, m = 700, 500
        a, b, C = ot.synthetic_instance(n, m, 11)
        return dict(kind="dense", a=a, b=b, C=C, eps=2e-2, tol=1e-9, iters=40)
    if case == "f32_dense_fallback":  # small eps: columns underflow at v = 0
        n, m = 900, 640
        x, y = ot.gen_config(3, n, m, 7)
        from oracle import oracle as O
        C, _ = O.cost_sqeuclid_max_f32(x, y)
        return dict(kind="dense", a=np.full(n, 1 / n), b=np.full(m, 1 / m), C=C, eps=2e-3,
                    tol=1e-6, iters=50, sweep="two_pass")
    raise ValueError(case)


def make(inst, **kw):
    from paper_2605_30267_b200 import ot
    if inst["kind"] == "points":
        return ot.TransportProblem.from_points(inst["a"], inst["b"], inst["x"], inst["y"],
                                               inst["eps"], storage=inst["storage"],
                                               norm=inst["norm"], sweep=inst.get("sweep", "auto"),
                                               **kw)
    p = ot.rescale_problem(ot.make_problem(inst["a"], inst["b"], inst["C"], inst["eps"]))
    return p.to_device(sweep=inst.get("sweep", "auto"), **kw)


def main():
    rank, world, port, case, out = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]),
                                    sys.argv[4], sys.argv[5])
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2605_30267_b200 import dist as D
    from paper_2605_30267_b200 import ot
    inst = instance(case)
    n = len(inst["a"])
    r0, r1 = D.shard_rows(n, world, rank)
    x_local = None
    kw = dict(world_size=world, rank=rank, row_begin=r0, row_end=r1,
              allreduce=D.gloo_allreduce())
    if inst["kind"] == "points":
        # the caller's local rows only (otg.h contract)
        x_local = np.ascontiguousarray(inst["x"][r0:r1])
        p = ot.TransportProblem.from_points(inst["a"], inst["b"], x_local, inst["y"],
                                            inst["eps"], storage=inst["storage"],
                                            norm=inst["norm"], sweep=inst.get("sweep", "auto"), **kw)
    else:
        p = make(inst, **kw)
    fixed = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300,
                                                   max_total_inner=inst["iters"]))
    tol = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=inst["tol"], max_total_inner=5000))
    st = ot.plan_stats(p, tol.potentials.u, tol.potentials.v)
    ev = ot.eval_normalized_step(p, fixed.potentials.v)
    np.savez(out, r0=r0, r1=r1, fixed_v=fixed.potentials.v, fixed_u=fixed.potentials.u,
             fixed_it=fixed.iterations, tol_v=tol.potentials.v, tol_u=tol.potentials.u,
             tol_it=tol.iterations, tol_conv=tol.converged, tol_fb=tol.fallback_columns,
             fixed_fb=fixed.fallback_columns, cost=st.primal_cost,
             viol=st.marginal_violation_l1, ev_v=ev.v_next, ev_u=ev.u, ev_f=ev.f_value,
             ev_g=ev.grad_l1, n_local=p.handle.info.n_local,
             culled=inst.get("storage") == "on_the_fly" and ot.cull_stats(p)[0] >= 0.0)
    p.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
