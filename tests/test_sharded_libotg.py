"""libotg's row-sharded path at world_size 2 (the column partial
sums of dual.cpp:41 are the all-reduced quantity).  Two processes share the
one GPU; their collective is a gloo host all-reduce passed through
otg_device_opts.allreduce, so the sharded data flow of the product library
(local rows through the C-ABI, one all-reduce per evaluation, the paused
chunk + eager cross-rank exact-LSE exchange for flagged columns, sharded plan
statistics) runs for real without a second GPU.

Bars: against the single-device solve with the same row split
(virtual_shards = 2: the per-shard partial sums combined in shard order,
which is exactly what the 2-rank SUM does) the column-side vectors and
iteration counts are bitwise equal; against the plain unsharded solve, 1e-12
(fp64 storage) / 1e-9 (fp32)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import sharded_worker as W  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_world2(case, tmp_path):
    port = _port()
    outs = [str(tmp_path / f"{case}_{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "sharded_worker.py"), str(r),
                               "2", str(port), case, outs[r]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out)
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(o)) for o in outs]


def _single(case, vshards):
    from paper_2605_30267_b200 import ot
    inst = W.instance(case)
    p = W.make(inst, virtual_shards=vshards)
    fixed = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-300, max_total_inner=inst["iters"]))
    tol = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=inst["tol"], max_total_inner=5000))
    st = ot.plan_stats(p, tol.potentials.u, tol.potentials.v)
    ev = ot.eval_normalized_step(p, fixed.potentials.v)
    r = dict(fixed_v=fixed.potentials.v, fixed_u=fixed.potentials.u, fixed_it=fixed.iterations,
             tol_v=tol.potentials.v, tol_u=tol.potentials.u, tol_it=tol.iterations,
             tol_conv=tol.converged, tol_fb=tol.fallback_columns, cost=st.primal_cost,
             viol=st.marginal_violation_l1, ev_v=ev.v_next, ev_u=ev.u, ev_f=ev.f_value,
             ev_g=ev.grad_l1,
             culled=inst.get("storage") == "on_the_fly" and ot.cull_stats(p)[0] >= 0.0)
    p.close()
    return r


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1.0, np.max(np.abs(b))))


@pytest.mark.parametrize("case", ["f32_points", "otf_points", "f64_dense"])
def test_world2_bitwise_vs_virtual_shards(case, tmp_path):
    r = _run_world2(case, tmp_path)
    v2 = _single(case, 2)
    assert r[0]["n_local"] + r[1]["n_local"] == len(W.instance(case)["a"])
    for k in range(2):  # every rank holds the same m-vectors
        assert int(r[k]["fixed_it"]) == v2["fixed_it"]
        assert int(r[k]["tol_it"]) == v2["tol_it"]
        assert np.array_equal(r[k]["fixed_v"], v2["fixed_v"])
        assert np.array_equal(r[k]["tol_v"], v2["tol_v"])
        assert np.array_equal(r[k]["ev_v"], v2["ev_v"])
    u = np.concatenate([r[0]["fixed_u"], r[1]["fixed_u"]])
    assert np.array_equal(u, v2["fixed_u"])
    assert np.array_equal(np.concatenate([r[0]["ev_u"], r[1]["ev_u"]]), v2["ev_u"])
    # sharded plan statistics are all-reduced: within rounding of the summation order
    assert abs(float(r[0]["cost"]) - v2["cost"]) <= 1e-12 * abs(v2["cost"])
    assert float(r[0]["cost"]) == float(r[1]["cost"])


@pytest.mark.parametrize("case,tol", [("f64_dense", 1e-12), ("f32_points", 1e-9),
                                      ("f32_points_sp", 1e-9)])
def test_world2_matches_unsharded(case, tol, tmp_path):
    """f32_points_sp: each rank runs the single-pass sweep on its own rows
    (its column partials all-reduced), against the single-pass sweep of the
    whole matrix on one device."""
    r = _run_world2(case, tmp_path)
    s = _single(case, 1)
    assert int(r[0]["tol_it"]) == s["tol_it"] and bool(r[0]["tol_conv"])
    assert rel(r[0]["tol_v"], s["tol_v"]) <= tol
    assert rel(np.concatenate([r[0]["tol_u"], r[1]["tol_u"]]), s["tol_u"]) <= tol
    assert abs(float(r[0]["ev_f"]) - s["ev_f"]) <= tol * max(1.0, abs(s["ev_f"]))


def test_world2_fallback_exchange(tmp_path):
    """eps small enough that columns underflow at v = 0: the sharded chunk
    pauses at those evaluations and the host runs the cross-rank exact LSE;
    the solve matches the unsharded one (whose fallback sums all rows on one
    device) to rounding, iteration count exactly."""
    r = _run_world2("f32_dense_fallback", tmp_path)
    s = _single("f32_dense_fallback", 1)
    assert s["tol_fb"] > 0 and int(r[0]["tol_fb"]) == s["tol_fb"]
    assert int(r[0]["tol_it"]) == s["tol_it"] and int(r[1]["tol_it"]) == s["tol_it"]
    assert np.array_equal(r[0]["tol_v"], r[1]["tol_v"])
    # (fp32 storage: the two fallback combinations round differently, and 50+
    # iterations carry that forward)
    assert rel(r[0]["tol_v"], s["tol_v"]) <= 1e-8
    assert abs(float(r[0]["cost"]) - s["cost"]) <= 1e-8 * abs(s["cost"])


def test_world2_culled_on_the_fly_matches_unsharded(tmp_path):
    """cfg5's sharded path: each rank runs the culled on-the-fly sweeps (its
    own Morton order of its local rows, exact FTZ skips) and the column
    partials are all-reduced; against the one-device culled solve the
    summation orders differ, so the bar is the fp32 parity bar: iteration
    count within 1%, potentials and transport cost to 1e-6."""
    r = _run_world2("otf_cull", tmp_path)
    s = _single("otf_cull", 1)
    assert s["culled"] and bool(r[0]["culled"]) and bool(r[1]["culled"])
    for k in range(2):
        assert bool(r[k]["tol_conv"])
        assert abs(int(r[k]["tol_it"]) - s["tol_it"]) <= max(1, s["tol_it"] // 100)
    assert np.array_equal(r[0]["tol_v"], r[1]["tol_v"])  # replicated m-vector epilogue
    assert rel(r[0]["fixed_v"], s["fixed_v"]) <= 1e-6
    assert rel(r[0]["tol_v"], s["tol_v"]) <= 1e-5
    assert abs(float(r[0]["cost"]) - s["cost"]) <= 1e-6 * abs(s["cost"])
