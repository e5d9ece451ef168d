"""Plan consumers on the device (csrc/consumers.cu) over the implicit plan:
the reference's test_pipelines.cpp cases replayed through the C-ABI, then
parity with the oracle on solved problems (fp64 stored, fp32 stored, on the
fly)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot
from test_oracle_consumers import plan_problem

pytestmark = pytest.mark.gpu


def dev_plan(entries, n, m):
    q, u, v = plan_problem(entries, n, m)
    p = ot.make_problem(q.a, q.b, q.C, 1.0)
    return ot.rescale_problem(p), u, v


def test_barycentric_kats(kat):
    src = np.array(kat["pipelines_barycentric_src"]["value"])
    pl = kat["pipelines_barycentric_plans"]
    p, u, v = dev_plan(pl["diagonal"], 2, 2)
    assert np.max(np.abs(ot.barycentric_projection(p, u, v, src) - src)) <= pl["tol"]
    p, u, v = dev_plan(pl["antidiagonal"], 2, 2)
    out = ot.barycentric_projection(p, u, v, src)
    assert np.max(np.abs(out[0] - src[1])) <= pl["tol"] and np.max(np.abs(out[1] - src[0])) <= pl["tol"]
    p, u, v = dev_plan(pl["uniform"], 2, 2)
    out = ot.barycentric_projection(p, u, v, src)
    assert np.allclose(out[:, 0], 0.5, rtol=1e-15) and np.allclose(out[:, 2], 0.5, rtol=1e-15)
    p, u, v = dev_plan(pl["zero_column"], 2, 2)
    with pytest.raises(ot.DegenerateColumn):
        ot.barycentric_projection(p, u, v, src)
    p, u, v = dev_plan(pl["diagonal"], 2, 2)
    with pytest.raises(ot.DimensionMismatch):
        ot.barycentric_projection(p, u, v, np.zeros((3, 3)))


def test_predict_translations_and_topk_kats(kat):
    k = kat["pipelines_predict_translations"]
    p, u, v = dev_plan(k["plan"], 3, 3)
    assert ot.predict_translations(p, u, v) == k["expected"]
    t = kat["pipelines_topk"]
    p, u, v = dev_plan(t["plan"], 3, 3)
    diag = [(0, 0), (1, 1), (2, 2)]
    assert ot.topk_accuracy(p, u, v, diag, 1) == t["diag_top1"]
    assert ot.topk_accuracy(p, u, v, diag, 5) == t["diag_top5"]
    assert ot.topk_accuracy(p, u, v, [(0, 1), (0, 2)], 1) == t["multi_top1"]
    assert ot.topk_accuracy(p, u, v, [(0, 1), (0, 2)], 2) == t["multi_top2"]
    mixed = [(0, 2), (1, 1), (2, 0)]
    assert ot.topk_accuracy(p, u, v, mixed, 1) <= ot.topk_accuracy(p, u, v, mixed, 5)
    assert ot.topk_accuracy(p, u, v, [], 1) is None
    with pytest.raises(ot.DimensionMismatch):
        ot.topk_accuracy(p, u, v, [(0, 5)], 1)
    with pytest.raises(ot.OtError):
        ot.topk_accuracy(p, u, v, [(0, 0)], 0)


def test_nn_propagate_kats(kat):
    k = kat["pipelines_nn"]
    c = round(k["single_color"] * 255)
    img = np.full((4, 3), c, dtype=np.uint8)
    sample = np.full((1, 3), c / 255.0)
    out = ot.nn_propagate(img, sample, [k["single_transferred"]])
    assert (out == np.array(k["single_expected"], dtype=np.uint8)).all()
    colors = np.array([[0, 0, 0], [128, 128, 128]], dtype=np.float64) / 255.0
    pixels = np.array([[0, 0, 0], [128, 128, 128], [64, 64, 64]], dtype=np.uint8)
    out = ot.nn_propagate(pixels, colors, [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    assert out[0, 0] == 255 and out[1, 1] == 255 and out[2, 0] == 255 and out[2, 1] == 0
    out = ot.nn_propagate(np.zeros((1, 3), np.uint8), np.zeros((1, 3)), [k["clip_transferred"]])
    assert list(out[0]) == k["clip_expected"]
    with pytest.raises(ot.DimensionMismatch):
        ot.nn_propagate(np.zeros((1, 3), np.uint8), np.zeros((2, 3)), np.zeros((1, 3)))


def _solved(kind, n, m, seed):
    if kind == "f64":
        a, b, Cm = ot.synthetic_instance(n, m, seed)
        p = ot.rescale_problem(ot.make_problem(a, b, Cm, 0.02))
        q = O.synthetic_rescaled(n, m, seed, 0.02)
    else:
        x, y = ot.gen_config(3 if kind == "f32" else 5, n, m, seed)
        a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
        if kind == "f32":
            p = ot.TransportProblem.from_points(a, b, x, y, 5e-3)
            q = O.Problem(a, b, p.stored_cost(), cost_div=5e-3)
        else:
            p = ot.TransportProblem.from_points(a, b, x, y, 5e-3, norm="none", storage="on_the_fly")
            q = O.Problem(a, b, O.cost_sqeuclid_f32(x.astype(np.float32), y.astype(np.float32)),
                          cost_div=ot.otf_epsilon(5e-3))
    r = ot.homotopy_solve(p, ot.HomotopyConfig(tol_l1=1e-6, max_total_inner=400))
    return p, q, r.potentials.u, r.potentials.v


@pytest.mark.parametrize("kind,n,m", [("f64", 300, 200), ("f32", 512, 700), ("otf", 400, 333)])
def test_consumers_match_oracle(kind, n, m):
    p, q, u, v = _solved(kind, n, m, 3)
    rng = np.random.default_rng(1)
    src = rng.random((n, 3))
    bg = ot.barycentric_projection(p, u, v, src)
    bo = O.barycentric_projection(q, u, v, src)
    assert np.max(np.abs(bg - bo)) <= 1e-12 * max(1.0, np.max(np.abs(bo)))
    pg = np.array(ot.predict_translations(p, u, v))
    po = O.predict_translations(q, u, v)
    assert (pg == po).mean() >= 0.999  # fp64 exp last-bit ties may differ
    rows = np.arange(0, n, 7)
    tg = ot.plan_topk(p, u, v, rows, 5)
    to = O.plan_topk(q, u, v, rows, 5)
    assert (tg == to).mean() >= 0.999
    pairs = [(int(i), int(po[i])) for i in rows]
    assert ot.topk_accuracy(p, u, v, pairs, 1) >= 0.99


def test_consumer_overflow_guard():
    p, u, v = dev_plan([0.5, 0.5, 0.5, 0.5], 2, 2)
    with pytest.raises(ot.PotentialOverflow):
        ot.predict_translations(p, np.full(2, 800.0), v)
    with pytest.raises(ot.PotentialOverflow):
        ot.barycentric_projection(p, np.full(2, 800.0), v, np.zeros((2, 3)))


def test_nn_assign_matches_oracle():
    rng = np.random.default_rng(5)
    refs = np.round(rng.random((3000, 3)) * 255) / 255.0
    q = np.round(rng.random((20000, 3)) * 255) / 255.0
    assert (ot.nn_assign(q, refs) == O.nn_assign(q, refs)).all()
