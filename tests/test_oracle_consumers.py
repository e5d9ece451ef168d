"""Plan consumers (pipelines.cpp:58-145) in the CPU oracle, pinned by the
reference's test_pipelines.cpp cases (tests/golden/kat.json); the plans are
realised as implicit plans P = exp(u + v - C') with u = v = 0 and
C' = -log(entry) (1000 for a zero entry: exp(-1000) is exactly 0)."""
import numpy as np
import pytest

from oracle import oracle as O


def plan_problem(entries, n, m):
    P = np.asarray(entries, dtype=np.float64).reshape(n, m)
    with np.errstate(divide="ignore"):
        Cp = np.where(P > 0, -np.log(np.where(P > 0, P, 1.0)), 1000.0)
    return O.Problem(np.full(n, 1.0 / n), np.full(m, 1.0 / m), Cp), np.zeros(n), np.zeros(m)


def test_barycentric_kats(kat):
    src = np.array(kat["pipelines_barycentric_src"]["value"])
    pl = kat["pipelines_barycentric_plans"]
    q, u, v = plan_problem(pl["diagonal"], 2, 2)
    assert np.max(np.abs(O.barycentric_projection(q, u, v, src) - src)) <= pl["tol"]
    q, u, v = plan_problem(pl["antidiagonal"], 2, 2)
    out = O.barycentric_projection(q, u, v, src)
    assert np.max(np.abs(out[0] - src[1])) <= pl["tol"] and np.max(np.abs(out[1] - src[0])) <= pl["tol"]
    q, u, v = plan_problem(pl["uniform"], 2, 2)
    out = O.barycentric_projection(q, u, v, src)
    assert np.allclose(out[:, 0], 0.5, rtol=1e-15) and np.allclose(out[:, 2], 0.5, rtol=1e-15)
    q, u, v = plan_problem(pl["zero_column"], 2, 2)
    with pytest.raises(O.OracleError) as e:
        O.barycentric_projection(q, u, v, src)
    assert e.value.kind == "DegenerateColumn"


def test_barycentric_hull(kat):
    pl = kat["pipelines_barycentric_plans"]
    rng = O.Rng(pl["hull_seed"])
    wide = np.array([[rng.next_double() for _ in range(3)] for _ in range(4)])
    P = np.array([[pl["hull_offset"] + rng.next_double() for _ in range(3)] for _ in range(4)])
    P /= P.sum()
    q, u, v = plan_problem(P.ravel(), 4, 3)
    out = O.barycentric_projection(q, u, v, wide)
    for ch in range(3):
        assert out[:, ch].min() >= wide[:, ch].min() - 1e-12
        assert out[:, ch].max() <= wide[:, ch].max() + 1e-12


def test_predict_translations_kat(kat):
    k = kat["pipelines_predict_translations"]
    q, u, v = plan_problem(k["plan"], 3, 3)
    assert list(O.predict_translations(q, u, v)) == k["expected"]


def test_topk_kat(kat):
    k = kat["pipelines_topk"]
    q, u, v = plan_problem(k["plan"], 3, 3)
    top = O.plan_topk(q, u, v, [0, 1, 2], 5)
    assert [list(t) for t in top] == [[0, 1, 2, -1, -1], [1, 0, 2, -1, -1], [2, 0, 1, -1, -1]]
    assert list(O.plan_topk(q, u, v, [0], 2)[0]) == [0, 1]


def test_nn_assign_ties_lowest_index(kat):
    k = kat["pipelines_nn"]
    colors = np.array(k["tie_colors"]) / np.array([1.0, 255.0])[[0, 1]][:, None]
    tied = np.full((1, 3), k["tie_pixel"] / 255.0)
    q = np.vstack([colors, tied])
    assert list(O.nn_assign(q, colors)) == [0, 1, 0]
