"""The oracle's own BASELINE config samplers (oracle/otoracle.cpp
orc_gen_config*) against the product library's otg_gen_config*: bitwise
equal, so the CPU legs (fixtures, bench.py --impl reference) can generate the
same inputs without loading libotg.  Also: the oracle's threaded sweep is
deterministic and equal to the reference's single-threaded order to rounding,
and the fp32 stored cost it builds is the device's definition."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_30267_b200 import ot


@pytest.mark.parametrize("cfg,n,m,seed", [(1, 37, 41, 1), (2, 300, 257, 2), (3, 211, 199, 3),
                                          (5, 403, 517, 5), (5, 20000, 20000, 5)])
def test_gen_config_bitwise(cfg, n, m, seed):
    a = O.gen_config(cfg, n, m, seed)
    b = ot.gen_config(cfg, n, m, seed)
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_gen_config4_bitwise():
    n1, m1, x1, y1 = O.gen_config4(64, 4, d=96)
    n2, m2, x2, y2 = ot.gen_config4(64, 4, d=96)
    assert np.array_equal(n1, n2) and np.array_equal(m1, m2)
    assert np.array_equal(x1.view(np.uint32), x2.view(np.uint32))
    assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))


def test_cost_sqeuclid_max_f32_matches_float64_definition():
    x, y = O.gen_config(3, 123, 77, 9)
    C64, _, mx = None, None, None
    raw = ((x[:, None, :] - y[None, :, :]) ** 2)
    # coordinate-ordered fp64 sum (no reassociation), as the device computes it
    acc = np.zeros(raw.shape[:2])
    for k in range(3):
        acc = acc + raw[:, :, k]
    ref = (acc / acc.max()).astype(np.float32)
    for th in (1, 3):
        Cm, mx = O.cost_sqeuclid_max_f32(x, y, threads=th)
        assert mx == acc.max()
        assert np.array_equal(Cm, ref)


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_threaded_oracle_matches_single_thread(threads):
    x, y = O.gen_config(2, 301, 263, 2)
    Cm, _ = O.cost_sqeuclid_max_f32(x, y)
    p = O.Problem(np.full(301, 1 / 301), np.full(263, 1 / 263), Cm, cost_div=1e-2)
    v = O.random_zero_sum(O.Rng(4), 263, 5.0)
    with O.threads(1):
        e1 = O.eval_normalized_step(p, v)
        h1 = O.homotopy_solve(p, tol_l1=1e-7)
        s1 = O.plan_stats(p, h1.u, h1.v, 1e-2)
    with O.threads(threads):
        e2 = O.eval_normalized_step(p, v)
        e3 = O.eval_normalized_step(p, v)
        h2 = O.homotopy_solve(p, tol_l1=1e-7)
        s2 = O.plan_stats(p, h2.u, h2.v, 1e-2)
    for k in ("v_next", "u", "grad"):
        assert np.array_equal(e2[k], e3[k])  # deterministic for a given count
        assert np.max(np.abs(e2[k] - e1[k])) <= 1e-15 * max(1.0, np.max(np.abs(e1[k])))
    assert h1.iterations == h2.iterations
    assert abs(s1["primal_cost"] - s2["primal_cost"]) <= 1e-13 * abs(s1["primal_cost"])
    assert np.max(np.abs(h1.v - h2.v)) <= 1e-12 * max(1.0, np.max(np.abs(h1.v)))


def test_threaded_fallback_columns():
    """Extreme potentials flag columns for the exact LSE fallback; the threaded
    fallback is bitwise the sequential one (columns are independent)."""
    a, b, Cm = O.gen_config(1, 50, 60, 3)
    p = O.Problem(a, b, Cm, cost_div=1e-3)
    v = np.zeros(60)
    v[::7] = -900.0
    v = v - v.mean()
    with O.threads(1):
        r1 = O.row_solve_marginals_log(p, v)
    with O.threads(4):
        r2 = O.row_solve_marginals_log(p, v)
    for x1, x2 in zip(r1, r2):
        assert np.allclose(x1, x2, rtol=1e-15, atol=0)
