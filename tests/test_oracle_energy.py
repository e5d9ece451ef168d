"""Energy / radius instrumentation (diag.cpp:76-105, 206-215; accel.cpp:38-114)
in the CPU oracle, pinned by the reference's own checks (test_diag.cpp:85-131,
test_accel.cpp:272-348): zero at the optimum, the mu = 0 value gap, the
parts form, the rejected reference, nonnegativity along runs, the radius
bound r_hat, the rate constant, and the geometric single-stage decay."""
import math

import numpy as np
import pytest

from oracle import oracle as O


def skewed():
    return O.skewed_2x2()


def test_energy_zero_at_the_anchored_optimum():  # test_diag.cpp:88-92
    p = skewed()
    vs, fs = O.reference_solve(p, 1e-13)
    ev = O.eval_normalized_step(p, vs)
    for mu in (0.5, 0.0):
        e = O.lyapunov_energy_from_parts(p.b, ev["f_value"], ev["grad"], vs, mu, (vs, fs))
        assert abs(e) <= 1e-9


def test_energy_mu0_is_value_gap_and_manual_assembly():  # test_diag.cpp:93-105
    p = skewed()
    vs, fs = O.reference_solve(p, 1e-13)
    v = np.zeros(2)
    ev = O.eval_normalized_step(p, v)
    e0 = O.lyapunov_energy_from_parts(p.b, ev["f_value"], ev["grad"], v, 0.0, (vs, fs))
    assert e0 == pytest.approx(ev["f_value"] - fs, rel=1e-13)
    g = ev["grad"]
    z = np.log1p(g / p.b)
    D = p.b * np.expm1(z) / z
    expect = ev["f_value"] - fs + 0.25 * np.sum(D * (v - vs) ** 2)
    e = O.lyapunov_energy_from_parts(p.b, ev["f_value"], g, v, 0.5, (vs, fs))
    assert e == pytest.approx(expect, rel=1e-13)


def test_energy_rejects_a_reference_above_f():  # test_diag.cpp:114-117
    p = skewed()
    vs, fs = O.reference_solve(p, 1e-13)
    ev = O.eval_normalized_step(p, np.zeros(2))
    with pytest.raises(O.OracleError) as err:
        O.lyapunov_energy_from_parts(p.b, ev["f_value"], ev["grad"], np.zeros(2), 0.5,
                                     (vs, ev["f_value"] + 1.0))
    assert err.value.kind == "OtError"


def test_instrumented_homotopy_energies_radii_and_rate():  # test_accel.cpp:272-313
    p = O.synthetic_rescaled(8, 8, 27, 0.2)
    ref = O.reference_solve(p, 1e-12)
    h = O.homotopy_solve(p, tol_l1=1e-9, record_trace=True, stability=True, reference=ref)
    assert h.converged and h.r_hat > 0.0
    assert h.conditions_checked > 0 and h.conditions_held <= h.conditions_checked
    tr = h.trace
    assert np.all(np.isfinite(tr[:, 12])) and np.all(tr[:, 12] >= -1e-9)
    assert np.all(tr[:, 13] >= 0.0)
    assert np.all(tr[:, 13] <= h.r_hat + 1e-15) and np.all(tr[:, 14] <= h.r_hat + 1e-15)
    assert max(tr[:, 13].max(), tr[:, 14].max()) == pytest.approx(h.r_hat, rel=1e-12)
    assert np.all(np.isfinite(h.boundaries[:, 4])) and np.all(h.boundaries[:, 4] >= -1e-9)
    c = O.homotopy_rate_constant(0.5, h.r_hat)
    assert c == pytest.approx((math.sqrt(2) - 1) / ((math.sqrt(2) + 1) * math.log(2 * (h.r_hat ** 2 + 1))),
                              rel=1e-15)


def test_single_stage_energy_gap_decays_geometrically():  # test_accel.cpp:326-348
    p = O.synthetic_rescaled(5, 5, 66, 0.005)
    ref = O.reference_solve(p, 1e-13)
    mu = 0.2
    alpha = math.sqrt(2 * mu)
    run = O.acc_run(p, np.zeros(5), np.zeros(5), mu, 60, record_trace=True, reference=ref)
    e = run.trace[:, 12]
    floor = e.min()
    d0 = e[0] - floor
    assert d0 > 0
    ks, ls = [], []
    for k, ek in enumerate(e):
        d = ek - floor
        if d <= 1e-3 * d0:
            break
        ks.append(k)
        ls.append(math.log(d))
    assert len(ks) >= 8
    slope = np.polyfit(ks, ls, 1)[0]
    assert math.exp(slope) <= 1.0 / (1.0 + alpha) + 0.05
