"""The C-ABI contract when called directly (no Python-side validation in
front): every entry point returns a status code and sets otg_last_error()
instead of crashing or throwing across the boundary ("No
exception crosses the ABI"), for NULL handles / outputs, invalid configs and
non-finite inputs."""
import ctypes as C

import numpy as np
import pytest

from paper_2605_30267_b200 import _capi, ot

pytestmark = pytest.mark.gpu

OK, E_OT, E_DOMAIN, E_DIMENSION, E_TOO_LARGE = 0, 1, 3, 7, 8


def lib():
    return ot._lib()


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def handle():
    a, b, Cm = ot.synthetic_instance(6, 5, 3)
    return ot.rescale_problem(ot.make_problem(a, b, Cm, 0.3))


def solve_cfg(**kw):
    c = _capi.SolveConfigC()
    c.tol_l1, c.max_iters, c.record_trace, c.trace_stride = 1e-8, 100, 0, 1
    c.reference_v, c.reference_f = None, 0.0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_null_handle_and_outputs():
    res = _capi.SolveResultC()
    v0 = np.zeros(5)
    rc = lib().otg_sinkhorn_solve(None, ptr(v0), C.byref(solve_cfg()), C.byref(res))
    assert rc == E_DIMENSION and b"NULL" in lib().otg_last_error()
    p = handle()
    H = p.handle
    rc = lib().otg_eval_normalized_step(H.raw, None, None)  # the point is required
    assert rc == E_DIMENSION and b"NULL" in lib().otg_last_error()
    assert lib().otg_eval_normalized_step(H.raw, ptr(v0), None) == OK  # outputs optional
    rc = lib().otg_hessian_f(H.raw, ptr(v0), None)
    assert rc == E_DIMENSION


@pytest.mark.parametrize("field,value", [("tol_l1", 0.0), ("tol_l1", -1.0), ("tol_l1", float("nan")),
                                         ("max_iters", 0), ("trace_stride", 0)])
def test_invalid_solve_config(field, value):  # sinkhorn.cpp:29-33
    p = handle()
    res = _capi.SolveResultC()
    v0 = np.zeros(5)
    cfg = solve_cfg(**{field: value})
    if field == "trace_stride":
        cfg.record_trace = 1
    rc = lib().otg_sinkhorn_solve(p.handle.raw, ptr(v0), C.byref(cfg), C.byref(res))
    assert rc == E_OT, lib().otg_last_error()
    # the handle stays usable after a refused call
    rc = lib().otg_sinkhorn_solve(p.handle.raw, ptr(v0), C.byref(solve_cfg()), C.byref(res))
    assert rc == OK and res.converged


def test_non_finite_point_is_refused():  # dual.cpp:13-18
    p = handle()
    v = np.zeros(5)
    v[2] = np.nan
    out = _capi.StepEvalC()
    bufs = [np.empty(5), np.empty(6), np.empty(5)]
    out.v_next, out.u, out.grad = ptr(bufs[0]), ptr(bufs[1]), ptr(bufs[2])
    rc = lib().otg_eval_normalized_step(p.handle.raw, ptr(v), C.byref(out))
    assert rc != OK and lib().otg_last_error()


def test_homotopy_config_refusals():  # accel.cpp:234-250
    p = handle()
    res = _capi.SolveResultC()
    for mu0, m0, max_outer in ((1.0, 4, 64), (0.0, 4, 64), (0.5, 0, 64), (0.5, 4, 0)):
        c = _capi.HomotopyConfigC()
        c.mu0, c.m0, c.max_outer, c.tol_l1, c.max_total_inner = mu0, m0, max_outer, 1e-8, 100
        c.rescale_w_across_stages, c.record_trace, c.trace_stride = 0, 0, 1
        rc = lib().otg_homotopy_solve(p.handle.raw, C.byref(c), None, C.byref(res))
        assert rc == E_OT, (mu0, m0, max_outer, lib().otg_last_error())
