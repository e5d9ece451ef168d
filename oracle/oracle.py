"""ctypes front-end to the CPU oracle (oracle/otoracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
timed CPU baseline, never as part of the product path.  The oracle restates
the reference's fp64 single-threaded solver (see otoracle.h for the file:line
map) and is pinned by the reference's known-answer tests
(tests/golden/kat.json, tests/test_oracle_kat.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

TRACE_COLS = 15
TRACE_FIELDS = ("iter", "wall_time_s", "marginal_violation_l1", "grad_f_l1", "reduced_f",
                "mu", "alpha", "cond1_lhs", "cond1_rhs", "cond2_lhs", "cond2_rhs",
                "metric_drift_inf")

_ERR_NAMES = {1: "OtError", 2: "PotentialOverflow", 3: "DomainViolation", 4: "GaugeViolation",
              5: "InvalidMarginals", 6: "NonPositiveEntry", 7: "DimensionMismatch",
              8: "DimensionTooLarge", 9: "OracleUnavailable", 10: "DegenerateColumn"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = _ERR_NAMES.get(code, str(code))


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("a", C.c_void_p), ("b", C.c_void_p),
                ("C64", C.c_void_p), ("C32", C.c_void_p), ("ldc", C.c_int64),
                ("cost_div", C.c_double)]


class _SolveConfig(C.Structure):
    _fields_ = [("tol_l1", C.c_double), ("max_iters", C.c_int64), ("record_trace", C.c_int),
                ("trace_stride", C.c_int64)]


class _HomotopyConfig(C.Structure):
    _fields_ = [("mu0", C.c_double), ("m0", C.c_int64), ("max_outer", C.c_int64),
                ("tol_l1", C.c_double), ("max_total_inner", C.c_int64),
                ("rescale_w_across_stages", C.c_int), ("record_trace", C.c_int),
                ("trace_stride", C.c_int64), ("stability", C.c_int)]


class _SolveResult(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int64), ("evaluations", C.c_int64),
                ("outer_stages", C.c_int64), ("final_violation", C.c_double),
                ("final_reduced_f", C.c_double), ("max_v_inf", C.c_double),
                ("conditions_checked", C.c_int64), ("conditions_held", C.c_int64),
                ("trace_len", C.c_int64), ("r_max_x", C.c_double), ("r_max_y", C.c_double)]


class _Reference(C.Structure):  # ReferenceSolution (diag.hpp:46-49)
    _fields_ = [("v_star", C.c_void_p), ("f_star", C.c_double)]


def _ref(reference):
    """reference = (v_star, f_star) or None -> (ctypes struct or None, keep-alive)."""
    if reference is None:
        return None, None
    vs = _f64(reference[0])
    return _Reference(vs.ctypes.data_as(C.c_void_p), float(reference[1])), vs


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_rng_next_u64.restype = C.c_uint64
        _lib.orc_rng_next_double.restype = C.c_double
        _lib.orc_rng_next_below.restype = C.c_uint64
        _lib.orc_rng_next_below.argtypes = [C.c_void_p, C.c_uint64]
        _lib.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        _lib.orc_homotopy_rate_constant.restype = C.c_double
        _lib.orc_homotopy_rate_constant.argtypes = [C.c_double] * 3
        _lib.orc_sqeuclid_max.restype = C.c_double
        _lib.orc_sqeuclid_max.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                          C.c_int64, C.c_int]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


class Rng:
    """rng.hpp:11-58 restated (xoshiro256++ / splitmix64)."""

    def __init__(self, seed: int):
        self._st = (C.c_uint64 * 4)()
        lib().orc_rng_seed(self._st, C.c_uint64(seed))

    def next_u64(self) -> int:
        return lib().orc_rng_next_u64(self._st)

    def next_double(self) -> float:
        return lib().orc_rng_next_double(self._st)

    def next_below(self, bound: int) -> int:
        return lib().orc_rng_next_below(self._st, C.c_uint64(bound))


@dataclass
class Problem:
    """A rescaled instance as the solvers see it: C' = C / cost_div."""
    a: np.ndarray
    b: np.ndarray
    C: np.ndarray  # (n, m) float64 or float32
    cost_div: float = 1.0
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        self.a = _f64(self.a)
        self.b = _f64(self.b)
        if self.C.dtype == np.float32:
            self.C = np.ascontiguousarray(self.C)
        else:
            self.C = _f64(self.C)
        self._s = _Problem(self.a.size, self.b.size, _p(self.a), _p(self.b),
                           _p(self.C) if self.C.dtype == np.float64 else None,
                           _p(self.C) if self.C.dtype == np.float32 else None,
                           self.C.shape[1], float(self.cost_div))

    @property
    def n(self):
        return self.a.size

    @property
    def m(self):
        return self.b.size

    @property
    def ref(self):
        return C.byref(self._s)


@dataclass
class Result:
    converged: bool
    iterations: int
    evaluations: int
    outer_stages: int
    final_violation: float
    final_reduced_f: float
    max_v_inf: float
    conditions_checked: int
    conditions_held: int
    u: np.ndarray = None
    v: np.ndarray = None
    w: np.ndarray = None
    trace: np.ndarray = None
    boundaries: np.ndarray = None
    r_max_x: float = 0.0
    r_max_y: float = 0.0

    @property
    def r_hat(self) -> float:  # RadiusTracker::r_hat (diag.hpp:130)
        return max(self.r_max_x, self.r_max_y)


def _result(r: _SolveResult, **kw) -> Result:
    return Result(bool(r.converged), r.iterations, r.evaluations, r.outer_stages,
                  r.final_violation, r.final_reduced_f, r.max_v_inf, r.conditions_checked,
                  r.conditions_held, r_max_x=r.r_max_x, r_max_y=r.r_max_y, **kw)


def synthetic_instance(n: int, m: int, seed: int):
    a, b, Cm = np.empty(n), np.empty(m), np.empty((n, m))
    _check(lib().orc_synthetic_instance(C.c_int64(n), C.c_int64(m), C.c_uint64(seed),
                                        _p(a), _p(b), _p(Cm)))
    return a, b, Cm


def synthetic_rescaled(n, m, seed, eps) -> Problem:
    """helpers.hpp:30-33: rescale_problem(with_epsilon(synthetic_instance(...), eps))."""
    a, b, Cm = synthetic_instance(n, m, seed)
    return Problem(a, b, Cm / eps)


def cost_sqeuclidean(x, y):
    x, y = _f64(x), _f64(y)
    n, d = x.shape
    m = y.shape[0]
    Cm = np.empty((n, m))
    lo, hi = C.c_double(), C.c_double()
    _check(lib().orc_cost_sqeuclidean(_p(x), _p(y), C.c_int64(n), C.c_int64(m), C.c_int64(d),
                                      _p(Cm), C.byref(lo), C.byref(hi)))
    return Cm, lo.value, hi.value


def cost_cosine(x, y, norm: int = 0):
    x, y = _f64(x), _f64(y)
    n, d = x.shape
    m = y.shape[0]
    Cm = np.empty((n, m))
    lo, hi = C.c_double(), C.c_double()
    _check(lib().orc_cost_cosine(_p(x), _p(y), C.c_int64(n), C.c_int64(m), C.c_int64(d),
                                 C.c_int(norm), _p(Cm), C.byref(lo), C.byref(hi)))
    return Cm, lo.value, hi.value


def validate_problem(p: Problem, epsilon: float = 1.0):
    _check(lib().orc_validate_problem(p.ref, C.c_double(epsilon)))


def row_solve_marginals(p: Problem, v):
    v = _f64(v)
    u, col = np.empty(p.n), np.empty(p.m)
    _check(lib().orc_row_solve_marginals(p.ref, _p(v), _p(u), _p(col)))
    return u, col


def row_solve_marginals_log(p: Problem, v):
    v = _f64(v)
    u, col, cl = np.empty(p.n), np.empty(p.m), np.empty(p.m)
    _check(lib().orc_row_solve_marginals_log(p.ref, _p(v), _p(u), _p(col), _p(cl)))
    return u, col, cl


def row_solve(p, v):
    return row_solve_marginals(p, v)[0]


def grad_f(p, v):
    return row_solve_marginals(p, v)[1] - p.b


def reduced_f(p, v):
    v = _f64(v)
    u = row_solve(p, v)
    return 1.0 - u.dot(p.a) - v.dot(p.b)


def dual_F(p: Problem, u, v) -> float:
    out = C.c_double()
    u, v = _f64(u), _f64(v)
    _check(lib().orc_dual_F(p.ref, _p(u), _p(v), C.byref(out)))
    return out.value


def hessian_f(p: Problem, v):
    v = _f64(v)
    H = np.empty((p.m, p.m))
    _check(lib().orc_hessian_f(p.ref, _p(v), _p(H)))
    return H


def eval_normalized_step(p: Problem, v):
    v = _f64(v)
    vn, u, g = np.empty(p.m), np.empty(p.n), np.empty(p.m)
    gl, f = C.c_double(), C.c_double()
    _check(lib().orc_eval_normalized_step(p.ref, _p(v), _p(vn), _p(u), _p(g), C.byref(gl),
                                          C.byref(f)))
    return dict(v_next=vn, u=u, grad=g, grad_l1=gl.value, f_value=f.value)


def normalized_sinkhorn_map(p, v):
    v = _f64(v)
    if abs(v.sum()) > 1e-9:
        raise OracleError(4, "normalized map fed an off-gauge v")
    return eval_normalized_step(p, v)["v_next"]


def sinkhorn_v_step(p, v):
    v = _f64(v)
    _, _, cl = row_solve_marginals_log(p, v)
    return v + (np.log(p.b) - cl)


def plan_stats(p: Problem, u, v, eps_ratio: float = 1.0):
    u, v = _f64(u), _f64(v)
    rs, cs = np.empty(p.n), np.empty(p.m)
    viol, cost = C.c_double(), C.c_double()
    _check(lib().orc_plan_stats(p.ref, _p(u), _p(v), C.c_double(eps_ratio), _p(rs), _p(cs),
                                C.byref(viol), C.byref(cost)))
    return dict(row_sums=rs, col_sums=cs, marginal_violation_l1=viol.value,
                primal_cost=cost.value)


def entropic_objective(p: Problem, u, v, epsilon: float = 1.0) -> float:
    out = C.c_double()
    u, v = _f64(u), _f64(v)
    _check(lib().orc_entropic_objective(p.ref, _p(u), _p(v), C.c_double(epsilon), C.byref(out)))
    return out.value


def _trace_buf(record, cap):
    return np.full((cap, TRACE_COLS), np.nan) if record else None


def sinkhorn_solve(p: Problem, v0=None, tol_l1=1e-6, max_iters=200000, record_trace=False,
                   trace_stride=1, trace_cap=100000) -> Result:
    v0 = np.zeros(p.m) if v0 is None else _f64(v0)
    cfg = _SolveConfig(tol_l1, max_iters, int(record_trace), trace_stride)
    r = _SolveResult()
    u, v = np.empty(p.n), np.empty(p.m)
    tr = _trace_buf(record_trace, trace_cap)
    _check(lib().orc_sinkhorn_solve(p.ref, _p(v0), C.byref(cfg), C.byref(r), _p(u), _p(v),
                                    _p(tr), C.c_int64(trace_cap if record_trace else 0)))
    return _result(r, u=u, v=v, trace=None if tr is None else tr[:min(r.trace_len, trace_cap)])


def acc_solve(p: Problem, v0=None, mu=0.5, tol_l1=1e-6, max_iters=200000, record_trace=False,
              trace_stride=1, trace_cap=100000, reference=None) -> Result:
    v0 = np.zeros(p.m) if v0 is None else _f64(v0)
    cfg = _SolveConfig(tol_l1, max_iters, int(record_trace), trace_stride)
    r = _SolveResult()
    u, v = np.empty(p.n), np.empty(p.m)
    tr = _trace_buf(record_trace, trace_cap)
    ref, keep = _ref(reference)
    _check(lib().orc_acc_solve(p.ref, _p(v0), C.c_double(mu), C.byref(cfg), C.byref(r), _p(u),
                               _p(v), _p(tr), C.c_int64(trace_cap if record_trace else 0),
                               None if ref is None else C.byref(ref)))
    return _result(r, u=u, v=v, trace=None if tr is None else tr[:min(r.trace_len, trace_cap)])


def acc_step(p: Problem, x, w, mu, Sx=None):
    x, w = _f64(x), _f64(w)
    Sx = None if Sx is None else _f64(Sx)
    xo, wo, so = np.empty(p.m), np.empty(p.m), np.empty(p.m)
    ev = C.c_int64(0)
    _check(lib().orc_acc_step(p.ref, _p(x), _p(w), _p(Sx), C.c_double(mu), _p(xo), _p(wo),
                              _p(so), C.byref(ev)))
    return xo, wo, so, ev.value


def acc_run(p: Problem, x0, w0, mu, msteps, record_trace=False, trace_stride=1, stability=False,
            trace_cap=100000, reference=None) -> Result:
    x0, w0 = _f64(x0), _f64(w0)
    r = _SolveResult()
    x, w = np.empty(p.m), np.empty(p.m)
    tr = _trace_buf(record_trace, trace_cap)
    ref, keep = _ref(reference)
    _check(lib().orc_acc_run(p.ref, _p(x0), _p(w0), C.c_double(mu), C.c_int64(msteps),
                             C.c_int(int(record_trace)), C.c_int64(trace_stride),
                             C.c_int(int(stability)), C.byref(r), _p(x), _p(w), _p(tr),
                             C.c_int64(trace_cap if record_trace else 0),
                             None if ref is None else C.byref(ref)))
    return _result(r, v=x, w=w, trace=None if tr is None else tr[:min(r.trace_len, trace_cap)])


def homotopy_solve(p: Problem, mu0=0.5, m0=4, max_outer=64, tol_l1=1e-6,
                   max_total_inner=20000000, rescale_w_across_stages=False, record_trace=False,
                   trace_stride=1, stability=False, trace_cap=100000, bcap=256,
                   reference=None) -> Result:
    cfg = _HomotopyConfig(mu0, m0, max_outer, tol_l1, max_total_inner,
                          int(rescale_w_across_stages), int(record_trace), trace_stride,
                          int(stability))
    r = _SolveResult()
    u, v = np.empty(p.n), np.empty(p.m)
    bd = np.full((bcap, 5), np.nan)
    tr = _trace_buf(record_trace, trace_cap)
    ref, keep = _ref(reference)
    _check(lib().orc_homotopy_solve(p.ref, C.byref(cfg), C.byref(r), _p(u), _p(v), _p(bd),
                                    C.c_int64(bcap), _p(tr),
                                    C.c_int64(trace_cap if record_trace else 0),
                                    None if ref is None else C.byref(ref)))
    return _result(r, u=u, v=v, boundaries=bd[:min(r.outer_stages, bcap)],
                   trace=None if tr is None else tr[:min(r.trace_len, trace_cap)])


def lyapunov_energy_from_parts(b, f_x, grad_x, y, mu, reference) -> float:
    """diag.cpp:76-88."""
    b, g, y = _f64(b), _f64(grad_x), _f64(y)
    ref, keep = _ref(reference)
    out = C.c_double(0.0)
    _check(lib().orc_lyapunov_energy(_p(b), C.c_int64(b.size), C.c_double(f_x), _p(g), _p(y),
                                     C.c_double(mu), C.byref(ref), C.byref(out)))
    return out.value


def reference_solve(p: Problem, tol=1e-12, max_iters=4000000):
    """helpers.hpp:37-45: the ReferenceSolution of the reference's tests."""
    r = sinkhorn_solve(p, np.zeros(p.m), tol_l1=tol, max_iters=max_iters)
    return r.v, r.final_reduced_f


def homotopy_rate_constant(mu0, r_hat, l_f=1.0) -> float:
    return lib().orc_homotopy_rate_constant(mu0, r_hat, l_f)


# mirror helpers -----------------------------------------------------------
def _vec_call(fn, b, x):
    b, x = _f64(b), _f64(x)
    out = np.empty(b.size)
    _check(fn(_p(b), C.c_int64(b.size), _p(x), _p(out)))
    return out


def grad_phi(b, v):
    return _vec_call(lib().orc_grad_phi, b, v)


def grad_phi_star(b, xi):
    return _vec_call(lib().orc_grad_phi_star, b, xi)


def metric_D(b, z):
    return _vec_call(lib().orc_metric_D, b, z)


def phi_star(b, xi) -> float:
    b, xi = _f64(b), _f64(xi)
    out = C.c_double()
    _check(lib().orc_phi_star(_p(b), C.c_int64(b.size), _p(xi), C.byref(out)))
    return out.value


def bregman_phi_star_from_zero(b, eta) -> float:
    b, eta = _f64(b), _f64(eta)
    out = C.c_double()
    _check(lib().orc_bregman_phi_star_from_zero(_p(b), C.c_int64(b.size), _p(eta),
                                                C.byref(out)))
    return out.value


def project_zero_sum(x):
    x = _f64(x)
    out = np.empty(x.size)
    lib().orc_project_zero_sum(_p(x), C.c_int64(x.size), _p(out))
    return out


def stability_conditions_from_grads(b, gk, gk1, xk, xk1, yk, yk1, alpha):
    arrs = [_f64(t) for t in (b, gk, gk1, xk, xk1, yk, yk1)]
    out = (C.c_double * 4)()
    both, skipped, drift = C.c_int(), C.c_int(), C.c_double()
    _check(lib().orc_stability_conditions_from_grads(
        _p(arrs[0]), C.c_int64(arrs[0].size), *[_p(t) for t in arrs[1:]], C.c_double(alpha),
        out, C.byref(both), C.byref(skipped), C.byref(drift)))
    return dict(c1_lhs=out[0], c1_rhs=out[1], c2_lhs=out[2], c2_rhs=out[3],
                both_hold=bool(both.value), skipped=bool(skipped.value), drift=drift.value)


def sweep_rows_mt(p: Problem, v, row0, row1, nthreads):
    v = _f64(v)
    u = np.empty(row1 - row0)
    col = np.empty(p.m)
    _check(lib().orc_sweep_rows_mt(p.ref, _p(v), C.c_int64(row0), C.c_int64(row1),
                                   C.c_int(nthreads), _p(u), _p(col)))
    return u, col


def cost_sqeuclid_f32(x, y):
    """fp32 on-the-fly cost (config 5 definition, otoracle.h)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    Cm = np.empty((x.shape[0], y.shape[0]), dtype=np.float32)
    lib().orc_cost_sqeuclid_f32(_p(x), _p(y), C.c_int64(x.shape[0]), C.c_int64(y.shape[0]),
                                C.c_int64(x.shape[1]), _p(Cm))
    return Cm


def sqeuclid_max(x, y, threads=1) -> float:
    x, y = _f64(x), _f64(y)
    return lib().orc_sqeuclid_max(_p(x), _p(y), x.shape[0], y.shape[0], x.shape[1], threads)


# plan consumers (pipelines.cpp:58-145) on the plan of plan_from_potentials ---
def barycentric_projection(p: Problem, u, v, src):
    src = np.ascontiguousarray(src, dtype=np.float64)
    d = src.shape[1]
    out = np.empty((p.m, d))
    _check(lib().orc_barycentric_projection(p.ref, _p(_f64(u)), _p(_f64(v)), _p(src), C.c_int(d),
                                            _p(out)))
    return out


def predict_translations(p: Problem, u, v):
    out = np.empty(p.n, dtype=np.int32)
    _check(lib().orc_predict_translations(p.ref, _p(_f64(u)), _p(_f64(v)), _p(out)))
    return out


def plan_topk(p: Problem, u, v, rows, k):
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.empty((len(rows), k), dtype=np.int32)
    _check(lib().orc_plan_topk(p.ref, _p(_f64(u)), _p(_f64(v)), _p(rows), C.c_int64(len(rows)),
                               C.c_int(k), _p(out)))
    return out


def nn_assign(q, ref):
    q = np.ascontiguousarray(q, dtype=np.float64)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    out = np.empty(q.shape[0], dtype=np.int32)
    lib().orc_nn_assign(_p(q), C.c_int64(q.shape[0]), _p(ref), C.c_int64(ref.shape[0]),
                        C.c_int(q.shape[1]), _p(out))
    return out


# fixtures (helpers.hpp:14-27) ----------------------------------------------
def skewed_2x2() -> Problem:
    return Problem(np.array([0.7, 0.3]), np.array([0.5, 0.5]), np.array([[0.0, 1.0], [1.0, 0.0]]))


def flat_2x2() -> Problem:
    return Problem(np.array([0.5, 0.5]), np.array([0.5, 0.5]), np.zeros((2, 2)))


def random_zero_sum(rng: Rng, m: int, scale: float) -> np.ndarray:
    """helpers.hpp:48-52."""
    v = np.array([scale * (2.0 * rng.next_double() - 1.0) for _ in range(m)])
    return project_zero_sum(v)


# ---- threads, config generators, device-equivalent fp32 cost ----
def set_threads(nthreads: int) -> None:
    """Worker threads of the oracle's O(nm) loops (1 = the reference's single
    thread); deterministic for a given count."""
    lib().orc_set_threads(C.c_int(int(nthreads)))


def get_threads() -> int:
    return int(lib().orc_get_threads())


class threads:
    """with O.threads(8): ... — scoped worker count."""

    def __init__(self, n: int):
        self.n = n

    def __enter__(self):
        self.prev = get_threads()
        set_threads(self.n)
        return self

    def __exit__(self, *exc):
        set_threads(self.prev)


def gen_config(cfg: int, n: int, m: int, seed: int):
    """BASELINE config inputs: cfg 1 -> (a, b, C); cfg 2/3/5 -> (x, y)."""
    if cfg == 1:
        a, b, Cm = np.empty(n), np.empty(m), np.empty((n, m))
        _check(lib().orc_gen_config(C.c_int(1), C.c_int64(n), C.c_int64(m), C.c_uint64(seed),
                                    _p(a), _p(b), _p(Cm)))
        return a, b, Cm
    d = {2: 2, 3: 3, 5: 3}.get(cfg)
    if d is None:
        raise OracleError(1, "cfg must be 1, 2, 3 or 5")
    x, y = np.empty((n, d)), np.empty((m, d))
    _check(lib().orc_gen_config(C.c_int(cfg), C.c_int64(n), C.c_int64(m), C.c_uint64(seed),
                                _p(x), _p(y), None))
    return x, y


def gen_config4(count: int, seed: int, d: int = 768):
    n = np.empty(count, dtype=np.int32)
    m = np.empty(count, dtype=np.int32)
    _check(lib().orc_gen_config4(C.c_int64(count), C.c_uint64(seed), C.c_int64(d), _p(n), _p(m),
                                 None, None))
    x = np.empty((int(n.sum()), d), dtype=np.float32)
    y = np.empty((int(m.sum()), d), dtype=np.float32)
    _check(lib().orc_gen_config4(C.c_int64(count), C.c_uint64(seed), C.c_int64(d), _p(n), _p(m),
                                 _p(x), _p(y)))
    return n, m, x, y


def cost_sqeuclid_max_f32(x, y, threads: int = 1, ldc: int = None):
    """The fp32 cost a points instance stores on the device (SQEUCLID, NORM_MAX,
    storage F32): fl32(sum_k (x_ik - y_jk)^2 / max).  Returns (C, raw_max)."""
    x, y = _f64(x), _f64(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    ldc = m if ldc is None else ldc
    Cm = np.empty((n, ldc), dtype=np.float32)
    mx = C.c_double()
    _check(lib().orc_cost_sqeuclid_max_f32(_p(x), _p(y), C.c_int64(n), C.c_int64(m), C.c_int64(d),
                                           C.c_int64(ldc), C.c_int(threads), _p(Cm),
                                           C.byref(mx)))
    return (Cm if ldc == m else Cm[:, :m]), mx.value
