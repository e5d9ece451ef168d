"""Host-side mirror of the reference solver API (otaccel ``ot::``) over libotg.

Same names, argument meaning and error behaviour as the reference C++ API
(paths under /root/reference/proj): include/ot/core.hpp, dual.hpp,
sinkhorn.hpp, accel.hpp, pipelines.hpp.  Every numerical call goes through
the C-ABI of include/otg.h into the sm_100a kernels; this module only holds
host bookkeeping (validation, result structs, the rescale fold).  There is no
CPU fallback: without libotg.so or a CUDA device the calls raise.

Rescaling.  As in the reference, solvers run on the instance's stored cost
treated as already divided by epsilon (dual.hpp:9-13); ``rescale_problem``
(core.cpp:42-49) returns a problem whose cost is C / epsilon.  Here the
division is not applied to a host copy: it is recorded in ``cost_div`` and
folded into the device upload (fp64: the same IEEE division on the device;
fp32: multiplication by 1/epsilon on load).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi

# --------------------------------------------------------------- errors ----


class OtError(RuntimeError):
    """types.hpp:21-23."""


class PotentialOverflow(OtError):
    pass


class DomainViolation(OtError):
    pass


class GaugeViolation(OtError):
    pass


class InvalidMarginals(OtError):
    pass


class NonPositiveEntry(OtError):
    pass


class DimensionMismatch(OtError):
    pass


class DimensionTooLarge(OtError):
    pass


class DegenerateColumn(OtError):
    pass


class MalformedLine(OtError):
    pass


class IoError(OtError):
    pass


class DeviceError(OtError):
    """CUDA / NCCL / allocation failures of the device path (no reference analogue)."""


class Unsupported(DeviceError):
    pass


_ERRORS = {1: OtError, 2: PotentialOverflow, 3: DomainViolation, 4: GaugeViolation,
           5: InvalidMarginals, 6: NonPositiveEntry, 7: DimensionMismatch,
           8: DimensionTooLarge, 9: DegenerateColumn, 20: DeviceError, 21: DeviceError, 22: DeviceError,
           23: Unsupported}


def _lib():
    return _capi.load()


def _check(rc: int):
    if rc != 0:
        msg = _lib().otg_last_error().decode()
        raise _ERRORS.get(rc, OtError)(msg)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


LOG2E = 1.4426950408889634074  # log2(e), the double of common.cuh kLog2e
STORAGE = {"f64": 0, "f32": 1, "on_the_fly": 2}
NORM = {"none": 0, "max": 1, "minmax": 2, "halfrange": 3}
COST = {"sqeuclidean": 0, "cosine": 1}

# --------------------------------------------------------------- problem ---


def _validate(a, b, C_shape, epsilon, C_arr=None):
    """core.cpp:9-29 (host side, before any upload)."""
    n, m = a.size, b.size
    if n == 0 or m == 0:
        raise DimensionMismatch("empty marginal")
    if C_shape != (n, m):
        raise DimensionMismatch(f"cost is {C_shape[0]}x{C_shape[1]} but marginals are {n} and {m}")
    if not (epsilon > 0.0) or not math.isfinite(epsilon):
        raise OtError("epsilon must be positive and finite")
    if C_arr is not None and not np.all(np.isfinite(C_arr)):
        raise OtError("cost matrix has non-finite entries")
    for w in (a, b):
        if not (w.min() > 0.0):
            raise InvalidMarginals("marginals must be strictly positive")
        s = 0.0
        for x in w:  # sequential sum like the reference loop order
            s += x
        if abs(s - 1.0) > 1e-9:
            raise InvalidMarginals(f"marginal sums to {s:.17g}, expected 1")


class TransportProblem:
    """core.hpp:15-27.  Holds a, b, the stored cost and epsilon; the device
    copy (a libotg handle) is created lazily and cached.

    The cost the solvers see is ``C_stored / cost_div``.  Built from points
    (``from_points``) the cost exists only on the device.
    """

    def __init__(self, a, b, C=None, epsilon=1.0, epsilon_original=None, cost_div=1.0,
                 _points=None, _opts=None):
        self.a = _f64(a)
        self.b = _f64(b)
        self._C = None if C is None else (np.ascontiguousarray(C) if np.asarray(C).dtype == np.float32
                                          else _f64(C))
        self.epsilon = float(epsilon)
        self.epsilon_original = float(epsilon if epsilon_original is None else epsilon_original)
        self.cost_div = float(cost_div)
        self._points = _points
        self._opts = _opts
        self._handle = None

    # sizes (core.hpp:22-23)
    def n(self) -> int:
        return self.a.size

    def m(self) -> int:
        return self.b.size

    @property
    def C(self) -> np.ndarray:
        """The solver-unit cost C_stored / cost_div as a host array."""
        if self._C is None:
            raise DimensionMismatch("cost lives on the device only (built from points)")
        return self._C / self.cost_div if self.cost_div != 1.0 else self._C

    def original_cost(self) -> np.ndarray:  # core.hpp:26
        return self.C * (self.epsilon_original / self.epsilon)

    # device handle -----------------------------------------------------
    @property
    def handle(self):
        if self._handle is None:
            self._handle = _DeviceHandle.dense(self)
        return self._handle

    @classmethod
    def from_points(cls, a, b, x, y, epsilon, cost="sqeuclidean", norm="max", storage="f32",
                    device=0, world_size=1, rank=0, row_begin=0, row_end=None,
                    nccl_unique_id=None, virtual_shards=1, allreduce=None, sweep="auto"):
        """Rescaled instance whose cost is built on the device from points
        (cost_sqeuclid / cost_cosine, data.cpp:69-110, then rescale_problem).

        Row sharding (world_size > 1): the device handle holds rows
        [row_begin, row_end) of the sources; `x` may be those local rows
        (what the C-ABI takes, otg.h) or all n rows (sliced here).  a and b
        are always the full marginals."""
        a, b = _f64(a), _f64(b)
        x, y = _f64(x), _f64(y)
        if x.ndim != 2 or y.ndim != 2 or x.shape[1] != y.shape[1]:
            raise DimensionMismatch("point clouds have different dimensions")
        rb, re_ = row_begin, (a.size if row_end is None else row_end)
        if world_size > 1 and x.shape[0] == a.size:
            x_dev = np.ascontiguousarray(x[rb:re_])
        elif world_size > 1 and x.shape[0] == re_ - rb:
            x_dev = x
        else:
            x_dev = x
            _validate(a, b, (x.shape[0], y.shape[0]), epsilon)
        if y.shape[0] != b.size:
            raise DimensionMismatch("target points do not match b")
        _validate(a, b, (a.size, y.shape[0]), epsilon)
        p = cls(a, b, None, epsilon=1.0, epsilon_original=epsilon, cost_div=epsilon)
        p._points = (x_dev, y, COST[cost], NORM[norm], STORAGE[storage])
        p._opts = _device_opts(device, world_size, rank, row_begin, re_, nccl_unique_id,
                               virtual_shards, allreduce, sweep)
        p._handle = _DeviceHandle.points(p)
        return p

    def to_device(self, device=0, world_size=1, rank=0, row_begin=0, row_end=None,
                  nccl_unique_id=None, virtual_shards=1, allreduce=None, sweep="auto"):
        """Create the device handle now with explicit placement / sharding."""
        if self._handle is not None:
            self._handle.close()
        self._opts = _device_opts(device, world_size, rank, row_begin,
                                  self.n() if row_end is None else row_end, nccl_unique_id,
                                  virtual_shards, allreduce, sweep)
        self._handle = (_DeviceHandle.points(self) if self._points is not None
                        else _DeviceHandle.dense(self))
        return self

    def stored_cost(self, row0=0, nrows=None) -> np.ndarray:
        """Copy of the device-resident (unscaled) cost rows, storage dtype."""
        return self.handle.get_cost(row0, nrows)

    def close(self):
        if self._handle is not None:
            self._handle.close()
            self._handle = None


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)


SWEEPS = {"auto": 0, "two_pass": 1, "single_pass": 2}


def _device_opts(device, world_size, rank, row_begin, row_end, nccl_unique_id, vshards,
                 allreduce=None, sweep="auto"):
    """otg_device_opts.  `allreduce`: a Python callable (buf: np.ndarray of
    float64, op: 0 SUM / 1 MAX) -> None reducing `buf` in place across the
    ranks (instead of NCCL; e.g. dist.gloo_allreduce()).  `sweep` (fp32 stored
    cost): "auto" (the single-HBM-pass sweep for long runs of row bands, else
    the two-pass kernels), "two_pass", or "single_pass" (whenever its column
    layout applies: tests and A/B)."""
    if sweep not in SWEEPS:
        raise OtError(f"unknown sweep '{sweep}'")
    o = _capi.DeviceOpts()
    o.sweep = SWEEPS[sweep]
    o.device = device
    o.world_size = world_size
    o.rank = rank
    o.row_begin = row_begin
    o.row_end = row_end
    o.virtual_shards = vshards
    if nccl_unique_id is not None:
        buf = C.create_string_buffer(bytes(nccl_unique_id), 128)
        o._uid = buf  # keep alive
        o.nccl_unique_id = C.cast(buf, C.c_void_p)
    if allreduce is not None:
        def _tramp(ptr, count, op, ctx, fn=allreduce):
            try:
                arr = np.ctypeslib.as_array((C.c_double * int(count)).from_address(ptr))
                fn(arr, int(op))
                return 0
            except Exception:  # reported by libotg as OTG_E_NCCL
                import traceback
                traceback.print_exc()
                return 1
        cb = ALLREDUCE_FN(_tramp)
        o._cb = cb  # keep alive as long as the options (and the handle holding them)
        o.allreduce = C.cast(cb, C.c_void_p)
    return o


class _DeviceHandle:
    def __init__(self, raw, info):
        self.raw = raw
        self.info = info

    @classmethod
    def dense(cls, p: TransportProblem):
        if p._C is None:
            raise DimensionMismatch("no cost matrix")
        Cs = p._C
        opts = p._opts
        if opts is not None and opts.world_size > 1:  # the handle's rows only (otg.h)
            Cs = Cs[opts.row_begin:opts.row_end]
        dtype = 1 if Cs.dtype == np.float32 else 0
        h = C.c_void_p()
        _check(_lib().otg_problem_create_dense(p.n(), p.m(), _ptr(p.a), _ptr(p.b), _ptr(Cs),
                                               dtype, Cs.shape[1], p.cost_div,
                                               None if opts is None else C.byref(opts),
                                               C.byref(h)))
        return cls._wrap(h)

    @classmethod
    def points(cls, p: TransportProblem):
        x, y, cost, norm, storage = p._points
        h = C.c_void_p()
        _check(_lib().otg_problem_create_points(
            p.n(), y.shape[0], x.shape[1], _ptr(p.a), _ptr(p.b), _ptr(x), _ptr(y), cost,
            norm, storage, p.cost_div, None if p._opts is None else C.byref(p._opts),
            C.byref(h)))
        return cls._wrap(h)

    @classmethod
    def _wrap(cls, h):
        info = _capi.ProblemInfo()
        _check(_lib().otg_problem_info_get(h, C.byref(info)))
        return cls(h, info)

    @property
    def n_local(self):
        return self.info.n_local

    def get_cost(self, row0=0, nrows=None):
        nrows = self.info.n_local - row0 if nrows is None else nrows
        dt = np.float64 if self.info.storage == 0 else np.float32
        out = np.empty((nrows, self.info.m), dtype=dt)
        _check(_lib().otg_problem_get_cost(self.raw, row0, nrows, _ptr(out)))
        return out

    def close(self):
        if self.raw:
            _lib().otg_problem_destroy(self.raw)
            self.raw = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_problem(a, b, C, epsilon) -> TransportProblem:
    """core.cpp:31-40."""
    p = TransportProblem(a, b, C, epsilon=epsilon)
    _validate(p.a, p.b, p._C.shape, p.epsilon, p._C)
    return p


def validate_problem(p: TransportProblem):
    _validate(p.a, p.b, (p.n(), p.m()) if p._C is None else p._C.shape, p.epsilon,
              p._C)


def rescale_problem(p: TransportProblem) -> TransportProblem:
    """core.cpp:42-49: C / epsilon with epsilon = 1; idempotent."""
    validate_problem(p)
    q = TransportProblem(p.a, p.b, p._C, epsilon=1.0, epsilon_original=p.epsilon_original,
                         cost_div=p.cost_div * p.epsilon)
    q._opts = p._opts
    return q


def with_epsilon(p: TransportProblem, epsilon) -> TransportProblem:
    """data.cpp:34-41."""
    if not (epsilon > 0.0) or not math.isfinite(epsilon):
        raise OtError("epsilon must be positive and finite")
    q = TransportProblem(p.a, p.b, p._C, epsilon=epsilon, epsilon_original=epsilon,
                         cost_div=p.cost_div)
    return q


# --------------------------------------------------------------- results ---


@dataclass
class DualPotentials:
    u: np.ndarray
    v: np.ndarray


@dataclass
class StepEval:  # sinkhorn.hpp:18-24
    v_next: np.ndarray
    u: np.ndarray
    grad: np.ndarray
    grad_l1: float
    f_value: float


@dataclass
class ReferenceSolution:  # diag.hpp:46-49 (the yardstick of the energy / radius columns)
    v_star: np.ndarray
    f_star: float


@dataclass
class SolveConfig:  # sinkhorn.hpp:29-39
    tol_l1: float = 1e-6
    max_iters: int = 200000
    record_trace: bool = False
    trace_stride: int = 1
    wall_clock: bool = True
    reference: Optional[ReferenceSolution] = None  # acc_solve energy / radius columns


@dataclass
class HomotopyConfig:  # accel.hpp:68-81
    mu0: float = 0.5
    m0: int = 4
    max_outer: int = 64
    tol_l1: float = 1e-6
    max_total_inner: int = 20000000
    rescale_w_across_stages: bool = False
    record_trace: bool = False
    trace_stride: int = 1
    wall_clock: bool = True


@dataclass
class AccelInstrumentation:  # accel.hpp:37-40
    reference: Optional[ReferenceSolution] = None  # energy + radius columns
    stability: bool = False                        # condition columns


TRACE_FIELDS = ("iter", "wall_time_s", "marginal_violation_l1", "grad_f_l1", "reduced_f", "mu",
                "alpha", "cond1_lhs", "cond1_rhs", "cond2_lhs", "cond2_rhs", "metric_drift_inf",
                "energy", "radius_x_d", "radius_y")


@dataclass
class TraceRecord:  # diag.hpp:15-33
    iter: int
    wall_time_s: float
    marginal_violation_l1: float
    grad_f_l1: float
    reduced_f: float
    mu: float
    alpha: float
    cond1_lhs: Optional[float] = None
    cond1_rhs: Optional[float] = None
    cond2_lhs: Optional[float] = None
    cond2_rhs: Optional[float] = None
    metric_drift_inf: Optional[float] = None
    energy: Optional[float] = None
    radius_x_d: Optional[float] = None
    radius_y: Optional[float] = None


@dataclass
class SolverTrace:
    records: List[TraceRecord] = field(default_factory=list)

    @staticmethod
    def csv_header() -> str:  # diag.cpp:32-36
        return ("iter,wall_time_s,marginal_violation_l1,grad_f_l1,reduced_f,mu,alpha,"
                "energy,cond1_lhs,cond1_rhs,cond2_lhs,cond2_rhs,metric_drift_inf,"
                "radius_x_d,radius_y")

    def to_csv(self) -> str:  # diag.cpp:38-54, %.17g
        def num(x):
            return "%.17g" % x

        def opt(x):
            return "" if x is None else num(x)
        lines = [self.csv_header()]
        for r in self.records:
            lines.append(",".join([str(r.iter), num(r.wall_time_s), num(r.marginal_violation_l1),
                                   num(r.grad_f_l1), num(r.reduced_f), num(r.mu), num(r.alpha),
                                   opt(r.energy), opt(r.cond1_lhs), opt(r.cond1_rhs),
                                   opt(r.cond2_lhs), opt(r.cond2_rhs), opt(r.metric_drift_inf),
                                   opt(r.radius_x_d), opt(r.radius_y)]))
        return "\n".join(lines) + "\n"

    def as_array(self) -> np.ndarray:
        return np.array([[np.nan if getattr(r, f) is None else getattr(r, f)
                          for f in TRACE_FIELDS] for r in self.records]).reshape(-1, len(TRACE_FIELDS))


@dataclass
class SolveResult:  # sinkhorn.hpp:44-54
    potentials: DualPotentials
    converged: bool = False
    iterations: int = 0
    evaluations: int = 0
    outer_stages: int = 0
    final_violation: float = 0.0
    final_reduced_f: float = 0.0
    max_v_inf: float = 0.0
    trace: SolverTrace = field(default_factory=SolverTrace)
    device_seconds: float = 0.0
    row_pass_seconds: float = 0.0
    col_pass_seconds: float = 0.0
    kernel_launches: int = 0
    row_redos: int = 0
    epilogue_seconds: float = 0.0
    fallback_columns: int = 0


@dataclass
class StageBoundary:  # accel.hpp:84-90
    stage: int
    mu: float
    alpha: float
    inner_before: int
    energy: Optional[float] = None  # E(x, w / alpha; mu) when a reference is given


@dataclass
class HomotopyResult:  # accel.hpp:92-99
    result: SolveResult
    boundaries: List[StageBoundary] = field(default_factory=list)
    conditions_checked: int = 0
    conditions_held: int = 0
    r_hat: float = 0.0   # max tracked radius, with a reference
    c_star: float = 0.0  # homotopy_rate_constant(mu0, r_hat), with a reference


@dataclass
class AccelState:  # accel.hpp:11-20 (final state of acc_run)
    x: np.ndarray
    w: np.ndarray
    mu: float
    alpha: float


@dataclass
class AccRun:  # accel.hpp:42-50
    state: AccelState
    evaluations: int = 0
    final_violation: float = 0.0
    trace: SolverTrace = field(default_factory=SolverTrace)
    conditions_checked: int = 0
    conditions_held: int = 0
    device_seconds: float = 0.0
    row_pass_seconds: float = 0.0
    col_pass_seconds: float = 0.0
    max_radius_x_d: float = 0.0  # RadiusTracker (diag.hpp:120-135), with a reference
    max_radius_y: float = 0.0


def _records(tr: np.ndarray, n: int) -> SolverTrace:
    out = SolverTrace()
    for row in tr[:n]:
        vals = [None if np.isnan(x) else float(x) for x in row]
        out.records.append(TraceRecord(int(vals[0]), *vals[1:7], *vals[7:15]))
    return out


def _instr_c(instr):
    """AccelInstrumentation -> (InstrC, keep-alive)."""
    ins = _capi.InstrC(0, None, 0.0)
    keep = None
    if instr is not None:
        ins.stability = int(bool(instr.stability))
        if instr.reference is not None:
            keep = _f64(instr.reference.v_star)
            ins.reference_v = _ptr(keep)
            ins.reference_f = float(instr.reference.f_star)
    return ins, keep


class _Res:
    """Owns the output buffers handed to otg_solve_result."""

    def __init__(self, h, record_trace, trace_cap, time_sweeps=False, boundaries_cap=0):
        self.r = _capi.SolveResultC()
        self.u = np.empty(h.n_local)
        self.v = np.empty(h.info.m)
        self.w = np.empty(h.info.m)
        self.r.u, self.r.v, self.r.w = _ptr(self.u), _ptr(self.v), _ptr(self.w)
        self.trace = np.full((trace_cap, _capi.TRACE_COLS), np.nan) if record_trace else None
        self.r.trace = _ptr(self.trace)
        self.r.trace_cap = trace_cap if record_trace else 0
        self.bounds = np.full((boundaries_cap, 5), np.nan) if boundaries_cap else None
        self.r.boundaries = _ptr(self.bounds)
        self.r.boundaries_cap = boundaries_cap
        self.r.time_sweeps = int(time_sweeps)

    def solve_result(self) -> SolveResult:
        r = self.r
        tr = _records(self.trace, min(r.trace_len, r.trace_cap)) if self.trace is not None else SolverTrace()
        return SolveResult(DualPotentials(self.u, self.v), bool(r.converged), r.iterations,
                           r.evaluations, r.outer_stages, r.final_violation, r.final_reduced_f,
                           r.max_v_inf, tr, r.device_seconds, r.row_pass_seconds,
                           r.col_pass_seconds, r.kernel_launches, r.row_redos,
                           r.epilogue_seconds, r.fallback_columns)


def _trace_cap(max_iters, stride):
    return int(min(max_iters // max(stride, 1) + 2, 1_000_000))


# ----------------------------------------------------------- dual.hpp ----


def row_solve_marginals(p: TransportProblem, v):
    """dual.cpp:29-42 -> (u, col_sums)."""
    h = p.handle
    v = _f64(v)
    if v.size != p.m():
        raise DimensionMismatch(f"v has size {v.size}, expected {p.m()}")
    u, col = np.empty(h.n_local), np.empty(p.m())
    _check(_lib().otg_row_solve_marginals(h.raw, _ptr(v), _ptr(u), _ptr(col)))
    return u, col


def row_solve_marginals_log(p: TransportProblem, v):
    """dual.cpp:44-70 -> (u, col_sums, col_log)."""
    h = p.handle
    v = _f64(v)
    if v.size != p.m():
        raise DimensionMismatch(f"v has size {v.size}, expected {p.m()}")
    u, col, cl = np.empty(h.n_local), np.empty(p.m()), np.empty(p.m())
    _check(_lib().otg_row_solve_marginals_log(h.raw, _ptr(v), _ptr(u), _ptr(col), _ptr(cl)))
    return u, col, cl


def row_solve(p, v):  # dual.cpp:80-86
    return row_solve_marginals(p, v)[0]


def grad_f(p, v):  # dual.cpp:110-116
    return row_solve_marginals(p, v)[1] - p.b


def reduced_f(p, v) -> float:  # dual.cpp:103-108
    v = _f64(v)
    u = row_solve(p, v)
    return 1.0 - u.dot(p.a) - v.dot(p.b)


def dual_F(p: TransportProblem, u, v) -> float:
    """dual.cpp:88-101: exp(LSE(u_i + v_j - C'_ij)) - <u, a> - <v, b>."""
    h = p.handle
    u, v = _f64(u), _f64(v)
    if u.size != h.n_local or v.size != p.m():
        raise DimensionMismatch(f"(u, v) sizes ({u.size}, {v.size}), expected ({h.n_local}, {p.m()})")
    out = C.c_double()
    _check(_lib().otg_dual_F(h.raw, _ptr(u), _ptr(v), C.byref(out)))
    return out.value


def hessian_f(p: TransportProblem, v) -> np.ndarray:
    """dual.cpp:118-136: diag(c(v)) - P^T diag(a)^-1 P, dense m x m (m <= 2000)."""
    h = p.handle
    v = _f64(v)
    if v.size != p.m():
        raise DimensionMismatch(f"v has size {v.size}, expected {p.m()}")
    H = np.empty((p.m(), p.m()))
    _check(_lib().otg_hessian_f(h.raw, _ptr(v), _ptr(H)))
    return H


# ------------------------------------------------------- sinkhorn.hpp ----


def eval_normalized_step(p: TransportProblem, v) -> StepEval:
    """sinkhorn.cpp:51-63."""
    h = p.handle
    v = _f64(v)
    if v.size != p.m():
        raise DimensionMismatch(f"v has size {v.size}, expected {p.m()}")
    out = _capi.StepEvalC()
    vn, u, g = np.empty(p.m()), np.empty(h.n_local), np.empty(p.m())
    out.v_next, out.u, out.grad = _ptr(vn), _ptr(u), _ptr(g)
    _check(_lib().otg_eval_normalized_step(h.raw, _ptr(v), C.byref(out)))
    return StepEval(vn, u, g, out.grad_l1, out.f_value)


def sinkhorn_v_step(p, v):  # sinkhorn.cpp:35-42
    v = _f64(v)
    _, _, cl = row_solve_marginals_log(p, v)
    if not np.all(np.isfinite(cl)):
        raise DomainViolation("column log-mass degenerated")
    return v + (np.log(p.b) - cl)


def normalized_sinkhorn_map(p, v):  # sinkhorn.cpp:44-49
    v = _f64(v)
    s = float(np.sum(v))
    if abs(s) > 1e-9:
        raise GaugeViolation(f"normalized map fed sum(v) = {s:.3g}")
    return eval_normalized_step(p, v).v_next


def _solve_cfg(cfg: SolveConfig):
    c = _capi.SolveConfigC()
    c.tol_l1, c.max_iters = cfg.tol_l1, cfg.max_iters
    c.record_trace, c.trace_stride = int(cfg.record_trace), cfg.trace_stride
    c._keep = None
    if cfg.reference is not None:
        c._keep = _f64(cfg.reference.v_star)
        c.reference_v = _ptr(c._keep)
        c.reference_f = float(cfg.reference.f_star)
    return c


def validate_solve_config(cfg: SolveConfig):  # sinkhorn.cpp:29-33
    if not (cfg.tol_l1 > 0.0):
        raise OtError("tol_l1 must be positive")
    if cfg.max_iters < 1:
        raise OtError("max_iters must be at least 1")
    if cfg.trace_stride < 1:
        raise OtError("trace_stride must be at least 1")


def sinkhorn_solve(p: TransportProblem, v0=None, cfg: SolveConfig = SolveConfig(),
                   time_sweeps=False) -> SolveResult:
    """sinkhorn.cpp:65-115."""
    validate_solve_config(cfg)
    h = p.handle
    v0 = np.zeros(p.m()) if v0 is None else _f64(v0)
    if v0.size != p.m():
        raise DimensionMismatch("v0 size does not match b")
    res = _Res(h, cfg.record_trace, _trace_cap(cfg.max_iters, cfg.trace_stride), time_sweeps)
    c = _solve_cfg(cfg)
    _check(_lib().otg_sinkhorn_solve(h.raw, _ptr(v0), C.byref(c), C.byref(res.r)))
    return res.solve_result()


# ---------------------------------------------------------- accel.hpp ----


def acc_solve(p: TransportProblem, v0=None, mu=0.5, cfg: SolveConfig = SolveConfig(),
              time_sweeps=False) -> SolveResult:
    """accel.cpp:200-232."""
    validate_solve_config(cfg)
    h = p.handle
    v0 = np.zeros(p.m()) if v0 is None else _f64(v0)
    if v0.size != p.m():
        raise DimensionMismatch("accelerated state size does not match b")
    res = _Res(h, cfg.record_trace, _trace_cap(cfg.max_iters, cfg.trace_stride), time_sweeps)
    c = _solve_cfg(cfg)
    _check(_lib().otg_acc_solve(h.raw, _ptr(v0), float(mu), C.byref(c), C.byref(res.r)))
    return res.solve_result()


def acc_run(p: TransportProblem, x0, w0, mu, m, record_trace=False, trace_stride=1,
            wall_clock=True, instr: Optional[AccelInstrumentation] = None,
            time_sweeps=False) -> AccRun:
    """accel.cpp:174-198: m accelerated steps, m + 1 evaluations."""
    h = p.handle
    x0, w0 = _f64(x0), _f64(w0)
    if x0.size != p.m() or w0.size != p.m():
        raise DimensionMismatch("accelerated state size does not match b")
    res = _Res(h, record_trace, _trace_cap(max(m, 1), trace_stride), time_sweeps)
    ins, keep = _instr_c(instr)
    _check(_lib().otg_acc_run(h.raw, _ptr(x0), _ptr(w0), float(mu), int(m), int(record_trace),
                              int(trace_stride), C.byref(ins), C.byref(res.r)))
    r = res.r
    sr = res.solve_result()
    return AccRun(AccelState(res.v, res.w, mu, math.sqrt(2.0 * mu)), r.evaluations,
                  r.final_violation, sr.trace, r.conditions_checked, r.conditions_held,
                  r.device_seconds, r.row_pass_seconds, r.col_pass_seconds, r.radius_x_max,
                  r.radius_y_max)


def homotopy_solve_instrumented(p: TransportProblem, cfg: HomotopyConfig = HomotopyConfig(),
                                instr: Optional[AccelInstrumentation] = None,
                                time_sweeps=False) -> HomotopyResult:
    """accel.cpp:234-301, with the stability and energy / radius instrumentation."""
    h = p.handle
    c = _capi.HomotopyConfigC(cfg.mu0, cfg.m0, cfg.max_outer, cfg.tol_l1, cfg.max_total_inner,
                              int(cfg.rescale_w_across_stages), int(cfg.record_trace),
                              cfg.trace_stride)
    ins, keep = _instr_c(instr)
    bcap = int(min(max(cfg.max_outer, 1), 4096))
    res = _Res(h, cfg.record_trace, _trace_cap(min(cfg.max_total_inner, 10_000_000), cfg.trace_stride),
               time_sweeps, boundaries_cap=bcap)
    _check(_lib().otg_homotopy_solve(h.raw, C.byref(c), C.byref(ins), C.byref(res.r)))
    sr = res.solve_result()
    nb = min(res.r.outer_stages, bcap)
    bounds = [StageBoundary(int(b[0]), float(b[1]), float(b[2]), int(b[3]),
                            None if np.isnan(b[4]) else float(b[4]))
              for b in res.bounds[:nb]]
    out = HomotopyResult(sr, bounds, res.r.conditions_checked, res.r.conditions_held)
    if instr is not None and instr.reference is not None:
        out.r_hat = max(res.r.radius_x_max, res.r.radius_y_max)
        out.c_star = homotopy_rate_constant(cfg.mu0, out.r_hat)
    return out


def homotopy_solve(p: TransportProblem, cfg: HomotopyConfig = HomotopyConfig(),
                   time_sweeps=False) -> SolveResult:
    """accel.cpp:303-305."""
    return homotopy_solve_instrumented(p, cfg, None, time_sweeps).result


def homotopy_rate_constant(mu0, r_hat, l_f=1.0) -> float:  # accel.cpp:307-311
    return (math.sqrt(2.0) - 1.0) / ((math.sqrt(2.0 * l_f) + math.sqrt(2.0 * mu0))
                                     * math.log(2.0 * (r_hat * r_hat + 1.0)))


# ------------------------------------------------------ pipelines.hpp ----

SOLVER_KINDS = ("sinkhorn", "acc", "acc-homotopy")


@dataclass
class SolverSpec:  # pipelines.hpp:16-25
    kind: str = "acc-homotopy"
    mu: float = 0.5
    mu0: float = 0.5
    m0: int = 4
    max_iters: int = 2000000
    record_trace: bool = False
    trace_stride: int = 1
    wall_clock: bool = True


def solver_kind_from_name(name: str) -> str:  # pipelines.cpp:20-26
    if name not in SOLVER_KINDS:
        raise OtError(f"unknown solver '{name}'")
    return name


def run_solver(rescaled: TransportProblem, spec: SolverSpec, tol_l1: float,
               time_sweeps=False) -> SolveResult:
    """pipelines.cpp:28-56: dispatch from v0 = 0 with the given tolerance."""
    cfg = SolveConfig(tol_l1, spec.max_iters, spec.record_trace, spec.trace_stride,
                      spec.wall_clock)
    v0 = np.zeros(rescaled.m())
    kind = solver_kind_from_name(spec.kind)
    if kind == "sinkhorn":
        return sinkhorn_solve(rescaled, v0, cfg, time_sweeps)
    if kind == "acc":
        return acc_solve(rescaled, v0, spec.mu, cfg, time_sweeps)
    h = HomotopyConfig(spec.mu0, spec.m0, 64, tol_l1, spec.max_iters, False, spec.record_trace,
                       spec.trace_stride, spec.wall_clock)
    return homotopy_solve(rescaled, h, time_sweeps)


# --------------------------------------------------- plan statistics ----


@dataclass
class PlanStats:
    marginal_violation_l1: float
    primal_cost: float
    max_exponent: float
    row_sums: np.ndarray
    col_sums: np.ndarray


def plan_stats(p: TransportProblem, u, v) -> PlanStats:
    """plan_from_potentials + marginal_violation_l1 + primal_cost (core.cpp:59-79)
    over the implicit plan; P is never materialised.  Raises PotentialOverflow
    when an exponent exceeds 700 (core.cpp:66-69)."""
    h = p.handle
    u, v = _f64(u), _f64(v)
    if u.size != h.n_local or v.size != p.m():
        raise DimensionMismatch("potential sizes do not match the instance")
    out = _capi.PlanSummaryC()
    rs, cs = np.empty(h.n_local), np.empty(p.m())
    out.row_sums, out.col_sums = _ptr(rs), _ptr(cs)
    _check(_lib().otg_plan_stats(h.raw, _ptr(u), _ptr(v), C.byref(out)))
    # primal_cost comes back as sum C'P * cost_div; the reference reports
    # <C, P> * (epsilon_original / epsilon) with C the stored (scaled) cost.
    scale = (p.epsilon_original / p.epsilon) / p.cost_div
    return PlanStats(out.marginal_violation_l1, out.primal_cost * scale, out.max_exponent, rs, cs)


# ------------------------------------------ plan consumers (pipelines.hpp) ----
# The reference consumes a materialised PlanDense; these take the potentials
# and stream the cost once on the device (P is never stored).

def _uv(p: TransportProblem, u, v):
    h = p.handle
    u, v = _f64(u), _f64(v)
    if u.size != h.n_local or v.size != p.m():
        raise DimensionMismatch("potential sizes do not match the instance")
    return h, u, v


def barycentric_projection(p: TransportProblem, u, v, src_colors) -> np.ndarray:
    """pipelines.cpp:58-71 on the implicit plan: (P^T src) / column mass, m x d.
    DimensionMismatch if src rows != n; DegenerateColumn on a zero-mass column."""
    h, u, v = _uv(p, u, v)
    src = np.ascontiguousarray(src_colors, dtype=np.float64)
    if src.ndim != 2 or src.shape[0] != h.n_local:
        raise DimensionMismatch("plan rows and source colors disagree")
    out = np.empty((p.m(), src.shape[1]))
    _check(_lib().otg_plan_barycentric(h.raw, _ptr(u), _ptr(v), _ptr(src), src.shape[1],
                                       _ptr(out), None))
    return out


def predict_translations(p: TransportProblem, u, v) -> List[int]:
    """pipelines.cpp:101-111: row argmax of the plan, ties to the lowest index."""
    h, u, v = _uv(p, u, v)
    out = np.empty(h.n_local, dtype=np.int32)
    _check(_lib().otg_plan_row_argmax(h.raw, _ptr(u), _ptr(v), _ptr(out)))
    return [int(x) for x in out]


def plan_topk(p: TransportProblem, u, v, rows, k: int) -> np.ndarray:
    """Top-k columns of the given rows (value descending, index ascending);
    -1 past m."""
    h, u, v = _uv(p, u, v)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.empty((len(rows), max(int(k), 1)), dtype=np.int32)
    _check(_lib().otg_plan_topk(h.raw, _ptr(u), _ptr(v), _ptr(rows), len(rows), int(k),
                                _ptr(out)))
    return out


def topk_accuracy(p: TransportProblem, u, v, pairs, k: int) -> Optional[float]:
    """pipelines.cpp:113-145: fraction of dictionary source words whose
    top-k plan columns contain one of their targets; None for an empty
    dictionary; OtError for k < 1; DimensionMismatch for indices outside."""
    if k < 1:
        raise OtError("topk_accuracy needs k >= 1")
    pairs = list(pairs)
    if not pairs:
        return None
    n, m = p.handle.n_local, p.m()
    targets = {}
    for s_, t_ in pairs:
        if s_ < 0 or s_ >= n or t_ < 0 or t_ >= m:
            raise DimensionMismatch("dictionary index outside the plan")
        targets.setdefault(int(s_), set()).add(int(t_))
    srcs = sorted(targets)
    top = plan_topk(p, u, v, srcs, k)
    correct = sum(1 for b, s_ in enumerate(srcs) if any(int(j) in targets[s_] for j in top[b] if j >= 0))
    return correct / len(srcs)


def nn_assign(queries, refs, device: int = 0) -> np.ndarray:
    """Nearest reference point of every query (squared distance in fp64,
    strict <: ties to the lowest index) -- the search of nn_propagate."""
    q = np.ascontiguousarray(queries, dtype=np.float64)
    r = np.ascontiguousarray(refs, dtype=np.float64)
    if q.ndim != 2 or r.ndim != 2 or q.shape[1] != r.shape[1]:
        raise DimensionMismatch("query and reference dimensions disagree")
    out = np.empty(q.shape[0], dtype=np.int32)
    _check(_lib().otg_nn_assign(_ptr(q), q.shape[0], _ptr(r), r.shape[0], q.shape[1], device,
                                _ptr(out)))
    return out


def nn_propagate(target_pixels, sampled_tgt_colors, transferred, device: int = 0) -> np.ndarray:
    """pipelines.cpp:73-99 on raw pixels: target_pixels (npix x 3 uint8) are
    matched to their nearest sampled target colour (values in [0, 1]) and take
    that sample's transferred colour, clipped to [0, 1] and rounded to uint8."""
    sampled = np.asarray(sampled_tgt_colors, dtype=np.float64)
    tr = np.asarray(transferred, dtype=np.float64)
    if sampled.shape[0] != tr.shape[0] or sampled.shape[1:] != (3,) or tr.shape[1:] != (3,):
        raise DimensionMismatch("sampled colors and transferred colors disagree")
    px = np.asarray(target_pixels, dtype=np.uint8).reshape(-1, 3)
    best = nn_assign(px.astype(np.float64) / 255.0, sampled, device)
    vals = np.clip(tr[best], 0.0, 1.0) * 255.0
    return np.floor(vals + 0.5).astype(np.uint8)  # std::lround of a non-negative value


def marginal_violation_l1(p, u, v) -> float:
    return plan_stats(p, u, v).marginal_violation_l1


def primal_cost(p, u, v) -> float:
    return plan_stats(p, u, v).primal_cost


def time_sweeps(p: TransportProblem, v, reps=10):
    """Device time (ms) of one (exact, first-evaluation) row pass, column pass
    and merge at v, plus the algorithmic HBM bytes of one row pass, one column
    pass and one steady-state single-pass launch (0 if none)."""
    h = p.handle
    v = _f64(v)
    ms = (C.c_double * 3)()
    by = (C.c_double * 3)()
    _check(_lib().otg_time_sweeps(h.raw, _ptr(v), int(reps), ms, by))
    return list(ms), list(by)


def cull_stats(p: TransportProblem):
    """On-the-fly handles with culled sweeps: the fraction of (warp tile x
    block) pairs the row / column pass visits at the handle's current state
    (otg_cull_stats); (-1, -1) when the handle is not culled."""
    out = (C.c_double * 2)()
    _check(_lib().otg_cull_stats(p.handle.raw, out))
    return float(out[0]), float(out[1])


# ------------------------------------------------------------ inputs -----


# -------------------------------------------- instance CSV (data.cpp:203-271) ----

def write_instance_csv(path, p: TransportProblem):
    """data.cpp:203-218: name,index,value rows; n, m, epsilon, a, b, C row-major,
    every double as %.17g (exact round trip)."""
    validate_problem(p)
    C_ = p.C  # the solver-unit cost (DimensionMismatch for a device-only cost)
    lines = ["name,index,value", f"n,0,{p.n()}", f"m,0,{p.m()}", "epsilon,0,%.17g" % p.epsilon]
    lines += ["a,%d,%.17g" % (i, x) for i, x in enumerate(p.a)]
    lines += ["b,%d,%.17g" % (j, x) for j, x in enumerate(p.b)]
    flat = np.asarray(C_, dtype=np.float64).ravel()
    lines += ["C,%d,%.17g" % (k, x) for k, x in enumerate(flat)]
    try:
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")
    except OSError as e:
        raise IoError(f"cannot write {path}") from e


def read_instance_csv(path) -> TransportProblem:
    """data.cpp:220-269 (MalformedLine for any structural problem)."""
    try:
        fh = open(path)
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    with fh:
        first = fh.readline().rstrip("\n")
        if first != "name,index,value":
            raise MalformedLine(f"{path}: missing 'name,index,value' header")
        n = m = -1
        eps = -1.0
        vals = {"a": [], "b": [], "C": []}
        for line_no, line in enumerate(fh, start=2):
            line = line.rstrip("\n")
            if not line:
                continue
            parts = line.split(",", 2)
            if len(parts) < 3:
                raise MalformedLine(f"{path}:{line_no}: expected three fields")
            name, idx, value = parts[0], _strtol(parts[1]), _strtod(parts[2])
            if name == "n":
                n = int(value)
            elif name == "m":
                m = int(value)
            elif name == "epsilon":
                eps = value
            elif name in vals:
                if idx != len(vals[name]):
                    raise MalformedLine(f"{path}:{line_no}: {name} index {idx} out of order")
                vals[name].append(value)
            else:
                raise MalformedLine(f"{path}:{line_no}: unknown field '{name}'")
    if n < 1 or m < 1 or not eps > 0.0:
        raise MalformedLine(f"{path}: missing n / m / epsilon")
    if len(vals["a"]) != n or len(vals["b"]) != m or len(vals["C"]) != n * m:
        raise MalformedLine(f"{path}: entry counts do not match n = {n}, m = {m}")
    return make_problem(np.array(vals["a"]), np.array(vals["b"]),
                        np.array(vals["C"]).reshape(n, m), eps)


def _strtol(t: str) -> int:  # std::strtol: leading integer, else 0
    import re as _re
    mt = _re.match(r"\s*[-+]?\d+", t)
    return int(mt.group(0)) if mt else 0


def _strtod(t: str) -> float:  # std::strtod: leading number, else 0
    import re as _re
    mt = _re.match(r"\s*[-+]?(?:inf(?:inity)?|nan|(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?)", t,
                   _re.IGNORECASE)
    return float(mt.group(0)) if mt else 0.0


def synthetic_instance(n, m, seed):
    """data.cpp:17-32 -> (a, b, C) numpy arrays."""
    a, b, Cm = np.empty(n), np.empty(m), np.empty((n, m))
    _check(_lib().otg_gen_synthetic_instance(n, m, seed, _ptr(a), _ptr(b), _ptr(Cm)))
    return a, b, Cm


def synthetic_rescaled(n, m, seed, eps) -> TransportProblem:
    """helpers.hpp:30-33."""
    a, b, Cm = synthetic_instance(n, m, seed)
    return rescale_problem(with_epsilon(make_problem(a, b, Cm, 1.0), eps))


def otf_epsilon(epsilon: float) -> float:
    """The INTERNAL epsilon of the on-the-fly sweeps: log2(e) / fl32(log2(e) /
    epsilon), within 2^-25 relative of `epsilon`.  The sweeps scale the fp32
    cost by the single fp32 number fl32(log2(e) / epsilon) (one FMA per
    exponent instead of a hi/lo pair), and every device kernel of the handle
    uses this same scale.  The instance itself keeps `epsilon` (reported, and
    the unit of the primal cost); parity is tested against the oracle at the
    true epsilon.  Tests that compare plan consumers bit-for-bit on the
    device's own model build the oracle problem with this value."""
    kh = float(np.float32(LOG2E / float(epsilon)))
    return LOG2E / kh


def gen_config(cfg: int, n: int, m: int, seed: int):
    """BASELINE config inputs (SURVEY §8d draw orders)."""
    if cfg == 1:
        a, b, Cm = np.empty(n), np.empty(m), np.empty((n, m))
        _check(_lib().otg_gen_config(1, n, m, seed, _ptr(a), _ptr(b), _ptr(Cm)))
        return a, b, Cm
    d = {2: 2, 3: 3, 5: 3}[cfg]
    x, y = np.empty((n, d)), np.empty((m, d))
    _check(_lib().otg_gen_config(cfg, n, m, seed, _ptr(x), _ptr(y), None))
    return x, y


def gen_config4(count: int, seed: int, d: int = 768):
    n = np.empty(count, dtype=np.int32)
    m = np.empty(count, dtype=np.int32)
    _check(_lib().otg_gen_config4(count, seed, d, _ptr(n), _ptr(m), None, None))
    x = np.empty((int(n.sum()), d), dtype=np.float32)
    y = np.empty((int(m.sum()), d), dtype=np.float32)
    _check(_lib().otg_gen_config4(count, seed, d, _ptr(n), _ptr(m), _ptr(x), _ptr(y)))
    return n, m, x, y


def device_count() -> int:
    c = C.c_int()
    _check(_lib().otg_device_count(C.byref(c)))
    return c.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().otg_nccl_get_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------- batched ---


@dataclass
class BatchResult:
    converged: np.ndarray
    iterations: np.ndarray
    final_violation: np.ndarray
    final_reduced_f: np.ndarray
    u: List[np.ndarray]
    v: List[np.ndarray]
    device_seconds: float
    total_iterations: int


class BatchProblem:
    """Many small independent (rescaled) problems, n, m <= 64 each, solved one
    CTA per problem (BASELINE config 4).  a_list / b_list: per-problem
    marginals; costs either dense fp32 (C_list) or built on the device as
    1 - <x, y> from unit embeddings (``cosine``)."""

    def __init__(self, raw, n, m):
        self.raw = raw
        self.n = np.asarray(n, dtype=np.int32)
        self.m = np.asarray(m, dtype=np.int32)

    @classmethod
    def dense(cls, a_list, b_list, C_list, epsilon, device=0):
        n = np.array([len(a) for a in a_list], dtype=np.int32)
        m = np.array([len(b) for b in b_list], dtype=np.int32)
        a = _f64(np.concatenate(a_list))
        b = _f64(np.concatenate(b_list))
        Cc = np.ascontiguousarray(np.concatenate([np.asarray(c, np.float32).ravel() for c in C_list]))
        h = C.c_void_p()
        opts = _device_opts(device, 1, 0, 0, 0, None, 1)
        _check(_lib().otg_batch_create_dense(len(n), _ptr(n), _ptr(m), _ptr(a), _ptr(b), _ptr(Cc),
                                             float(epsilon), C.byref(opts), C.byref(h)))
        return cls(h, n, m)

    @classmethod
    def cosine(cls, n, m, x_cat, y_cat, epsilon, a_cat=None, b_cat=None, norm="none", device=0):
        n = np.ascontiguousarray(n, dtype=np.int32)
        m = np.ascontiguousarray(m, dtype=np.int32)
        x = np.ascontiguousarray(x_cat, dtype=np.float32)
        y = np.ascontiguousarray(y_cat, dtype=np.float32)
        a = _f64(a_cat) if a_cat is not None else np.concatenate([np.full(k, 1.0 / k) for k in n])
        b = _f64(b_cat) if b_cat is not None else np.concatenate([np.full(k, 1.0 / k) for k in m])
        h = C.c_void_p()
        opts = _device_opts(device, 1, 0, 0, 0, None, 1)
        _check(_lib().otg_batch_create_cosine(len(n), _ptr(n), _ptr(m), x.shape[1], _ptr(a), _ptr(b),
                                              _ptr(x), _ptr(y), NORM[norm], float(epsilon),
                                              C.byref(opts), C.byref(h)))
        return cls(h, n, m)

    def stored_cost(self):
        out = np.empty(int((self.n.astype(np.int64) * self.m).sum()), dtype=np.float32)
        _check(_lib().otg_batch_get_cost(self.raw, _ptr(out)))
        res, off = [], 0
        for k in range(len(self.n)):
            sz = int(self.n[k]) * int(self.m[k])
            res.append(out[off:off + sz].reshape(self.n[k], self.m[k]))
            off += sz
        return res

    def homotopy_solve(self, cfg: HomotopyConfig = HomotopyConfig()) -> BatchResult:
        cnt = len(self.n)
        conv = np.empty(cnt, dtype=np.int32)
        it = np.empty(cnt, dtype=np.int64)
        fv, ff = np.empty(cnt), np.empty(cnt)
        u, v = np.empty(int(self.n.sum())), np.empty(int(self.m.sum()))
        r = _capi.BatchResultC(_ptr(conv), _ptr(it), _ptr(fv), _ptr(ff), _ptr(u), _ptr(v), 0.0, 0)
        c = _capi.HomotopyConfigC(cfg.mu0, cfg.m0, cfg.max_outer, cfg.tol_l1, cfg.max_total_inner,
                                  int(cfg.rescale_w_across_stages), 0, 1)
        _check(_lib().otg_batch_homotopy_solve(self.raw, C.byref(c), C.byref(r)))
        us = np.split(u, np.cumsum(self.n)[:-1])
        vs = np.split(v, np.cumsum(self.m)[:-1])
        return BatchResult(conv.astype(bool), it, fv, ff, us, vs, r.device_seconds,
                           r.total_iterations)

    def close(self):
        if self.raw:
            _lib().otg_batch_destroy(self.raw)
            self.raw = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
