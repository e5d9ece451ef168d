"""ctypes binding of include/otg.h (the C-ABI of libotg.so).

The library is built in-tree (paper_2605_30267_b200/libotg.so) by
``__graft_entry__.build()``.  There is no fallback: importing the product API
without the library, or calling a solver without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OTG_LIB") or os.path.join(_HERE, "libotg.so")  # (OTG_LIB: A/B builds)

c_double_p = C.POINTER(C.c_double)


class DeviceOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("world_size", C.c_int), ("rank", C.c_int),
                ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("nccl_unique_id", C.c_void_p), ("virtual_shards", C.c_int),
                ("allreduce", C.c_void_p), ("allreduce_ctx", C.c_void_p), ("sweep", C.c_int)]


class ProblemInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("n_local", C.c_int64),
                ("row_begin", C.c_int64), ("storage", C.c_int), ("epsilon", C.c_double),
                ("cost_raw_min", C.c_double), ("cost_raw_max", C.c_double),
                ("device_bytes", C.c_int64), ("world_size", C.c_int), ("rank", C.c_int),
                ("device", C.c_int), ("sweep_mode", C.c_int), ("sweep_clusters", C.c_int),
                ("col_splits", C.c_int)]


class StepEvalC(C.Structure):
    _fields_ = [("v_next", C.c_void_p), ("u", C.c_void_p), ("grad", C.c_void_p),
                ("grad_l1", C.c_double), ("f_value", C.c_double)]


TRACE_COLS = 15  # OTG_TRACE_COLS


class SolveConfigC(C.Structure):
    _fields_ = [("tol_l1", C.c_double), ("max_iters", C.c_int64), ("record_trace", C.c_int),
                ("trace_stride", C.c_int64), ("reference_v", C.c_void_p),
                ("reference_f", C.c_double)]


class HomotopyConfigC(C.Structure):
    _fields_ = [("mu0", C.c_double), ("m0", C.c_int64), ("max_outer", C.c_int64),
                ("tol_l1", C.c_double), ("max_total_inner", C.c_int64),
                ("rescale_w_across_stages", C.c_int), ("record_trace", C.c_int),
                ("trace_stride", C.c_int64)]


class InstrC(C.Structure):
    _fields_ = [("stability", C.c_int), ("reference_v", C.c_void_p), ("reference_f", C.c_double)]


class SolveResultC(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int64), ("evaluations", C.c_int64),
                ("outer_stages", C.c_int64), ("final_violation", C.c_double),
                ("final_reduced_f", C.c_double), ("max_v_inf", C.c_double),
                ("conditions_checked", C.c_int64), ("conditions_held", C.c_int64),
                ("u", C.c_void_p), ("v", C.c_void_p), ("w", C.c_void_p),
                ("trace", C.c_void_p), ("trace_cap", C.c_int64), ("trace_len", C.c_int64),
                ("boundaries", C.c_void_p), ("boundaries_cap", C.c_int64),
                ("time_sweeps", C.c_int), ("device_seconds", C.c_double),
                ("row_pass_seconds", C.c_double), ("col_pass_seconds", C.c_double),
                ("kernel_launches", C.c_int64), ("row_redos", C.c_int64),
                ("epilogue_seconds", C.c_double), ("fallback_columns", C.c_int64),
                ("radius_x_max", C.c_double), ("radius_y_max", C.c_double)]


class PlanSummaryC(C.Structure):
    _fields_ = [("marginal_violation_l1", C.c_double), ("primal_cost", C.c_double),
                ("max_exponent", C.c_double), ("row_sums", C.c_void_p),
                ("col_sums", C.c_void_p)]


class BatchResultC(C.Structure):
    _fields_ = [("converged", C.c_void_p), ("iterations", C.c_void_p),
                ("final_violation", C.c_void_p), ("final_reduced_f", C.c_void_p),
                ("u_cat", C.c_void_p), ("v_cat", C.c_void_p), ("device_seconds", C.c_double),
                ("total_iterations", C.c_int64)]


# Every symbol include/otg.h declares, with its ctypes signature.
H = C.c_void_p
I64 = C.c_int64
VP = C.c_void_p
SIGNATURES = {
    "otg_last_error": (C.c_char_p, []),
    "otg_abi_version": (C.c_int, []),
    "otg_device_count": (C.c_int, [VP]),
    "otg_nccl_get_unique_id": (C.c_int, [VP]),
    "otg_problem_create_dense": (C.c_int, [I64, I64, VP, VP, VP, C.c_int, I64, C.c_double, VP, VP]),
    "otg_problem_create_points": (C.c_int, [I64, I64, I64, VP, VP, VP, VP, C.c_int, C.c_int,
                                            C.c_int, C.c_double, VP, VP]),
    "otg_problem_destroy": (C.c_int, [H]),
    "otg_problem_info_get": (C.c_int, [H, VP]),
    "otg_problem_get_cost": (C.c_int, [H, I64, I64, VP]),
    "otg_row_solve_marginals": (C.c_int, [H, VP, VP, VP]),
    "otg_row_solve_marginals_log": (C.c_int, [H, VP, VP, VP, VP]),
    "otg_eval_normalized_step": (C.c_int, [H, VP, VP]),
    "otg_sinkhorn_solve": (C.c_int, [H, VP, VP, VP]),
    "otg_acc_solve": (C.c_int, [H, VP, C.c_double, VP, VP]),
    "otg_acc_run": (C.c_int, [H, VP, VP, C.c_double, I64, C.c_int, I64, VP, VP]),
    "otg_homotopy_solve": (C.c_int, [H, VP, VP, VP]),
    "otg_plan_stats": (C.c_int, [H, VP, VP, VP]),
    "otg_time_sweeps": (C.c_int, [H, VP, C.c_int, VP, VP]),
    "otg_plan_barycentric": (C.c_int, [H, VP, VP, VP, C.c_int, VP, VP]),
    "otg_plan_row_argmax": (C.c_int, [H, VP, VP, VP]),
    "otg_plan_topk": (C.c_int, [H, VP, VP, VP, C.c_int64, C.c_int, VP]),
    "otg_nn_assign": (C.c_int, [VP, C.c_int64, VP, C.c_int64, C.c_int, C.c_int, VP]),
    "otg_dual_F": (C.c_int, [H, VP, VP, VP]),
    "otg_hessian_f": (C.c_int, [H, VP, VP]),
    "otg_batch_create_dense": (C.c_int, [I64, VP, VP, VP, VP, VP, C.c_double, VP, VP]),
    "otg_batch_create_cosine": (C.c_int, [I64, VP, VP, I64, VP, VP, VP, VP, C.c_int,
                                          C.c_double, VP, VP]),
    "otg_batch_destroy": (C.c_int, [H]),
    "otg_batch_get_cost": (C.c_int, [H, VP]),
    "otg_batch_homotopy_solve": (C.c_int, [H, VP, VP]),
    "otg_gen_synthetic_instance": (C.c_int, [I64, I64, C.c_uint64, VP, VP, VP]),
    "otg_gen_config": (C.c_int, [C.c_int, I64, I64, C.c_uint64, VP, VP, VP]),
    "otg_gen_config4": (C.c_int, [I64, C.c_uint64, I64, VP, VP, VP, VP]),
    "otg_debug_cull": (C.c_int, [C.c_int]),
    "otg_cull_stats": (C.c_int, [H, VP]),
}

_lib = None


def load():
    """Load libotg.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                          "(libotg has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def header_symbols(header: str | None = None):
    """Function names declared in include/otg.h (for the export test)."""
    import re
    header = header or os.path.join(os.path.dirname(_HERE), "include", "otg.h")
    text = open(header).read()
    return sorted(set(re.findall(r"\b(otg_[a-z0-9_]+)\s*\(", text)) - {"otg_status"})
