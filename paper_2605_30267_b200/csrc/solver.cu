// solver.cu — solver entry points of the C-ABI: one-shot evaluations and the
// device-resident Sinkhorn / Acc-Sinkhorn / homotopy loops.
//
// The loop body (row pass, column pass, merge, fallback, finalize, apply) is
// captured once per handle into a CUDA graph holding kChunk evaluations; the
// host replays the graph and reads the 300-byte control block once per
// chunk.  All stop / schedule decisions are taken on the device by the
// finalize kernel (sweep.cu: control_step), so there is no per-iteration
// host round trip; evaluations past the stop point are no-ops.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstring>

#include "common.cuh"

namespace otg {

namespace {

constexpr int kChunk = 8;
constexpr int kT = 256;

void check_finite_vec(const double* v, int64_t m, const char* what) {  // dual.cpp:13-18
  if (!v) fail(OTG_E_DIMENSION, std::string(what) + " is NULL");
  for (int64_t j = 0; j < m; ++j)
    if (!std::isfinite(v[j])) fail(OTG_E_OT, std::string(what) + " has non-finite entries");
}

std::vector<double> project_zero_sum(const double* x, int64_t m) {  // mirror.cpp:103-105
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) s += x[j];
  const double mean = s / static_cast<double>(m);
  std::vector<double> out(m);
  for (int64_t j = 0; j < m; ++j) out[j] = x[j] - mean;
  return out;
}

void check_zero_sum(const double* x, int64_t m, const char* what) {  // accel.cpp:21-25
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) s += x[j];
  if (std::abs(s) > 1e-9) fail(OTG_E_GAUGE, std::string(what) + " must be zero-sum");
}

void validate_solve_config(const otg_solve_config* c) {  // sinkhorn.cpp:29-33
  if (!c) fail(OTG_E_OT, "solve config is NULL");
  if (!(c->tol_l1 > 0.0)) fail(OTG_E_OT, "tol_l1 must be positive");
  if (c->max_iters < 1) fail(OTG_E_OT, "max_iters must be at least 1");
  if (c->trace_stride < 1) fail(OTG_E_OT, "trace_stride must be at least 1");
}

// A solve on a single-pass handle whose first evaluation point is the zero
// point starts with the single pass: the rows' statistics at p = 0 (upper
// bound of the base-2 max and the argmin column, fused.cu k_zero_rowstats,
// computed once with the cost) stand in for the previous evaluation's, with
// a zero step -- so no exact two-pass seed evaluation (~2.2 ms at 65536^2).
void zero_start(Problem& P, Ctrl& c, const double* x0) {
  if (!P.fused || !P.sp_zM2) return;
  for (int64_t j = 0; j < P.m; ++j)
    if (x0[j] != 0.0) return;
  OTG_CUDA(cudaMemcpyAsync(P.rowM2, P.sp_zM2, P.n_local * sizeof(double), cudaMemcpyDeviceToDevice,
                           P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.rowJ, P.sp_zJ, P.n_local * sizeof(int), cudaMemcpyDeviceToDevice,
                           P.stream));
  OTG_CUDA(cudaMemsetAsync(P.dq, 0, P.mpad * sizeof(double), P.stream));
  c.shift_valid = 1;
  c.dmax2 = 0.0;
}

Ctrl base_ctrl(const Problem& P) {
  Ctrl c;
  std::memset(&c, 0, sizeof c);
  c.tiny = P.storage == OTG_STORE_F64 ? kTinyPrecise : kTinyFast;
  c.trace_cap = 4096;
  c.boundary_cap = 4096;
  c.trace_stride = 1;
  return c;
}

void put_ctrl(Problem& P, const Ctrl& c) {
  std::memcpy(P.ctrl_host, &c, sizeof c);
  OTG_CUDA(cudaMemcpyAsync(P.ctrl, P.ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice, P.stream));
}

void get_ctrl(Problem& P) {
  OTG_CUDA(cudaMemcpyAsync(P.ctrl_host, P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, P.stream));
  comm_sync(P);  // (sharded NCCL handles: polls the communicator's async error state)
}

void h2d(Problem& P, double* dst, const double* src, int64_t count) {
  OTG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyHostToDevice, P.stream));
}
// New evaluation point from the host: p and its fp32 split (row pass input).
void set_point(Problem& P, const double* v) {
  h2d(P, P.p, v, P.m);
  launch_split_p(P);
}
void d2h(Problem& P, double* dst, const double* src, int64_t count) {
  if (dst) OTG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToHost, P.stream));
}

void raise_device_error(const Ctrl& c) {
  if (c.error == OTG_E_DOMAIN) fail(OTG_E_DOMAIN, "column log-mass degenerated (non-finite log c)");
  if (c.error == OTG_E_OT)
    fail(OTG_E_OT, "reference value f* exceeds f(x) (lyapunov_energy_from_parts, diag.cpp:78-81)");
  if (c.error) fail(static_cast<otg_status>(c.error), "device-side error");
}

void build_graph(Problem& P, bool timed, bool steady = false) {
  cudaGraphExec_t& exec = steady ? P.chunk_exec_steady : (timed ? P.chunk_exec_timed : P.chunk_exec);
  if (exec) return;
  if (timed && P.chunk_events.empty()) {
    P.chunk_events.resize(5 * kChunk);
    for (auto& e : P.chunk_events) OTG_CUDA(cudaEventCreate(&e));
  }
  cudaGraph_t g = nullptr;
  OTG_CUDA(cudaStreamBeginCapture(P.stream, cudaStreamCaptureModeThreadLocal));
  P.capturing = 1;
  P.steady_capture = steady ? 1 : 0;
  try {
    for (int k = 0; k < kChunk; ++k) {
      launch_eval(P, true, timed, timed ? &P.chunk_events[5 * k] : nullptr);
      launch_apply(P);
      if (timed)
        OTG_CUDA(cudaEventRecordWithFlags(P.chunk_events[5 * k + 4], P.stream,
                                          cudaEventRecordExternal));
    }
  } catch (...) {
    P.capturing = 0;
    P.steady_capture = 0;
    cudaStreamEndCapture(P.stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  P.capturing = 0;
  P.steady_capture = 0;
  OTG_CUDA(cudaStreamEndCapture(P.stream, &g));
  size_t nn = 0;
  OTG_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  OTG_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
  int kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    OTG_CUDA(cudaGraphNodeGetType(nd, &t));
    kernels += (t == cudaGraphNodeTypeKernel);
  }
  (steady ? P.chunk_kernels_steady : (timed ? P.chunk_kernels_timed : P.chunk_kernels)) = kernels;
  OTG_CUDA(cudaGraphInstantiate(&exec, g, 0));
  cudaGraphDestroy(g);
  P.chunk_len = kChunk;
}

struct LoopOut {
  double device_s = 0.0, row_s = 0.0, col_s = 0.0, epi_s = 0.0;
  int64_t trace_len = 0;
  int64_t launches = 0;  // kernel nodes executed (every replayed chunk)
  int64_t pauses = 0;    // sharded: chunks paused for an eager fallback exchange
};

// Replays the chunk graph until the device control block says done; drains
// the trace ring into res->trace after every chunk.
LoopOut run_loop(Problem& P, otg_solve_result* res, bool timed) {
  build_graph(P, timed);
  // unsharded single-pass handles replay the steady graph (no exact-path
  // kernels, merge in the patch kernel) for chunks that start after an
  // evaluation (or at the zero point: zero_start)
  const bool use_steady = patch_merges(P) && !timed;
  if (use_steady) build_graph(P, false, true);
  cudaEvent_t t0, t1;
  OTG_CUDA(cudaEventCreate(&t0));
  OTG_CUDA(cudaEventCreate(&t1));
  LoopOut lo;
  int64_t drained = 0;
  long long ev_before = P.ctrl_host->evaluations;
  OTG_CUDA(cudaEventRecord(t0, P.stream));
  for (;;) {
    {
      OTG_RANGE("otg chunk (8 evaluations)");
      const bool steady = use_steady && P.ctrl_host->shift_valid;
      OTG_CUDA(cudaGraphLaunch(steady ? P.chunk_exec_steady
                                      : (timed ? P.chunk_exec_timed : P.chunk_exec),
                               P.stream));
      lo.launches += steady ? P.chunk_kernels_steady
                            : (timed ? P.chunk_kernels_timed : P.chunk_kernels);
      get_ctrl(P);
    }
    if (P.sharded && comm_failed(P)) fail(OTG_E_NCCL, "host all-reduce callback failed");
    if (P.ctrl_host->done == kPaused) {
      // a sharded evaluation flagged columns: finish it eagerly (exact
      // cross-rank LSE exchange, finalize, apply), then keep replaying
      OTG_CUDA(cudaMemsetAsync(&P.ctrl->done, 0, sizeof(int), P.stream));
      launch_fallback_and_finalize(P);
      launch_apply(P);
      get_ctrl(P);
      ++lo.pauses;
    }
    const Ctrl& c = *P.ctrl_host;
    if (timed) {
      const long long live = c.evaluations - ev_before;
      for (long long k = 0; k < live && k < kChunk; ++k) {
        float a = 0.f, b = 0.f, e = 0.f;
        const cudaEvent_t* ev = &P.chunk_events[5 * k];
        OTG_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
        OTG_CUDA(cudaEventElapsedTime(&b, ev[2], ev[3]));
        OTG_CUDA(cudaEventElapsedTime(&e, ev[3], ev[4]));
        lo.row_s += a * 1e-3;
        lo.col_s += b * 1e-3;
        lo.epi_s += e * 1e-3;
      }
      ev_before = c.evaluations;
    }
    if (c.trace_count > drained) {
      const int64_t cap = c.trace_cap;
      std::vector<double> ring(static_cast<size_t>(cap) * kTraceCols);
      OTG_CUDA(cudaMemcpyAsync(ring.data(), P.trace, ring.size() * sizeof(double),
                               cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      for (int64_t r = drained; r < c.trace_count; ++r) {
        if (res && res->trace && r < res->trace_cap)
          std::memcpy(res->trace + r * kTraceCols, ring.data() + (r % cap) * kTraceCols,
                      kTraceCols * sizeof(double));
      }
      drained = c.trace_count;
    }
    if (c.done == 1) break;
  }
  OTG_CUDA(cudaEventRecord(t1, P.stream));
  OTG_CUDA(cudaEventSynchronize(t1));
  float ms = 0.f;
  OTG_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  lo.device_s = ms * 1e-3;
  lo.trace_len = drained;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  return lo;
}

void fill_result(Problem& P, otg_solve_result* res, const LoopOut& lo) {
  const Ctrl& c = *P.ctrl_host;
  raise_device_error(c);
  if (!res) return;
  res->converged = c.converged;
  res->iterations = c.iterations;
  res->evaluations = c.evaluations;
  res->outer_stages = c.outer_stages;
  res->final_violation = c.final_violation;
  res->final_reduced_f = c.final_f;
  res->max_v_inf = c.max_v_inf;
  res->conditions_checked = c.cond_checked;
  res->conditions_held = c.cond_held;
  res->trace_len = lo.trace_len;
  res->device_seconds = lo.device_s;
  res->row_pass_seconds = lo.row_s;
  res->col_pass_seconds = lo.col_s;
  res->epilogue_seconds = lo.epi_s;
  res->kernel_launches = lo.launches;
  res->row_redos = c.redo_total;
  res->fallback_columns = c.fb_total;
  res->radius_x_max = c.rmax_x;
  res->radius_y_max = c.rmax_y;
  d2h(P, res->u, P.u, P.n_local);
  d2h(P, res->v, P.p, P.m);
  d2h(P, res->w, P.wacc, P.m);
  if (res->boundaries && res->boundaries_cap > 0) {
    const int64_t nb = std::min<int64_t>(c.boundary_count, std::min<int64_t>(res->boundaries_cap, c.boundary_cap));
    if (nb > 0) d2h(P, res->boundaries, P.bounds, nb * kBoundCols);
  }
  OTG_CUDA(cudaStreamSynchronize(P.stream));
}

Problem& get(otg_problem h) {
  if (!h) fail(OTG_E_DIMENSION, "NULL problem handle");
  OTG_CUDA(cudaSetDevice(h->P.device));
  return h->P;
}

// One evaluation at v (host), outputs left on the device.
void one_eval(Problem& P, const double* v, bool with_log) {
  check_finite_vec(v, P.m, "v");
  Ctrl c = base_ctrl(P);
  c.mode = MODE_EVAL;
  put_ctrl(P, c);
  set_point(P, v);
  launch_eval(P, with_log, false, nullptr);
  if (with_log) launch_apply(P);
  get_ctrl(P);
  raise_device_error(*P.ctrl_host);
}

__global__ void k_plan_rows(const double* __restrict__ C64, const float* __restrict__ C32,
                            const float4* __restrict__ X, const float4* __restrict__ Y,
                            int64_t ldc, int64_t n, int64_t m, double kappa,
                            const double* __restrict__ u, const double* __restrict__ v,
                            double* __restrict__ rowsum, double* __restrict__ rowcost,
                            double* __restrict__ rowmax) {
  __shared__ double s1[kT], s2[kT], s3[kT];
  const int64_t i = blockIdx.x;
  double rs = 0.0, cs = 0.0, mx = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < m; j += kT) {
    const double c = cost_at(C64, C32, X, Y, ldc, kappa, i, j);
    const double e = ((-c) + u[i]) + v[j];  // core.cpp:63-65
    const double P = exp(e);
    mx = fmax(mx, e);
    rs += P;
    cs += c * P;
  }
  s1[threadIdx.x] = rs;
  s2[threadIdx.x] = cs;
  s3[threadIdx.x] = mx;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
      s3[threadIdx.x] = fmax(s3[threadIdx.x], s3[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rowsum[i] = s1[0];
    rowcost[i] = s2[0];
    rowmax[i] = s3[0];
  }
}

__global__ void k_plan_cols(const double* __restrict__ C64, const float* __restrict__ C32,
                            const float4* __restrict__ X, const float4* __restrict__ Y,
                            int64_t ldc, int64_t n, int64_t m, double kappa,
                            const double* __restrict__ u, const double* __restrict__ v,
                            double* __restrict__ colsum) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double c = cost_at(C64, C32, X, Y, ldc, kappa, i, j);
    s += exp(((-c) + u[i]) + v[j]);
  }
  colsum[j] = s;
}

}  // namespace

Problem& problem_of(otg_problem h) { return get(h); }

}  // namespace otg

using namespace otg;

extern "C" {

otg_status otg_row_solve_marginals(otg_problem h, const double* v, double* u, double* col) {
  return guard([&] {
    OTG_RANGE("otg_row_solve_marginals");
    Problem& P = get(h);
    check_finite_vec(v, P.m, "v");
    Ctrl c = base_ctrl(P);
    c.mode = MODE_EVAL;
    put_ctrl(P, c);
    set_point(P, v);
    launch_sweeps(P, false, nullptr);
    launch_merge_nolog(P);
    if (P.sharded) comm_allreduce_sum(P, P.col, static_cast<size_t>(P.mpad + 1));
    d2h(P, u, P.u, P.n_local);
    d2h(P, col, P.col, P.m);
    OTG_CUDA(cudaStreamSynchronize(P.stream));
  });
}

otg_status otg_row_solve_marginals_log(otg_problem h, const double* v, double* u, double* col,
                                       double* col_log) {
  return guard([&] {
    OTG_RANGE("otg_row_solve_marginals_log");
    Problem& P = get(h);
    one_eval(P, v, true);
    d2h(P, u, P.u, P.n_local);
    d2h(P, col, P.col, P.m);
    d2h(P, col_log, P.col_log, P.m);
    OTG_CUDA(cudaStreamSynchronize(P.stream));
  });
}

otg_status otg_eval_normalized_step(otg_problem h, const double* v, otg_step_eval* out) {
  return guard([&] {
    OTG_RANGE("otg_eval_normalized_step");
    Problem& P = get(h);
    one_eval(P, v, true);
    if (out) {
      d2h(P, out->v_next, P.y, P.m);
      d2h(P, out->u, P.u, P.n_local);
      d2h(P, out->grad, P.grad, P.m);
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      out->grad_l1 = P.ctrl_host->grad_l1;
      out->f_value = P.ctrl_host->f_value;
    }
  });
}

otg_status otg_sinkhorn_solve(otg_problem h, const double* v0, const otg_solve_config* cfg,
                              otg_solve_result* res) {
  return guard([&] {
    OTG_RANGE("otg_sinkhorn_solve");
    Problem& P = get(h);
    validate_solve_config(cfg);
    std::vector<double> zero;
    if (!v0) {
      zero.assign(P.m, 0.0);
      v0 = zero.data();
    }
    check_finite_vec(v0, P.m, "v0");
    const std::vector<double> v = project_zero_sum(v0, P.m);  // sinkhorn.cpp:77
    Ctrl c = base_ctrl(P);
    c.mode = MODE_SINKHORN;
    c.tol = cfg->tol_l1;
    c.max_iters = cfg->max_iters;
    c.record_trace = cfg->record_trace;
    c.trace_stride = cfg->trace_stride;
    zero_start(P, c, v.data());
    put_ctrl(P, c);
    set_point(P, v.data());
    const LoopOut lo = run_loop(P, res, res && res->time_sweeps);
    fill_result(P, res, lo);
  });
}

// ReferenceSolution (diag.hpp:46-49) for the energy / radius columns.
static void attach_reference(Problem& P, Ctrl& c, const double* v_star, double f_star) {
  if (!v_star) return;
  check_finite_vec(v_star, P.m, "reference v_star");
  if (!std::isfinite(f_star)) fail(OTG_E_OT, "reference f_star is not finite");
  h2d(P, P.vstar, v_star, P.m);
  c.have_ref = 1;
  c.f_star = f_star;
}

static void start_acc(Problem& P, Ctrl& c, const double* x0, const double* w0, double mu) {
  c.mu = mu;
  c.alpha_next = std::sqrt(2.0 * mu);  // accel.cpp:149
  c.alpha_step = c.alpha_next;
  // (the first evaluation point is x0: the extrapolation of x0 with w0 is x0)
  zero_start(P, c, x0);
  put_ctrl(P, c);
  set_point(P, x0);
  if (w0)
    h2d(P, P.wacc, w0, P.m);
  else
    OTG_CUDA(cudaMemsetAsync(P.wacc, 0, P.m * sizeof(double), P.stream));
}

otg_status otg_acc_solve(otg_problem h, const double* v0, double mu, const otg_solve_config* cfg,
                         otg_solve_result* res) {
  return guard([&] {
    OTG_RANGE("otg_acc_solve");
    Problem& P = get(h);
    validate_solve_config(cfg);
    if (!(mu > 0.0) || !(mu < 1.0)) fail(OTG_E_OT, "mu must lie in (0, 1)");
    std::vector<double> zero;
    if (!v0) {
      zero.assign(P.m, 0.0);
      v0 = zero.data();
    }
    check_finite_vec(v0, P.m, "v0");
    const std::vector<double> x0 = project_zero_sum(v0, P.m);  // accel.cpp:207
    Ctrl c = base_ctrl(P);
    c.mode = MODE_ACC;
    c.tol = cfg->tol_l1;
    c.max_iters = cfg->max_iters;
    c.record_trace = cfg->record_trace;
    c.trace_stride = cfg->trace_stride;
    attach_reference(P, c, cfg->reference_v, cfg->reference_f);  // accel.cpp:211-213
    start_acc(P, c, x0.data(), nullptr, mu);
    const LoopOut lo = run_loop(P, res, res && res->time_sweeps);
    fill_result(P, res, lo);
  });
}

otg_status otg_acc_run(otg_problem h, const double* x0, const double* w0, double mu,
                       int64_t m_steps, int record_trace, int64_t trace_stride,
                       const otg_instr* instr, otg_solve_result* res) {
  return guard([&] {
    OTG_RANGE("otg_acc_run");
    Problem& P = get(h);
    if (m_steps < 0) fail(OTG_E_OT, "acc_run needs m >= 0");
    check_finite_vec(x0, P.m, "x0");
    check_finite_vec(w0, P.m, "w0");
    if (!(mu > 0.0) || !(mu < 1.0)) fail(OTG_E_OT, "mu must lie in (0, 1)");
    check_zero_sum(x0, P.m, "x0");
    check_zero_sum(w0, P.m, "w0");
    Ctrl c = base_ctrl(P);
    c.mode = MODE_ACC_RUN;
    c.msteps = m_steps;
    c.record_trace = record_trace;
    c.trace_stride = trace_stride > 0 ? trace_stride : 1;
    c.stability = instr && instr->stability;
    if (instr) attach_reference(P, c, instr->reference_v, instr->reference_f);
    start_acc(P, c, x0, w0, mu);
    const LoopOut lo = run_loop(P, res, res && res->time_sweeps);
    fill_result(P, res, lo);
  });
}

otg_status otg_homotopy_solve(otg_problem h, const otg_homotopy_config* cfg,
                              const otg_instr* instr, otg_solve_result* res) {
  return guard([&] {
    OTG_RANGE("otg_homotopy_solve");
    Problem& P = get(h);
    if (!cfg) fail(OTG_E_OT, "homotopy config is NULL");
    if (!(cfg->mu0 > 0.0) || !(cfg->mu0 < 1.0) || cfg->m0 < 1 || cfg->max_outer < 1)
      fail(OTG_E_OT, "homotopy schedule needs mu0 in (0, 1), m0 >= 1, max_outer >= 1");
    if (!(cfg->tol_l1 > 0.0)) fail(OTG_E_OT, "tol_l1 must be positive");
    if (cfg->max_total_inner < 1) fail(OTG_E_OT, "max_total_inner must be at least 1");
    if (cfg->trace_stride < 1) fail(OTG_E_OT, "trace_stride must be at least 1");
    Ctrl c = base_ctrl(P);
    c.mode = MODE_HOMOTOPY;
    c.tol = cfg->tol_l1;
    c.m0 = cfg->m0;
    c.max_outer = cfg->max_outer;
    c.max_total_inner = cfg->max_total_inner;
    c.rescale_w = cfg->rescale_w_across_stages;
    c.record_trace = cfg->record_trace;
    c.trace_stride = cfg->trace_stride;
    c.stability = instr && instr->stability;
    if (instr) attach_reference(P, c, instr->reference_v, instr->reference_f);
    c.mu0 = cfg->mu0;
    const std::vector<double> zero(P.m, 0.0);
    start_acc(P, c, zero.data(), nullptr, cfg->mu0);
    const LoopOut lo = run_loop(P, res, res && res->time_sweeps);
    fill_result(P, res, lo);
  });
}

otg_status otg_plan_stats(otg_problem h, const double* u, const double* v, otg_plan_summary* out) {
  return guard([&] {
    OTG_RANGE("otg_plan_stats");
    Problem& P = get(h);
    if (!out) fail(OTG_E_DIMENSION, "NULL output");
    check_finite_vec(u, P.n_local, "u");
    check_finite_vec(v, P.m, "v");
    const int64_t n = P.n_local, m = P.m;
    double *du = nullptr, *dv = nullptr, *rs = nullptr, *rc = nullptr, *rm = nullptr, *cs = nullptr;
    OTG_CUDA(cudaMalloc(&du, n * sizeof(double)));
    OTG_CUDA(cudaMalloc(&dv, m * sizeof(double)));
    OTG_CUDA(cudaMalloc(&rs, std::max<int64_t>(n, 2) * sizeof(double)));
    OTG_CUDA(cudaMalloc(&rc, n * sizeof(double)));
    OTG_CUDA(cudaMalloc(&rm, n * sizeof(double)));
    OTG_CUDA(cudaMalloc(&cs, m * sizeof(double)));
    h2d(P, du, u, n);
    h2d(P, dv, v, m);
    const float4* X4 = reinterpret_cast<const float4*>(P.X);
    const float4* Y4 = reinterpret_cast<const float4*>(P.Y);
    k_plan_rows<<<static_cast<unsigned>(n), kT, 0, P.stream>>>(P.C64, P.C32, X4, Y4, P.ldc, n, m,
                                                               P.kappa, du, dv, rs, rc, rm);
    k_plan_cols<<<static_cast<unsigned>((m + kT - 1) / kT), kT, 0, P.stream>>>(
        P.C64, P.C32, X4, Y4, P.ldc, n, m, P.kappa, du, dv, cs);
    OTG_CUDA(cudaGetLastError());
    if (P.sharded) comm_allreduce_sum(P, cs, static_cast<size_t>(m));  // global column sums
    std::vector<double> hrs(n), hrc(n), hrm(n), hcs(m);
    d2h(P, hrs.data(), rs, n);
    d2h(P, hrc.data(), rc, n);
    d2h(P, hrm.data(), rm, n);
    d2h(P, hcs.data(), cs, m);
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    double top = -DBL_MAX, cost = 0.0, viol = 0.0, vc = 0.0;
    for (int64_t i = 0; i < n; ++i) top = std::max(top, hrm[i]);
    std::vector<double> hb(m), ha(n);
    OTG_CUDA(cudaMemcpy(hb.data(), P.b, m * sizeof(double), cudaMemcpyDeviceToHost));
    OTG_CUDA(cudaMemcpy(ha.data(), P.a, n * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      cost += hrc[i];
      viol += std::abs(hrs[i] - ha[i]);
    }
    if (P.sharded) {  // row-local scalars: sum the cost and the row violation, max the exponent
      double hsum[2] = {cost, viol}, hmax[1] = {top};
      OTG_CUDA(cudaMemcpyAsync(rs, hsum, sizeof hsum, cudaMemcpyHostToDevice, P.stream));
      OTG_CUDA(cudaMemcpyAsync(rm, hmax, sizeof hmax, cudaMemcpyHostToDevice, P.stream));
      comm_allreduce_sum(P, rs, 2);
      comm_allreduce_max(P, rm, 1);
      OTG_CUDA(cudaMemcpyAsync(hsum, rs, sizeof hsum, cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaMemcpyAsync(hmax, rm, sizeof hmax, cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      cost = hsum[0];
      viol = hsum[1];
      top = hmax[0];
    }
    for (double* q : {du, dv, rs, rc, rm, cs}) cudaFree(q);
    out->max_exponent = top;
    if (top > kExpOverflowBound) fail(OTG_E_OVERFLOW, "plan exponent exceeds bound");
    for (int64_t j = 0; j < m; ++j) vc += std::abs(hcs[j] - hb[j]);
    out->marginal_violation_l1 = viol + vc;
    // (eps_original / eps) with eps = 1 (core.cpp:77-79); on the fly the
    // internal scale is kappa (within 2^-25 of 1 / epsilon), so undo exactly that
    out->primal_cost = P.storage == OTG_STORE_ON_THE_FLY ? cost / P.kappa : cost * P.epsilon;
    if (out->row_sums) std::memcpy(out->row_sums, hrs.data(), n * sizeof(double));
    if (out->col_sums) std::memcpy(out->col_sums, hcs.data(), m * sizeof(double));
  });
}

otg_status otg_time_sweeps(otg_problem h, const double* v, int reps, double ms[3],
                           double bytes[3]) {
  return guard([&] {
    Problem& P = get(h);
    if (reps < 1) reps = 1;
    one_eval(P, v, true);  // warm
    cudaEvent_t e[4];
    for (auto& x : e) OTG_CUDA(cudaEventCreate(&x));
    double acc[3] = {0, 0, 0};
    for (int r = 0; r < reps; ++r) {
      Ctrl c = base_ctrl(P);
      c.mode = MODE_EVAL;
      put_ctrl(P, c);
      set_point(P, v);
      OTG_CUDA(cudaEventRecord(e[0], P.stream));
      launch_row_pass(P);  // exact first-evaluation kernels (no shift estimate here)
      OTG_CUDA(cudaEventRecord(e[1], P.stream));
      launch_col_pass(P);
      OTG_CUDA(cudaEventRecord(e[2], P.stream));
      launch_merge_nolog(P);
      OTG_CUDA(cudaEventRecord(e[3], P.stream));
      OTG_CUDA(cudaEventSynchronize(e[3]));
      float a = 0, b = 0, c2 = 0;
      OTG_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
      OTG_CUDA(cudaEventElapsedTime(&b, e[1], e[2]));
      OTG_CUDA(cudaEventElapsedTime(&c2, e[2], e[3]));
      acc[0] += a;
      acc[1] += b;
      acc[2] += c2;
    }
    for (auto& x : e) cudaEventDestroy(x);
    if (ms)
      for (int k = 0; k < 3; ++k) ms[k] = acc[k] / reps;
    if (bytes) {
      const double elem = P.storage == OTG_STORE_F64 ? 8.0 : 4.0;
      const double nm = static_cast<double>(P.n_local) * static_cast<double>(P.m);
      bytes[0] = nm * elem + P.m * 8.0 + P.n_local * (2 * 8.0 + 4 * 8.0 + 16.0);
      bytes[1] = nm * elem + P.m * 8.0 + P.n_local * 16.0 +
                 static_cast<double>(P.col_splits) * P.vshards * P.m * 8.0;  // C + aux + partials
      bytes[2] = 0.0;
      if (P.fused) {
        // in-solve single pass: C once, split p (8 B), row state in/out
        // (rowM2, rowJ, a, log a in; u, M, S, w, M2, J, aux out), cluster partials
        bytes[2] = nm * elem + P.m * 8.0 + P.n_local * (8.0 + 4 + 16.0 + 5 * 8.0 + 4 + 16.0) +
                   static_cast<double>(P.fused_clusters + 1) * P.m * 8.0;
      }
    }
  });
}

}  // extern "C"
