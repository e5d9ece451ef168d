// common.cuh — shared internals of libotg (B200 / sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/otg.h"

// Compile-time tuning defaults (A/B builds: tools/ab_build.sh NAME SRC "-DOTG_...=x").
// The shipped library reads no environment knobs that change its behaviour.
#ifndef OTG_PDL
#define OTG_PDL 1            // programmatic dependent launch on every graph kernel
#endif
#ifndef OTG_ROW_R
#define OTG_ROW_R 0          // fp32 row pass rows per CTA (0 = auto: 4 stored, 8 on the fly)
#endif
#ifndef OTG_ONLINE_FIRST
#define OTG_ONLINE_FIRST 1   // first evaluation with the fp32 online-shift row pass
#endif
#ifndef OTG_COL_T
#define OTG_COL_T 0          // column-pass CTA width (0 = auto: 256)
#endif
#ifndef OTG_COL_SPLITS
#define OTG_COL_SPLITS 0     // column-pass row splits (0 = auto: whole waves)
#endif
#ifndef OTG_ROW_OTF_T
#define OTG_ROW_OTF_T 1      // on the fly: the transposed row pass
#endif
#ifndef OTG_ROW_PF
#define OTG_ROW_PF -1        // row-pass L2 prefetch (-1 = auto)
#endif
#ifndef OTG_CULL
#define OTG_CULL 1  // on-the-fly sweeps: Morton-ordered, exact (FTZ) block culling
#endif
#ifndef OTG_CULL_COL_SPLITS
#define OTG_CULL_COL_SPLITS 64  // culled on-the-fly column pass: row splits
#endif
#ifndef OTG_CULL_ROW_WAVES
#define OTG_CULL_ROW_WAVES 16   // culled on-the-fly row pass: waves of column splits
#endif
#ifndef OTG_CULL_ROW_T
#define OTG_CULL_ROW_T 128  // culled row pass: threads per CTA (warps are independent)
#endif
#ifndef OTG_CULL_RT
#define OTG_CULL_RT 4       // culled row pass: rows per thread (warp tile = 32 x this)
#endif
#ifndef OTG_CULL_COL_T
#define OTG_CULL_COL_T 128  // culled column pass: threads per CTA
#endif
#ifndef OTG_FIN_SORTED_FB
#define OTG_FIN_SORTED_FB 0  // k_finalize's folded fallback: column-sorted work items (32 KB smem)
#endif

#include <nvtx3/nvToolsExt.h>  // (header-only NVTX v3: ranges cost nothing without a tool)

namespace otg {

// NVTX range over a C-ABI call or a chunk replay (nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define OTG_RANGE(name) ::otg::NvtxRange otg_nvtx_range_(name)

// ---------------------------------------------------------------- errors --
struct Error {
  otg_status code;
  std::string msg;
};

[[noreturn]] inline void fail(otg_status code, const std::string& msg) { throw Error{code, msg}; }

void set_last_error(const std::string& msg);

#define OTG_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess)                                                          \
      ::otg::fail(_e == cudaErrorMemoryAllocation ? OTG_E_OOM : OTG_E_CUDA,         \
                  std::string(#call) + ": " + cudaGetErrorString(_e));              \
  } while (0)

template <class F>
otg_status guard(F&& f) {
  try {
    f();
    return OTG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return OTG_E_OT;
  }
}

// --------------------------------------------------------------- numerics --
constexpr double kLog2e = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;
constexpr double kExpOverflowBound = 700.0;  // types.hpp:15
constexpr double kGradFloor = 1e-12;         // types.hpp:19
constexpr double kTinyPrecise = 1e-280;      // dual.cpp:53 (fp64 path: same threshold)
constexpr double kTinyFast = 1e-30;          // fp32 ex2.ftz path: flushed mass <= 1.2e-38
constexpr float kQuant = 256.0f;             // 2^8 quantum of the split shifts

// On-the-fly squared-Euclidean cost of fp32 points (x, y, z, 0): the
// definition of the instance for OTG_STORE_ON_THE_FLY (the oracle evaluates
// the same fp32 operations in the same order).
#ifdef __CUDACC__
__device__ __forceinline__ float otf_sqeuclid(const float4& x, const float4& y) {
  const float dx = __fsub_rn(x.x, y.x), dy = __fsub_rn(x.y, y.y), dz = __fsub_rn(x.z, y.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// C'_ij of any storage, in fp64: fp64 C' (stored divided), fp32 C x 1/eps, or
// the on-the-fly fp32 cost of the points x 1/eps (plan statistics, consumers).
__device__ __forceinline__ double cost_at(const double* __restrict__ C64,
                                          const float* __restrict__ C32,
                                          const float4* __restrict__ X,
                                          const float4* __restrict__ Y, int64_t ldc, double kappa,
                                          int64_t i, int64_t j) {
  if (C64) return C64[i * ldc + j];
  if (C32) return static_cast<double>(C32[i * ldc + j]) * kappa;
  return static_cast<double>(otf_sqeuclid(X[i], Y[j])) * kappa;
}
#endif

// -------------------------------------------- programmatic dependent launch --
// Every graph kernel is launched with programmatic stream serialization and
// starts with griddepcontrol.wait: the next kernel's grid is set up while the
// previous one drains (no early trigger, so no resource contention), then it
// waits for the previous grid's completion and memory flush before touching
// its outputs.  OTG_PDL=0 turns the attribute off (plain stream order).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  OTG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// ------------------------------------------------------------ loop control --
enum Mode : int {
  MODE_EVAL = 0,       // one eval_normalized_step
  MODE_SINKHORN = 1,   // sinkhorn.cpp:65-115
  MODE_ACC = 2,        // acc_solve accel.cpp:200-232
  MODE_ACC_RUN = 3,    // acc_run accel.cpp:174-198
  MODE_HOMOTOPY = 4,   // homotopy_solve_instrumented accel.cpp:234-301
};

// Device-resident control block.  The last CTA of the finalize epilogue runs
// the solver's scalar control flow (stop test, homotopy schedule, trace) so
// the iteration never round-trips to the host.
// Ctrl::done values: 0 running, 1 finished (stop rule / cap / error), and
// kPaused: a sharded chunk graph stopped at an evaluation whose flagged
// columns need the cross-rank exact-LSE exchange (run eagerly by the host).
constexpr int kPaused = 2;

struct Ctrl {
  // --- status (device-written) ---
  int done;
  int converged;
  int capped;
  int error;          // otg_status raised on the device (DomainViolation, ...)
  int stage_changed;  // this eval closed a homotopy stage
  int is_step;        // the eval in flight is an accelerated step (not a seed)
  int have_prev;      // stability: previous observation stored
  int live_e2;        // finalize -> apply handoff for the current eval
  int fin_done;       // steady single pass: k_sp_patch_merge finalized this eval (no flags)
  long long k;        // observation index (sinkhorn / acc / acc_run)
  long long evaluations;
  long long iterations;
  long long total_inner, stage, inner_i, m_stage, outer_stages;
  double mu, alpha_step, alpha_next;
  double grad_l1, f_value, mean_y, max_v_inf;
  double final_violation, final_f;
  long long trace_count;   // records produced
  long long trace_row;     // ring slot of the current eval's record, -1 none
  long long boundary_count;
  long long cond_checked, cond_held;
  long long live_kernels;
  unsigned int e1_counter, e2_counter, fb_count, redo_count;
  unsigned int bar_count, bar_gen;  // (unused: the round-1 one-kernel epilogue's grid barrier)
  // fp32 row pass: shift estimate from the previous evaluation (sweep.cu)
  int shift_valid;    // rowM2 / vq describe the previous point, dmax2 the step
  int pad1;
  double dmax2;       // max_j (p_new - p_old)_j * log2(e)
  long long redo_total;  // rows redone exactly over the solve (diagnostic)
  // ReferenceSolution instrumentation (energy / radii, diag.cpp:76-88, 206-215)
  int have_ref;
  int boundary_pending;  // control_step pushed a boundary row this evaluation
  double f_star;
  double mu_step;        // mu of the evaluation being observed (before a halving)
  double rmax_x, rmax_y;
  long long fb_total;    // columns that took the exact LSE fallback (diagnostic)
  // --- configuration (host-written) ---
  int mode;
  int record_trace;
  int stability;
  int rescale_w;
  double tol;
  long long max_iters;       // sinkhorn / acc
  long long trace_stride;
  long long max_outer;
  long long max_total_inner;
  long long m0;
  long long msteps;          // acc_run
  double mu0;
  double tiny;               // fallback threshold for c_j
  long long trace_cap;       // ring capacity
  long long boundary_cap;
};

constexpr int kTraceCols = OTG_TRACE_COLS;
constexpr int kBoundCols = 5;  // stage, mu, alpha, inner_before, energy
constexpr int kEpiMaxGrid = 296;  // CTAs of the single-kernel epilogue, at most

// ---------------------------------------------------------------- problem --
struct Shard {
  int64_t row0 = 0;  // first local row of the shard
  int64_t rows = 0;
};

struct Problem {
  // sizes
  int64_t n = 0, m = 0, n_local = 0, row_begin = 0;
  int64_t ldc = 0;  // row stride of C in elements (multiple of 4)
  int storage = OTG_STORE_F64;
  double epsilon = 1.0;   // epsilon_original
  double kappa = 1.0;     // 1 / epsilon (fp32 path multiplies on load)
  double raw_min = 0.0, raw_max = 0.0;
  int device = 0;
  int world = 1, rank = 0;
  int sharded = 0;  // rows split across ranks; column sums all-reduced over NCCL
  double* fbA = nullptr;  // sharded fallback: per-column global top (MAX all-reduce)
  double* fbS = nullptr;  //                   per-column rescaled sums (SUM all-reduce)
  double* fbT = nullptr;  //                   per-column local top
  int vshards = 1;

  cudaStream_t stream = nullptr;

  // cost
  double* C64 = nullptr;  // fp64: C' = C / eps (pre-divided, core.cpp:42-49)
  float* C32 = nullptr;   // fp32: raw C
  float* X = nullptr;     // on-the-fly: x (n_local x 4 padded), y (m x 4)
  float* Y = nullptr;
  float* Yn = nullptr;    // on-the-fly: -y as SoA [x | y | z], stride mpad (packed kernels)
  // on the fly, culled sweeps (sweep.cu: k_row_otf<true>, k_col_fast<true, T, true>):
  // Morton orders of the rows and columns, the points in those orders, the
  // static boxes of the culling blocks and their per-evaluation potential bounds
  int cull = 0;
  int* perm_r = nullptr;
  int* perm_c = nullptr;
  float* Xs = nullptr;    // n_local x 4, sorted rows
  float* Yns = nullptr;   // -y SoA in sorted column order, stride mpad
  float* cbox = nullptr;  // 2 float4 per 64 sorted columns
  float* rbox = nullptr;  // 2 float4 per 16 sorted rows
  float* cvmax = nullptr;
  float* rnegm = nullptr;
  float* ves = nullptr;   // float2 per sorted column: (V, 2^F), per evaluation
  float* auxs = nullptr;  // float4 per sorted row: aux (w pre-scaled), per evaluation

  // marginals (fp64)
  double *a = nullptr, *loga = nullptr, *b = nullptr, *logb = nullptr;

  // per-row state (n_local)
  double *rowM = nullptr, *rowS = nullptr, *u = nullptr, *wrow = nullptr;
  float4* aux = nullptr;  // fast path: {Mc, mf, w, 0} (base-2 split row shift)
  double* rowM2 = nullptr;  // fast path: base-2 row max of the previous evaluation
  int* rowJ = nullptr;      // fast path: its argmax column
  double* dq = nullptr;     // fast path: (p_new - p_old) * log2(e) per column
  int* redo_rows = nullptr; // rows whose shift estimate was off (exact redo)
  float* vq = nullptr;      // fast path: split column potential (Vc[mpad], vf[mpad], 2^vf[mpad])

  // per-column state (m, padded)
  double *p = nullptr, *wacc = nullptr, *col = nullptr, *col_log = nullptr, *y = nullptr,
         *grad = nullptr;
  double *prev_grad = nullptr, *prev_x = nullptr, *prev_y = nullptr;
  int* flag_idx = nullptr;  // fallback slot per column (-1 none)
  int* fb_cols = nullptr;   // flagged column list (m)
  double2* fb_part = nullptr;  // (max, sum) per flagged column per row chunk

  // single-pass sweep (fused.cu), fp32 storage only.  fused_clusters = H
  // groups of sp_group CTAs (one per SM); each group streams every H-th row
  // band and writes one row of column partials (merge sums H + 1 rows).
  int fused = 0, fused_slots = 0, fused_smem = 0, fused_clusters = 0;
  int two_pass = 0;             // otg_device_opts.sweep == 1: never the single pass
  int force_single_pass = 0;    // otg_device_opts.sweep == 2: single pass whenever it applies
  int sp_group = 0;             // CTAs (SMs) sharing one row band
  int sp_fix = 28;              // fixed-point scale 2^sp_fix of the row sums
  int sp_bw = 0, sp_nbox = 0;   // TMA box: chunk width (columns), chunks per slice
  alignas(64) unsigned char sp_tmap[128] = {};  // CUtensorMap of the stored cost (2-D)
  int64_t sp_cap = 0;           // capacity of each CTA's loose-row list
  double* sp_rec = nullptr;     // per-row 32-byte records (shift estimate, a, log a)
  int* sp_bad_rows = nullptr;   // rows whose shift estimate was loose, per CTA (row order)
  int* sp_bad_count = nullptr;
  void* sp_sums = nullptr;      // [2][n] fixed-point row sums, [2][n] (max, argmax) keys
  unsigned* sp_cnt = nullptr;   // [0] buffer parity of the next launch, [1] finished CTAs
  // the row statistics at the zero point (p = 0): base-2 row max upper bound
  // and argmin column of the stored cost, so a solve that starts at 0 runs
  // the single pass from its first evaluation (no exact two-pass seed)
  double* sp_zM2 = nullptr;
  int* sp_zJ = nullptr;

  // on-the-fly transposed row pass (k_row_otf): column splits and their
  // per-row partials (row_splits x n_local records of 16 B)
  int row_splits = 0;  // 0: the row_shift_block kernel instead
  int64_t row_cols_per_split = 0;
  void* rpart = nullptr;

  // column-pass partials
  int col_splits = 1;
  int col_threads = 128;  // fp32 column pass CTA width (4 columns per thread)
  int epi_grid = 0;       // single-kernel epilogue CTAs (0 = unset, -1 = unavailable)
  int apply_pending = 0;  // launch_eval left the vector update to launch_apply
  int64_t rows_per_split = 0;
  double* part = nullptr;  // (vshards * col_splits) x mpad

  // epilogue scratch
  int e_blocks = 1;
  double* e1_part = nullptr;  // e_blocks x 8
  double* e2_part = nullptr;  // e_blocks x 8
  Ctrl* ctrl = nullptr;
  Ctrl* ctrl_host = nullptr;  // pinned mirror
  double* trace = nullptr;    // ring: trace_cap x kTraceCols
  double* vstar = nullptr;    // ReferenceSolution v* (m), allocated on first use
  double* bounds = nullptr;   // boundary_cap x 4

  int64_t mpad = 0;
  int64_t device_bytes = 0;

  // captured solver chunk graphs (lazily built)
  cudaGraphExec_t chunk_exec = nullptr;
  cudaGraphExec_t chunk_exec_timed = nullptr;
  int chunk_len = 0;
  int chunk_kernels = 0, chunk_kernels_timed = 0;  // kernel nodes per chunk graph
  std::vector<cudaEvent_t> chunk_events;  // 5 per iteration (timed graph)

  // collective of a sharded handle: NCCL, or a caller-supplied host
  // all-reduce (otg_device_opts.allreduce) staged through pinned memory
  void* nccl_comm = nullptr;
  otg_allreduce_fn ar_fn = nullptr;
  void* ar_ctx = nullptr;
  double* ar_host = nullptr;  // pinned staging of the host all-reduce
  size_t ar_host_len = 0;
  double* red = nullptr;      // sharded: this rank's merged column partials (+ <u, a>)
  int capturing = 0;          // launch_eval is being captured into the chunk graph
  // single-pass handles: a second chunk graph for evaluations that follow one
  // (shift estimates valid): no exact-path kernels, merge folded into the patch
  int steady_capture = 0;     // the steady graph is being captured
  cudaGraphExec_t chunk_exec_steady = nullptr;
  int chunk_kernels_steady = 0;
};

// allocation helpers (track bytes)
template <class T>
T* dalloc(Problem& P, size_t count) {
  if (count == 0) count = 1;
  void* ptr = nullptr;
  OTG_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
  P.device_bytes += static_cast<int64_t>(count * sizeof(T));
  // per-row / per-column state starts zeroed (no kernel or diagnostic can
  // read uninitialised indices); the cost itself (>= 1 GiB) is written in full
  if (count * sizeof(T) < (size_t{1} << 30))
    OTG_CUDA(cudaMemsetAsync(ptr, 0, count * sizeof(T), P.stream));
  return static_cast<T*>(ptr);
}

void problem_free(Problem& P);
// E1 (finalize) partials: one per group of 32 consecutive columns
__host__ __device__ inline int64_t e1_groups_of(int64_t m) { return (m + 31) / 32; }
Problem& problem_of(otg_problem h);  // handle -> problem (sets the device)
void problem_alloc_state(Problem& P);

// sweeps / epilogue (sweep.cu)
void launch_eval(Problem& P, bool with_log, bool timed, cudaEvent_t* ev4);
void launch_apply(Problem& P);
void launch_fallback_and_finalize(Problem& P);  // sharded pause: the eager rest of an eval
void launch_row_pass(Problem& P);
void launch_col_pass(Problem& P);
void launch_merge_nolog(Problem& P);
void launch_sweeps(Problem& P, bool timed, cudaEvent_t* ev4);
void launch_split_p(Problem& P);  // vq <- split of p (after the host sets p)
struct SpLayout {  // column layout of the single-pass sweep (fused.cu)
  bool ok = false;
  int H = 0, group = 0, cw = 0, nch = 0;
};
SpLayout sp_layout(int64_t m, int sms);
bool fused_configure(Problem& P);
void fused_alloc(Problem& P);
void launch_fused(Problem& P, float kh, float kl);
void launch_sp_redo(Problem& P, const int* bad_rows, const int* bad_count, int ncl, int64_t cap);
// unsharded single pass: the loose rows' column patch + the merge of the
// partial rows + the underflow flags + <u, a> in one kernel (sweep.cu)
void launch_sp_patch_merge(Problem& P, float kh, float kl, int nlists);
inline bool patch_merges(const Problem& P) { return P.fused && !P.sharded; }
int partial_rows(const Problem& P);  // rows of P.part the merge sums

// collectives of a sharded handle (comm.cpp).  recv may equal send.  Both
// are stream-ordered on P.stream and capturable into the chunk graph.
void comm_init(Problem& P, const otg_device_opts* opts);
void comm_destroy(Problem& P);
int comm_failed(Problem& P);  // a host all-reduce callback returned non-zero
void comm_sync(Problem& P);    // stream wait; sharded NCCL handles poll the async error state
void comm_allreduce_sum(Problem& P, const double* send, double* recv, size_t count);
void comm_allreduce_max(Problem& P, const double* send, double* recv, size_t count);
inline void comm_allreduce_sum(Problem& P, double* buf, size_t count) {
  comm_allreduce_sum(P, buf, buf, count);
}
inline void comm_allreduce_max(Problem& P, double* buf, size_t count) {
  comm_allreduce_max(P, buf, buf, count);
}

inline int64_t round_up(int64_t x, int64_t k) { return (x + k - 1) / k * k; }

}  // namespace otg

struct otg_problem_s {
  otg::Problem P;
};
