/*
 * otg.h — C-ABI of the B200-native Sinkhorn / Acc-Sinkhorn hot path.
 *
 * Drop-in boundary for the reference solver API (otaccel, arXiv 2605.30267;
 * paths below are under /root/reference/proj).  Every entry point names the
 * reference interface it replaces.  No C++ types cross this boundary: plain
 * pointers, sizes and POD structs; errors are status codes, never exceptions.
 *
 * Semantics shared by all solver entry points
 * -------------------------------------------
 * A problem handle owns a device-resident instance.  The solvers always run
 * on the RESCALED instance C' = C / epsilon, epsilon = 1, exactly as the
 * reference requires its callers to apply rescale_problem first
 * (include/ot/dual.hpp:9-13, src/core.cpp:42-49); the handle folds that
 * division into its loads (fp32 storage) or applies it once on upload
 * (fp64 storage), so callers pass the UNSCALED cost and its epsilon.
 * Pass epsilon = 1 for a cost that is already rescaled.
 *
 * Potentials are fp64 on both sides of the boundary.  u has the handle's
 * LOCAL row count (n for an unsharded handle, row_end - row_begin for a
 * row shard), v / x / w / grad have length m.
 *
 * Error mapping (include/ot/types.hpp:21-89): each OTG_E_* code corresponds
 * to the reference exception named beside it; otg_last_error() returns the
 * message of the calling thread's last failure.  Non-convergence is not an
 * error (converged = 0), as in include/ot/sinkhorn.hpp:46.
 *
 * Threading: one handle = one owner (one host thread at a time).  Distinct
 * handles may be used concurrently.  Each handle owns one CUDA stream.
 */
#ifndef OTG_H
#define OTG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTG_ABI_VERSION 1
#define OTG_TRACE_COLS 15 /* see otg_solve_result.trace */

typedef enum {
  OTG_OK = 0,
  OTG_E_OT = 1,                /* OtError (config, non-finite input, generic) */
  OTG_E_OVERFLOW = 2,          /* PotentialOverflow                           */
  OTG_E_DOMAIN = 3,            /* DomainViolation                             */
  OTG_E_GAUGE = 4,             /* GaugeViolation                              */
  OTG_E_INVALID_MARGINALS = 5, /* InvalidMarginals                            */
  OTG_E_NONPOSITIVE = 6,       /* NonPositiveEntry                            */
  OTG_E_DIMENSION = 7,         /* DimensionMismatch                           */
  OTG_E_TOO_LARGE = 8,         /* DimensionTooLarge                           */
  OTG_E_DEGENERATE = 9,        /* DegenerateColumn                            */
  OTG_E_CUDA = 20,             /* CUDA runtime / launch failure               */
  OTG_E_NCCL = 21,             /* NCCL failure (sharded handles)              */
  OTG_E_OOM = 22,              /* device allocation failed                    */
  OTG_E_UNSUPPORTED = 23       /* no CUDA device / feature not built          */
} otg_status;

typedef enum { OTG_F64 = 0, OTG_F32 = 1 } otg_dtype;

/* Cost families of data.cpp:69-110. */
typedef enum { OTG_COST_SQEUCLID = 0, OTG_COST_COSINE = 1 } otg_cost;

/* Normalisation of a cost built from points (data.hpp:59-69):
 * NONE = raw values, MAX = divide by max (cost_sqeuclidean),
 * MINMAX / HALFRANGE = cost_cosine's two modes. */
typedef enum {
  OTG_NORM_NONE = 0,
  OTG_NORM_MAX = 1,
  OTG_NORM_MINMAX = 2,
  OTG_NORM_HALFRANGE = 3
} otg_norm;

/* How a cost built from points is held on the device. */
typedef enum {
  OTG_STORE_F64 = 0,       /* dense fp64 C' (fp64 path: exact exp)          */
  OTG_STORE_F32 = 1,       /* dense fp32 C, fp64 accumulation               */
  OTG_STORE_ON_THE_FLY = 2 /* squared-Euclidean recomputed per tile         */
} otg_storage;

/* Host all-reduce for sharded handles without NCCL (e.g. a torch.distributed
 * gloo group, tests/test_sharded_libotg.py): reduce `count` doubles of `buf`
 * in place across the ranks (op 0 = SUM, 1 = MAX); return 0 on success.
 * libotg stages the device buffer through pinned host memory and calls it
 * from a CUDA host node (cudaLaunchHostFunc), so it must not call CUDA. */
typedef int (*otg_allreduce_fn)(double* buf, int64_t count, int op, void* ctx);

/* Device placement and row sharding.  NULL means { device = current,
 * world_size = 1 }.  Row sharding (world_size > 1, or a 1-rank NCCL id):
 * every rank creates the handle with the FULL a and b and ITS OWN rows
 * [row_begin, row_end) of the row-indexed data -- C (otg_problem_create_dense)
 * or the source points x (otg_problem_create_points) are passed as those
 * n_local = row_end - row_begin rows only.  The ranks agree on the
 * collective: the same 128-byte ncclUniqueId, or the same `allreduce`
 * callback group (then nccl_unique_id is NULL).  The length-m column partial
 * sums (+ <u, a>) are then all-reduced ONCE per evaluation; columns whose
 * global sum underflows take an exact cross-rank LSE exchange that runs only
 * in evaluations that flag some.
 * virtual_shards > 1 splits an unsharded handle's rows into that many shards
 * on ONE device whose partial column sums are combined by an on-device sum
 * standing in for the allreduce (tests the sharded data flow on one GPU). */
typedef struct {
  int device;
  int world_size;
  int rank;
  int64_t row_begin;
  int64_t row_end;
  const void* nccl_unique_id;
  int virtual_shards;
  otg_allreduce_fn allreduce; /* optional host collective (instead of NCCL) */
  void* allreduce_ctx;
  int sweep;                  /* fp32 stored cost: 0 = auto (the single-HBM-pass
                                 sweep for long row-band runs, else two-pass),
                                 1 = the two-pass kernels, 2 = the single pass
                                 whenever its column layout applies */
} otg_device_opts;

typedef struct otg_problem_s* otg_problem;

typedef struct {
  int64_t n, m;            /* global sizes                                  */
  int64_t n_local;         /* rows held by this handle                      */
  int64_t row_begin;       /* first global row held                         */
  int storage;             /* otg_storage                                   */
  double epsilon;          /* epsilon_original of the instance              */
  double cost_raw_min;     /* CostMatrix::raw_min when built from points    */
  double cost_raw_max;     /* CostMatrix::raw_max                           */
  int64_t device_bytes;    /* device memory held by the handle              */
  int world_size, rank, device;
  int sweep_mode;          /* 0: fp64 two-pass, 1: fp32 two-pass, 2: fp32 single pass (k_sweep1) */
  int sweep_clusters;      /* fused: co-resident 8-CTA clusters (persistent)  */
  int col_splits;          /* two-pass: row splits of the column pass         */
} otg_problem_info;

/* StepEval (sinkhorn.hpp:18-24): caller-owned output buffers, any may be NULL. */
typedef struct {
  double* v_next; /* m       */
  double* u;      /* n_local */
  double* grad;   /* m       */
  double grad_l1;
  double f_value;
} otg_step_eval;

/* SolveConfig (sinkhorn.hpp:29-39).  reference_v (m, or NULL) and
 * reference_f form the optional ReferenceSolution (diag.hpp:46-49) that adds
 * the energy / radius trace columns to acc_solve (accel.cpp:211-213). */
typedef struct {
  double tol_l1;
  int64_t max_iters;
  int record_trace;
  int64_t trace_stride;
  const double* reference_v;
  double reference_f;
} otg_solve_config;

/* HomotopyConfig (accel.hpp:68-81). */
typedef struct {
  double mu0;
  int64_t m0;
  int64_t max_outer;
  double tol_l1;
  int64_t max_total_inner;
  int rescale_w_across_stages;
  int record_trace;
  int64_t trace_stride;
} otg_homotopy_config;

/* AccelInstrumentation (accel.hpp:37-40): the stability conditions
 * (diag.cpp:107-146) and, with a ReferenceSolution (reference_v != NULL,
 * diag.hpp:46-49), the Lyapunov energy and radii (diag.cpp:76-88, 206-215),
 * all fused into the evaluation epilogue. */
typedef struct {
  int stability;
  const double* reference_v; /* m, or NULL */
  double reference_f;
} otg_instr;

/* SolveResult (sinkhorn.hpp:44-54) + HomotopyResult (accel.hpp:92-99)
 * scalars.  Output buffers are caller-owned; set the ones you want.
 * trace rows hold OTG_TRACE_COLS doubles: iter, wall_time_s (always 0:
 * byte-stable traces), marginal_violation_l1, grad_f_l1, reduced_f, mu,
 * alpha, cond1_lhs, cond1_rhs, cond2_lhs, cond2_rhs, metric_drift_inf,
 * energy, radius_x_d, radius_y (NaN marks an empty optional cell,
 * diag.hpp:15-33).
 * boundaries rows hold (stage, mu, alpha, inner_before, energy)
 * (accel.hpp:84-90). */
typedef struct {
  int converged;
  int64_t iterations;
  int64_t evaluations;
  int64_t outer_stages;
  double final_violation;
  double final_reduced_f;
  double max_v_inf;
  int64_t conditions_checked;
  int64_t conditions_held;
  double* u;          /* n_local: u(x) of the final evaluation              */
  double* v;          /* m: final potential (v for Sinkhorn, x for Acc)     */
  double* w;          /* m: final momentum w (acc_run / acc solves)         */
  double* trace;      /* trace_cap rows, or NULL                            */
  int64_t trace_cap;
  int64_t trace_len;  /* rows produced (may exceed trace_cap)               */
  double* boundaries; /* boundaries_cap rows of 4, or NULL                  */
  int64_t boundaries_cap;
  int time_sweeps;       /* in: record CUDA events around every row / column
                            pass launch inside the solve                    */
  double device_seconds; /* device time of the whole solve (CUDA events)    */
  double row_pass_seconds; /* summed row-pass launch times (time_sweeps)    */
  double col_pass_seconds; /* summed column-pass launch times (time_sweeps) */
  int64_t kernel_launches; /* kernel nodes replayed by the solve loop        */
  int64_t row_redos;     /* fp32 row pass: rows recomputed exactly because
                            the shift estimate was loose (diagnostic)       */
  double epilogue_seconds; /* summed merge + fallback + finalize + apply
                              times (time_sweeps)                           */
  int64_t fallback_columns; /* columns whose mass underflowed and took the
                               exact log-sum-exp (dual.cpp:54-69), summed
                               over the evaluations (diagnostic)            */
  double radius_x_max;      /* RadiusTracker maxima (diag.hpp:120-135), with a */
  double radius_y_max;      /* reference; r_hat = max of the two            */
} otg_solve_result;

/* plan_from_potentials + marginal_violation_l1 + primal_cost
 * (core.cpp:59-79) evaluated on the implicit plan P = exp(u + v - C'),
 * never materialised.  row_sums (n_local) / col_sums (m) optional. */
typedef struct {
  double marginal_violation_l1;
  double primal_cost;   /* <C, P> in the instance's original cost units */
  double max_exponent;  /* max_ij u_i + v_j - C'_ij                     */
  double* row_sums;
  double* col_sums;
} otg_plan_summary;

/* ---------------------------------------------------------------- */
const char* otg_last_error(void);
int otg_abi_version(void);
otg_status otg_device_count(int* count);
/* ncclGetUniqueId for sharded handles (rank 0 calls it and broadcasts the
 * 128 bytes, e.g. over torch.distributed). */
otg_status otg_nccl_get_unique_id(void* out128);

/* make_problem + rescale_problem (core.cpp:31-49), dense cost.
 * C: n_local x m row-major with row stride ldc (0 = m), dtype fp64 or fp32. */
otg_status otg_problem_create_dense(int64_t n, int64_t m, const double* a, const double* b,
                                    const void* C, otg_dtype dtype, int64_t ldc,
                                    double epsilon, const otg_device_opts* opts,
                                    otg_problem* out);

/* Cost built on the device from points (data.cpp:69-110): x is n_local x d,
 * y is m x d, fp64 row-major.  SQEUCLID with NORM_MAX = cost_sqeuclidean;
 * COSINE with MINMAX / HALFRANGE / NONE = cost_cosine (+ raw, BASELINE cfg4).
 * The normaliser is a global reduction (MAX all-reduce when sharded).
 * STORAGE_ON_THE_FLY (SQEUCLID, NORM_NONE, d <= 3; BASELINE cfg5): the cost
 * fl32((x - y)^2) of the fp32-rounded points is recomputed per tile and never
 * stored.  The instance keeps `epsilon` (info.epsilon, primal-cost unit); the
 * device kernels all scale the cost by the internal 1 / epsilon_int with
 * epsilon_int = log2(e) / fl32(log2(e) / epsilon), within 2^-25 relative of
 * epsilon (the sweeps then multiply by one exact fp32 number).  Parity is
 * tested against the oracle at the true epsilon (tests/test_gpu_otf.py). */
otg_status otg_problem_create_points(int64_t n, int64_t m, int64_t d, const double* a,
                                     const double* b, const double* x, const double* y,
                                     otg_cost cost, otg_norm norm, otg_storage storage,
                                     double epsilon, const otg_device_opts* opts,
                                     otg_problem* out);

otg_status otg_problem_destroy(otg_problem h);
otg_status otg_problem_info_get(otg_problem h, otg_problem_info* out);

/* Copy rows [row0, row0 + nrows) of the stored (unscaled) cost back to the
 * host in its storage dtype (fp32 or fp64).  Parity tests feed this to the
 * oracle so both sides solve bit-identical instances. */
otg_status otg_problem_get_cost(otg_problem h, int64_t row0, int64_t nrows, void* out);

/* row_solve_marginals (dual.cpp:29-42): u(v) and the column sums c_P. */
otg_status otg_row_solve_marginals(otg_problem h, const double* v, double* u, double* col);

/* row_solve_marginals_log (dual.cpp:44-70): + log c_P with the exact
 * column log-sum-exp fallback for underflowed columns. */
otg_status otg_row_solve_marginals_log(otg_problem h, const double* v, double* u,
                                       double* col, double* col_log);

/* eval_normalized_step (sinkhorn.cpp:51-63). */
otg_status otg_eval_normalized_step(otg_problem h, const double* v, otg_step_eval* out);

/* sinkhorn_solve (sinkhorn.cpp:65-115); v0 may be NULL (= 0). */
otg_status otg_sinkhorn_solve(otg_problem h, const double* v0, const otg_solve_config* cfg,
                              otg_solve_result* res);

/* acc_solve (accel.cpp:200-232), fixed mu; v0 may be NULL. */
otg_status otg_acc_solve(otg_problem h, const double* v0, double mu,
                         const otg_solve_config* cfg, otg_solve_result* res);

/* acc_run (accel.cpp:174-198): exactly m_steps accelerated steps from
 * (x0, w0) (zero-sum), m_steps + 1 evaluations. */
otg_status otg_acc_run(otg_problem h, const double* x0, const double* w0, double mu,
                       int64_t m_steps, int record_trace, int64_t trace_stride,
                       const otg_instr* instr, otg_solve_result* res);

/* homotopy_solve_instrumented / homotopy_solve (accel.cpp:234-305). */
otg_status otg_homotopy_solve(otg_problem h, const otg_homotopy_config* cfg,
                              const otg_instr* instr, otg_solve_result* res);

/* Plan statistics over the implicit plan (core.cpp:59-79). */
otg_status otg_plan_stats(otg_problem h, const double* u, const double* v,
                          otg_plan_summary* out);

/* Device timing of the O(nm) sweep kernels at point v: reps launches of
 * each, CUDA events on the handle's stream.  These are the first-evaluation
 * (exact, two-pass) kernels.  ms[0] = row pass, ms[1] = column pass, ms[2] =
 * merge.  bytes[0..1] = algorithmic HBM bytes of one row / column pass
 * launch; bytes[2] = those of one steady-state single-pass launch (fused.cu;
 * 0 when the handle has no single-pass kernel). */
otg_status otg_time_sweeps(otg_problem h, const double* v, int reps, double ms[3],
                           double bytes[3]);

/* ---- plan consumers over the implicit plan P = exp(u + v - C') ----
 * (SURVEY §8f row 1).  P is never materialised: each call streams the cost
 * once and rebuilds P_ij = exp(((-C'_ij) + u_i) + v_j) (core.cpp:63-70) in
 * fp64; PotentialOverflow if an exponent exceeds 700 (core.cpp:66-69).  u is
 * the handle's local rows (row shard), v all m columns. */

/* barycentric_projection (pipelines.cpp:58-71): out[j][k] = sum_i P_ij src[i][k]
 * / sum_i P_ij, src is n_local x d row-major (1 <= d <= 8), out m x d;
 * DegenerateColumn (OTG_E_DEGENERATE) if a column has zero mass.  col_mass
 * (optional, m) receives sum_i P_ij.  Sharded handles all-reduce the sums. */
otg_status otg_plan_barycentric(otg_problem h, const double* u, const double* v,
                                const double* src, int d, double* out, double* col_mass);

/* predict_translations (pipelines.cpp:101-111): out[i] = argmax_j P_ij,
 * ties to the lowest index (n_local entries). */
otg_status otg_plan_row_argmax(otg_problem h, const double* u, const double* v, int* out);

/* The per-source ranking of topk_accuracy (pipelines.cpp:113-145): for each
 * row rows[b], the k columns with the largest P (value descending, index
 * ascending on ties) into out[b * k + r]; -1 past m.  OtError if k < 1. */
otg_status otg_plan_topk(otg_problem h, const double* u, const double* v, const int* rows,
                         int64_t nrows, int k, int* out);

/* The nearest-sample search of nn_propagate (pipelines.cpp:80-92): out[p] =
 * argmin_s ||queries[p] - refs[s]||^2 in fp64, strict < so ties go to the
 * lowest index; d in 1..4, row-major. */
otg_status otg_nn_assign(const double* queries, int64_t nq, const double* refs, int64_t nref,
                         int d, int device, int* out);

/* ---- diagnostics (dual.hpp) ---- */

/* dual_F (dual.cpp:88-101): exp(LSE_ij(u_i + v_j - C'_ij)) - <u, a> - <v, b>;
 * PotentialOverflow above exponent 700. */
otg_status otg_dual_F(otg_problem h, const double* u, const double* v, double* out);

/* hessian_f (dual.cpp:118-136): H = diag(c(v)) - P^T diag(a)^{-1} P at the row
 * solve of v, m x m row-major; DimensionTooLarge past m = 2000. */
otg_status otg_hessian_f(otg_problem h, const double* v, double* H);

/* ---- batched path: many small independent problems, one CTA each ---- */
typedef struct otg_batch_s* otg_batch;

/* Problems p = 0..count-1 with sizes n[p], m[p] <= 64; a, b concatenated;
 * C concatenated row-major per problem (fp32). */
otg_status otg_batch_create_dense(int64_t count, const int32_t* n, const int32_t* m,
                                  const double* a_cat, const double* b_cat,
                                  const float* C_cat, double epsilon,
                                  const otg_device_opts* opts, otg_batch* out);
/* Cosine costs from unit embeddings (fp32, d-dim): x_cat holds sum n[p] rows,
 * y_cat sum m[p] rows.  norm as otg_problem_create_points. */
otg_status otg_batch_create_cosine(int64_t count, const int32_t* n, const int32_t* m,
                                   int64_t d, const double* a_cat, const double* b_cat,
                                   const float* x_cat, const float* y_cat, otg_norm norm,
                                   double epsilon, const otg_device_opts* opts,
                                   otg_batch* out);
otg_status otg_batch_destroy(otg_batch h);
/* Copy the stored cost of the batch back (concatenated, fp32). */
otg_status otg_batch_get_cost(otg_batch h, float* out);

/* Per-problem homotopy_solve; arrays have `count` entries (or are NULL);
 * u_cat / v_cat are concatenated like a / b. */
typedef struct {
  int32_t* converged;
  int64_t* iterations;
  double* final_violation;
  double* final_reduced_f;
  double* u_cat;
  double* v_cat;
  double device_seconds;
  int64_t total_iterations;
} otg_batch_result;
otg_status otg_batch_homotopy_solve(otg_batch h, const otg_homotopy_config* cfg,
                                    otg_batch_result* res);

/* ---- seeded synthetic inputs (rng.hpp:11-58 xoshiro256++) ---- */
/* Reference generator data.cpp:17-32 (a, b, C ~ U[0,1), normalised, C to
 * total sum 1). */
otg_status otg_gen_synthetic_instance(int64_t n, int64_t m, uint64_t seed, double* a,
                                      double* b, double* C);
/* BASELINE config inputs.  cfg 1: a, b = 1 - 0.9 U normalised, C = U[0,1)
 * (out: a, b, C).  cfg 2: x ~ N(0, I2), y ~ N((2,0), diag(0.5, 2)).
 * cfg 3: x ~ Beta(2,5)^3, y ~ Beta(5,2)^3.  cfg 5: x ~ U[0,1]^3, y from a
 * 3-component Gaussian mixture (sigma 0.1) clipped to [0,1]^3.
 * For cfg 2/3/5: out0 = x (n x d), out1 = y (m x d), out2 unused. */
otg_status otg_gen_config(int cfg, int64_t n, int64_t m, uint64_t seed, double* out0,
                          double* out1, double* out2);
/* cfg 4: n[p], m[p] = 8 + next_below(57); embeddings N(0,I) normalised to
 * unit length, stored fp32.  Draw order: for p in 0..count-1: n_p, m_p, x_p (n_p x d normals, row-major),
 * y_p (m_p x d).  Call once with x_cat = y_cat = NULL to get the sizes, then
 * again with buffers of sum(n) x d and sum(m) x d floats. */
otg_status otg_gen_config4(int64_t count, uint64_t seed, int64_t d, int32_t* n, int32_t* m,
                           float* x_cat, float* y_cat);

/* ---- test hooks ---- */
/* On-the-fly handles visit rows and columns in Morton order in their
 * steady-state sweeps and skip blocks whose every exponent is provably below
 * -127 (ex2.approx.ftz returns +0 there: the skip is bitwise invisible).
 * mode 1 (default): culled; 0: same sorted order, every block visited (the
 * bitwise reference for the skip); -1: handles created afterwards keep the
 * caller's order (the dense original sweeps).  Returns the previous mode.
 * No reference counterpart (internal to the GPU sweeps). */
int otg_debug_cull(int mode);
/* Fraction of (warp tile x block) pairs the culled sweeps visit at the
 * handle's current state: out[0] row pass (256 sorted rows x 64 sorted
 * columns), out[1] column pass (128 sorted columns x 16 sorted rows); -1 when
 * the handle is not culled.  Diagnostic (bench roofline). */
otg_status otg_cull_stats(otg_problem h, double out[2]);

#ifdef __cplusplus
}
#endif
#endif /* OTG_H */
