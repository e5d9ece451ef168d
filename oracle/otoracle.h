/*
 * otoracle.h — CPU restatement of the reference solver (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle for the B200 path, NOT part of the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library (libotg.so)
 * never links or calls anything in oracle/.
 *
 * It restates, in plain C++ (std::vector<double>, <cmath>, no Eigen),
 * the reference's single-threaded fp64 algorithm for the hot path:
 *   core.cpp:9-93, dual.cpp:22-116, mirror.cpp:21-105, sinkhorn.cpp:20-115,
 *   accel.cpp:137-311, diag.cpp:107-146, rng.hpp:11-58, data.cpp:17-41,69-110
 * (all paths relative to /root/reference/proj/src or include/ot).
 *
 * Parity pinning: the reference cannot be compiled here (Eigen 3, libpng,
 * doctest, CLI11 absent; no network), so the oracle is pinned by the
 * reference's own known-answer tests (tests/golden/kat.json, each value
 * cited to its test file:line) — see tests/test_oracle_kat.py.
 *
 * Cost access: C'_ij = C_ij / cost_div with C given as fp64 (C64) or fp32
 * (C32, up-cast exactly); cost_div = 1 for an already rescaled instance,
 * = epsilon to fold rescale_problem (core.cpp:42-49) into the load.  The
 * division is the same IEEE operation the reference applies once to the
 * whole matrix, so the values are bit-identical to rescaling first.
 */
#ifndef OTORACLE_H
#define OTORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; same numbering as include/otg.h (otg_status). */
enum {
  ORC_OK = 0,
  ORC_E_OT = 1,                 /* plain OtError (config / generic)        */
  ORC_E_OVERFLOW = 2,           /* PotentialOverflow                        */
  ORC_E_DOMAIN = 3,             /* DomainViolation                          */
  ORC_E_GAUGE = 4,              /* GaugeViolation                           */
  ORC_E_INVALID_MARGINALS = 5,  /* InvalidMarginals                         */
  ORC_E_NONPOSITIVE = 6,        /* NonPositiveEntry                         */
  ORC_E_DIMENSION = 7,          /* DimensionMismatch                        */
  ORC_E_TOO_LARGE = 8,          /* DimensionTooLarge                        */
  ORC_E_ORACLE_UNAVAILABLE = 9, /* OracleUnavailable                        */
  ORC_E_DEGENERATE = 10         /* DegenerateColumn                         */
};

typedef struct {
  int64_t n, m;
  const double* a;     /* n */
  const double* b;     /* m */
  const double* C64;   /* n*m row-major, or NULL */
  const float* C32;    /* n*m row-major, or NULL */
  int64_t ldc;         /* row stride in elements (>= m); 0 means m */
  double cost_div;     /* C' = C / cost_div */
} orc_problem;

typedef struct {
  double tol_l1;
  int64_t max_iters;
  int record_trace;
  int64_t trace_stride;
} orc_solve_config;

typedef struct {
  double mu0;
  int64_t m0;
  int64_t max_outer;
  double tol_l1;
  int64_t max_total_inner;
  int rescale_w_across_stages;
  int record_trace;
  int64_t trace_stride;
  int stability;       /* AccelInstrumentation::stability */
} orc_homotopy_config;

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
  int64_t trace_len;     /* records produced (may exceed trace_cap) */
  double r_max_x;        /* RadiusTracker maxima (diag.hpp:120-135), with a reference */
  double r_max_y;
} orc_solve_result;

/* ReferenceSolution (diag.hpp:46-49): the energy / radius columns. */
typedef struct {
  const double* v_star;  /* m */
  double f_star;
} orc_reference;

/* Trace record layout: ORC_TRACE_COLS doubles per row:
 * iter, wall_time_s(=0), marginal_violation_l1, grad_f_l1, reduced_f, mu,
 * alpha, cond1_lhs, cond1_rhs, cond2_lhs, cond2_rhs, metric_drift_inf,
 * energy, radius_x_d, radius_y (NaN = empty optional cell, diag.hpp:15-33). */
#define ORC_TRACE_COLS 15

const char* orc_last_error(void);

/* Worker threads of the O(nm) loops (row sweep, fallback columns, plan
 * statistics); 1 (default) is the reference's single thread.  Deterministic
 * for a given count; equal to the 1-thread result to rounding. */
void orc_set_threads(int nthreads);
int orc_get_threads(void);

/* BASELINE config inputs (SURVEY §8d draw orders), restated independently of
 * the product library's otg_gen_config (bitwise equal, tests/test_oracle_gen.py).
 * cfg 1: out0 = a (n), out1 = b (m), out2 = C (n*m); cfg 2/3/5: out0 = x (n*d),
 * out1 = y (m*d), d = 2/3/3. */
int orc_gen_config(int cfg, int64_t n, int64_t m, uint64_t seed, double* out0, double* out1,
                   double* out2);
int orc_gen_config4(int64_t count, uint64_t seed, int64_t d, int32_t* n, int32_t* m,
                    float* x_cat, float* y_cat);
/* fp32 C = fl32(sum_k (x_ik - y_jk)^2 / max) with row stride ldc: the stored
 * cost of a points instance (SQEUCLID, NORM_MAX, storage F32). */
int orc_cost_sqeuclid_max_f32(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                              int64_t ldc, int nthreads, float* C, double* raw_max);

/* ---- rng.hpp:11-58 ---------------------------------------------------- */
void orc_rng_seed(uint64_t state[4], uint64_t seed);
uint64_t orc_rng_next_u64(uint64_t state[4]);
double orc_rng_next_double(uint64_t state[4]);
uint64_t orc_rng_next_below(uint64_t state[4], uint64_t bound);

/* ---- core.cpp / data.cpp ---------------------------------------------- */
int orc_validate_problem(const orc_problem* p, double epsilon);
int orc_synthetic_instance(int64_t n, int64_t m, uint64_t seed, double* a, double* b,
                           double* C);
int orc_cost_sqeuclidean(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                         double* C, double* raw_min, double* raw_max);
/* norm: 0 = MinMax, 1 = HalfRange, 2 = raw (1 - <x,y>, BASELINE cfg4) */
int orc_cost_cosine(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                    int norm, double* C, double* raw_min, double* raw_max);
/* plan_from_potentials + marginal_violation_l1 + primal_cost (core.cpp:59-79),
 * without keeping P.  eps_ratio = epsilon_original / epsilon. */
int orc_plan_stats(const orc_problem* p, const double* u, const double* v, double eps_ratio,
                   double* row_sums, double* col_sums, double* violation_l1,
                   double* primal_cost);
/* Plan consumers on the plan of plan_from_potentials (pipelines.cpp:58-145). */
int orc_barycentric_projection(const orc_problem* p, const double* u, const double* v,
                               const double* src, int d, double* out);
int orc_predict_translations(const orc_problem* p, const double* u, const double* v, int* out);
int orc_plan_topk(const orc_problem* p, const double* u, const double* v, const int* rows,
                  int64_t nrows, int k, int* out);
void orc_nn_assign(const double* q, int64_t nq, const double* ref, int64_t nref, int d,
                   int* out);

int orc_entropic_objective(const orc_problem* p, const double* u, const double* v,
                           double epsilon, double* out);

/* ---- dual.cpp --------------------------------------------------------- */
int orc_row_solve_marginals(const orc_problem* p, const double* v, double* u, double* col);
int orc_row_solve_marginals_log(const orc_problem* p, const double* v, double* u,
                                double* col, double* col_log);
int orc_dual_F(const orc_problem* p, const double* u, const double* v, double* out);
int orc_hessian_f(const orc_problem* p, const double* v, double* H /* m*m */);

/* ---- mirror.cpp ------------------------------------------------------- */
int orc_grad_phi(const double* b, int64_t m, const double* v, double* out);
int orc_grad_phi_star(const double* b, int64_t m, const double* xi, double* out);
int orc_phi_star(const double* b, int64_t m, const double* xi, double* out);
int orc_bregman_phi_star_from_zero(const double* b, int64_t m, const double* eta,
                                   double* out);
int orc_metric_D(const double* b, int64_t m, const double* z, double* d);
void orc_project_zero_sum(const double* x, int64_t m, double* out);

/* ---- diag.cpp:107-146 ------------------------------------------------- */
int orc_stability_conditions_from_grads(const double* b, int64_t m, const double* grad_k,
                                        const double* grad_k1, const double* x_k,
                                        const double* x_k1, const double* y_k,
                                        const double* y_k1, double alpha,
                                        double out[4] /* c1l c1r c2l c2r */,
                                        int* both_hold, int* skipped, double* drift);

/* ---- sinkhorn.cpp ----------------------------------------------------- */
int orc_eval_normalized_step(const orc_problem* p, const double* v, double* v_next,
                             double* u, double* grad, double* grad_l1, double* f_value);
int orc_sinkhorn_solve(const orc_problem* p, const double* v0, const orc_solve_config* cfg,
                       orc_solve_result* res, double* u_out, double* v_out,
                       double* trace, int64_t trace_cap);

/* ---- accel.cpp -------------------------------------------------------- */
/* One acc_step from (x, w) without a cache (2 evaluations) or with
 * Sx != NULL (cached map at x, 1 evaluation); returns x+, w+, S(x+). */
int orc_acc_step(const orc_problem* p, const double* x, const double* w, const double* Sx,
                 double mu, double* x_out, double* w_out, double* Sx_out,
                 int64_t* eval_count);
/* ref (optional): ReferenceSolution -> energy / radius trace columns. */
int orc_acc_run(const orc_problem* p, const double* x0, const double* w0, double mu,
                int64_t msteps, int record_trace, int64_t trace_stride, int stability,
                orc_solve_result* res, double* x_out, double* w_out, double* trace,
                int64_t trace_cap, const orc_reference* ref);
int orc_acc_solve(const orc_problem* p, const double* v0, double mu,
                  const orc_solve_config* cfg, orc_solve_result* res, double* u_out,
                  double* v_out, double* trace, int64_t trace_cap, const orc_reference* ref);
/* boundaries: up to bcap rows of (stage, mu, alpha, inner_before, energy). */
int orc_homotopy_solve(const orc_problem* p, const orc_homotopy_config* cfg,
                       orc_solve_result* res, double* u_out, double* v_out,
                       double* boundaries, int64_t bcap, double* trace,
                       int64_t trace_cap, const orc_reference* ref);
/* lyapunov_energy_from_parts (diag.cpp:76-88) at (f(x), grad f(x), y, mu). */
int orc_lyapunov_energy(const double* b, int64_t m, double f_x, const double* grad_x,
                        const double* y, double mu, const orc_reference* ref, double* out);
double orc_homotopy_rate_constant(double mu0, double r_hat, double l_f);

/* ---- CPU baseline helpers (bench.py cpu_baseline / --impl reference) ---- */
/* Timing-only variant of one evaluation's O(nm) sweep restricted to rows
 * [row0, row1) with nthreads workers (deterministic per-thread column
 * partials summed in thread order).  Same arithmetic as
 * orc_row_solve_marginals per element. */
int orc_sweep_rows_mt(const orc_problem* p, const double* v, int64_t row0, int64_t row1,
                      int nthreads, double* u, double* col_partial);

/* On-the-fly cost of the B200 path's config 5 (OTG_STORE_ON_THE_FLY): fp32
 * coordinates (d <= 3, missing coordinates 0), C_ij = fmaf(dz, dz, fmaf(dy,
 * dy, dx * dx)) in fp32 with d = x_i - y_j — data.cpp:75-77's squared norm
 * evaluated in this exact fp32 operation order, which defines that instance. */
void orc_cost_sqeuclid_f32(const float* x, const float* y, int64_t n, int64_t m, int64_t d,
                           float* C);

/* max_ij ||x_i - y_j||^2 (the cost_sqeuclidean normaliser, data.cpp:78-80),
 * nthreads workers. */
double orc_sqeuclid_max(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                        int nthreads);

#ifdef __cplusplus
}
#endif
#endif
