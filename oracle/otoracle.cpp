// otoracle.cpp — CPU restatement of the reference hot path (TEST INFRASTRUCTURE;
// see otoracle.h for the rules on who may load it).  Every function cites the
// reference file:line it follows (paths under /root/reference/proj).  The
// order of floating-point operations inside each element follows the
// reference expressions; only Eigen's internal reduction order (unpinned,
// SURVEY §8c) is replaced by plain left-to-right sums.
#include "otoracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using Vec = std::vector<double>;

thread_local std::string g_err;

struct OrcError : std::runtime_error {
  int code;
  OrcError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& what) { throw OrcError(code, what); }

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return ORC_OK;
  } catch (const OrcError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_E_OT;
  }
}

constexpr double kExpOverflowBound = 700.0;  // types.hpp:15
constexpr double kGradFloor = 1e-12;         // types.hpp:19

// C'_ij with the fold of rescale_problem (core.cpp:42-49).
struct Cost {
  const double* c64;
  const float* c32;
  int64_t ld;
  double div;
  double operator()(int64_t i, int64_t j) const {
    const double c = c64 ? c64[i * ld + j] : static_cast<double>(c32[i * ld + j]);
    return div == 1.0 ? c : c / div;
  }
};

struct Prob {
  int64_t n, m;
  const double* a;
  const double* b;
  Cost C;
};

Prob wrap(const orc_problem* p) {
  if (!p || p->n < 1 || p->m < 1) fail(ORC_E_DIMENSION, "empty marginal");
  if (!p->C64 && !p->C32) fail(ORC_E_DIMENSION, "no cost matrix");
  Prob q;
  q.n = p->n;
  q.m = p->m;
  q.a = p->a;
  q.b = p->b;
  q.C = Cost{p->C64, p->C32, p->ldc > 0 ? p->ldc : p->m, p->cost_div};
  return q;
}

double sum(const Vec& x) {
  double s = 0.0;
  for (double v : x) s += v;
  return s;
}

double inf_norm(const double* x, int64_t m) {
  double r = 0.0;
  for (int64_t j = 0; j < m; ++j) r = std::max(r, std::abs(x[j]));
  return r;
}

// mirror.cpp:103-105
Vec project_zero_sum(const Vec& x) {
  const double mean = sum(x) / static_cast<double>(x.size());
  Vec out(x.size());
  for (size_t j = 0; j < x.size(); ++j) out[j] = x[j] - mean;
  return out;
}

void check_zero_sum(const Vec& x, const char* what) {  // accel.cpp:21-25
  const double s = sum(x);
  if (std::abs(s) > 1e-9) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "%s must be zero-sum, got sum %.3g", what, s);
    fail(ORC_E_GAUGE, buf);
  }
}

// core.cpp:9-29 (+ epsilon check)
void validate(const Prob& p, double epsilon) {
  if (!(epsilon > 0.0) || !std::isfinite(epsilon)) fail(ORC_E_OT, "epsilon must be positive and finite");
  for (int64_t i = 0; i < p.n; ++i)
    for (int64_t j = 0; j < p.m; ++j)
      if (!std::isfinite(p.C(i, j))) fail(ORC_E_OT, "cost matrix has non-finite entries");
  const double* ms[2] = {p.a, p.b};
  const int64_t ls[2] = {p.n, p.m};
  for (int k = 0; k < 2; ++k) {
    double mn = ms[k][0], s = 0.0;
    for (int64_t j = 0; j < ls[k]; ++j) {
      mn = std::min(mn, ms[k][j]);
      s += ms[k][j];
    }
    if (!(mn > 0.0)) fail(ORC_E_INVALID_MARGINALS, "marginals must be strictly positive");
    if (std::abs(s - 1.0) > 1e-9) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "marginal sums to %.17g, expected 1", s);
      fail(ORC_E_INVALID_MARGINALS, buf);
    }
  }
}

// dual.cpp:13-18
void check_v(const Prob& p, const double* v) {
  for (int64_t j = 0; j < p.m; ++j)
    if (!std::isfinite(v[j])) fail(ORC_E_OT, "v has non-finite entries");
}

// Worker count for the O(nm) loops (orc_set_threads; 1 = the reference's
// single thread).  Rows are split into T contiguous blocks; every thread keeps
// its own column partial and the partials are summed in thread order, so a
// run is deterministic for a given T and equals the T = 1 result to rounding
// (tests/test_oracle_kat.py checks 1e-15).
int g_threads = 1;

template <class F>
void parallel_blocks(int64_t n, int T, F&& fn) {
  if (T <= 1 || n < 2 * T) {
    fn(0, int64_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back([&, t] { fn(t, n * t / T, n * (t + 1) / T); });
  fn(0, int64_t{0}, n / T);
  for (auto& x : th) x.join();
}

// dual.cpp:29-42 — streamed one row at a time (T never materialised; the
// per-element arithmetic and the i-ordered GEMV accumulation are unchanged).
void row_block(const Prob& p, const double* v, int64_t lo, int64_t hi, double* u, double* col) {
  Vec T(p.m);
  for (int64_t i = lo; i < hi; ++i) {
    double mx = -std::numeric_limits<double>::infinity();
    for (int64_t j = 0; j < p.m; ++j) {
      T[j] = (-p.C(i, j)) + v[j];  // (-C).rowwise() + v^T   dual.cpp:34
      mx = std::max(mx, T[j]);     // rowwise maxCoeff        dual.cpp:35
    }
    double rs = 0.0;
    for (int64_t j = 0; j < p.m; ++j) {
      T[j] = std::exp(T[j] - mx);  // dual.cpp:36
      rs += T[j];                  // dual.cpp:37
    }
    u[i] = (std::log(p.a[i]) - mx) - std::log(rs);  // dual.cpp:38
    const double wi = p.a[i] / rs;                   // a.cwiseQuotient(row_sum)
    for (int64_t j = 0; j < p.m; ++j) col[j] += T[j] * wi;  // T^T w  dual.cpp:41
  }
}

void row_solve_marginals(const Prob& p, const double* v, double* u, double* col) {
  check_v(p, v);
  for (int64_t j = 0; j < p.m; ++j) col[j] = 0.0;
  const int T = static_cast<int>(std::min<int64_t>(g_threads, p.n));
  if (T <= 1) {
    row_block(p, v, 0, p.n, u, col);
    return;
  }
  std::vector<Vec> parts(T, Vec(p.m, 0.0));
  parallel_blocks(p.n, T, [&](int t, int64_t lo, int64_t hi) {
    row_block(p, v, lo, hi, u, parts[t].data());
  });
  for (int64_t j = 0; j < p.m; ++j) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += parts[t][j];
    col[j] = s;
  }
}

// dual.cpp:44-70 (the exact column LSE of each flagged column is independent:
// flagged columns are spread over the workers, each column summed in i order)
void row_solve_marginals_log(const Prob& p, const double* v, double* u, double* col,
                             double* col_log) {
  row_solve_marginals(p, v, u, col);
  constexpr double tiny = 1e-280;
  std::vector<int64_t> flagged;
  for (int64_t j = 0; j < p.m; ++j) {
    if (col[j] >= tiny)
      col_log[j] = std::log(col[j]);
    else
      flagged.push_back(j);
  }
  const int64_t nf = static_cast<int64_t>(flagged.size());
  parallel_blocks(nf, g_threads, [&](int, int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t j = flagged[k];
      double top = -std::numeric_limits<double>::infinity();
      for (int64_t i = 0; i < p.n; ++i) top = std::max(top, u[i] + v[j] - p.C(i, j));
      double s = 0.0;
      for (int64_t i = 0; i < p.n; ++i) s += std::exp(u[i] + v[j] - p.C(i, j) - top);
      col_log[j] = top + std::log(s);
      col[j] = std::exp(col_log[j]);
    }
  });
}

struct StepEval {  // sinkhorn.hpp:18-24
  Vec v_next, u, grad;
  double grad_l1 = 0.0, f_value = 0.0;
};

// sinkhorn.cpp:51-63
StepEval eval_normalized_step(const Prob& p, const double* v) {
  StepEval e;
  e.u.assign(p.n, 0.0);
  Vec col(p.m), col_log(p.m);
  row_solve_marginals_log(p, v, e.u.data(), col.data(), col_log.data());
  for (int64_t j = 0; j < p.m; ++j)  // check_col_log_finite sinkhorn.cpp:20-25
    if (!std::isfinite(col_log[j])) fail(ORC_E_DOMAIN, "column log-mass degenerated");
  e.grad.resize(p.m);
  double gl = 0.0;
  for (int64_t j = 0; j < p.m; ++j) {
    e.grad[j] = col[j] - p.b[j];
    gl += std::abs(e.grad[j]);
  }
  e.grad_l1 = gl;
  double ua = 0.0, vb = 0.0;
  for (int64_t i = 0; i < p.n; ++i) ua += e.u[i] * p.a[i];
  for (int64_t j = 0; j < p.m; ++j) vb += v[j] * p.b[j];
  e.f_value = 1.0 - ua - vb;
  Vec y(p.m);
  for (int64_t j = 0; j < p.m; ++j) y[j] = v[j] + (std::log(p.b[j]) - col_log[j]);
  e.v_next = project_zero_sum(y);
  return e;
}

// mirror.cpp:21-24
double expm1_over_z(double z) {
  if (std::abs(z) < 1e-8) return 1.0 + z / 2.0 + z * z / 6.0;
  return std::expm1(z) / z;
}

// mirror.cpp:46-58
Vec grad_phi_star(const double* b, int64_t m, const double* xi) {
  Vec out(m);
  for (int64_t j = 0; j < m; ++j) {
    const double r = xi[j] / b[j];
    if (r <= -1.0) fail(ORC_E_DOMAIN, "grad_phi_star: argument out of domain");
    out[j] = std::log1p(r);
  }
  return out;
}

// mirror.cpp:94-101
Vec metric_D(const double* b, int64_t m, const double* z) {
  Vec d(m);
  for (int64_t j = 0; j < m; ++j) d[j] = b[j] * expm1_over_z(z[j]);
  return d;
}

// mirror.cpp:80-92
double bregman_from_zero(const double* b, int64_t m, const double* eta) {
  double acc = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double r = eta[j] / b[j];
    if (r <= -1.0) fail(ORC_E_DOMAIN, "bregman_phi_star_from_zero: out of domain");
    acc += eta[j] - b[j] * std::log1p(r);
  }
  return acc;
}

struct Stab {
  double c1l = 0, c1r = 0, c2l = 0, c2r = 0, drift = 0;
  bool both = false, skipped = false;
};

// diag.cpp:107-146
Stab stability_from_grads(const double* b, int64_t m, const double* gk, const double* gk1,
                          const double* xk, const double* xk1, const double* yk,
                          const double* yk1, double alpha) {
  if (!(alpha > 0.0) || !(alpha < 2.0)) fail(ORC_E_OT, "stability conditions need alpha in (0, 2)");
  Stab r;
  if (inf_norm(gk, m) < kGradFloor) {
    r.skipped = true;
    r.both = true;
    r.drift = 0.0;
    return r;
  }
  const Vec pk = grad_phi_star(b, m, gk), pk1 = grad_phi_star(b, m, gk1);
  const Vec Dk = metric_D(b, m, pk.data()), Dk1 = metric_D(b, m, pk1.data());
  double drift = 0.0;
  for (int64_t j = 0; j < m; ++j) drift = std::max(drift, std::abs(Dk1[j] - Dk[j]));
  r.drift = drift;
  double c1 = 0.0;
  for (int64_t j = 0; j < m; ++j) c1 += gk[j] * gk[j] * Dk1[j] / (Dk[j] * Dk[j]);
  r.c1l = c1;
  const double coef = (4.0 - alpha * alpha - 2.0 * std::sqrt(alpha)) /
                      (2.0 * alpha * (1.0 + alpha) * (1.0 + alpha));
  r.c1r = coef * bregman_from_zero(b, m, gk);
  double c2 = 0.0, q = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double vk = yk[j] - xk[j], vk1 = yk1[j] - xk1[j];
    c2 += (Dk1[j] - Dk[j]) * (vk * vk);
    q += Dk1[j] * (vk1 * vk1);
  }
  r.c2l = c2;
  r.c2r = std::pow(alpha, 1.5) * q;
  r.both = r.c1l < r.c1r && r.c2l < r.c2r;
  return r;
}

// diag.cpp:76-88: E(x, y; mu) = f(x) - f* + mu/2 ||y - v*||^2_{D(p(x))}
double lyapunov_from_parts(const double* b, int64_t m, double f_x, const double* grad_x,
                           const double* y, double mu, const orc_reference& ref) {
  if (ref.f_star > f_x + 1e-9) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "reference value %.17g exceeds f(x) = %.17g", ref.f_star, f_x);
    fail(ORC_E_OT, buf);
  }
  double e = f_x - ref.f_star;
  if (mu != 0.0) {
    const Vec pz = grad_phi_star(b, m, grad_x);
    const Vec D = metric_D(b, m, pz.data());
    double q = 0.0;  // MetricDiag::quad
    for (int64_t j = 0; j < m; ++j) {
      const double z = y[j] - ref.v_star[j];
      q += D[j] * (z * z);
    }
    e += 0.5 * mu * q;
  }
  return e;
}

// diag.cpp:206-215 RadiusTracker::observe
std::pair<double, double> radii(const double* b, int64_t m, const double* grad_x,
                                const double* x, const double* y, const orc_reference& ref) {
  const Vec pz = grad_phi_star(b, m, grad_x);
  const Vec D = metric_D(b, m, pz.data());
  double qx = 0.0, qy = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double zx = x[j] - ref.v_star[j], zy = y[j] - ref.v_star[j];
    qx += D[j] * (zx * zx);
    qy += zy * zy;
  }
  return {std::sqrt(qx), std::sqrt(qy)};
}

// Trace writer (diag.hpp:15-42; optional cells as NaN).
struct TraceOut {
  double* buf;
  int64_t cap;
  int64_t len = 0;
  void push(const double row[ORC_TRACE_COLS]) {
    if (buf && len < cap) std::memcpy(buf + len * ORC_TRACE_COLS, row, sizeof(double) * ORC_TRACE_COLS);
    ++len;
  }
};

const double kNaN = std::numeric_limits<double>::quiet_NaN();

// accel.cpp:11-20, 137-151
struct AccelState {
  Vec x, w;
  double mu = 0.0, alpha = 0.0;
  bool has_cache = false;
  StepEval cache;
};

AccelState make_accel_state(const Prob& p, const Vec& x0, const Vec& w0, double mu) {
  if ((int64_t)x0.size() != p.m || (int64_t)w0.size() != p.m)
    fail(ORC_E_DIMENSION, "accelerated state size does not match b");
  if (!(mu > 0.0) || !(mu < 1.0)) fail(ORC_E_OT, "mu must lie in (0, 1)");
  check_zero_sum(x0, "x0");
  check_zero_sum(w0, "w0");
  AccelState s;
  s.x = x0;
  s.w = w0;
  s.mu = mu;
  s.alpha = std::sqrt(2.0 * mu);
  return s;
}

// accel.cpp:153-172
AccelState acc_step(const Prob& p, const AccelState& s, int64_t& evals) {
  const double al = s.alpha;
  Vec Sx;
  if (s.has_cache) {
    Sx = s.cache.v_next;
  } else {
    Sx = eval_normalized_step(p, s.x.data()).v_next;
    ++evals;
  }
  AccelState next;
  next.mu = s.mu;
  next.alpha = al;
  next.x.resize(p.m);
  for (int64_t j = 0; j < p.m; ++j) next.x[j] = (s.w[j] + Sx[j]) / (1.0 + al);
  StepEval e1 = eval_normalized_step(p, next.x.data());
  ++evals;
  next.w.resize(p.m);
  for (int64_t j = 0; j < p.m; ++j)
    next.w[j] = (s.w[j] + (al * al - 2.0) * next.x[j] + 2.0 * e1.v_next[j]) / (1.0 + al);
  next.cache = std::move(e1);
  next.has_cache = true;
  return next;
}

// accel.cpp:27-133 (AccObserver): scalar trace, stability counters, and with a
// ReferenceSolution the energy / radius columns.
class Observer {
 public:
  Observer(const Prob& p, bool trace, int64_t stride, bool stability, TraceOut* out,
           const orc_reference* ref = nullptr)
      : p_(p), trace_(trace), stride_(stride > 0 ? stride : 1), stab_(stability), out_(out),
        ref_(ref) {}

  void observe(int64_t iter, const AccelState& s, bool terminal) {
    const StepEval& e = s.cache;
    max_v_inf_ = std::max(max_v_inf_, inf_norm(s.x.data(), p_.m));
    double c[5] = {kNaN, kNaN, kNaN, kNaN, kNaN};
    double energy = kNaN, rx = kNaN, ry = kNaN;
    const bool want = trace_ && (iter % stride_ == 0 || terminal);
    if (stab_ || ref_) {
      Vec y(p_.m);
      for (int64_t j = 0; j < p_.m; ++j) y[j] = s.w[j] / s.alpha;
      if (ref_) {
        try {
          energy = lyapunov_from_parts(p_.b, p_.m, e.f_value, e.grad.data(), y.data(), s.mu, *ref_);
          auto r = radii(p_.b, p_.m, e.grad.data(), s.x.data(), y.data(), *ref_);
          max_x_ = std::max(max_x_, r.first);
          max_y_ = std::max(max_y_, r.second);
          rx = r.first;
          ry = r.second;
        } catch (const OrcError& err) {
          if (err.code != ORC_E_DOMAIN) throw;
          energy = kNaN;
        }
      }
      if (stab_ && have_prev_) {
        try {
          Stab r = stability_from_grads(p_.b, p_.m, prev_grad_.data(), e.grad.data(),
                                        prev_x_.data(), s.x.data(), prev_y_.data(), y.data(),
                                        s.alpha);
          c[0] = r.c1l; c[1] = r.c1r; c[2] = r.c2l; c[3] = r.c2r; c[4] = r.drift;
          checked_ += r.skipped ? 0 : 1;
          held_ += (!r.skipped && r.both) ? 1 : 0;
        } catch (const OrcError& err) {
          if (err.code != ORC_E_DOMAIN) throw;
        }
      }
      prev_grad_ = e.grad;
      prev_x_ = s.x;
      prev_y_ = y;
      have_prev_ = true;
    }
    if (want) {
      double row[ORC_TRACE_COLS] = {static_cast<double>(iter), 0.0, e.grad_l1, e.grad_l1,
                                    e.f_value, s.mu, s.alpha, c[0], c[1], c[2], c[3], c[4],
                                    energy, rx, ry};
      out_->push(row);
    }
  }
  // accel.cpp:104-114
  double stage_energy(const AccelState& s) const {
    if (!ref_) return kNaN;
    Vec y(p_.m);
    for (int64_t j = 0; j < p_.m; ++j) y[j] = s.w[j] / s.alpha;
    try {
      return lyapunov_from_parts(p_.b, p_.m, s.cache.f_value, s.cache.grad.data(), y.data(), s.mu,
                                 *ref_);
    } catch (const OrcError& err) {
      if (err.code != ORC_E_DOMAIN) throw;
      return kNaN;
    }
  }
  double max_v_inf() const { return max_v_inf_; }
  int64_t checked() const { return checked_; }
  int64_t held() const { return held_; }
  double max_x() const { return max_x_; }
  double max_y() const { return max_y_; }

 private:
  const Prob& p_;
  bool trace_;
  int64_t stride_;
  bool stab_;
  TraceOut* out_;
  const orc_reference* ref_;
  Vec prev_grad_, prev_x_, prev_y_;
  bool have_prev_ = false;
  double max_v_inf_ = 0.0, max_x_ = 0.0, max_y_ = 0.0;
  int64_t checked_ = 0, held_ = 0;
};

void copy_out(const Vec& x, double* dst) {
  if (dst) std::memcpy(dst, x.data(), sizeof(double) * x.size());
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_set_threads(int nthreads) { g_threads = std::max(1, nthreads); }
int orc_get_threads(void) { return g_threads; }

// rng.hpp:11-58 (xoshiro256++ seeded by splitmix64)
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
void orc_rng_seed(uint64_t st[4], uint64_t seed) {
  uint64_t x = seed;
  for (int k = 0; k < 4; ++k) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    st[k] = z ^ (z >> 31);
  }
}
uint64_t orc_rng_next_u64(uint64_t s[4]) {
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
double orc_rng_next_double(uint64_t s[4]) {
  return static_cast<double>(orc_rng_next_u64(s) >> 11) * 0x1.0p-53;
}
uint64_t orc_rng_next_below(uint64_t s[4], uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t r = orc_rng_next_u64(s);
    if (r >= threshold) return r % bound;
  }
}

// ---- BASELINE config samplers (SURVEY §8d draw orders) --------------------
// Restated here so that the CPU legs (tests' fixtures, bench.py --impl
// reference) never load the product library; tests/test_oracle_gen.py checks
// them bitwise against libotg's otg_gen_config.  Gaussian / Beta / mixture
// draws are not in the reference (it has uniform and bounded draws only,
// rng.hpp:38-50):
//   Gaussian  — Box–Muller cosine branch, first uniform taken as 1 - U so the
//               logarithm never sees 0; the sine branch is not drawn;
//   Beta(k, 7-k) — k-th smallest of six uniforms;
//   mixture   — component by next_below(3), then three Gaussian offsets.
static double orc_gauss(uint64_t s[4]) {
  const double one_minus_u = 1.0 - orc_rng_next_double(s);
  const double angle_u = orc_rng_next_double(s);
  const double radius = std::sqrt(-2.0 * std::log(one_minus_u));
  return radius * std::cos(2.0 * M_PI * angle_u);
}

static double orc_order_stat6(uint64_t s[4], int k) {
  double draws[6];
  for (int t = 0; t < 6; ++t) draws[t] = orc_rng_next_double(s);
  // insertion sort: only the order statistic matters
  for (int t = 1; t < 6; ++t)
    for (int q = t; q > 0 && draws[q] < draws[q - 1]; --q) std::swap(draws[q], draws[q - 1]);
  return draws[k - 1];
}

static void orc_normalise_sum(double* x, int64_t n) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += x[i];
  for (int64_t i = 0; i < n; ++i) x[i] /= total;
}

int orc_gen_config(int cfg, int64_t n, int64_t m, uint64_t seed, double* out0, double* out1,
                   double* out2) {
  return guard([&] {
    if (n < 1 || m < 1) fail(ORC_E_DIMENSION, "config needs n, m >= 1");
    uint64_t s[4];
    orc_rng_seed(s, seed);
    if (cfg == 1) {  // a, b ~ U(0.1, 1] normalised; C ~ U[0, 1) raw, row-major
      for (int64_t i = 0; i < n; ++i) out0[i] = 1.0 - 0.9 * orc_rng_next_double(s);
      for (int64_t j = 0; j < m; ++j) out1[j] = 1.0 - 0.9 * orc_rng_next_double(s);
      for (int64_t k = 0; k < n * m; ++k) out2[k] = orc_rng_next_double(s);
      orc_normalise_sum(out0, n);
      orc_normalise_sum(out1, m);
    } else if (cfg == 2) {  // x ~ N(0, I2); y ~ N((2, 0), diag(0.5, 2))
      for (int64_t k = 0; k < 2 * n; ++k) out0[k] = orc_gauss(s);
      const double sd0 = std::sqrt(0.5), sd1 = std::sqrt(2.0);
      for (int64_t j = 0; j < m; ++j) {
        const double g0 = orc_gauss(s);
        out1[2 * j] = 2.0 + sd0 * g0;
        const double g1 = orc_gauss(s);
        out1[2 * j + 1] = sd1 * g1;
      }
    } else if (cfg == 3) {  // Beta(2,5)^3 sources, Beta(5,2)^3 targets
      for (int64_t k = 0; k < 3 * n; ++k) out0[k] = orc_order_stat6(s, 2);
      for (int64_t k = 0; k < 3 * m; ++k) out1[k] = orc_order_stat6(s, 5);
    } else if (cfg == 5) {  // U[0,1]^3 sources; 3-Gaussian mixture targets (sigma 0.1), clipped
      for (int64_t k = 0; k < 3 * n; ++k) out0[k] = orc_rng_next_double(s);
      double means[3][3];
      for (auto& mu : means)
        for (double& c : mu) c = orc_rng_next_double(s);
      for (int64_t j = 0; j < m; ++j) {
        const uint64_t comp = orc_rng_next_below(s, 3);
        for (int k = 0; k < 3; ++k) {
          const double t = means[comp][k] + 0.1 * orc_gauss(s);
          out1[3 * j + k] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        }
      }
    } else {
      fail(ORC_E_OT, "orc_gen_config: cfg must be 1, 2, 3 or 5");
    }
  });
}

int orc_gen_config4(int64_t count, uint64_t seed, int64_t d, int32_t* n, int32_t* m,
                    float* x_cat, float* y_cat) {
  return guard([&] {
    if (count < 1 || d < 1) fail(ORC_E_DIMENSION, "config 4 needs count, d >= 1");
    uint64_t s[4];
    orc_rng_seed(s, seed);
    Vec g(d);
    int64_t xrow = 0, yrow = 0;
    auto unit_rows = [&](int64_t rows, float* dst, int64_t& row) {
      for (int64_t r = 0; r < rows; ++r, ++row) {
        double ss = 0.0;
        for (int64_t k = 0; k < d; ++k) {
          g[k] = orc_gauss(s);
          ss += g[k] * g[k];
        }
        const double inv = 1.0 / std::sqrt(ss);
        if (dst)
          for (int64_t k = 0; k < d; ++k) dst[row * d + k] = static_cast<float>(g[k] * inv);
      }
    };
    for (int64_t p = 0; p < count; ++p) {
      n[p] = 8 + static_cast<int32_t>(orc_rng_next_below(s, 57));
      m[p] = 8 + static_cast<int32_t>(orc_rng_next_below(s, 57));
      unit_rows(n[p], x_cat, xrow);
      unit_rows(m[p], y_cat, yrow);
    }
  });
}

// cost_sqeuclidean (data.cpp:69-82) stored as fp32 the way the B200 path
// stores a points instance (storage F32, norm MAX): raw fp64 sum of squared
// differences in coordinate order, divided by the global maximum, rounded to
// fp32.  nthreads workers (rows are independent; the result does not depend on
// the thread count).  C has row stride ldc.
int orc_cost_sqeuclid_max_f32(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                              int64_t ldc, int nthreads, float* C, double* raw_max) {
  return guard([&] {
    const double mx = orc_sqeuclid_max(x, y, n, m, d, nthreads);
    parallel_blocks(n, std::max(1, nthreads), [&](int, int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i)
        for (int64_t j = 0; j < m; ++j) {
          double acc = 0.0;
          for (int64_t k = 0; k < d; ++k) {
            const double diff = x[i * d + k] - y[j * d + k];
            acc += diff * diff;
          }
          const double c = mx > 0.0 ? acc / mx : acc;
          C[i * ldc + j] = static_cast<float>(c);
        }
    });
    if (raw_max) *raw_max = mx;
  });
}

int orc_validate_problem(const orc_problem* pp, double epsilon) {
  return guard([&] { validate(wrap(pp), epsilon); });
}

// data.cpp:17-32
int orc_synthetic_instance(int64_t n, int64_t m, uint64_t seed, double* a, double* b,
                           double* C) {
  return guard([&] {
    if (n < 1 || m < 1) fail(ORC_E_DIMENSION, "synthetic instance needs n, m >= 1");
    uint64_t st[4];
    orc_rng_seed(st, seed);
    for (int64_t i = 0; i < n; ++i) a[i] = orc_rng_next_double(st);
    for (int64_t j = 0; j < m; ++j) b[j] = orc_rng_next_double(st);
    for (int64_t k = 0; k < n * m; ++k) C[k] = orc_rng_next_double(st);
    double sa = 0, sb = 0, sc = 0;
    for (int64_t i = 0; i < n; ++i) sa += a[i];
    for (int64_t j = 0; j < m; ++j) sb += b[j];
    for (int64_t k = 0; k < n * m; ++k) sc += C[k];
    for (int64_t i = 0; i < n; ++i) a[i] /= sa;
    for (int64_t j = 0; j < m; ++j) b[j] /= sb;
    for (int64_t k = 0; k < n * m; ++k) C[k] /= sc;
  });
}

// data.cpp:69-82
int orc_cost_sqeuclidean(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                         double* C, double* raw_min, double* raw_max) {
  return guard([&] {
    double mn = std::numeric_limits<double>::infinity(), mx = -mn;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) {
          const double diff = x[i * d + k] - y[j * d + k];
          s += diff * diff;
        }
        C[i * m + j] = s;
        mn = std::min(mn, s);
        mx = std::max(mx, s);
      }
    if (raw_min) *raw_min = mn;
    if (raw_max) *raw_max = mx;
    if (mx > 0.0)
      for (int64_t k = 0; k < n * m; ++k) C[k] /= mx;
  });
}

// data.cpp:84-110 (+ norm 2 = raw 1 - <x,y>, BASELINE cfg4)
int orc_cost_cosine(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                    int norm, double* C, double* raw_min, double* raw_max) {
  return guard([&] {
    for (int side = 0; side < 2; ++side) {
      const double* Z = side ? y : x;
      const int64_t rows = side ? m : n;
      for (int64_t i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) s += Z[i * d + k] * Z[i * d + k];
        if (std::abs(std::sqrt(s) - 1.0) > 1e-6) fail(ORC_E_OT, "cosine cost expects unit rows");
      }
    }
    double mn = std::numeric_limits<double>::infinity(), mx = -mn;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double dot = 0.0;
        for (int64_t k = 0; k < d; ++k) dot += x[i * d + k] * y[j * d + k];
        const double c = -dot + 1.0;
        C[i * m + j] = c;
        mn = std::min(mn, c);
        mx = std::max(mx, c);
      }
    if (raw_min) *raw_min = mn;
    if (raw_max) *raw_max = mx;
    if (norm == 1) {
      for (int64_t k = 0; k < n * m; ++k) C[k] /= 2.0;
    } else if (norm == 0) {
      if (mx - mn > 1e-15)
        for (int64_t k = 0; k < n * m; ++k) C[k] = (C[k] - mn) / (mx - mn);
      else
        for (int64_t k = 0; k < n * m; ++k) C[k] = 0.0;
    }
  });
}

// core.cpp:59-79
int orc_plan_stats(const orc_problem* pp, const double* u, const double* v, double eps_ratio,
                   double* row_sums, double* col_sums, double* violation, double* primal) {
  return guard([&] {
    Prob p = wrap(pp);
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g_threads, p.n)));
    Vec tops(T, -std::numeric_limits<double>::infinity());
    parallel_blocks(p.n, T, [&](int t, int64_t lo, int64_t hi) {
      double top = -std::numeric_limits<double>::infinity();
      for (int64_t i = lo; i < hi; ++i)
        for (int64_t j = 0; j < p.m; ++j) top = std::max(top, ((-p.C(i, j)) + u[i]) + v[j]);
      tops[t] = top;
    });
    const double top = *std::max_element(tops.begin(), tops.end());
    if (top > kExpOverflowBound) fail(ORC_E_OVERFLOW, "plan exponent exceeds bound");
    Vec rs(p.n, 0.0);
    std::vector<Vec> cs_t(T, Vec(p.m, 0.0));
    Vec cost_t(T, 0.0);
    parallel_blocks(p.n, T, [&](int t, int64_t lo, int64_t hi) {
      Vec& cs = cs_t[t];
      double cost = 0.0;
      for (int64_t i = lo; i < hi; ++i)
        for (int64_t j = 0; j < p.m; ++j) {
          const double P = std::exp(((-p.C(i, j)) + u[i]) + v[j]);
          rs[i] += P;
          cs[j] += P;
          cost += p.C(i, j) * P;
        }
      cost_t[t] = cost;
    });
    Vec cs(p.m, 0.0);
    double cost = 0.0;
    for (int t = 0; t < T; ++t) {
      cost += cost_t[t];
      for (int64_t j = 0; j < p.m; ++j) cs[j] += cs_t[t][j];
    }
    double viol = 0.0;
    for (int64_t i = 0; i < p.n; ++i) viol += std::abs(rs[i] - p.a[i]);
    double vc = 0.0;
    for (int64_t j = 0; j < p.m; ++j) vc += std::abs(cs[j] - p.b[j]);
    if (violation) *violation = viol + vc;
    if (primal) *primal = cost * eps_ratio;
    copy_out(rs, row_sums);
    copy_out(cs, col_sums);
  });
}

// ---- plan consumers (pipelines.cpp) on the plan of plan_from_potentials ----
// P_ij = exp(((-C'_ij) + u_i) + v_j) with the 700 overflow guard (core.cpp:59-71).
static Vec plan_dense(const Prob& p, const double* u, const double* v) {
  double top = -std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < p.n; ++i)
    for (int64_t j = 0; j < p.m; ++j) top = std::max(top, ((-p.C(i, j)) + u[i]) + v[j]);
  if (top > kExpOverflowBound) fail(ORC_E_OVERFLOW, "plan exponent exceeds bound");
  Vec P(static_cast<size_t>(p.n * p.m));
  for (int64_t i = 0; i < p.n; ++i)
    for (int64_t j = 0; j < p.m; ++j) P[i * p.m + j] = std::exp(((-p.C(i, j)) + u[i]) + v[j]);
  return P;
}

// pipelines.cpp:58-71
int orc_barycentric_projection(const orc_problem* pp, const double* u, const double* v,
                               const double* src, int d, double* out) {
  return guard([&] {
    Prob p = wrap(pp);
    const Vec P = plan_dense(p, u, v);
    Vec col(p.m, 0.0);  // make_plan: column sums
    for (int64_t i = 0; i < p.n; ++i)
      for (int64_t j = 0; j < p.m; ++j) col[j] += P[i * p.m + j];
    for (int64_t j = 0; j < p.m; ++j)
      if (!(col[j] > 0.0)) fail(ORC_E_DEGENERATE, "plan column has zero mass");
    for (int64_t j = 0; j < p.m; ++j)
      for (int k = 0; k < d; ++k) {
        double t = 0.0;  // (P^T src)(j, k)
        for (int64_t i = 0; i < p.n; ++i) t += P[i * p.m + j] * src[i * d + k];
        out[j * d + k] = t / col[j];
      }
  });
}

// pipelines.cpp:101-111
int orc_predict_translations(const orc_problem* pp, const double* u, const double* v,
                             int* out) {
  return guard([&] {
    Prob p = wrap(pp);
    const Vec P = plan_dense(p, u, v);
    for (int64_t i = 0; i < p.n; ++i) {
      int64_t best = 0;
      for (int64_t j = 1; j < p.m; ++j)
        if (P[i * p.m + j] > P[i * p.m + best]) best = j;
      out[i] = static_cast<int>(best);
    }
  });
}

// pipelines.cpp:113-145: per-row top-k (value descending, index ascending)
int orc_plan_topk(const orc_problem* pp, const double* u, const double* v, const int* rows,
                  int64_t nrows, int k, int* out) {
  return guard([&] {
    Prob p = wrap(pp);
    if (k < 1) fail(ORC_E_OT, "topk_accuracy needs k >= 1");
    const Vec P = plan_dense(p, u, v);
    std::vector<int> order(static_cast<size_t>(p.m));
    const int64_t kk = std::min<int64_t>(k, p.m);
    for (int64_t b = 0; b < nrows; ++b) {
      const int64_t s = rows[b];
      if (s < 0 || s >= p.n) fail(ORC_E_DIMENSION, "dictionary index outside the plan");
      for (size_t j = 0; j < order.size(); ++j) order[j] = static_cast<int>(j);
      std::partial_sort(order.begin(), order.begin() + kk, order.end(), [&](int x, int y) {
        const double px = P[s * p.m + x], py = P[s * p.m + y];
        return px > py || (px == py && x < y);
      });
      for (int64_t r = 0; r < k; ++r) out[b * k + r] = r < kk ? order[r] : -1;
    }
  });
}

// pipelines.cpp:80-92: nearest sample, squared distance, strict < (lowest index)
void orc_nn_assign(const double* q, int64_t nq, const double* ref, int64_t nref, int d,
                   int* out) {
  for (int64_t a = 0; a < nq; ++a) {
    int64_t best = 0;
    double best_d2 = 0.0;
    for (int64_t s = 0; s < nref; ++s) {
      double d2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double dd = q[a * d + k] - ref[s * d + k];
        d2 += dd * dd;
      }
      if (s == 0 || d2 < best_d2) {
        best_d2 = d2;
        best = s;
      }
    }
    out[a] = static_cast<int>(best);
  }
}

// core.cpp:81-93
int orc_entropic_objective(const orc_problem* pp, const double* u, const double* v,
                           double epsilon, double* out) {
  return guard([&] {
    Prob p = wrap(pp);
    double ent = 0.0, cost = 0.0;
    for (int64_t i = 0; i < p.n; ++i)
      for (int64_t j = 0; j < p.m; ++j) {
        const double q = std::exp(((-p.C(i, j)) + u[i]) + v[j]);
        if (!(q > 0.0)) fail(ORC_E_NONPOSITIVE, "plan entry is not positive");
        ent += q * (std::log(q) - 1.0);
        cost += p.C(i, j) * q;
      }
    *out = cost + epsilon * ent;
  });
}

int orc_row_solve_marginals(const orc_problem* pp, const double* v, double* u, double* col) {
  return guard([&] { row_solve_marginals(wrap(pp), v, u, col); });
}

int orc_row_solve_marginals_log(const orc_problem* pp, const double* v, double* u,
                                double* col, double* col_log) {
  return guard([&] { row_solve_marginals_log(wrap(pp), v, u, col, col_log); });
}

// dual.cpp:88-101
int orc_dual_F(const orc_problem* pp, const double* u, const double* v, double* out) {
  return guard([&] {
    Prob p = wrap(pp);
    double top = -std::numeric_limits<double>::infinity();
    for (int64_t i = 0; i < p.n; ++i)
      for (int64_t j = 0; j < p.m; ++j) top = std::max(top, ((-p.C(i, j)) + u[i]) + v[j]);
    double s = 0.0;
    for (int64_t i = 0; i < p.n; ++i)
      for (int64_t j = 0; j < p.m; ++j) s += std::exp((((-p.C(i, j)) + u[i]) + v[j]) - top);
    const double lse = top + std::log(s);
    if (lse > kExpOverflowBound) fail(ORC_E_OVERFLOW, "dual mass exponent exceeds bound");
    double ua = 0.0, vb = 0.0;
    for (int64_t i = 0; i < p.n; ++i) ua += u[i] * p.a[i];
    for (int64_t j = 0; j < p.m; ++j) vb += v[j] * p.b[j];
    *out = std::exp(lse) - ua - vb;
  });
}

// dual.cpp:118-136
int orc_hessian_f(const orc_problem* pp, const double* v, double* H) {
  return guard([&] {
    Prob p = wrap(pp);
    if (p.m > 2000) fail(ORC_E_TOO_LARGE, "dense reduced Hessian capped at m = 2000");
    Vec u(p.n), col(p.m);
    row_solve_marginals(p, v, u.data(), col.data());
    std::vector<double> P(p.n * p.m);
    for (int64_t i = 0; i < p.n; ++i) {
      double mx = -std::numeric_limits<double>::infinity();
      for (int64_t j = 0; j < p.m; ++j) mx = std::max(mx, (-p.C(i, j)) + v[j]);
      double rs = 0.0;
      for (int64_t j = 0; j < p.m; ++j) rs += std::exp(((-p.C(i, j)) + v[j]) - mx);
      for (int64_t j = 0; j < p.m; ++j)
        P[i * p.m + j] = std::exp(((-p.C(i, j)) + v[j]) - mx) * (p.a[i] / rs);
    }
    for (int64_t j = 0; j < p.m; ++j)
      for (int64_t k = 0; k < p.m; ++k) {
        double s = 0.0;
        for (int64_t i = 0; i < p.n; ++i) s += P[i * p.m + j] * (P[i * p.m + k] / p.a[i]);
        H[j * p.m + k] = -s + (j == k ? col[j] : 0.0);
      }
  });
}

int orc_grad_phi(const double* b, int64_t m, const double* v, double* out) {  // mirror.cpp:37-44
  return guard([&] {
    for (int64_t j = 0; j < m; ++j)
      if (v[j] > kExpOverflowBound) fail(ORC_E_OVERFLOW, "grad_phi argument exceeds the exponent bound");
    for (int64_t j = 0; j < m; ++j) out[j] = b[j] * std::expm1(v[j]);
  });
}
int orc_grad_phi_star(const double* b, int64_t m, const double* xi, double* out) {
  return guard([&] { copy_out(grad_phi_star(b, m, xi), out); });
}
int orc_phi_star(const double* b, int64_t m, const double* xi, double* out) {  // mirror.cpp:60-71
  return guard([&] {
    double acc = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      const double r = xi[j] / b[j];
      if (r <= -1.0) fail(ORC_E_DOMAIN, "phi_star: out of domain");
      acc += (b[j] + xi[j]) * std::log1p(r) - xi[j];
    }
    *out = acc;
  });
}
int orc_bregman_phi_star_from_zero(const double* b, int64_t m, const double* eta, double* out) {
  return guard([&] { *out = bregman_from_zero(b, m, eta); });
}
int orc_metric_D(const double* b, int64_t m, const double* z, double* d) {
  return guard([&] { copy_out(metric_D(b, m, z), d); });
}
void orc_project_zero_sum(const double* x, int64_t m, double* out) {
  copy_out(project_zero_sum(Vec(x, x + m)), out);
}

int orc_stability_conditions_from_grads(const double* b, int64_t m, const double* gk,
                                        const double* gk1, const double* xk,
                                        const double* xk1, const double* yk,
                                        const double* yk1, double alpha, double out[4],
                                        int* both, int* skipped, double* drift) {
  return guard([&] {
    Stab r = stability_from_grads(b, m, gk, gk1, xk, xk1, yk, yk1, alpha);
    out[0] = r.c1l; out[1] = r.c1r; out[2] = r.c2l; out[3] = r.c2r;
    if (both) *both = r.both;
    if (skipped) *skipped = r.skipped;
    if (drift) *drift = r.drift;
  });
}

int orc_eval_normalized_step(const orc_problem* pp, const double* v, double* v_next,
                             double* u, double* grad, double* grad_l1, double* f_value) {
  return guard([&] {
    Prob p = wrap(pp);
    if (!v) fail(ORC_E_DIMENSION, "v missing");
    StepEval e = eval_normalized_step(p, v);
    copy_out(e.v_next, v_next);
    copy_out(e.u, u);
    copy_out(e.grad, grad);
    if (grad_l1) *grad_l1 = e.grad_l1;
    if (f_value) *f_value = e.f_value;
  });
}

static void validate_solve_config(const orc_solve_config* c) {  // sinkhorn.cpp:29-33
  if (!(c->tol_l1 > 0.0)) fail(ORC_E_OT, "tol_l1 must be positive");
  if (c->max_iters < 1) fail(ORC_E_OT, "max_iters must be at least 1");
  if (c->trace_stride < 1) fail(ORC_E_OT, "trace_stride must be at least 1");
}

// sinkhorn.cpp:65-115
int orc_sinkhorn_solve(const orc_problem* pp, const double* v0, const orc_solve_config* cfg,
                       orc_solve_result* res, double* u_out, double* v_out, double* trace,
                       int64_t trace_cap) {
  return guard([&] {
    Prob p = wrap(pp);
    validate(p, 1.0);
    validate_solve_config(cfg);
    TraceOut tr{trace, trace_cap};
    *res = orc_solve_result{};
    Vec v = project_zero_sum(Vec(v0, v0 + p.m));
    const int64_t stride = cfg->trace_stride;
    for (int64_t k = 0;; ++k) {
      StepEval e = eval_normalized_step(p, v.data());
      ++res->evaluations;
      res->max_v_inf = std::max(res->max_v_inf, inf_norm(v.data(), p.m));
      const double violation = e.grad_l1;
      const bool done = violation < cfg->tol_l1 || k >= cfg->max_iters;
      if (cfg->record_trace && (k % stride == 0 || done)) {
        double row[ORC_TRACE_COLS] = {static_cast<double>(k), 0.0, violation, e.grad_l1,
                                      e.f_value, 0.0, 0.0, kNaN, kNaN, kNaN, kNaN, kNaN};
        tr.push(row);
      }
      if (done) {
        res->converged = violation < cfg->tol_l1;
        res->iterations = k;
        res->final_violation = violation;
        res->final_reduced_f = e.f_value;
        copy_out(e.u, u_out);
        copy_out(v, v_out);
        break;
      }
      v = std::move(e.v_next);
    }
    res->trace_len = tr.len;
  });
}

int orc_acc_step(const orc_problem* pp, const double* x, const double* w, const double* Sx,
                 double mu, double* x_out, double* w_out, double* Sx_out, int64_t* evals) {
  return guard([&] {
    Prob p = wrap(pp);
    AccelState s = make_accel_state(p, Vec(x, x + p.m), Vec(w, w + p.m), mu);
    if (Sx) {
      s.has_cache = true;
      s.cache.v_next.assign(Sx, Sx + p.m);
    }
    int64_t e = 0;
    AccelState nx = acc_step(p, s, e);
    copy_out(nx.x, x_out);
    copy_out(nx.w, w_out);
    copy_out(nx.cache.v_next, Sx_out);
    if (evals) *evals += e;
  });
}

// accel.cpp:174-198
int orc_acc_run(const orc_problem* pp, const double* x0, const double* w0, double mu,
                int64_t msteps, int record_trace, int64_t trace_stride, int stability,
                orc_solve_result* res, double* x_out, double* w_out, double* trace,
                int64_t trace_cap, const orc_reference* ref) {
  return guard([&] {
    Prob p = wrap(pp);
    validate(p, 1.0);
    if (msteps < 0) fail(ORC_E_OT, "acc_run needs m >= 0");
    *res = orc_solve_result{};
    TraceOut tr{trace, trace_cap};
    AccelState s = make_accel_state(p, Vec(x0, x0 + p.m), Vec(w0, w0 + p.m), mu);
    s.cache = eval_normalized_step(p, s.x.data());
    s.has_cache = true;
    ++res->evaluations;
    Observer obs(p, record_trace != 0, trace_stride, stability != 0, &tr, ref);
    obs.observe(0, s, msteps == 0);
    for (int64_t k = 0; k < msteps; ++k) {
      s = acc_step(p, s, res->evaluations);
      obs.observe(k + 1, s, k + 1 == msteps);
    }
    res->final_violation = s.cache.grad_l1;
    res->final_reduced_f = s.cache.f_value;
    res->iterations = msteps;
    res->max_v_inf = obs.max_v_inf();
    res->conditions_checked = obs.checked();
    res->conditions_held = obs.held();
    res->trace_len = tr.len;
    res->r_max_x = obs.max_x();
    res->r_max_y = obs.max_y();
    copy_out(s.x, x_out);
    copy_out(s.w, w_out);
  });
}

// accel.cpp:200-232
int orc_acc_solve(const orc_problem* pp, const double* v0, double mu,
                  const orc_solve_config* cfg, orc_solve_result* res, double* u_out,
                  double* v_out, double* trace, int64_t trace_cap, const orc_reference* ref) {
  return guard([&] {
    Prob p = wrap(pp);
    validate(p, 1.0);
    validate_solve_config(cfg);
    *res = orc_solve_result{};
    TraceOut tr{trace, trace_cap};
    AccelState s = make_accel_state(p, project_zero_sum(Vec(v0, v0 + p.m)), Vec(p.m, 0.0), mu);
    s.cache = eval_normalized_step(p, s.x.data());
    s.has_cache = true;
    ++res->evaluations;
    Observer obs(p, cfg->record_trace != 0, cfg->trace_stride, false, &tr, ref);
    for (int64_t k = 0;; ++k) {
      const double violation = s.cache.grad_l1;
      const bool done = violation < cfg->tol_l1 || k >= cfg->max_iters;
      obs.observe(k, s, done);
      if (done) {
        res->converged = violation < cfg->tol_l1;
        res->iterations = k;
        res->final_violation = violation;
        res->final_reduced_f = s.cache.f_value;
        copy_out(s.cache.u, u_out);
        copy_out(s.x, v_out);
        break;
      }
      s = acc_step(p, s, res->evaluations);
    }
    res->max_v_inf = obs.max_v_inf();
    res->trace_len = tr.len;
    res->r_max_x = obs.max_x();
    res->r_max_y = obs.max_y();
  });
}

// accel.cpp:234-301
int orc_homotopy_solve(const orc_problem* pp, const orc_homotopy_config* cfg,
                       orc_solve_result* res, double* u_out, double* v_out,
                       double* boundaries, int64_t bcap, double* trace, int64_t trace_cap,
                       const orc_reference* ref) {
  return guard([&] {
    Prob p = wrap(pp);
    validate(p, 1.0);
    if (!(cfg->mu0 > 0.0) || !(cfg->mu0 < 1.0) || cfg->m0 < 1 || cfg->max_outer < 1)
      fail(ORC_E_OT, "homotopy schedule needs mu0 in (0, 1), m0 >= 1, max_outer >= 1");
    if (!(cfg->tol_l1 > 0.0)) fail(ORC_E_OT, "tol_l1 must be positive");
    if (cfg->max_total_inner < 1) fail(ORC_E_OT, "max_total_inner must be at least 1");
    if (cfg->trace_stride < 1) fail(ORC_E_OT, "trace_stride must be at least 1");
    *res = orc_solve_result{};
    TraceOut tr{trace, trace_cap};
    AccelState s = make_accel_state(p, Vec(p.m, 0.0), Vec(p.m, 0.0), cfg->mu0);
    s.cache = eval_normalized_step(p, s.x.data());
    s.has_cache = true;
    ++res->evaluations;
    Observer obs(p, cfg->record_trace != 0, cfg->trace_stride, cfg->stability != 0, &tr, ref);
    obs.observe(0, s, false);
    int64_t total_inner = 0, m = cfg->m0, nb = 0;
    bool converged = s.cache.grad_l1 < cfg->tol_l1;
    bool capped = false;
    for (int64_t stage = 0; stage < cfg->max_outer && !converged && !capped; ++stage) {
      ++res->outer_stages;
      if (boundaries && nb < bcap) {
        double* row = boundaries + 5 * nb;
        row[0] = static_cast<double>(stage);
        row[1] = s.mu;
        row[2] = s.alpha;
        row[3] = static_cast<double>(total_inner);
        row[4] = obs.stage_energy(s);
      }
      ++nb;
      for (int64_t i = 0; i < m; ++i) {
        if (total_inner >= cfg->max_total_inner) {
          capped = true;
          break;
        }
        s = acc_step(p, s, res->evaluations);
        ++total_inner;
        converged = s.cache.grad_l1 < cfg->tol_l1;
        obs.observe(total_inner, s, converged || total_inner >= cfg->max_total_inner);
        if (converged) break;
      }
      if (converged || capped) break;
      const double alpha_old = s.alpha;
      s.mu /= 2.0;
      s.alpha = std::sqrt(2.0 * s.mu);
      if (cfg->rescale_w_across_stages)
        for (double& wj : s.w) wj *= s.alpha / alpha_old;
      m = static_cast<int64_t>(std::floor(std::sqrt(2.0) * static_cast<double>(m))) + 1;
    }
    res->converged = converged;
    res->iterations = total_inner;
    res->final_violation = s.cache.grad_l1;
    res->final_reduced_f = s.cache.f_value;
    res->max_v_inf = obs.max_v_inf();
    res->conditions_checked = obs.checked();
    res->conditions_held = obs.held();
    res->trace_len = tr.len;
    res->r_max_x = obs.max_x();
    res->r_max_y = obs.max_y();
    copy_out(s.cache.u, u_out);
    copy_out(s.x, v_out);
  });
}

int orc_lyapunov_energy(const double* b, int64_t m, double f_x, const double* grad_x,
                        const double* y, double mu, const orc_reference* ref, double* out) {
  return guard([&] {
    if (!ref || !out) fail(ORC_E_DIMENSION, "NULL reference / output");
    *out = lyapunov_from_parts(b, m, f_x, grad_x, y, mu, *ref);
  });
}

// accel.cpp:307-311
double orc_homotopy_rate_constant(double mu0, double r_hat, double l_f) {
  const double denom = (std::sqrt(2.0 * l_f) + std::sqrt(2.0 * mu0)) *
                       std::log(2.0 * (r_hat * r_hat + 1.0));
  return (std::sqrt(2.0) - 1.0) / denom;
}

int orc_sweep_rows_mt(const orc_problem* pp, const double* v, int64_t row0, int64_t row1,
                      int nthreads, double* u, double* col_partial) {
  return guard([&] {
    Prob p = wrap(pp);
    if (row0 < 0 || row1 > p.n || row0 > row1) fail(ORC_E_DIMENSION, "row range");
    const int T = std::max(1, nthreads);
    std::vector<Vec> parts(T, Vec(p.m, 0.0));
    auto work = [&](int t) {
      const int64_t span = row1 - row0;
      const int64_t lo = row0 + span * t / T, hi = row0 + span * (t + 1) / T;
      Vec Tr(p.m);
      Vec& col = parts[t];
      for (int64_t i = lo; i < hi; ++i) {
        double mx = -std::numeric_limits<double>::infinity();
        for (int64_t j = 0; j < p.m; ++j) {
          Tr[j] = (-p.C(i, j)) + v[j];
          mx = std::max(mx, Tr[j]);
        }
        double rs = 0.0;
        for (int64_t j = 0; j < p.m; ++j) {
          Tr[j] = std::exp(Tr[j] - mx);
          rs += Tr[j];
        }
        u[i - row0] = (std::log(p.a[i]) - mx) - std::log(rs);
        const double wi = p.a[i] / rs;
        for (int64_t j = 0; j < p.m; ++j) col[j] += Tr[j] * wi;
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int64_t j = 0; j < p.m; ++j) {
      double s = 0.0;
      for (int t = 0; t < T; ++t) s += parts[t][j];
      col_partial[j] = s;
    }
  });
}

void orc_cost_sqeuclid_f32(const float* x, const float* y, int64_t n, int64_t m, int64_t d,
                           float* C) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      float dv[3] = {0.f, 0.f, 0.f};
      for (int64_t k = 0; k < d && k < 3; ++k) dv[k] = x[i * d + k] - y[j * d + k];
      const float dx2 = dv[0] * dv[0];
      C[i * m + j] = std::fmaf(dv[2], dv[2], std::fmaf(dv[1], dv[1], dx2));
    }
}

double orc_sqeuclid_max(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                        int nthreads) {
  const int T = std::max(1, nthreads);
  std::vector<double> best(T, 0.0);
  auto work = [&](int t) {
    double mx = 0.0;
    for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) {
          const double diff = x[i * d + k] - y[j * d + k];
          s += diff * diff;
        }
        mx = std::max(mx, s);
      }
    best[t] = mx;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& q : th) q.join();
  return *std::max_element(best.begin(), best.end());
}

}  // extern "C"
