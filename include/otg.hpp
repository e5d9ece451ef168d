// otg.hpp — header-only C++ mirror of the reference `ot::` solver API over the
// C-ABI of otg.h (link with libotg.so).
//
// Same names, argument meaning and error classes as the reference
// (/root/reference/proj/include/ot/{types,core,dual,sinkhorn,accel}.hpp), with
// std::vector<double> in place of Eigen vectors.  A reference caller switches
// backends by replacing `ot::` with `otg::` for the hot-path calls (see
// INTEGRATION.md); exceptions thrown here derive from otg::OtError exactly as
// the reference's derive from ot::OtError (types.hpp:21-89), so doctest's
// CHECK_THROWS_AS ports unchanged.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "otg.h"

namespace otg {

using Vec = std::vector<double>;

// ------------------------------------------------------------ errors (types.hpp:21-89)
struct OtError : std::runtime_error {
  explicit OtError(const std::string& w) : std::runtime_error(w) {}
};
struct PotentialOverflow : OtError { using OtError::OtError; };
struct DomainViolation : OtError { using OtError::OtError; };
struct GaugeViolation : OtError { using OtError::OtError; };
struct InvalidMarginals : OtError { using OtError::OtError; };
struct NonPositiveEntry : OtError { using OtError::OtError; };
struct DimensionMismatch : OtError { using OtError::OtError; };
struct DimensionTooLarge : OtError { using OtError::OtError; };
struct DegenerateColumn : OtError { using OtError::OtError; };
struct MalformedLine : OtError { using OtError::OtError; };
struct IoError : OtError { using OtError::OtError; };
struct DeviceError : OtError { using OtError::OtError; };  // CUDA / NCCL / OOM / no device

inline void check(otg_status s) {
  if (s == OTG_OK) return;
  const std::string m = otg_last_error();
  switch (s) {
    case OTG_E_OVERFLOW: throw PotentialOverflow(m);
    case OTG_E_DOMAIN: throw DomainViolation(m);
    case OTG_E_GAUGE: throw GaugeViolation(m);
    case OTG_E_INVALID_MARGINALS: throw InvalidMarginals(m);
    case OTG_E_NONPOSITIVE: throw NonPositiveEntry(m);
    case OTG_E_DIMENSION: throw DimensionMismatch(m);
    case OTG_E_TOO_LARGE: throw DimensionTooLarge(m);
    case OTG_E_DEGENERATE: throw DegenerateColumn(m);
    case OTG_E_CUDA:
    case OTG_E_NCCL:
    case OTG_E_OOM:
    case OTG_E_UNSUPPORTED: throw DeviceError(m);
    default: throw OtError(m);
  }
}

// ------------------------------------------------------------ problem (core.hpp:15-49)
// The rescaled instance the solvers run on: cost C / epsilon (rescale_problem
// folded into the upload).  Move-only owner of a device handle.
class TransportProblem {
 public:
  TransportProblem() = default;
  // make_problem(a, b, C, eps) + rescale_problem, dense fp64 or fp32 cost.
  static TransportProblem dense(const Vec& a, const Vec& b, const std::vector<double>& C,
                                double epsilon, const otg_device_opts* opts = nullptr) {
    return make_dense(a, b, C.data(), OTG_F64, C.size(), epsilon, opts);
  }
  static TransportProblem dense(const Vec& a, const Vec& b, const std::vector<float>& C,
                                double epsilon, const otg_device_opts* opts = nullptr) {
    return make_dense(a, b, C.data(), OTG_F32, C.size(), epsilon, opts);
  }
  // cost_sqeuclidean / cost_cosine on the device from points (data.cpp:69-110).
  static TransportProblem points(const Vec& a, const Vec& b, const Vec& x, const Vec& y,
                                 int64_t d, double epsilon, otg_cost cost = OTG_COST_SQEUCLID,
                                 otg_norm norm = OTG_NORM_MAX,
                                 otg_storage storage = OTG_STORE_F32,
                                 const otg_device_opts* opts = nullptr) {
    TransportProblem p;
    p.a_ = a;
    p.b_ = b;
    check(otg_problem_create_points(static_cast<int64_t>(a.size()),
                                    static_cast<int64_t>(b.size()), d, a.data(), b.data(),
                                    x.data(), y.data(), cost, norm, storage, epsilon, opts,
                                    &p.h_));
    return p;
  }
  TransportProblem(TransportProblem&& o) noexcept { *this = std::move(o); }
  TransportProblem& operator=(TransportProblem&& o) noexcept {
    std::swap(h_, o.h_);
    a_ = std::move(o.a_);
    b_ = std::move(o.b_);
    return *this;
  }
  TransportProblem(const TransportProblem&) = delete;
  TransportProblem& operator=(const TransportProblem&) = delete;
  ~TransportProblem() {
    if (h_) otg_problem_destroy(h_);
  }
  int64_t n() const { return static_cast<int64_t>(a_.size()); }
  int64_t m() const { return static_cast<int64_t>(b_.size()); }
  const Vec& a() const { return a_; }
  const Vec& b() const { return b_; }
  otg_problem handle() const { return h_; }
  otg_problem_info info() const {
    otg_problem_info i{};
    check(otg_problem_info_get(h_, &i));
    return i;
  }

 private:
  static TransportProblem make_dense(const Vec& a, const Vec& b, const void* C, otg_dtype dt,
                                     size_t count, double eps, const otg_device_opts* opts) {
    if (count != a.size() * b.size()) throw DimensionMismatch("cost size != n * m");
    TransportProblem p;
    p.a_ = a;
    p.b_ = b;
    check(otg_problem_create_dense(static_cast<int64_t>(a.size()),
                                   static_cast<int64_t>(b.size()), a.data(), b.data(), C, dt, 0,
                                   eps, opts, &p.h_));
    return p;
  }
  otg_problem h_ = nullptr;
  Vec a_, b_;
};

// ------------------------------------------------------------ instance CSV (data.cpp:203-271)
// The host instance (a, b, row-major C, epsilon) as the reference writes it;
// TransportProblem::dense(inst.a, inst.b, inst.C, inst.epsilon) uploads it.
struct Instance {
  Vec a, b, C;
  double epsilon = 1.0;
};

inline void write_instance_csv(const std::string& path, const Instance& p) {
  if (p.a.empty() || p.b.empty() || p.C.size() != p.a.size() * p.b.size())
    throw DimensionMismatch("instance sizes do not match");
  std::ofstream os(path);
  if (!os) throw IoError("cannot write " + path);
  char buf[64];
  auto num = [&](double x) {
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return std::string(buf);
  };
  os << "name,index,value\n";
  os << "n,0," << p.a.size() << "\n";
  os << "m,0," << p.b.size() << "\n";
  os << "epsilon,0," << num(p.epsilon) << "\n";
  for (size_t i = 0; i < p.a.size(); ++i) os << "a," << i << "," << num(p.a[i]) << "\n";
  for (size_t j = 0; j < p.b.size(); ++j) os << "b," << j << "," << num(p.b[j]) << "\n";
  for (size_t k = 0; k < p.C.size(); ++k) os << "C," << k << "," << num(p.C[k]) << "\n";
  if (!os) throw IoError("short write to " + path);
}

namespace detail {
// One record of the instance format: "name,index,value" (the value field
// keeps anything after the second comma, as the writer never emits one).
struct CsvRecord {
  std::string name;
  long index = 0;
  double value = 0.0;
};

// Leading integer / number of a field, 0 when there is none (the format's
// reader is lenient about trailing text, data.cpp:220-269).
inline long leading_long(const std::string& f) {
  std::istringstream in(f);
  long x = 0;
  return (in >> x) ? x : 0L;
}
inline double leading_double(const std::string& f) {
  char* end = nullptr;
  const double x = std::strtod(f.c_str(), &end);
  return end == f.c_str() ? 0.0 : x;
}

inline bool parse_record(const std::string& line, CsvRecord& rec) {
  const size_t first = line.find(',');
  if (first == std::string::npos) return false;
  const size_t second = line.find(',', first + 1);
  if (second == std::string::npos) return false;
  rec.name.assign(line, 0, first);
  rec.index = leading_long(line.substr(first + 1, second - first - 1));
  rec.value = leading_double(line.substr(second + 1));
  return true;
}
}  // namespace detail

// Instance CSV (data.cpp:203-271): header "name,index,value", then n, m,
// epsilon and the a / b / C entries in index order.
inline Instance read_instance_csv(const std::string& path) {
  std::ifstream file(path);
  if (!file) throw IoError("cannot read instance file " + path);
  std::string text;
  if (!std::getline(file, text) || text != "name,index,value")
    throw MalformedLine(path + ": the first line must be the header name,index,value");
  Instance inst;
  inst.epsilon = -1.0;
  long rows = -1, cols = -1;
  long lineno = 1;
  auto where = [&] { return path + " line " + std::to_string(lineno); };
  while (std::getline(file, text)) {
    ++lineno;
    if (text.empty()) continue;
    detail::CsvRecord rec;
    if (!detail::parse_record(text, rec)) throw MalformedLine(where() + ": not a name,index,value record");
    if (rec.name == "n" || rec.name == "m") {
      (rec.name == "n" ? rows : cols) = static_cast<long>(rec.value);
      continue;
    }
    if (rec.name == "epsilon") {
      inst.epsilon = rec.value;
      continue;
    }
    Vec* target = rec.name == "a" ? &inst.a : rec.name == "b" ? &inst.b
                : rec.name == "C" ? &inst.C : nullptr;
    if (!target) throw MalformedLine(where() + ": unknown record name '" + rec.name + "'");
    if (rec.index != static_cast<long>(target->size()))
      throw MalformedLine(where() + ": " + rec.name + "[" + std::to_string(rec.index) +
                          "] is not the next entry");
    target->push_back(rec.value);
  }
  if (rows < 1 || cols < 1 || !(inst.epsilon > 0.0))
    throw MalformedLine(path + ": n, m or epsilon missing");
  if (static_cast<long>(inst.a.size()) != rows || static_cast<long>(inst.b.size()) != cols ||
      static_cast<long>(inst.C.size()) != rows * cols)
    throw MalformedLine(path + ": the a / b / C entries do not match n and m");
  return inst;
}

// ------------------------------------------------------------ configs / results
struct ReferenceSolution {  // diag.hpp:46-49
  Vec v_star;
  double f_star = 0.0;
};

struct SolveConfig {  // sinkhorn.hpp:29-39
  double tol_l1 = 1e-6;
  long max_iters = 200000;
  bool record_trace = false;
  long trace_stride = 1;
  bool wall_clock = true;  // traces always carry wall_time_s = 0 (byte-stable)
  const ReferenceSolution* reference = nullptr;  // acc_solve energy / radius columns
};

struct HomotopyConfig {  // accel.hpp:68-81
  double mu0 = 0.5;
  long m0 = 4;
  long max_outer = 64;
  double tol_l1 = 1e-6;
  long max_total_inner = 20000000;
  bool rescale_w_across_stages = false;
  bool record_trace = false;
  long trace_stride = 1;
  bool wall_clock = true;
};

struct AccelInstrumentation {  // accel.hpp:37-40
  const ReferenceSolution* reference = nullptr;  // energy + radius columns
  bool stability = false;                        // condition columns
};

struct TraceRecord {  // diag.hpp:15-33; NaN marks an empty optional cell
  long iter = 0;
  double wall_time_s = 0, marginal_violation_l1 = 0, grad_f_l1 = 0, reduced_f = 0, mu = 0,
         alpha = 0, cond1_lhs = NAN, cond1_rhs = NAN, cond2_lhs = NAN, cond2_rhs = NAN,
         metric_drift_inf = NAN, energy = NAN, radius_x_d = NAN, radius_y = NAN;
};

struct DualPotentials {
  Vec u, v;
};

struct SolveResult {  // sinkhorn.hpp:44-54
  DualPotentials potentials;
  bool converged = false;
  long iterations = 0, evaluations = 0, outer_stages = 0;
  double final_violation = 0, final_reduced_f = 0, max_v_inf = 0;
  std::vector<TraceRecord> trace;
  double device_seconds = 0;
};

struct StageBoundary {  // accel.hpp:84-90
  long stage = 0;
  double mu = 0, alpha = 0;
  long inner_before = 0;
  double energy = NAN;  // E(x, w / alpha; mu) when a reference is given
};

struct HomotopyResult {  // accel.hpp:92-99
  SolveResult result;
  std::vector<StageBoundary> boundaries;
  long conditions_checked = 0, conditions_held = 0;
  double r_hat = 0, c_star = 0;  // with a reference
};

struct AccelState {  // accel.hpp:11-20 (final state of acc_run)
  Vec x, w;
  double mu = 0, alpha = 0;
};

struct AccRun {  // accel.hpp:42-50
  AccelState state;
  long evaluations = 0;
  double final_violation = 0;
  std::vector<TraceRecord> trace;
  long conditions_checked = 0, conditions_held = 0;
  double max_radius_x_d = 0, max_radius_y = 0;  // RadiusTracker, with a reference
};

struct StepEval {  // sinkhorn.hpp:18-24
  Vec v_next, u, grad;
  double grad_l1 = 0, f_value = 0;
};

namespace detail {
struct Out {
  otg_solve_result r{};
  Vec u, v, w, trace, bounds;
  Out(const TransportProblem& p, bool trace_on, long cap, long bcap = 0)
      : u(p.info().n_local), v(p.m()), w(p.m()), trace(trace_on ? cap * OTG_TRACE_COLS : 0),
        bounds(bcap * 5) {
    r.u = u.data();
    r.v = v.data();
    r.w = w.data();
    r.trace = trace_on ? trace.data() : nullptr;
    r.trace_cap = trace_on ? cap : 0;
    r.boundaries = bcap ? bounds.data() : nullptr;
    r.boundaries_cap = bcap;
  }
  std::vector<TraceRecord> records() const {
    std::vector<TraceRecord> out;
    const long n = r.trace_len < r.trace_cap ? r.trace_len : r.trace_cap;
    for (long k = 0; k < n; ++k) {
      const double* t = trace.data() + k * OTG_TRACE_COLS;
      TraceRecord rec;
      rec.iter = static_cast<long>(t[0]);
      rec.wall_time_s = t[1];
      rec.marginal_violation_l1 = t[2];
      rec.grad_f_l1 = t[3];
      rec.reduced_f = t[4];
      rec.mu = t[5];
      rec.alpha = t[6];
      rec.cond1_lhs = t[7];
      rec.cond1_rhs = t[8];
      rec.cond2_lhs = t[9];
      rec.cond2_rhs = t[10];
      rec.metric_drift_inf = t[11];
      rec.energy = t[12];
      rec.radius_x_d = t[13];
      rec.radius_y = t[14];
      out.push_back(rec);
    }
    return out;
  }
  SolveResult result() {
    SolveResult s;
    s.potentials = {u, v};
    s.converged = r.converged != 0;
    s.iterations = r.iterations;
    s.evaluations = r.evaluations;
    s.outer_stages = r.outer_stages;
    s.final_violation = r.final_violation;
    s.final_reduced_f = r.final_reduced_f;
    s.max_v_inf = r.max_v_inf;
    s.trace = records();
    s.device_seconds = r.device_seconds;
    return s;
  }
};
inline long trace_cap(long iters, long stride) { return iters / (stride > 0 ? stride : 1) + 2; }
inline otg_instr instr_of(const AccelInstrumentation* instr) {
  otg_instr in{0, nullptr, 0.0};
  if (instr) {
    in.stability = instr->stability;
    if (instr->reference) {
      in.reference_v = instr->reference->v_star.data();
      in.reference_f = instr->reference->f_star;
    }
  }
  return in;
}
}  // namespace detail

// ------------------------------------------------------------ dual.hpp / sinkhorn.hpp
inline std::pair<Vec, Vec> row_solve_marginals(const TransportProblem& p, const Vec& v) {
  if (static_cast<int64_t>(v.size()) != p.m()) throw DimensionMismatch("v size");
  Vec u(p.info().n_local), col(p.m());
  check(otg_row_solve_marginals(p.handle(), v.data(), u.data(), col.data()));
  return {u, col};
}
inline Vec row_solve(const TransportProblem& p, const Vec& v) { return row_solve_marginals(p, v).first; }
inline Vec grad_f(const TransportProblem& p, const Vec& v) {
  Vec g = row_solve_marginals(p, v).second;
  for (size_t j = 0; j < g.size(); ++j) g[j] -= p.b()[j];
  return g;
}
inline double reduced_f(const TransportProblem& p, const Vec& v) {  // dual.cpp:103-108
  const Vec u = row_solve(p, v);
  double ua = 0, vb = 0;
  for (size_t i = 0; i < u.size(); ++i) ua += u[i] * p.a()[i];
  for (size_t j = 0; j < v.size(); ++j) vb += v[j] * p.b()[j];
  return 1.0 - ua - vb;
}

inline double dual_F(const TransportProblem& p, const Vec& u, const Vec& v) {  // dual.cpp:88-101
  if (static_cast<int64_t>(u.size()) != p.info().n_local || static_cast<int64_t>(v.size()) != p.m())
    throw DimensionMismatch("(u, v) size");
  double out = 0;
  check(otg_dual_F(p.handle(), u.data(), v.data(), &out));
  return out;
}
inline Vec hessian_f(const TransportProblem& p, const Vec& v) {  // dual.cpp:118-136, row-major m x m
  if (static_cast<int64_t>(v.size()) != p.m()) throw DimensionMismatch("v size");
  Vec H(static_cast<size_t>(p.m()) * p.m());
  check(otg_hessian_f(p.handle(), v.data(), H.data()));
  return H;
}

inline StepEval eval_normalized_step(const TransportProblem& p, const Vec& v) {
  if (static_cast<int64_t>(v.size()) != p.m()) throw DimensionMismatch("v size");
  StepEval e;
  e.v_next.resize(p.m());
  e.u.resize(p.info().n_local);
  e.grad.resize(p.m());
  otg_step_eval out{e.v_next.data(), e.u.data(), e.grad.data(), 0, 0};
  check(otg_eval_normalized_step(p.handle(), v.data(), &out));
  e.grad_l1 = out.grad_l1;
  e.f_value = out.f_value;
  return e;
}

inline Vec normalized_sinkhorn_map(const TransportProblem& p, const Vec& v) {  // sinkhorn.cpp:44-49
  double s = 0;
  for (double x : v) s += x;
  if (std::abs(s) > 1e-9) throw GaugeViolation("normalized map fed an off-gauge v");
  return eval_normalized_step(p, v).v_next;
}

inline SolveResult sinkhorn_solve(const TransportProblem& p, const Vec& v0,
                                  const SolveConfig& cfg) {
  detail::Out o(p, cfg.record_trace, detail::trace_cap(cfg.max_iters, cfg.trace_stride));
  const otg_solve_config c{cfg.tol_l1, cfg.max_iters, cfg.record_trace, cfg.trace_stride,
                           cfg.reference ? cfg.reference->v_star.data() : nullptr,
                           cfg.reference ? cfg.reference->f_star : 0.0};
  check(otg_sinkhorn_solve(p.handle(), v0.empty() ? nullptr : v0.data(), &c, &o.r));
  return o.result();
}

// ------------------------------------------------------------ accel.hpp
inline SolveResult acc_solve(const TransportProblem& p, const Vec& v0, double mu,
                             const SolveConfig& cfg) {
  detail::Out o(p, cfg.record_trace, detail::trace_cap(cfg.max_iters, cfg.trace_stride));
  const otg_solve_config c{cfg.tol_l1, cfg.max_iters, cfg.record_trace, cfg.trace_stride,
                           cfg.reference ? cfg.reference->v_star.data() : nullptr,
                           cfg.reference ? cfg.reference->f_star : 0.0};
  check(otg_acc_solve(p.handle(), v0.empty() ? nullptr : v0.data(), mu, &c, &o.r));
  return o.result();
}

inline AccRun acc_run(const TransportProblem& p, const Vec& x0, const Vec& w0, double mu, long m,
                      bool record_trace = false, long trace_stride = 1, bool /*wall_clock*/ = true,
                      const AccelInstrumentation* instr = nullptr) {
  detail::Out o(p, record_trace, detail::trace_cap(m > 0 ? m : 1, trace_stride));
  const otg_instr in = detail::instr_of(instr);
  check(otg_acc_run(p.handle(), x0.data(), w0.data(), mu, m, record_trace, trace_stride, &in,
                    &o.r));
  AccRun a;
  a.state = {o.v, o.w, mu, std::sqrt(2.0 * mu)};
  a.evaluations = o.r.evaluations;
  a.final_violation = o.r.final_violation;
  a.trace = o.records();
  a.conditions_checked = o.r.conditions_checked;
  a.conditions_held = o.r.conditions_held;
  a.max_radius_x_d = o.r.radius_x_max;
  a.max_radius_y = o.r.radius_y_max;
  return a;
}

inline HomotopyResult homotopy_solve_instrumented(const TransportProblem& p,
                                                  const HomotopyConfig& cfg,
                                                  const AccelInstrumentation* instr = nullptr) {
  const long bcap = cfg.max_outer < 4096 ? cfg.max_outer : 4096;
  const long iters = cfg.max_total_inner < 10000000 ? cfg.max_total_inner : 10000000;
  detail::Out o(p, cfg.record_trace, detail::trace_cap(iters, cfg.trace_stride), bcap);
  const otg_homotopy_config c{cfg.mu0,    cfg.m0, cfg.max_outer, cfg.tol_l1, cfg.max_total_inner,
                              cfg.rescale_w_across_stages, cfg.record_trace, cfg.trace_stride};
  const otg_instr in = detail::instr_of(instr);
  check(otg_homotopy_solve(p.handle(), &c, &in, &o.r));
  HomotopyResult h;
  h.result = o.result();
  const long nb = o.r.outer_stages < bcap ? o.r.outer_stages : bcap;
  for (long k = 0; k < nb; ++k) {
    const double* b = o.bounds.data() + 5 * k;
    h.boundaries.push_back({static_cast<long>(b[0]), b[1], b[2], static_cast<long>(b[3]), b[4]});
  }
  h.conditions_checked = o.r.conditions_checked;
  h.conditions_held = o.r.conditions_held;
  if (instr && instr->reference) {
    h.r_hat = o.r.radius_x_max > o.r.radius_y_max ? o.r.radius_x_max : o.r.radius_y_max;
    h.c_star = (std::sqrt(2.0) - 1.0) /  // homotopy_rate_constant (accel.cpp:307-311), L = 1
               ((std::sqrt(2.0) + std::sqrt(2.0 * cfg.mu0)) * std::log(2.0 * (h.r_hat * h.r_hat + 1.0)));
  }
  return h;
}

inline SolveResult homotopy_solve(const TransportProblem& p, const HomotopyConfig& cfg) {
  return homotopy_solve_instrumented(p, cfg, nullptr).result;
}

// ------------------------------------------------------------ core.hpp plan statistics
struct PlanStats {
  double marginal_violation_l1 = 0, primal_cost = 0, max_exponent = 0;
  Vec row_sums, col_sums;
};
inline PlanStats plan_stats(const TransportProblem& p, const Vec& u, const Vec& v) {
  PlanStats s;
  s.row_sums.resize(p.info().n_local);
  s.col_sums.resize(p.m());
  otg_plan_summary out{0, 0, 0, s.row_sums.data(), s.col_sums.data()};
  check(otg_plan_stats(p.handle(), u.data(), v.data(), &out));
  s.marginal_violation_l1 = out.marginal_violation_l1;
  s.primal_cost = out.primal_cost;
  s.max_exponent = out.max_exponent;
  return s;
}

// ------------------------------------------------------------ pipelines.hpp plan consumers
// Over the implicit plan of the potentials (the reference takes a PlanDense).
// src is n x d row-major; the result m x d row-major.
inline Vec barycentric_projection(const TransportProblem& p, const Vec& u, const Vec& v,
                                  const Vec& src, int d) {  // pipelines.cpp:58-71
  if (static_cast<long>(src.size()) != p.info().n_local * d)
    throw DimensionMismatch("plan rows and source colors disagree");
  Vec out(static_cast<size_t>(p.m()) * d);
  check(otg_plan_barycentric(p.handle(), u.data(), v.data(), src.data(), d, out.data(), nullptr));
  return out;
}
inline std::vector<int> predict_translations(const TransportProblem& p, const Vec& u,
                                             const Vec& v) {  // pipelines.cpp:101-111
  std::vector<int> out(static_cast<size_t>(p.info().n_local));
  check(otg_plan_row_argmax(p.handle(), u.data(), v.data(), out.data()));
  return out;
}
inline std::vector<int> plan_topk(const TransportProblem& p, const Vec& u, const Vec& v,
                                  const std::vector<int>& rows, int k) {
  std::vector<int> out(rows.size() * static_cast<size_t>(k > 0 ? k : 1));
  check(otg_plan_topk(p.handle(), u.data(), v.data(), rows.data(),
                      static_cast<int64_t>(rows.size()), k, out.data()));
  return out;
}

// ------------------------------------------------------------ pipelines.hpp run_solver
enum class SolverKind { Sinkhorn, Acc, AccHomotopy };
struct SolverSpec {  // pipelines.hpp:16-25
  SolverKind kind = SolverKind::AccHomotopy;
  double mu = 0.5, mu0 = 0.5;
  long m0 = 4;
  long max_iters = 2000000;
  bool record_trace = false;
  long trace_stride = 1;
  bool wall_clock = true;
};
inline SolveResult run_solver(const TransportProblem& rescaled, const SolverSpec& spec,
                              double tol_l1) {  // pipelines.cpp:28-56
  SolveConfig cfg{tol_l1, spec.max_iters, spec.record_trace, spec.trace_stride, spec.wall_clock};
  const Vec v0(static_cast<size_t>(rescaled.m()), 0.0);
  switch (spec.kind) {
    case SolverKind::Sinkhorn: return sinkhorn_solve(rescaled, v0, cfg);
    case SolverKind::Acc: return acc_solve(rescaled, v0, spec.mu, cfg);
    case SolverKind::AccHomotopy: {
      HomotopyConfig h;
      h.mu0 = spec.mu0;
      h.m0 = spec.m0;
      h.tol_l1 = tol_l1;
      h.max_total_inner = spec.max_iters;
      h.record_trace = spec.record_trace;
      h.trace_stride = spec.trace_stride;
      return homotopy_solve(rescaled, h);
    }
  }
  throw OtError("unreachable solver kind");
}

}  // namespace otg
