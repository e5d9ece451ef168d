// test_kat.cpp — the reference's known-answer tests replayed through the C++
// mirror (include/otg.hpp) of the C-ABI, written the way the reference's
// doctest suites are (values and tolerances from proj/tests/*.cpp, see
// tests/golden/kat.json).  `--cpu` runs only the checks that need no device
// (input validation maps onto the reference's exception classes).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/otg.hpp"

static int g_fail = 0, g_pass = 0;

#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool ok_ = false;                                                      \
    try {                                                                  \
      expr;                                                                \
    } catch (const type&) {                                                \
      ok_ = true;                                                          \
    } catch (...) {                                                        \
    }                                                                      \
    CHECK(ok_);                                                            \
  } while (0)

// doctest::Approx(b).epsilon(e)
static bool approx(double a, double b, double eps) {
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

using otg::Vec;

static otg::TransportProblem skewed_2x2() {  // helpers.hpp:14-21
  return otg::TransportProblem::dense({0.7, 0.3}, {0.5, 0.5}, std::vector<double>{0, 1, 1, 0}, 1.0);
}

static otg::TransportProblem synthetic_rescaled(int64_t n, int64_t m, uint64_t seed, double eps) {
  Vec a(n), b(m), C(n * m);
  otg::check(otg_gen_synthetic_instance(n, m, seed, a.data(), b.data(), C.data()));
  return otg::TransportProblem::dense(a, b, C, eps);
}

static void cpu_checks() {  // test_core.cpp:30-71 through the C-ABI
  const std::vector<double> Z(4, 0.0);
  CHECK_THROWS_AS(otg::TransportProblem::dense({1.2, -0.2}, {0.5, 0.5}, Z, 1.0),
                  otg::InvalidMarginals);
  CHECK_THROWS_AS(otg::TransportProblem::dense({0.7, 0.4}, {0.5, 0.5}, Z, 1.0),
                  otg::InvalidMarginals);
  CHECK_THROWS_AS(otg::TransportProblem::dense({0.7, 0.3}, {0.5, 0.5}, Z, 0.0), otg::OtError);
  CHECK_THROWS_AS(otg::TransportProblem::dense({0.7, 0.3}, {0.5, 0.5}, std::vector<double>(6, 0.0), 1.0),
                  otg::DimensionMismatch);
  CHECK(otg_abi_version() == OTG_ABI_VERSION);
  Vec a(2), b(3), C(6);
  otg::check(otg_gen_synthetic_instance(2, 3, 7, a.data(), b.data(), C.data()));
  CHECK(approx(C[0], 0.17316924621916613, 1e-15));  // test_data.cpp:84
  CHECK(approx(a[1], 0.75663205931103994, 1e-15));  // test_data.cpp:80
  // instance CSV round trip is exact (test_data.cpp:310-336)
  otg::Instance inst;
  inst.a.resize(3);
  inst.b.resize(4);
  inst.C.resize(12);
  otg::check(otg_gen_synthetic_instance(3, 4, 99, inst.a.data(), inst.b.data(), inst.C.data()));
  inst.epsilon = 0.037;
  const std::string path = "/tmp/otg_test_instance.csv";
  otg::write_instance_csv(path, inst);
  const otg::Instance back = otg::read_instance_csv(path);
  CHECK(back.a == inst.a && back.b == inst.b && back.C == inst.C && back.epsilon == inst.epsilon);
  {
    std::FILE* f = std::fopen(path.c_str(), "w");
    std::fputs("name,index,value\nn,0,1\nm,0,1\nepsilon,0,1\na,1,1\n", f);
    std::fclose(f);
  }
  CHECK_THROWS_AS(otg::read_instance_csv(path), otg::MalformedLine);
  CHECK_THROWS_AS(otg::read_instance_csv("/nonexistent/otg.csv"), otg::IoError);
}

static void gpu_checks() {
  {  // test_dual.cpp:68-74, 131-138, 245-252
    auto p = skewed_2x2();
    auto uc = otg::row_solve_marginals(p, {0.0, 0.0});
    CHECK(approx(uc.first[0], -0.66993663145695526, 1e-14));
    CHECK(approx(uc.first[1], -1.5172344918441589, 1e-14));
    CHECK(approx(uc.second[0], 0.59242343145200194, 1e-14));
    CHECK(approx(uc.second[1], 0.40757656854799801, 1e-14));
    const Vec g = otg::grad_f(p, {0.0, 0.0});
    CHECK(approx(g[0], 0.092423431452001936, 1e-13));
    CHECK(approx(otg::reduced_f(p, {0.0, 0.0}), 1.9241259895731164, 1e-14));
  }
  {  // test_sinkhorn.cpp:42-58
    auto p = skewed_2x2();
    const Vec z = otg::normalized_sinkhorn_map(p, {0.0, 0.0});
    CHECK(approx(z[0], -0.18699641086700131, 1e-13));
    CHECK(approx(z[1], 0.18699641086700131, 1e-13));
    CHECK_THROWS_AS(otg::normalized_sinkhorn_map(p, {0.5, 0.4}), otg::GaugeViolation);
  }
  {  // test_accel.cpp:36-50
    auto p = skewed_2x2();
    const auto r = otg::acc_run(p, {0.0, 0.0}, {0.0, 0.0}, 0.5, 1);
    CHECK(r.evaluations == 2);
    CHECK(approx(r.state.x[0], -0.093498205433500653, 1e-13));
    CHECK(approx(r.state.w[1], 0.1573243605054549, 1e-13));
  }
  {  // test_accel.cpp:164-191
    auto p = synthetic_rescaled(6, 6, 18, 0.5);
    otg::HomotopyConfig cfg;
    cfg.max_outer = 3;
    cfg.tol_l1 = 1e-15;
    const auto h = otg::homotopy_solve_instrumented(p, cfg);
    CHECK(!h.result.converged);
    CHECK(h.result.iterations == 19);
    CHECK(h.result.outer_stages == 3);
    CHECK(h.boundaries.size() == 3);
    CHECK(h.boundaries[1].mu == 0.25 && h.boundaries[1].inner_before == 4);
    CHECK(h.boundaries[2].mu == 0.125 && h.boundaries[2].inner_before == 10);
  }
  {  // test_sinkhorn.cpp:160-184 / test_core.cpp:131-190
    auto p = skewed_2x2();
    otg::SolveConfig cfg;
    cfg.tol_l1 = 1e-8;
    const auto r = otg::sinkhorn_solve(p, {0.0, 0.0}, cfg);
    CHECK(r.converged && r.evaluations == r.iterations + 1 && r.final_violation < 1e-8);
    const auto st = otg::plan_stats(p, otg::row_solve(p, {0.0, 0.0}), {0.0, 0.0});
    CHECK(approx(st.marginal_violation_l1, 0.18484686290400393, 1e-13));
    CHECK(approx(st.primal_cost, 0.2689414213699951, 1e-13));
    CHECK_THROWS_AS(otg::plan_stats(p, {800.0, 800.0}, {0.0, 0.0}), otg::PotentialOverflow);
  }
  {  // run_solver dispatch (pipelines.cpp:28-56)
    auto p = synthetic_rescaled(20, 30, 4, 0.1);
    otg::SolverSpec s;
    const auto h = otg::run_solver(p, s, 1e-9);
    s.kind = otg::SolverKind::Sinkhorn;
    const auto k = otg::run_solver(p, s, 1e-9);
    CHECK(h.converged && k.converged);
    CHECK(h.final_violation < 1e-9 && k.final_violation < 1e-9);
    CHECK(h.evaluations == h.iterations + 1 && k.evaluations == k.iterations + 1);
  }
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  cpu_checks();
  if (!cpu_only) gpu_checks();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
