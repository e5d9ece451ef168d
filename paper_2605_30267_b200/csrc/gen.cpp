// gen.cpp — seeded synthetic inputs (host code of the product library).
//
// Rng restates rng.hpp:11-58 (xoshiro256++ seeded by splitmix64; golden
// sequence pinned by test_data.cpp:47-58).  The config samplers follow the
// draw orders proposed in SURVEY §8(d); Gaussian / Beta / mixture draws are
// new (the reference has only uniform and bounded-integer draws):
//   normal(): u1 = 1 - next_double(), u2 = next_double(),
//             sqrt(-2 ln u1) cos(2 pi u2)  (sine discarded)
//   Beta(2,5) / Beta(5,2): 2nd / 5th order statistic of 6 uniforms.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "common.cuh"

namespace otg {
namespace {

class Rng {
 public:
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s_) {
      x += 0x9e3779b97f4a7c15ULL;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      w = z ^ (z >> 31);
    }
  }
  uint64_t next_u64() {
    const uint64_t r = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return r;
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % bound;
    }
  }
  double normal() {
    const double u1 = 1.0 - next_double();
    const double u2 = next_double();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  // k-th order statistic (1-based) of 6 uniforms: Beta(k, 7 - k)
  double beta_os6(int k) {
    double u[6];
    for (double& x : u) x = next_double();
    std::sort(u, u + 6);
    return u[k - 1];
  }

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t s_[4];
};

void normalize(double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i];
  for (int64_t i = 0; i < n; ++i) x[i] /= s;
}

}  // namespace
}  // namespace otg

using namespace otg;

extern "C" {

// data.cpp:17-32
otg_status otg_gen_synthetic_instance(int64_t n, int64_t m, uint64_t seed, double* a, double* b,
                                      double* C) {
  return guard([&] {
    if (n < 1 || m < 1) fail(OTG_E_DIMENSION, "synthetic instance needs n, m >= 1");
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) a[i] = rng.next_double();
    for (int64_t j = 0; j < m; ++j) b[j] = rng.next_double();
    for (int64_t k = 0; k < n * m; ++k) C[k] = rng.next_double();
    normalize(a, n);
    normalize(b, m);
    double s = 0.0;
    for (int64_t k = 0; k < n * m; ++k) s += C[k];
    for (int64_t k = 0; k < n * m; ++k) C[k] /= s;
  });
}

otg_status otg_gen_config(int cfg, int64_t n, int64_t m, uint64_t seed, double* out0,
                          double* out1, double* out2) {
  return guard([&] {
    if (n < 1 || m < 1) fail(OTG_E_DIMENSION, "config needs n, m >= 1");
    Rng rng(seed);
    switch (cfg) {
      case 1: {  // a, b = 1 - 0.9 U (i.e. U(0.1, 1]) normalised; C = U[0,1) raw
        for (int64_t i = 0; i < n; ++i) out0[i] = 1.0 - 0.9 * rng.next_double();
        for (int64_t j = 0; j < m; ++j) out1[j] = 1.0 - 0.9 * rng.next_double();
        for (int64_t k = 0; k < n * m; ++k) out2[k] = rng.next_double();
        normalize(out0, n);
        normalize(out1, m);
        break;
      }
      case 2: {  // x ~ N(0, I2); y ~ N((2,0), diag(0.5, 2)) (variances)
        for (int64_t i = 0; i < n; ++i) {
          out0[2 * i] = rng.normal();
          out0[2 * i + 1] = rng.normal();
        }
        for (int64_t j = 0; j < m; ++j) {
          out1[2 * j] = 2.0 + std::sqrt(0.5) * rng.normal();
          out1[2 * j + 1] = std::sqrt(2.0) * rng.normal();
        }
        break;
      }
      case 3: {  // Beta(2,5)^3 sources, Beta(5,2)^3 targets
        for (int64_t i = 0; i < 3 * n; ++i) out0[i] = rng.beta_os6(2);
        for (int64_t j = 0; j < 3 * m; ++j) out1[j] = rng.beta_os6(5);
        break;
      }
      case 5: {  // U[0,1]^3 sources; 3-component mixture targets, sigma 0.1, clipped
        for (int64_t i = 0; i < 3 * n; ++i) out0[i] = rng.next_double();
        double mu[9];
        for (double& x : mu) x = rng.next_double();
        for (int64_t j = 0; j < m; ++j) {
          const uint64_t c = rng.next_below(3);
          for (int k = 0; k < 3; ++k) {
            const double v = mu[3 * c + k] + 0.1 * rng.normal();
            out1[3 * j + k] = std::min(1.0, std::max(0.0, v));
          }
        }
        break;
      }
      default:
        fail(OTG_E_OT, "otg_gen_config: cfg must be 1, 2, 3 or 5");
    }
  });
}

otg_status otg_gen_config4(int64_t count, uint64_t seed, int64_t d, int32_t* n, int32_t* m,
                           float* x_cat, float* y_cat) {
  return guard([&] {
    if (count < 1 || d < 1) fail(OTG_E_DIMENSION, "config 4 needs count, d >= 1");
    Rng rng(seed);
    std::vector<double> row(d);
    int64_t xo = 0, yo = 0;
    auto draw_rows = [&](int64_t rows, float* dst, int64_t& off) {
      for (int64_t r = 0; r < rows; ++r) {
        double ss = 0.0;
        for (int64_t k = 0; k < d; ++k) {
          row[k] = rng.normal();
          ss += row[k] * row[k];
        }
        const double inv = 1.0 / std::sqrt(ss);
        if (dst)
          for (int64_t k = 0; k < d; ++k) dst[(off + r) * d + k] = static_cast<float>(row[k] * inv);
      }
      off += rows;
    };
    for (int64_t p = 0; p < count; ++p) {
      const int32_t np = 8 + static_cast<int32_t>(rng.next_below(57));
      const int32_t mp = 8 + static_cast<int32_t>(rng.next_below(57));
      n[p] = np;
      m[p] = mp;
      draw_rows(np, x_cat, xo);
      draw_rows(mp, y_cat, yo);
    }
  });
}

}  // extern "C"
