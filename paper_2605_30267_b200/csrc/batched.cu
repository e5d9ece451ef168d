// batched.cu — many small independent OT problems (BASELINE config 4:
// 4096 problems, n, m <= 64), one CTA per problem.
//
// Each CTA pulls problems from an atomic queue (iteration counts differ per
// problem), stages the problem's cost in shared memory (fp32 in
// HBM, up-cast and divided by epsilon once: the oracle's C32 / eps), and runs
// the whole homotopy Acc-Sinkhorn solve (accel.cpp:234-301) inside the CTA:
// row log-sum-exp (warp per row), column sums (64 columns x 4 row groups,
// fixed-order combine), exact column LSE fallback (dual.cpp:53-69), the
// normalised map (sinkhorn.cpp:51-63), the Hessian-driven extrapolation
// (accel.cpp:153-172) and the stage schedule.  All arithmetic fp64 with IEEE
// exp / log, so results match the CPU oracle to ~1e-13 and iteration counts
// exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace otg {
namespace {

constexpr int kBT = 256;     // threads per CTA
constexpr int kBMax = 64;    // max n, m per problem
constexpr int kBGroups = kBT / kBMax;

struct BatchDev {
  int64_t count = 0;
  int32_t* n = nullptr;
  int32_t* m = nullptr;
  int64_t* off_a = nullptr;  // prefix sums of n
  int64_t* off_b = nullptr;  // prefix sums of m
  int64_t* off_c = nullptr;  // prefix sums of n*m
  double* a = nullptr;
  double* b = nullptr;
  float* C = nullptr;
  double eps = 1.0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t total_n = 0, total_m = 0, total_c = 0;
};

struct BatchOut {
  int32_t* converged;
  int64_t* iterations;
  double* final_violation;
  double* final_f;
  double* u;
  double* v;
};

struct BatchCfg {
  double mu0, tol;
  long long m0, max_outer, cap;
  int rescale_w;
};

struct Smem {
  double C[kBMax * kBMax];  // C' = C32 / eps
  double a[kBMax], loga[kBMax], b[kBMax], logb[kBMax];
  double x[kBMax], w[kBMax], pt[kBMax];  // state x, momentum w, evaluation point
  double S[kBMax];                       // normalised map at the evaluation point
  double u[kBMax], M[kBMax], wr[kBMax];  // row solve
  double colp[kBGroups][kBMax];
  double red[kBT / 32][4];
  double scal[4];  // gl, f, mean
  int prob;
};

__device__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One eval_normalized_step at sm.pt: fills sm.S (projected step), sm.u and
// returns (grad_l1, f) in sm.scal[0..1].
__device__ void eval_step(Smem& sm, int n, int m) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // row pass: warp per row (dual.cpp:34-38)
  for (int i = warp; i < n; i += kBT / 32) {
    const double* Ci = sm.C + i * kBMax;
    double mx = -INFINITY;
    for (int j = lane; j < m; j += 32) mx = fmax(mx, (-Ci[j]) + sm.pt[j]);
    mx = warp_max(mx);
    double s = 0.0;
    for (int j = lane; j < m; j += 32) s += exp(((-Ci[j]) + sm.pt[j]) - mx);
    s = warp_sum(s);
    if (lane == 0) {
      sm.M[i] = mx;
      sm.u[i] = (sm.loga[i] - mx) - log(s);
      sm.wr[i] = sm.a[i] / s;
    }
  }
  __syncthreads();
  // column pass: c_j = sum_i T_ij w_i (dual.cpp:41), 4 row groups
  {
    const int j = tid % kBMax, g = tid / kBMax;
    double acc = 0.0;
    if (j < m) {
      // 4 rows' exponentials in flight, accumulated in the same order
      int i = g;
      for (; i + 3 * kBGroups < n; i += 4 * kBGroups) {
        double e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int ii = i + k * kBGroups;
          e[k] = exp(((-sm.C[ii * kBMax + j]) + sm.pt[j]) - sm.M[ii]) * sm.wr[ii];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += e[k];
      }
      for (; i < n; i += kBGroups)
        acc += exp(((-sm.C[i * kBMax + j]) + sm.pt[j]) - sm.M[i]) * sm.wr[i];
    }
    sm.colp[g][j] = acc;
  }
  __syncthreads();
  double labs = 0.0, ly = 0.0, lpb = 0.0, lua = 0.0;
  if (tid < m) {
    const int j = tid;
    double c = 0.0;
    for (int g = 0; g < kBGroups; ++g) c += sm.colp[g][j];
    double cl;
    if (c >= kTinyPrecise) {
      cl = log(c);
    } else {  // dual.cpp:54-69
      double top = -INFINITY;
      for (int i = 0; i < n; ++i) top = fmax(top, (sm.u[i] + sm.pt[j]) - sm.C[i * kBMax + j]);
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += exp(((sm.u[i] + sm.pt[j]) - sm.C[i * kBMax + j]) - top);
      cl = top + log(s);
      c = exp(cl);
    }
    const double g = c - sm.b[j];
    labs = fabs(g);
    const double y = sm.pt[j] + (sm.logb[j] - cl);
    sm.S[j] = y;
    ly = y;
    lpb = sm.pt[j] * sm.b[j];
  }
  if (tid < n) lua = sm.u[tid] * sm.a[tid];
  labs = warp_sum(labs);
  ly = warp_sum(ly);
  lpb = warp_sum(lpb);
  lua = warp_sum(lua);
  if (lane == 0) {
    sm.red[warp][0] = labs;
    sm.red[warp][1] = ly;
    sm.red[warp][2] = lpb;
    sm.red[warp][3] = lua;
  }
  __syncthreads();
  if (tid == 0) {
    double t[4] = {0, 0, 0, 0};
    for (int k = 0; k < kBT / 32; ++k)
      for (int q = 0; q < 4; ++q) t[q] += sm.red[k][q];
    sm.scal[0] = t[0];                                // grad_l1
    sm.scal[1] = (1.0 - t[3]) - t[2];                 // f = 1 - <u,a> - <v,b>
    sm.scal[2] = t[1] / static_cast<double>(m);       // mean(y)
  }
  __syncthreads();
  if (tid < m) sm.S[tid] -= sm.scal[2];  // project_zero_sum
  __syncthreads();
}

__global__ void __launch_bounds__(kBT)
k_batch_homotopy(int64_t count, const int32_t* __restrict__ nn, const int32_t* __restrict__ mm,
                 const int64_t* __restrict__ off_a, const int64_t* __restrict__ off_b,
                 const int64_t* __restrict__ off_c, const double* __restrict__ ga,
                 const double* __restrict__ gb, const float* __restrict__ gC, double eps,
                 BatchCfg cfg, BatchOut out, unsigned int* __restrict__ queue) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  for (;;) {
    if (tid == 0) sm.prob = static_cast<int>(atomicAdd(queue, 1u));
    __syncthreads();
    const int64_t p = sm.prob;
    if (p >= count) return;
    const int n = nn[p], m = mm[p];
    const double* a = ga + off_a[p];
    const double* b = gb + off_b[p];
    const float* C = gC + off_c[p];
    for (int k = tid; k < n * m; k += kBT) {
      const int i = k / m, j = k % m;
      sm.C[i * kBMax + j] = static_cast<double>(C[k]) / eps;
    }
    if (tid < n) {
      sm.a[tid] = a[tid];
      sm.loga[tid] = log(a[tid]);
    }
    if (tid < m) {
      sm.b[tid] = b[tid];
      sm.logb[tid] = log(b[tid]);
      sm.x[tid] = 0.0;
      sm.w[tid] = 0.0;
      sm.pt[tid] = 0.0;
    }
    __syncthreads();
    // seed evaluation at x0 = 0 (accel.cpp:244-246)
    eval_step(sm, n, m);
    double mu = cfg.mu0, alpha = sqrt(2.0 * mu);
    double gl = sm.scal[0], f = sm.scal[1];
    bool converged = gl < cfg.tol;
    long long total = 0, inner = 0, m_stage = cfg.m0, stage = 0;
    bool stop = converged;
    while (!stop) {
      // x+ = (w + S(x)) / (1 + alpha)   (accel.cpp:161)
      if (tid < m) {
        sm.pt[tid] = (sm.w[tid] + sm.S[tid]) / (1.0 + alpha);
        sm.x[tid] = sm.pt[tid];
      }
      __syncthreads();
      eval_step(sm, n, m);
      // w+ = (w + (alpha^2 - 2) x+ + 2 S(x+)) / (1 + alpha)   (accel.cpp:168)
      if (tid < m) sm.w[tid] = (sm.w[tid] + (alpha * alpha - 2.0) * sm.x[tid] + 2.0 * sm.S[tid]) /
                               (1.0 + alpha);
      gl = sm.scal[0];
      f = sm.scal[1];
      total += 1;
      inner += 1;
      converged = gl < cfg.tol;
      if (converged) break;
      if (inner == m_stage) {  // accel.cpp:276-285
        if (stage + 1 < cfg.max_outer) {
          stage += 1;
          const double alpha_old = alpha;
          mu /= 2.0;
          alpha = sqrt(2.0 * mu);
          if (cfg.rescale_w && tid < m) sm.w[tid] *= alpha / alpha_old;
          m_stage = static_cast<long long>(floor(sqrt(2.0) * static_cast<double>(m_stage))) + 1;
          inner = 0;
        } else {
          stop = true;
        }
      }
      if (total >= cfg.cap) stop = true;
      __syncthreads();
    }
    if (tid == 0) {
      out.converged[p] = converged ? 1 : 0;
      out.iterations[p] = total;
      out.final_violation[p] = gl;
      out.final_f[p] = f;
    }
    if (tid < n) out.u[off_a[p] + tid] = sm.u[tid];
    if (tid < m) out.v[off_b[p] + tid] = sm.x[tid];
    __syncthreads();
  }
}

// C = 1 - <x_i, y_j> per problem (data.cpp:84-110), fp64 dot without FMA
// contraction, then MinMax / HalfRange / raw; stored fp32.
__global__ void __launch_bounds__(kBT)
k_batch_cosine(int64_t count, const int32_t* __restrict__ nn, const int32_t* __restrict__ mm,
               const int64_t* __restrict__ off_a, const int64_t* __restrict__ off_b,
               const int64_t* __restrict__ off_c, const float* __restrict__ X,
               const float* __restrict__ Y, int64_t d, int norm, float* __restrict__ C) {
  __shared__ double sh_min[kBT / 32], sh_max[kBT / 32];
  __shared__ double rng[2];
  for (int64_t p = blockIdx.x; p < count; p += gridDim.x) {
    const int n = nn[p], m = mm[p];
    const float* x = X + off_a[p] * d;
    const float* y = Y + off_b[p] * d;
    float* Cp = C + off_c[p];
    double mn = DBL_MAX, mx = -DBL_MAX;
    for (int k = threadIdx.x; k < n * m; k += kBT) {
      const int i = k / m, j = k % m;
      double s = 0.0;
      for (int64_t t = 0; t < d; ++t)
        s = __dadd_rn(s, __dmul_rn(static_cast<double>(x[i * d + t]), static_cast<double>(y[j * d + t])));
      const double c = __dadd_rn(-s, 1.0);
      mn = fmin(mn, c);
      mx = fmax(mx, c);
      Cp[k] = static_cast<float>(c);  // raw for now
    }
    if (norm == OTG_NORM_MINMAX) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if ((threadIdx.x & 31) == 0) {
        sh_min[threadIdx.x >> 5] = mn;
        sh_max[threadIdx.x >> 5] = mx;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double a = DBL_MAX, b = -DBL_MAX;
        for (int k = 0; k < kBT / 32; ++k) {
          a = fmin(a, sh_min[k]);
          b = fmax(b, sh_max[k]);
        }
        rng[0] = a;
        rng[1] = b;
      }
      __syncthreads();
    }
    if (norm != OTG_NORM_NONE) {
      // recompute from the fp64 raw value (not from its fp32 rounding)
      for (int k = threadIdx.x; k < n * m; k += kBT) {
        const int i = k / m, j = k % m;
        double s = 0.0;
        for (int64_t t = 0; t < d; ++t)
          s = __dadd_rn(s, __dmul_rn(static_cast<double>(x[i * d + t]), static_cast<double>(y[j * d + t])));
        double c = __dadd_rn(-s, 1.0);
        if (norm == OTG_NORM_HALFRANGE) c = c / 2.0;
        else if (norm == OTG_NORM_MINMAX)
          c = (rng[1] - rng[0] > 1e-15) ? (c - rng[0]) / (rng[1] - rng[0]) : 0.0;
        Cp[k] = static_cast<float>(c);
      }
    }
    __syncthreads();
  }
}

void check_sizes(int64_t count, const int32_t* n, const int32_t* m) {
  if (count < 1 || !n || !m) fail(OTG_E_DIMENSION, "batch needs count >= 1 and sizes");
  for (int64_t p = 0; p < count; ++p)
    if (n[p] < 1 || m[p] < 1 || n[p] > kBMax || m[p] > kBMax)
      fail(OTG_E_DIMENSION, "batched problems need 1 <= n, m <= 64");
}

// Host validation of every problem's marginals (core.cpp:9-29).
void check_marginals(int64_t count, const int32_t* n, const int32_t* m, const double* a,
                     const double* b) {
  int64_t oa = 0, ob = 0;
  for (int64_t p = 0; p < count; ++p) {
    for (int side = 0; side < 2; ++side) {
      const double* w = side ? b + ob : a + oa;
      const int len = side ? m[p] : n[p];
      double mn = w[0], s = 0.0;
      for (int k = 0; k < len; ++k) {
        mn = std::min(mn, w[k]);
        s += w[k];
      }
      if (!(mn > 0.0)) fail(OTG_E_INVALID_MARGINALS, "marginals must be strictly positive");
      if (std::abs(s - 1.0) > 1e-9) fail(OTG_E_INVALID_MARGINALS, "marginal does not sum to 1");
    }
    oa += n[p];
    ob += m[p];
  }
}

template <class T>
T* upload(BatchDev& B, const T* src, size_t count) {
  T* d = nullptr;
  OTG_CUDA(cudaMalloc(&d, std::max<size_t>(count, 1) * sizeof(T)));
  if (src) OTG_CUDA(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, B.stream));
  return d;
}

void batch_begin(BatchDev& B, int64_t count, const int32_t* n, const int32_t* m, const double* a,
                 const double* b, double eps, const otg_device_opts* opts) {
  check_sizes(count, n, m);
  if (!a || !b) fail(OTG_E_DIMENSION, "marginals are NULL");
  check_marginals(count, n, m, a, b);
  if (!(eps > 0.0) || !std::isfinite(eps)) fail(OTG_E_OT, "epsilon must be positive and finite");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(OTG_E_UNSUPPORTED, "no CUDA device available (libotg has no CPU fallback)");
  B.device = (opts && opts->device >= 0) ? opts->device : 0;
  OTG_CUDA(cudaSetDevice(B.device));
  OTG_CUDA(cudaStreamCreateWithFlags(&B.stream, cudaStreamNonBlocking));
  B.count = count;
  B.eps = eps;
  std::vector<int64_t> oa(count), ob(count), oc(count);
  int64_t ta = 0, tb = 0, tc = 0;
  for (int64_t p = 0; p < count; ++p) {
    oa[p] = ta;
    ob[p] = tb;
    oc[p] = tc;
    ta += n[p];
    tb += m[p];
    tc += static_cast<int64_t>(n[p]) * m[p];
  }
  B.total_n = ta;
  B.total_m = tb;
  B.total_c = tc;
  B.n = upload(B, n, count);
  B.m = upload(B, m, count);
  B.off_a = upload(B, oa.data(), count);
  B.off_b = upload(B, ob.data(), count);
  B.off_c = upload(B, oc.data(), count);
  B.a = upload(B, a, ta);
  B.b = upload(B, b, tb);
  B.C = upload<float>(B, nullptr, tc);
  OTG_CUDA(cudaStreamSynchronize(B.stream));
}

void batch_free(BatchDev& B) {
  void* ptrs[] = {B.n, B.m, B.off_a, B.off_b, B.off_c, B.a, B.b, B.C};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (B.stream) cudaStreamDestroy(B.stream);
  B = BatchDev{};
}

}  // namespace
}  // namespace otg

struct otg_batch_s {
  otg::BatchDev B;
};

using namespace otg;

extern "C" {

otg_status otg_batch_create_dense(int64_t count, const int32_t* n, const int32_t* m,
                                  const double* a_cat, const double* b_cat, const float* C_cat,
                                  double epsilon, const otg_device_opts* opts, otg_batch* out) {
  BatchDev B;
  const otg_status st = guard([&] {
    if (!out) fail(OTG_E_DIMENSION, "NULL output");
    *out = nullptr;
    if (!C_cat) fail(OTG_E_DIMENSION, "cost is NULL");
    check_sizes(count, n, m);
    int64_t tc = 0;
    for (int64_t p = 0; p < count; ++p) tc += static_cast<int64_t>(n[p]) * m[p];
    for (int64_t k = 0; k < tc; ++k)
      if (!std::isfinite(C_cat[k])) fail(OTG_E_OT, "cost matrix has non-finite entries");
    batch_begin(B, count, n, m, a_cat, b_cat, epsilon, opts);
    OTG_CUDA(cudaMemcpyAsync(B.C, C_cat, tc * sizeof(float), cudaMemcpyHostToDevice, B.stream));
    OTG_CUDA(cudaStreamSynchronize(B.stream));
    auto* h = new otg_batch_s;
    h->B = B;
    *out = h;
  });
  if (st != OTG_OK) batch_free(B);
  return st;
}

otg_status otg_batch_create_cosine(int64_t count, const int32_t* n, const int32_t* m, int64_t d,
                                   const double* a_cat, const double* b_cat, const float* x_cat,
                                   const float* y_cat, otg_norm norm, double epsilon,
                                   const otg_device_opts* opts, otg_batch* out) {
  BatchDev B;
  const otg_status st = guard([&] {
    if (!out) fail(OTG_E_DIMENSION, "NULL output");
    *out = nullptr;
    if (d < 1 || !x_cat || !y_cat) fail(OTG_E_DIMENSION, "embeddings need d >= 1 and data");
    if (norm != OTG_NORM_NONE && norm != OTG_NORM_MINMAX && norm != OTG_NORM_HALFRANGE)
      fail(OTG_E_OT, "cosine cost supports NONE, MINMAX and HALFRANGE");
    check_sizes(count, n, m);
    int64_t tn = 0, tm = 0;
    for (int64_t p = 0; p < count; ++p) {
      tn += n[p];
      tm += m[p];
    }
    for (int side = 0; side < 2; ++side) {  // data.cpp:89-96 unit rows
      const float* Z = side ? y_cat : x_cat;
      const int64_t rows = side ? tm : tn;
      for (int64_t i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) s += static_cast<double>(Z[i * d + k]) * Z[i * d + k];
        if (std::abs(std::sqrt(s) - 1.0) > 1e-6) fail(OTG_E_OT, "cosine cost expects unit rows");
      }
    }
    batch_begin(B, count, n, m, a_cat, b_cat, epsilon, opts);
    float* dx = upload(B, x_cat, tn * d);
    float* dy = upload(B, y_cat, tm * d);
    k_batch_cosine<<<static_cast<unsigned>(std::min<int64_t>(count, 148 * 8)), kBT, 0, B.stream>>>(
        count, B.n, B.m, B.off_a, B.off_b, B.off_c, dx, dy, d, norm, B.C);
    OTG_CUDA(cudaGetLastError());
    OTG_CUDA(cudaStreamSynchronize(B.stream));
    cudaFree(dx);
    cudaFree(dy);
    auto* h = new otg_batch_s;
    h->B = B;
    *out = h;
  });
  if (st != OTG_OK) batch_free(B);
  return st;
}

otg_status otg_batch_destroy(otg_batch h) {
  return guard([&] {
    if (!h) return;
    cudaSetDevice(h->B.device);
    cudaStreamSynchronize(h->B.stream);
    batch_free(h->B);
    delete h;
  });
}

otg_status otg_batch_get_cost(otg_batch h, float* out) {
  return guard([&] {
    if (!h || !out) fail(OTG_E_DIMENSION, "NULL argument");
    BatchDev& B = h->B;
    OTG_CUDA(cudaSetDevice(B.device));
    OTG_CUDA(cudaMemcpyAsync(out, B.C, B.total_c * sizeof(float), cudaMemcpyDeviceToHost, B.stream));
    OTG_CUDA(cudaStreamSynchronize(B.stream));
  });
}

otg_status otg_batch_homotopy_solve(otg_batch h, const otg_homotopy_config* cfg,
                                    otg_batch_result* res) {
  return guard([&] {
    OTG_RANGE("otg_batch_homotopy_solve");
    if (!h || !cfg || !res) fail(OTG_E_DIMENSION, "NULL argument");
    if (!(cfg->mu0 > 0.0) || !(cfg->mu0 < 1.0) || cfg->m0 < 1 || cfg->max_outer < 1)
      fail(OTG_E_OT, "homotopy schedule needs mu0 in (0, 1), m0 >= 1, max_outer >= 1");
    if (!(cfg->tol_l1 > 0.0)) fail(OTG_E_OT, "tol_l1 must be positive");
    if (cfg->max_total_inner < 1) fail(OTG_E_OT, "max_total_inner must be at least 1");
    BatchDev& B = h->B;
    OTG_CUDA(cudaSetDevice(B.device));
    int32_t* d_conv = nullptr;
    int64_t* d_it = nullptr;
    double *d_fv = nullptr, *d_ff = nullptr, *d_u = nullptr, *d_v = nullptr;
    unsigned int* d_q = nullptr;
    OTG_CUDA(cudaMalloc(&d_conv, B.count * sizeof(int32_t)));
    OTG_CUDA(cudaMalloc(&d_it, B.count * sizeof(int64_t)));
    OTG_CUDA(cudaMalloc(&d_fv, B.count * sizeof(double)));
    OTG_CUDA(cudaMalloc(&d_ff, B.count * sizeof(double)));
    OTG_CUDA(cudaMalloc(&d_u, B.total_n * sizeof(double)));
    OTG_CUDA(cudaMalloc(&d_v, B.total_m * sizeof(double)));
    OTG_CUDA(cudaMalloc(&d_q, sizeof(unsigned int)));
    OTG_CUDA(cudaMemsetAsync(d_q, 0, sizeof(unsigned int), B.stream));
    const BatchCfg bc{cfg->mu0, cfg->tol_l1, cfg->m0, cfg->max_outer, cfg->max_total_inner,
                      cfg->rescale_w_across_stages};
    const BatchOut bo{d_conv, d_it, d_fv, d_ff, d_u, d_v};
    const int smem = static_cast<int>(sizeof(Smem));
    OTG_CUDA(cudaFuncSetAttribute(k_batch_homotopy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_batch_homotopy, kBT, smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, B.device);
    const int64_t grid = std::min<int64_t>(B.count, static_cast<int64_t>(std::max(per_sm, 1)) * sms);
    cudaEvent_t e0, e1;
    OTG_CUDA(cudaEventCreate(&e0));
    OTG_CUDA(cudaEventCreate(&e1));
    OTG_CUDA(cudaEventRecord(e0, B.stream));
    k_batch_homotopy<<<static_cast<unsigned>(grid), kBT, smem, B.stream>>>(
        B.count, B.n, B.m, B.off_a, B.off_b, B.off_c, B.a, B.b, B.C, B.eps, bc, bo, d_q);
    OTG_CUDA(cudaGetLastError());
    OTG_CUDA(cudaEventRecord(e1, B.stream));
    OTG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    OTG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    res->device_seconds = ms * 1e-3;
    std::vector<int64_t> it(B.count);
    OTG_CUDA(cudaMemcpy(it.data(), d_it, B.count * sizeof(int64_t), cudaMemcpyDeviceToHost));
    int64_t tot = 0;
    for (int64_t k : it) tot += k;
    res->total_iterations = tot;
    if (res->iterations) std::memcpy(res->iterations, it.data(), B.count * sizeof(int64_t));
    if (res->converged)
      OTG_CUDA(cudaMemcpy(res->converged, d_conv, B.count * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (res->final_violation)
      OTG_CUDA(cudaMemcpy(res->final_violation, d_fv, B.count * sizeof(double), cudaMemcpyDeviceToHost));
    if (res->final_reduced_f)
      OTG_CUDA(cudaMemcpy(res->final_reduced_f, d_ff, B.count * sizeof(double), cudaMemcpyDeviceToHost));
    if (res->u_cat) OTG_CUDA(cudaMemcpy(res->u_cat, d_u, B.total_n * sizeof(double), cudaMemcpyDeviceToHost));
    if (res->v_cat) OTG_CUDA(cudaMemcpy(res->v_cat, d_v, B.total_m * sizeof(double), cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (void* q : {static_cast<void*>(d_conv), static_cast<void*>(d_it), static_cast<void*>(d_fv),
                    static_cast<void*>(d_ff), static_cast<void*>(d_u), static_cast<void*>(d_v),
                    static_cast<void*>(d_q)})
      cudaFree(q);
  });
}

}  // extern "C"
