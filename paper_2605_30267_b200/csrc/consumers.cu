// consumers.cu — plan consumers over the IMPLICIT plan P_ij = exp(u_i + v_j - C'_ij)
// (SURVEY §8f row 1).  The reference materialises P (plan_from_potentials,
// core.cpp:59-71: n x m fp64) and then reads it; here every consumer streams
// the stored (or on-the-fly) cost once and rebuilds P_ij in registers with the
// reference's expression ((-C'_ij) + u_i) + v_j and an fp64 exp, so P is never
// stored.  The 700 overflow guard of core.cpp:66-69 is applied to the same
// exponents.
//
//   otg_plan_barycentric   barycentric_projection (pipelines.cpp:58-71)
//   otg_plan_row_argmax    predict_translations   (pipelines.cpp:101-111)
//   otg_plan_topk          the per-source top-k of topk_accuracy (:113-145)
//   otg_nn_assign          the nearest-sample search of nn_propagate (:73-99)
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"

namespace otg {

namespace {

constexpr int kT = 256;
constexpr int kMaxFeat = 8;     // barycentric features per row
constexpr int kSplits = 64;     // row splits of the column reduction
constexpr double kOverflow = 700.0;  // types.hpp:15

struct Src {
  const double* C64;
  const float* C32;
  const float4* X;
  const float4* Y;
  int64_t ldc;
  double kappa;
};

Src src_of(const Problem& P) {
  return Src{P.C64, P.C32, reinterpret_cast<const float4*>(P.X),
             reinterpret_cast<const float4*>(P.Y), P.ldc, P.kappa};
}

__device__ __forceinline__ double exponent(const Src& s, const double* u, const double* v,
                                           int64_t i, int64_t j) {
  const double c = cost_at(s.C64, s.C32, s.X, s.Y, s.ldc, s.kappa, i, j);
  return ((-c) + u[i]) + v[j];  // core.cpp:63-65
}

// Column partials of [sum_i P_ij x_i (d features), sum_i P_ij] over row split
// blockIdx.y, plus the largest exponent seen (overflow guard).
__global__ void __launch_bounds__(kT)
k_bary_part(const Src s, int64_t n, int64_t m, const double* __restrict__ u,
            const double* __restrict__ v, const double* __restrict__ X, int d,
            int64_t rows_per_split, double* __restrict__ part, double* __restrict__ emax) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t i1 = min(n, i0 + rows_per_split);
  double acc[kMaxFeat + 1];
#pragma unroll
  for (int k = 0; k <= kMaxFeat; ++k) acc[k] = 0.0;
  double mx = -DBL_MAX;
  if (j < m) {
    for (int64_t i = i0; i < i1; ++i) {
      const double e = exponent(s, u, v, i, j);
      mx = fmax(mx, e);
      const double P = exp(e);
#pragma unroll
      for (int k = 0; k < kMaxFeat; ++k)
        if (k < d) acc[k] += P * X[i * d + k];
      acc[kMaxFeat] += P;
    }
    double* dst = part + (static_cast<int64_t>(blockIdx.y) * m + j) * (d + 1);
    for (int k = 0; k < d; ++k) dst[k] = acc[k];
    dst[d] = acc[kMaxFeat];
  }
  __shared__ double sh[kT];
  sh[threadIdx.x] = mx;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) emax[blockIdx.y * gridDim.x + blockIdx.x] = sh[0];
}

// Sum the row splits in order (deterministic).
__global__ void __launch_bounds__(kT)
k_bary_sum(int64_t m, int d, int splits, const double* __restrict__ part,
           double* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (j >= m) return;
  for (int k = 0; k <= d; ++k) {
    double t = 0.0;
    for (int sp = 0; sp < splits; ++sp) t += part[(static_cast<int64_t>(sp) * m + j) * (d + 1) + k];
    out[j * (d + 1) + k] = t;
  }
}

// Row argmax of P (strict >, so ties resolve to the lowest index) and the
// row's largest exponent; R rows per CTA.
__global__ void __launch_bounds__(kT)
k_row_argmax(const Src s, int64_t n, int64_t m, const double* __restrict__ u,
             const double* __restrict__ v, int* __restrict__ best, double* __restrict__ emax) {
  const int64_t i = blockIdx.x;
  double bp = -1.0, mx = -DBL_MAX;
  int64_t bj = m;
  for (int64_t j = threadIdx.x; j < m; j += kT) {
    const double e = exponent(s, u, v, i, j);
    mx = fmax(mx, e);
    const double P = exp(e);
    if (P > bp) {  // j increases along the thread's stride: first max kept
      bp = P;
      bj = j;
    }
  }
  __shared__ double sp[kT], sm[kT];
  __shared__ int64_t sj[kT];
  sp[threadIdx.x] = bp;
  sj[threadIdx.x] = bj;
  sm[threadIdx.x] = mx;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double p2 = sp[threadIdx.x + o];
      const int64_t j2 = sj[threadIdx.x + o];
      if (p2 > sp[threadIdx.x] || (p2 == sp[threadIdx.x] && j2 < sj[threadIdx.x])) {
        sp[threadIdx.x] = p2;
        sj[threadIdx.x] = j2;
      }
      sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    best[i] = static_cast<int>(sj[0]);
    emax[i] = sm[0];
  }
}

// Top-k of row rows[b] by (P descending, index ascending): k rounds, each the
// largest element strictly after the previous pick in that order.
__global__ void __launch_bounds__(kT)
k_row_topk(const Src s, int64_t m, const double* __restrict__ u, const double* __restrict__ v,
           const int* __restrict__ rows, int k, int* __restrict__ out,
           double* __restrict__ emax) {
  const int64_t i = rows[blockIdx.x];
  __shared__ double sp[kT], sm[kT];
  __shared__ int64_t sj[kT];
  double lastP = DBL_MAX;
  int64_t lastJ = -1;
  for (int r = 0; r < k; ++r) {
    double bp = -1.0, mx = -DBL_MAX;
    int64_t bj = m;
    for (int64_t j = threadIdx.x; j < m; j += kT) {
      const double e = exponent(s, u, v, i, j);
      mx = fmax(mx, e);
      const double P = exp(e);
      const bool after = P < lastP || (P == lastP && j > lastJ);
      if (after && P > bp) {
        bp = P;
        bj = j;
      }
    }
    sp[threadIdx.x] = bp;
    sj[threadIdx.x] = bj;
    sm[threadIdx.x] = mx;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const double p2 = sp[threadIdx.x + o];
        const int64_t j2 = sj[threadIdx.x + o];
        if (p2 > sp[threadIdx.x] || (p2 == sp[threadIdx.x] && j2 < sj[threadIdx.x])) {
          sp[threadIdx.x] = p2;
          sj[threadIdx.x] = j2;
        }
        sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
      }
      __syncthreads();
    }
    lastP = sp[0];
    lastJ = sj[0];
    if (threadIdx.x == 0) {
      out[static_cast<int64_t>(blockIdx.x) * k + r] = lastJ < m ? static_cast<int>(lastJ) : -1;
      if (r == 0) emax[blockIdx.x] = sm[0];
    }
    __syncthreads();
  }
}

// Nearest reference point (squared distance in fp64, strict <: lowest index
// on ties), reference points staged through shared memory.
template <int D>
__global__ void __launch_bounds__(kT)
k_nn(const double* __restrict__ q, int64_t nq, const double* __restrict__ ref, int64_t nref,
     int* __restrict__ out) {
  __shared__ double tile[kT * D];
  const int64_t p = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  double c[D];
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = p < nq ? q[p * D + k] : 0.0;
  double best_d2 = DBL_MAX;
  int64_t best = 0;
  for (int64_t t0 = 0; t0 < nref; t0 += kT) {
    const int64_t tn = min(static_cast<int64_t>(kT), nref - t0);
    __syncthreads();
    for (int64_t k = threadIdx.x; k < tn * D; k += kT) tile[k] = ref[t0 * D + k];
    __syncthreads();
    for (int64_t r = 0; r < tn; ++r) {
      double d2 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double dd = __dsub_rn(c[k], tile[r * D + k]);
        d2 = __dadd_rn(d2, __dmul_rn(dd, dd));
      }
      if (t0 + r == 0 || d2 < best_d2) {
        best_d2 = d2;
        best = t0 + r;
      }
    }
  }
  if (p < nq) out[p] = static_cast<int>(best);
}

// ---- diagnostics (dual.cpp:88-101, 118-136) ----

// Q_ij = P_ij / sqrt(a_i) with the plan of the row solve at v
// (plan_from_workspace, dual.cpp:72-78): P_ij = exp((-C'_ij + v_j) - M_i) a_i / S_i.
__global__ void __launch_bounds__(kT)
k_plan_q(const Src s, int64_t n, int64_t m, const double* __restrict__ v,
         const double* __restrict__ rowM, const double* __restrict__ wrow,
         const double* __restrict__ a, double* __restrict__ Q) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const double Mi = rowM[i], wi = wrow[i], ra = 1.0 / sqrt(a[i]);
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; j < m;
         j += static_cast<int64_t>(gridDim.x) * kT) {
      const double c = cost_at(s.C64, s.C32, s.X, s.Y, s.ldc, s.kappa, i, j);
      Q[i * m + j] = exp(((-c) + v[j]) - Mi) * wi * ra;
    }
  }
}

// H_jk = -sum_i Q_ij Q_ik (+ col_j on the diagonal, added on the host):
// 32 x 32 output tiles, rows of Q staged through shared memory.
constexpr int kHT = 32;
__global__ void __launch_bounds__(kHT * kHT)
k_syrk_neg(int64_t n, int64_t m, const double* __restrict__ Q, double* __restrict__ H) {
  __shared__ double qa[kHT][kHT + 1], qb[kHT][kHT + 1];
  const int tj = threadIdx.x % kHT, tk = threadIdx.x / kHT;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kHT, k0 = static_cast<int64_t>(blockIdx.y) * kHT;
  double acc = 0.0;
  for (int64_t i0 = 0; i0 < n; i0 += kHT) {
    const int64_t ir = i0 + tk;
    qa[tk][tj] = (ir < n && j0 + tj < m) ? Q[ir * m + j0 + tj] : 0.0;
    qb[tk][tj] = (ir < n && k0 + tj < m) ? Q[ir * m + k0 + tj] : 0.0;
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < kHT; ++r) acc += qa[r][tj] * qb[r][tk];
    __syncthreads();
  }
  if (j0 + tj < m && k0 + tk < m) H[(k0 + tk) * m + j0 + tj] = -acc;
}

// dual_F: per-row online (max, sum) of E_ij = ((-C'_ij) + u_i) + v_j.
__global__ void __launch_bounds__(kT)
k_dual_rows(const Src s, int64_t n, int64_t m, const double* __restrict__ u,
            const double* __restrict__ v, double2* __restrict__ out) {
  const int64_t i = blockIdx.x;
  double top = -DBL_MAX, sum = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += kT) {
    const double e = exponent(s, u, v, i, j);
    if (e > top) {
      sum = sum * exp(top - e) + 1.0;
      top = e;
    } else {
      sum += exp(e - top);
    }
  }
  __shared__ double st[kT], ss[kT];
  st[threadIdx.x] = top;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) st[threadIdx.x] = fmax(st[threadIdx.x], st[threadIdx.x + o]);
    __syncthreads();
  }
  const double T = st[0];
  __syncthreads();
  ss[threadIdx.x] = top > -DBL_MAX ? sum * exp(top - T) : 0.0;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) ss[threadIdx.x] += ss[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = make_double2(T, ss[0]);
}

void check_vec(const double* x, int64_t count, const char* what) {  // dual.cpp:13-18
  if (!x) fail(OTG_E_DIMENSION, std::string(what) + " is NULL");
  for (int64_t k = 0; k < count; ++k)
    if (!std::isfinite(x[k])) fail(OTG_E_OT, std::string(what) + " has non-finite entries");
}

// Upload u (local rows) and v into dst (n_local + m doubles).
void upload_uv(Problem& P, const double* u, const double* v, double* dst) {
  check_vec(u, P.n_local, "u");
  check_vec(v, P.m, "v");
  OTG_CUDA(cudaMemcpyAsync(dst, u, P.n_local * sizeof(double), cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(dst + P.n_local, v, P.m * sizeof(double), cudaMemcpyHostToDevice,
                           P.stream));
}

void check_overflow(const std::vector<double>& emax) {  // core.cpp:66-69
  double top = -DBL_MAX;
  for (double e : emax) top = std::max(top, e);
  if (top > kOverflow) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "plan exponent %.3g exceeds bound", top);
    fail(OTG_E_OVERFLOW, buf);
  }
}

void check(otg_status st) {  // a nested C-ABI call: propagate its status and message
  if (st != OTG_OK) fail(st, otg_last_error());
}

struct DevBuf {  // RAII for the consumers' scratch
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { OTG_CUDA(cudaMalloc(&p, bytes)); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

}  // namespace
}  // namespace otg

using namespace otg;

extern "C" {

otg_status otg_plan_barycentric(otg_problem h, const double* u, const double* v,
                                const double* src, int d, double* out, double* col_mass) {
  return guard([&] {
    OTG_RANGE("otg_plan_barycentric");
    Problem& P = problem_of(h);
    if (d < 1 || d > kMaxFeat) fail(OTG_E_DIMENSION, "barycentric features: 1 <= d <= 8");
    if (!src || !out) fail(OTG_E_DIMENSION, "NULL feature / output buffer");
    const int64_t n = P.n_local, m = P.m;
    DevBuf uvb(static_cast<size_t>(P.n_local + P.m) * sizeof(double));
    double* uv = uvb.as<double>();
    upload_uv(P, u, v, uv);
    DevBuf X(static_cast<size_t>(n) * d * sizeof(double));
    OTG_CUDA(cudaMemcpyAsync(X.p, src, static_cast<size_t>(n) * d * sizeof(double),
                             cudaMemcpyHostToDevice, P.stream));
    const int splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kSplits, n / 16)));
    const int64_t rps = (n + splits - 1) / splits;
    const unsigned gx = static_cast<unsigned>((m + kT - 1) / kT);
    DevBuf part(static_cast<size_t>(splits) * m * (d + 1) * sizeof(double));
    DevBuf sums(static_cast<size_t>(m) * (d + 1) * sizeof(double));
    DevBuf emax(static_cast<size_t>(splits) * gx * sizeof(double));
    k_bary_part<<<dim3(gx, splits), kT, 0, P.stream>>>(src_of(P), n, m, uv, uv + n, X.as<double>(),
                                                       d, rps, part.as<double>(),
                                                       emax.as<double>());
    k_bary_sum<<<gx, kT, 0, P.stream>>>(m, d, splits, part.as<double>(), sums.as<double>());
    OTG_CUDA(cudaGetLastError());
    if (P.sharded) {
      comm_allreduce_sum(P, sums.as<double>(), static_cast<size_t>(m) * (d + 1));
      comm_allreduce_max(P, emax.as<double>(), static_cast<size_t>(splits) * gx);
    }
    std::vector<double> hs(static_cast<size_t>(m) * (d + 1)), he(static_cast<size_t>(splits) * gx);
    OTG_CUDA(cudaMemcpyAsync(hs.data(), sums.p, hs.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaMemcpyAsync(he.data(), emax.p, he.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    check_overflow(he);
    for (int64_t j = 0; j < m; ++j) {  // pipelines.cpp:62-67
      const double c = hs[j * (d + 1) + d];
      if (!(c > 0.0)) fail(OTG_E_DEGENERATE, "plan column " + std::to_string(j) + " has zero mass");
    }
    for (int64_t j = 0; j < m; ++j) {  // out = P^T src, rows divided by the column mass
      const double c = hs[j * (d + 1) + d];
      for (int k = 0; k < d; ++k) out[j * d + k] = hs[j * (d + 1) + k] / c;
      if (col_mass) col_mass[j] = c;
    }
  });
}

otg_status otg_plan_row_argmax(otg_problem h, const double* u, const double* v, int* out) {
  return guard([&] {
    Problem& P = problem_of(h);
    if (!out) fail(OTG_E_DIMENSION, "NULL output buffer");
    const int64_t n = P.n_local, m = P.m;
    DevBuf uvb(static_cast<size_t>(P.n_local + P.m) * sizeof(double));
    double* uv = uvb.as<double>();
    upload_uv(P, u, v, uv);
    DevBuf best(static_cast<size_t>(n) * sizeof(int));
    DevBuf emax(static_cast<size_t>(n) * sizeof(double));
    k_row_argmax<<<static_cast<unsigned>(n), kT, 0, P.stream>>>(src_of(P), n, m, uv, uv + n,
                                                                 best.as<int>(), emax.as<double>());
    OTG_CUDA(cudaGetLastError());
    std::vector<double> he(n);
    OTG_CUDA(cudaMemcpyAsync(out, best.p, n * sizeof(int), cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaMemcpyAsync(he.data(), emax.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                             P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    check_overflow(he);
  });
}

otg_status otg_plan_topk(otg_problem h, const double* u, const double* v, const int* rows,
                         int64_t nrows, int k, int* out) {
  return guard([&] {
    OTG_RANGE("otg_plan_topk");
    Problem& P = problem_of(h);
    if (k < 1) fail(OTG_E_OT, "topk needs k >= 1");
    if (nrows < 0 || (nrows > 0 && (!rows || !out))) fail(OTG_E_DIMENSION, "NULL rows / output");
    for (int64_t b = 0; b < nrows; ++b)
      if (rows[b] < 0 || rows[b] >= P.n_local) fail(OTG_E_DIMENSION, "row index outside the plan");
    if (nrows == 0) return;
    const int kk = static_cast<int>(std::min<int64_t>(k, P.m));
    DevBuf uvb(static_cast<size_t>(P.n_local + P.m) * sizeof(double));
    double* uv = uvb.as<double>();
    upload_uv(P, u, v, uv);
    DevBuf drows(static_cast<size_t>(nrows) * sizeof(int));
    DevBuf dout(static_cast<size_t>(nrows) * kk * sizeof(int));
    DevBuf emax(static_cast<size_t>(nrows) * sizeof(double));
    OTG_CUDA(cudaMemcpyAsync(drows.p, rows, nrows * sizeof(int), cudaMemcpyHostToDevice,
                             P.stream));
    k_row_topk<<<static_cast<unsigned>(nrows), kT, 0, P.stream>>>(
        src_of(P), P.m, uv, uv + P.n_local, drows.as<int>(), kk, dout.as<int>(),
        emax.as<double>());
    OTG_CUDA(cudaGetLastError());
    std::vector<int> ho(static_cast<size_t>(nrows) * kk);
    std::vector<double> he(nrows);
    OTG_CUDA(cudaMemcpyAsync(ho.data(), dout.p, ho.size() * sizeof(int), cudaMemcpyDeviceToHost,
                             P.stream));
    OTG_CUDA(cudaMemcpyAsync(he.data(), emax.p, he.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    check_overflow(he);
    for (int64_t b = 0; b < nrows; ++b)  // out is nrows x k; picks beyond m are -1
      for (int r = 0; r < k; ++r) out[b * k + r] = r < kk ? ho[b * kk + r] : -1;
  });
}

otg_status otg_nn_assign(const double* queries, int64_t nq, const double* refs, int64_t nref,
                         int d, int device, int* out) {
  return guard([&] {
    if (d != 3 && d != 1 && d != 2 && d != 4) fail(OTG_E_DIMENSION, "nn_assign supports d in 1..4");
    if (nref < 1) fail(OTG_E_DIMENSION, "no reference points");
    if (nq < 0 || (nq > 0 && (!queries || !out)) || !refs) fail(OTG_E_DIMENSION, "NULL buffer");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1)
      fail(OTG_E_UNSUPPORTED, "no CUDA device (this library has no CPU fallback)");
    OTG_CUDA(cudaSetDevice(device));
    if (nq == 0) return;
    DevBuf dq(static_cast<size_t>(nq) * d * sizeof(double));
    DevBuf dr(static_cast<size_t>(nref) * d * sizeof(double));
    DevBuf dout(static_cast<size_t>(nq) * sizeof(int));
    OTG_CUDA(cudaMemcpy(dq.p, queries, static_cast<size_t>(nq) * d * sizeof(double),
                        cudaMemcpyHostToDevice));
    OTG_CUDA(cudaMemcpy(dr.p, refs, static_cast<size_t>(nref) * d * sizeof(double),
                        cudaMemcpyHostToDevice));
    const unsigned g = static_cast<unsigned>((nq + kT - 1) / kT);
    switch (d) {
      case 1: k_nn<1><<<g, kT>>>(dq.as<double>(), nq, dr.as<double>(), nref, dout.as<int>()); break;
      case 2: k_nn<2><<<g, kT>>>(dq.as<double>(), nq, dr.as<double>(), nref, dout.as<int>()); break;
      case 3: k_nn<3><<<g, kT>>>(dq.as<double>(), nq, dr.as<double>(), nref, dout.as<int>()); break;
      default: k_nn<4><<<g, kT>>>(dq.as<double>(), nq, dr.as<double>(), nref, dout.as<int>());
    }
    OTG_CUDA(cudaGetLastError());
    OTG_CUDA(cudaMemcpy(out, dout.p, static_cast<size_t>(nq) * sizeof(int), cudaMemcpyDeviceToHost));
  });
}

otg_status otg_dual_F(otg_problem h, const double* u, const double* v, double* out) {
  return guard([&] {  // dual.cpp:88-101
    Problem& P = problem_of(h);
    if (!out) fail(OTG_E_DIMENSION, "NULL output");
    const int64_t n = P.n_local, m = P.m;
    DevBuf uvb(static_cast<size_t>(n + m) * sizeof(double));
    double* uv = uvb.as<double>();
    upload_uv(P, u, v, uv);
    DevBuf rows(static_cast<size_t>(n) * sizeof(double2));
    k_dual_rows<<<static_cast<unsigned>(n), kT, 0, P.stream>>>(src_of(P), n, m, uv, uv + n,
                                                               rows.as<double2>());
    OTG_CUDA(cudaGetLastError());
    std::vector<double2> hr(n);
    OTG_CUDA(cudaMemcpyAsync(hr.data(), rows.p, n * sizeof(double2), cudaMemcpyDeviceToHost,
                             P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    double top = -DBL_MAX;
    for (const auto& r : hr) top = std::max(top, r.x);
    double sum = 0.0, ua = 0.0, vb = 0.0;
    for (const auto& r : hr) sum += r.y * std::exp(r.x - top);
    std::vector<double> ha(n), hb(m);
    OTG_CUDA(cudaMemcpy(ha.data(), P.a, n * sizeof(double), cudaMemcpyDeviceToHost));
    OTG_CUDA(cudaMemcpy(hb.data(), P.b, m * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) ua += u[i] * ha[i];
    for (int64_t j = 0; j < m; ++j) vb += v[j] * hb[j];
    if (P.sharded) {  // global max, then the rescaled sums and <u, a>
      DevBuf d(3 * sizeof(double));
      double hv[3] = {top, 0.0, 0.0};
      OTG_CUDA(cudaMemcpy(d.p, hv, sizeof(double), cudaMemcpyHostToDevice));
      comm_allreduce_max(P, d.as<double>(), 1);
      OTG_CUDA(cudaMemcpy(hv, d.p, sizeof(double), cudaMemcpyDeviceToHost));
      const double g = hv[0];
      hv[1] = sum * std::exp(top - g);
      hv[2] = ua;
      OTG_CUDA(cudaMemcpy(d.as<double>() + 1, hv + 1, 2 * sizeof(double), cudaMemcpyHostToDevice));
      comm_allreduce_sum(P, d.as<double>() + 1, 2);
      OTG_CUDA(cudaMemcpy(hv + 1, d.as<double>() + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost));
      top = g;
      sum = hv[1];
      ua = hv[2];
    }
    const double lse = top + std::log(sum);
    if (lse > kOverflow) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "dual mass exponent %.3g exceeds bound", lse);
      fail(OTG_E_OVERFLOW, buf);
    }
    *out = std::exp(lse) - ua - vb;
  });
}

otg_status otg_hessian_f(otg_problem h, const double* v, double* H) {
  return guard([&] {  // dual.cpp:118-136
    OTG_RANGE("otg_hessian_f");
    Problem& P = problem_of(h);
    if (!H) fail(OTG_E_DIMENSION, "NULL output");
    const int64_t n = P.n_local, m = P.m;
    if (m > 2000) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "dense reduced Hessian capped at m = 2000, got %lld",
                    static_cast<long long>(m));
      fail(OTG_E_TOO_LARGE, buf);
    }
    std::vector<double> u(n), col(m);
    check(otg_row_solve_marginals(h, v, u.data(), col.data()));  // rowM, wrow on the device
    DevBuf dv(static_cast<size_t>(m) * sizeof(double));
    OTG_CUDA(cudaMemcpyAsync(dv.p, v, m * sizeof(double), cudaMemcpyHostToDevice, P.stream));
    DevBuf Q(static_cast<size_t>(n) * m * sizeof(double));
    DevBuf dH(static_cast<size_t>(m) * m * sizeof(double));
    const dim3 gq(static_cast<unsigned>(std::min<int64_t>((m + kT - 1) / kT, 64)),
                  static_cast<unsigned>(std::min<int64_t>(n, 65535)));
    k_plan_q<<<gq, kT, 0, P.stream>>>(src_of(P), n, m, dv.as<double>(), P.rowM, P.wrow, P.a,
                                       Q.as<double>());
    const unsigned gt = static_cast<unsigned>((m + kHT - 1) / kHT);
    k_syrk_neg<<<dim3(gt, gt), kHT * kHT, 0, P.stream>>>(n, m, Q.as<double>(), dH.as<double>());
    OTG_CUDA(cudaGetLastError());
    if (P.sharded) comm_allreduce_sum(P, dH.as<double>(), static_cast<size_t>(m) * m);
    OTG_CUDA(cudaMemcpyAsync(H, dH.p, static_cast<size_t>(m) * m * sizeof(double),
                             cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    for (int64_t j = 0; j < m; ++j) H[j * m + j] += col[j];  // + col.asDiagonal()
  });
}

}  // extern "C"
