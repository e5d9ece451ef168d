// sweep.cu — the O(nm) evaluation of the normalised Sinkhorn map on sm_100a.
//
// One evaluation at the column potential p (reference: eval_normalized_step,
// sinkhorn.cpp:51-63 -> row_solve_marginals_log, dual.cpp:44-70 ->
// row_solve_marginals, dual.cpp:29-42) is this launch sequence on the
// handle's stream:
//
//   K1 row pass     M_i = max_j (p_j - C'_ij), S_i = sum_j exp(. - M_i),
//                   u_i = (log a_i - M_i) - log S_i, w_i = a_i / S_i
//   K2 column pass  partial c_j = sum_{i in split} w_i exp(p_j - C'_ij - M_i)
//   E1a merge       c_j = sum of partials (fixed order); flag c_j < tiny
//   K5 fallback     exact column log-sum-exp for flagged columns (dual.cpp:53-69)
//   E1b finalize    log c, grad = c - b, |grad|_1, mean(y), f; LAST CTA runs the
//                   solver's scalar control flow (stop test, homotopy schedule,
//                   trace) on the device
//   E2  apply       S(p) = y - mean(y) (mirror.cpp:103-105) fused with the
//                   Acc-Sinkhorn extrapolation (accel.cpp:161-169) and the
//                   stability-condition sums (diag.cpp:107-146)
//
// Two numeric paths:
//  * fp64 storage ("precise"): C' = C / eps stored in fp64, every exponential
//    is the IEEE fp64 exp of the reference's own expression -> per-iterate
//    parity to ~1e-13.
//  * fp32 storage ("fast"): C fp32 read once per pass with 128-bit streaming
//    loads.  Row pass: exponent argument formed in fp64 (DFMA) with an online
//    max, rounded to fp32 only after the max shift, MUFU ex2, fp64 partial
//    sums.  Column pass: all-fp32 exact cancellation - the row shift and the
//    column potential are split into a 2^-8-quantised part (exactly
//    representable, differences exact) and a small remainder, so
//    fmaf(-C, kappa_hi, Vc - Mc) cancels the large magnitudes inside one FMA
//    and only the small result is rounded; fp32 accumulation flushed into
//    fp64 every 16 rows.
//
// All kernels read the control block first and return at once after the
// solve stopped, so a captured chunk of evaluations can run past the stop
// point harmlessly.
#include <cuda_runtime.h>

#include <cfloat>

#include "common.cuh"

// resident CTAs per SM the stored fp32 row / column kernels are compiled for
// (the register cap follows: 4 -> 64, 5 -> 48 registers per thread)
#ifndef OTG_ROW_MINB
#define OTG_ROW_MINB 4
#endif
#ifndef OTG_COL_MINB
#define OTG_COL_MINB 5
#endif
#ifndef OTG_EXACT_MINB
#define OTG_EXACT_MINB 4
#endif
#ifndef OTG_ROW_OTF_MINB
#define OTG_ROW_OTF_MINB 2
#endif
#ifndef OTG_ROW_OTF_UNROLL
#define OTG_ROW_OTF_UNROLL 4
#endif
#ifndef OTG_COL_OTF_MINB
#define OTG_COL_OTF_MINB 1
#endif

namespace otg {

namespace {

constexpr int kRowThreads = 256;
constexpr int kColThreads = 128;
constexpr int kColUnroll = 8;
constexpr int kAuxTile = 256;
constexpr int kEThreads = 256;
constexpr int kFbChunks = 32;
constexpr int kFbUnroll = 8;
constexpr int kE2 = 16;  // doubles per CTA partial of the vector update (stability + energy)
constexpr int kFlushRows = 16;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float4 ld_stream(const float4* ptr) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(ptr));
  return r;
}

__device__ __forceinline__ void prefetch_l2(const void* ptr) {
  asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(ptr));
}
__device__ __forceinline__ float4 ld_stream256(const float4* ptr) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(ptr));
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions for blockDim == NT (multiple of 32); result valid in
// every thread.  Deterministic: fixed shuffle tree then fixed warp order.
template <int NT>
__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) r += sh[k];
  return r;
}
template <int NT>
__device__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = -DBL_MAX;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) r = fmax(r, sh[k]);
  return r;
}

// NS sums then NM maxima in one pass (two barriers instead of two per value);
// each value reduced exactly as block_sum / block_max would (same shuffle
// tree, same warp order), so results are bitwise those of separate calls.
template <int NT, int NS, int NM>
__device__ void block_multi(double (&v)[NS + NM], double* shm /* NT / 32 * (NS + NM) */) {
  constexpr int N = NS + NM, W = NT / 32;
#pragma unroll
  for (int q = 0; q < NS; ++q) v[q] = warp_sum(v[q]);
#pragma unroll
  for (int q = NS; q < N; ++q) v[q] = warp_max(v[q]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) shm[q * W + w] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double r = q < NS ? 0.0 : -DBL_MAX;
#pragma unroll
    for (int k = 0; k < W; ++k) r = q < NS ? r + shm[q * W + k] : fmax(r, shm[q * W + k]);
    v[q] = r;
  }
}

// Exact fp32 -> fp64 with integer ops (ALU pipe, no F2F on the XU pipe).
// Normal and zero inputs map exactly except +-0 and subnormals, which land
// within 2^-126 of their value (|error| < 1.2e-38; irrelevant for a cost).
__device__ __forceinline__ double f32_to_f64(float x) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t hi = (((b & 0x7fffffffu) >> 3) + 0x38000000u) | (b & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(b << 29));
}

// fp64 -> fp32 (round to nearest) for a value in [-2^127, 0] with integer ops;
// values above -2^-100 are clamped to -2^-100 (ex2 of it is 1.0f).
__device__ __forceinline__ float neg_f64_to_f32(double x) {
  x = fmin(x, -7.888609052210118e-31);  // -2^-100
  const uint32_t lo = static_cast<uint32_t>(__double2loint(x));
  const uint32_t hi = static_cast<uint32_t>(__double2hiint(x));
  const uint32_t w = __funnelshift_l(lo, hi, 3);  // exponent[8:0] | mantissa[51:29]
  const uint32_t rb = (lo >> 28) & 1u;            // round bit
  return __uint_as_float((w - 0xC0000000u + rb) | 0x80000000u);
}

// fp32 partial -> fp64 in the on-the-fly sweeps, whose XU pipe carries the
// ex2 stream: OTG_OTF_INT_CVT=1 converts with integer ops (f32_to_f64; a zero
// partial maps to 2^-127-scale, negligible in a sum), 0 with F2F.
#ifndef OTG_OTF_INT_CVT
#define OTG_OTF_INT_CVT 0
#endif
__device__ __forceinline__ double otf_cvt(float x) {
  return OTG_OTF_INT_CVT ? f32_to_f64(x) : static_cast<double>(x);
}

// Quantised split of a base-2 value: hi is a multiple of 2^-8 (exact in fp32
// for |x| < 2^15), lo = x - hi rounded to fp32 (|lo| <= 2^-9).
__device__ __forceinline__ void split_q(double x2, float& hi, float& lo) {
  const double h = rint(x2 * 256.0) * (1.0 / 256.0);
  hi = static_cast<float>(h);
  lo = static_cast<float>(x2 - h);
}

// The row pass's column potential, three planes of stride mpad: the quantised
// split (V, F) and 2^F (fp32 round of the fp64 power), which the on-the-fly
// kernels apply as a factor after the ex2 instead of adding F to the exponent.
__device__ __forceinline__ void split_store(double x2, float* vq, int64_t mpad, int64_t j) {
  float hi, lo;
  split_q(x2, hi, lo);
  vq[j] = hi;
  vq[mpad + j] = lo;
  vq[2 * mpad + j] = static_cast<float>(exp2(static_cast<double>(lo)));
}

// ------------------------------------------------------------------ K1 ----
// fp64 storage: exact restatement of dual.cpp:34-38 for one row per G threads.
template <int G>
__global__ void __launch_bounds__(kRowThreads)
k_row_precise(const double* __restrict__ C, int64_t ldc, int64_t n, int64_t m,
              const double* __restrict__ p, const double* __restrict__ a,
              const double* __restrict__ loga, double* __restrict__ rowM,
              double* __restrict__ rowS, double* __restrict__ u, double* __restrict__ wrow,
              double* __restrict__ rowpart, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  constexpr int RPB = kRowThreads / G;
  __shared__ double sh[kRowThreads / 32];
  __shared__ double ua_sh[RPB];
  const int sub = threadIdx.x / G, lane = threadIdx.x % G;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * RPB + sub;
  const bool valid = i < n;
  const double* Ci = C + (valid ? i : 0) * ldc;
  // the thread's first kRC exponents stay in registers (all loads in flight;
  // cfg1, 1000^2 with G = 128: the whole row); longer rows stream the rest in
  // kRC-wide chunks.  Sums in column order per thread, as the plain loop.
  constexpr int kRC = 8;
  double t0[kRC];
#pragma unroll
  for (int k = 0; k < kRC; ++k) {
    const int64_t j = lane + static_cast<int64_t>(k) * G;
    t0[k] = (valid && j < m) ? (-Ci[j]) + p[j] : -INFINITY;
  }
  double mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < kRC; ++k) mx = fmax(mx, t0[k]);
  if (valid)
    for (int64_t j0 = lane + kRC * G; j0 < m; j0 += kRC * G) {
      double t[kRC];
#pragma unroll
      for (int k = 0; k < kRC; ++k) {
        const int64_t j = j0 + static_cast<int64_t>(k) * G;
        t[k] = j < m ? (-Ci[j]) + p[j] : -INFINITY;
      }
#pragma unroll
      for (int k = 0; k < kRC; ++k) mx = fmax(mx, t[k]);
    }
  auto row_sum = [&](double mxr) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < kRC; ++k)
      if (lane + static_cast<int64_t>(k) * G < m) acc += exp(t0[k] - mxr);
    for (int64_t j0 = lane + kRC * G; j0 < m; j0 += kRC * G) {
      double t[kRC];
#pragma unroll
      for (int k = 0; k < kRC; ++k) {
        const int64_t j = j0 + static_cast<int64_t>(k) * G;
        t[k] = j < m ? (-Ci[j]) + p[j] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kRC; ++k)
        if (j0 + static_cast<int64_t>(k) * G < m) acc += exp(t[k] - mxr);
    }
    return acc;
  };
  double s = 0.0;
  if (G == 32) {
    mx = warp_max(mx);
    if (valid) s = row_sum(mx);
    s = warp_sum(s);
  } else if (G < kRowThreads) {
    // G / 32 warps per row: shuffle trees, then the group's warps in order
    constexpr int WG = G / 32;
    const int w0 = sub * WG;
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = -DBL_MAX;
#pragma unroll
    for (int k = 0; k < WG; ++k) mx = fmax(mx, sh[w0 + k]);
    if (valid) s = row_sum(mx);
    s = warp_sum(s);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    s = 0.0;
#pragma unroll
    for (int k = 0; k < WG; ++k) s += sh[w0 + k];
  } else {
    mx = block_max<kRowThreads>(mx, sh);
    s = row_sum(mx);
    s = block_sum<kRowThreads>(s, sh);
  }
  if (lane == 0) {
    double ua = 0.0;
    if (valid) {
      const double ui = (loga[i] - mx) - log(s);
      rowM[i] = mx;
      rowS[i] = s;
      u[i] = ui;
      wrow[i] = a[i] / s;
      ua = ui * a[i];
    }
    ua_sh[sub] = ua;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < RPB; ++k) t += ua_sh[k];
    rowpart[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------- cost sources ----
// The fp32 kernels read the cost either from the stored matrix (C, ldc) or
// recompute it per tile from fp32 points (BASELINE config 5, C never stored):
//   C_ij = fl32(fl32(dz^2 + fl32(dy^2 + fl32(dx^2))))  with d = x_i - y_j,
// the squared-Euclidean cost of data.cpp:69-82 evaluated in fp32 with this
// exact operation order, which is the definition the oracle reproduces.
struct CostSrc {
  const float* C;    // stored: n x ldc
  int64_t ldc;
  const float4* X;   // on-the-fly: n points (x, y, z, 0)
  const float4* Y;   // on-the-fly: m points (x, y, z, 0)
  const float* Yn;   // on-the-fly: the same points negated, SoA [-x | -y | -z], stride ypad
  int64_t ypad;
  // on the fly, spatially sorted sweeps with exact block culling (P.cull):
  // rows / columns visited in Morton order; a block is skipped when a bound
  // proves every exponent in it below -127 (ex2.approx.ftz returns +0 there,
  // so skipping is bitwise the same sum)
  const int* perm_r;   // sorted row position -> row
  const int* perm_c;   // sorted column position -> column
  const float4* Xs;    // rows in sorted order
  const float4* cbox;  // per kCullCB sorted columns: (lo, hi) boxes
  const float* cvmax;  // per kCullCB sorted columns: max V (this evaluation)
  const float4* rbox;  // per kCullRB sorted rows: (lo, hi) boxes
  const float* rnegm;  // per kCullRB sorted rows: max -M (this evaluation)
  int skip;            // 0: visit every block in the sorted order (test hook)
  const float2* ves;   // per sorted column: (V, 2^F) of this evaluation
  const float4* auxs;  // per sorted row: aux with w' = w 2^-mf, this evaluation
};

constexpr int kCullCB = 64;  // columns per culling block (row pass)
constexpr int kCullRowT = OTG_CULL_ROW_T;  // threads per CTA of the culled row pass (warp-independent)
constexpr int kCullColT = OTG_CULL_COL_T;  // threads per CTA of the culled column pass
constexpr int kCullRB = 16;  // rows per culling block (column pass)
constexpr float kCullT = -127.0f;  // bound below which a block is skipped (FTZ below -126)
constexpr float kCullSlack = 1.0f - 1.0f / 65536.0f;  // relative slack on the box distance

// squared distances of two points (packed) to an axis-aligned box (0 inside)
__device__ __forceinline__ float2 box_d2x2(float2 x, float2 y, float2 z, const float4& lo,
                                           const float4& hi) {
  const float2 gxa = __fadd2_rn(make_float2(lo.x, lo.x), make_float2(-x.x, -x.y));
  const float2 gxb = __fadd2_rn(x, make_float2(-hi.x, -hi.x));
  const float2 gya = __fadd2_rn(make_float2(lo.y, lo.y), make_float2(-y.x, -y.y));
  const float2 gyb = __fadd2_rn(y, make_float2(-hi.y, -hi.y));
  const float2 gza = __fadd2_rn(make_float2(lo.z, lo.z), make_float2(-z.x, -z.y));
  const float2 gzb = __fadd2_rn(z, make_float2(-hi.z, -hi.z));
  const float2 gx = make_float2(fmaxf(fmaxf(gxa.x, gxb.x), 0.f), fmaxf(fmaxf(gxa.y, gxb.y), 0.f));
  const float2 gy = make_float2(fmaxf(fmaxf(gya.x, gyb.x), 0.f), fmaxf(fmaxf(gya.y, gyb.y), 0.f));
  const float2 gz = make_float2(fmaxf(fmaxf(gza.x, gzb.x), 0.f), fmaxf(fmaxf(gza.y, gzb.y), 0.f));
  return __ffma2_rn(gz, gz, __ffma2_rn(gy, gy, __fmul2_rn(gx, gx)));
}
// squared distance from a point to an axis-aligned box (0 inside), fp32
__device__ __forceinline__ float box_d2(float x, float y, float z, const float4& lo, const float4& hi) {
  const float gx = fmaxf(fmaxf(lo.x - x, x - hi.x), 0.0f);
  const float gy = fmaxf(fmaxf(lo.y - y, y - hi.y), 0.0f);
  const float gz = fmaxf(fmaxf(lo.z - z, z - hi.z), 0.0f);
  return fmaf(gz, gz, fmaf(gy, gy, gx * gx));
}

__device__ __forceinline__ float otf_cost(const float4& x, const float4& y) {
  return otf_sqeuclid(x, y);
}

// The 4 columns 4q .. 4q+3 of an on-the-fly quad: negated coordinates, SoA,
// so that each coordinate pair is a packed f32x2 operand.
struct YQ {
  float4 x, y, z;
};

// One quad of row `i` (columns 4q .. 4q+3).  Stored: a 128-bit streaming load.
// On the fly: packed f32x2 form of otf_sqeuclid -- d = x_i + (-y_j) (exactly
// x_i - y_j), c = fma(dz, dz, fma(dy, dy, dx * dx)): bitwise the scalar cost.
template <bool OTF>
__device__ __forceinline__ float4 cost_quad(const CostSrc& s, int64_t i, int64_t q,
                                            const float4& xi, const YQ& yq) {
  if constexpr (OTF) {
    const float2 bx = make_float2(xi.x, xi.x), by = make_float2(xi.y, xi.y),
                 bz = make_float2(xi.z, xi.z);
    const float2 dx01 = __fadd2_rn(bx, make_float2(yq.x.x, yq.x.y));
    const float2 dx23 = __fadd2_rn(bx, make_float2(yq.x.z, yq.x.w));
    const float2 dy01 = __fadd2_rn(by, make_float2(yq.y.x, yq.y.y));
    const float2 dy23 = __fadd2_rn(by, make_float2(yq.y.z, yq.y.w));
    const float2 dz01 = __fadd2_rn(bz, make_float2(yq.z.x, yq.z.y));
    const float2 dz23 = __fadd2_rn(bz, make_float2(yq.z.z, yq.z.w));
    const float2 c01 = __ffma2_rn(dz01, dz01, __ffma2_rn(dy01, dy01, __fmul2_rn(dx01, dx01)));
    const float2 c23 = __ffma2_rn(dz23, dz23, __ffma2_rn(dy23, dy23, __fmul2_rn(dx23, dx23)));
    return make_float4(c01.x, c01.y, c23.x, c23.y);
  } else {
    return ld_stream(reinterpret_cast<const float4*>(s.C + i * s.ldc) + q);
  }
}
template <bool OTF>
__device__ __forceinline__ float cost_one(const CostSrc& s, int64_t i, int64_t j) {
  if constexpr (OTF) {
    return otf_cost(s.X[i], s.Y[j]);
  } else {
    return s.C[i * s.ldc + j];
  }
}
template <bool OTF>
__device__ __forceinline__ void load_y4(const CostSrc& s, int64_t q, YQ& yq) {
  if constexpr (OTF) {
    const float4* Yn = reinterpret_cast<const float4*>(s.Yn);
    const int64_t st = s.ypad >> 2;
    yq.x = __ldg(Yn + q);
    yq.y = __ldg(Yn + st + q);
    yq.z = __ldg(Yn + 2 * st + q);
  }
}

// fp32 storage, exact row statistics for R rows (fp64 exponent argument with an
// online max).  Every thread streams float4 columns of the R rows; the column
// potential is loaded once per column chunk and reused across the R rows.
// Used for the first evaluation of a solve (no shift estimate yet) and, in
// LIST mode, to redo the rows whose shift estimate failed (k_row_shift).
template <int R, bool OTF>
__device__ void row_exact_block(const int64_t* rows, const CostSrc src,
                                int64_t m, const double* __restrict__ p, double kappa,
                                const double* __restrict__ a, const double* __restrict__ loga,
                                double* __restrict__ rowM, double* __restrict__ rowS,
                                double* __restrict__ u, double* __restrict__ wrow,
                                float4* __restrict__ aux, double* __restrict__ rowM2,
                                int* __restrict__ rowJ, const bool* valid) {
  __shared__ double sh[kRowThreads / 32];
  __shared__ double resM[R], resS[R];
  __shared__ int resJ[R];
  float4 xr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) xr[r] = OTF ? src.X[rows[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
  double mr[R], sr[R];
  int jr[R];  // argmax column of the running max (next evaluation's shift estimate)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mr[r] = -INFINITY;
    sr[r] = 0.0;
    jr[r] = 0;
  }
  // Base-2 units: t2 = p_j log2e - C_ij kappa log2e (fp64 DFMA on an exactly
  // up-cast C), online max m2, ex2(t2 - m2) on MUFU; fp32 <-> fp64 conversions
  // with integer ops (ALU pipe) instead of F2F (XU pipe, shared with MUFU).
  const double k2 = kappa * kLog2e;
  const int64_t nq = m >> 2;
  const double2* p2 = reinterpret_cast<const double2*>(p);
  for (int64_t q = threadIdx.x; q < nq; q += kRowThreads) {
    const double2 pa = __ldg(p2 + 2 * q), pb = __ldg(p2 + 2 * q + 1);
    const double q0 = pa.x * kLog2e, q1 = pa.y * kLog2e, q2 = pb.x * kLog2e, q3 = pb.y * kLog2e;
    YQ y4;
    load_y4<OTF>(src, q, y4);
    float4 c[R];
#pragma unroll
    for (int r = 0; r < R; ++r) c[r] = cost_quad<OTF>(src, rows[r], q, xr[r], y4);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double t0 = fma(-f32_to_f64(c[r].x), k2, q0);
      const double t1 = fma(-f32_to_f64(c[r].y), k2, q1);
      const double t2 = fma(-f32_to_f64(c[r].z), k2, q2);
      const double t3 = fma(-f32_to_f64(c[r].w), k2, q3);
      const double cm = fmax(fmax(t0, t1), fmax(t2, t3));
      if (cm > mr[r]) {
        sr[r] *= exp2(mr[r] - cm);
        mr[r] = cm;
        jr[r] = static_cast<int>(4 * q) + (t0 == cm ? 0 : t1 == cm ? 1 : t2 == cm ? 2 : 3);
      }
      const double mm = mr[r];
      const float e = ex2_approx(neg_f64_to_f32(t0 - mm)) + ex2_approx(neg_f64_to_f32(t1 - mm)) +
                      ex2_approx(neg_f64_to_f32(t2 - mm)) + ex2_approx(neg_f64_to_f32(t3 - mm));
      sr[r] += static_cast<double>(e);
    }
  }
  for (int64_t j = 4 * nq + threadIdx.x; j < m; j += kRowThreads) {  // ragged tail
    const double pj = p[j] * kLog2e;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double t = fma(-f32_to_f64(cost_one<OTF>(src, rows[r], j)), k2, pj);
      if (t > mr[r]) {
        jr[r] = static_cast<int>(j);
        sr[r] *= exp2(mr[r] - t);
        mr[r] = t;
      }
      sr[r] += static_cast<double>(ex2_approx(neg_f64_to_f32(t - mr[r])));
    }
  }
  // per row: exact max, then each thread rescales its partial once (fp64 exp2)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double M2 = block_max<kRowThreads>(mr[r], sh);
    const double s = sr[r] > 0.0 ? sr[r] * exp2(mr[r] - M2) : 0.0;
    const double S = block_sum<kRowThreads>(s, sh);
    const double J = block_max<kRowThreads>(mr[r] == M2 ? -static_cast<double>(jr[r]) : -1e300, sh);
    if (threadIdx.x == 0) {
      resM[r] = M2;
      resS[r] = S;
      resJ[r] = static_cast<int>(-J);
    }
  }
  __syncthreads();
  if (threadIdx.x < R && valid[threadIdx.x]) {
    const int r = threadIdx.x;
    const int64_t i = rows[r];
    const double M2 = resM[r], S = resS[r];
    const double M = M2 * kLn2;
    const double ui = (loga[i] - M) - log(S);
    const double wi = a[i] / S;
    rowM[i] = M;
    rowS[i] = S;
    u[i] = ui;
    wrow[i] = wi;
    rowM2[i] = M2;
    rowJ[i] = resJ[r];
    // the column pass uses the S-consistent shift M2 split into hi + lo
    float hi, lo;
    split_q(M2, hi, lo);
    aux[i] = make_float4(hi, lo, static_cast<float>(wi), 0.0f);
  }
}

// Exact redo of the rows k_row_shift flagged (grid-stride over the list).
template <bool OTF>
__global__ void __launch_bounds__(kRowThreads)
k_row_redo(const CostSrc src, int64_t m, const double* __restrict__ p,
           double kappa, const double* __restrict__ a, const double* __restrict__ loga,
           double* __restrict__ rowM, double* __restrict__ rowS, double* __restrict__ u,
           double* __restrict__ wrow, float4* __restrict__ aux, double* __restrict__ rowM2,
           int* __restrict__ rowJ, const int* __restrict__ redo_rows,
           const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  const unsigned cnt = ctrl->redo_count;
  for (unsigned k = blockIdx.x; k < cnt; k += gridDim.x) {
    const int64_t rows[1] = {redo_rows[k]};
    const bool valid[1] = {true};
    row_exact_block<1, OTF>(rows, src, m, p, kappa, a, loga, rowM, rowS, u, wrow, aux, rowM2,
                            rowJ, valid);
    __syncthreads();
  }
}

// fp32 row pass with a shift ESTIMATE (all-fp32, no fp64 per element).  From
// the previous evaluation the row keeps its exact base-2 max M2_prev and the
// argmax column J; with dq_j = (p_new - p_old)_j log2e the new max satisfies
//   L = M2_prev + dq_J  <=  M2_new  <=  M2_prev + max_j dq_j = U.
// The shift s = min(L + 1, U), rounded up to a multiple of 2^-8, is an exact
// constant of the row, so every exponent t = Vc_j - s - C_ij kappa2 (+ small
// terms) is formed by the same exact-cancellation FMA as the column pass,
// S_i = sum_j ex2(t_ij) and u_i = log a_i - s ln2 - log S_i are the
// reference's quantities up to rounding.  Precision needs the dominant
// exponents small: rows whose true max T = M2_new - s falls outside
// [-kRedoLo, kRedoHi] (the argmax moved to a column whose potential moved
// much more) are listed for an exact redo (k_row_redo).  The kernel tracks the
// new argmax for the next evaluation.
__device__ __forceinline__ void quad_exponents(const float4& c, float2 V01, float2 V23, float2 F01,
                                               float2 F23, float2 nSc2, float2 nkh2, float2 nkl2,
                                               float2& t01, float2& t23) {
  const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
  t01 = __fadd2_rn(__ffma2_rn(c01, nkh2, __fadd2_rn(V01, nSc2)), __ffma2_rn(c01, nkl2, F01));
  t23 = __fadd2_rn(__ffma2_rn(c23, nkh2, __fadd2_rn(V23, nSc2)), __ffma2_rn(c23, nkl2, F23));
}

// On the fly (FMA-pipe bound, ncu: the packed FP32 pipe at 65-84 % with MUFU
// at 50-60 %): t = fmaf(-c, kl, fmaf(-c, kh, V - Sc)), the column's low part F
// applied after the ex2 as the factor 2^F (vq plane 2) -- three FP32 ops per
// element instead of four, each rounding at the scale of the small result.
__device__ __forceinline__ void quad_exponents_nf(const float4& c, float2 V01, float2 V23,
                                                  float2 nSc2, float2 nkh2, float2 nkl2,
                                                  float2& t01, float2& t23) {
  const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
  t01 = __ffma2_rn(c01, nkl2, __ffma2_rn(c01, nkh2, __fadd2_rn(V01, nSc2)));
  t23 = __ffma2_rn(c23, nkl2, __ffma2_rn(c23, nkh2, __fadd2_rn(V23, nSc2)));
}

constexpr float kRedoLo = 2.0f;
constexpr float kRedoHi = 6.0f;

template <int R, bool OTF, int PF>
__device__ __forceinline__ void row_shift_block(
    const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq,
    const double* __restrict__ dq, int64_t mpad, float kh, float kl, const double* __restrict__ a,
    const double* __restrict__ loga, double* __restrict__ rowM, double* __restrict__ rowS,
    double* __restrict__ u, double* __restrict__ wrow, float4* __restrict__ aux,
    double* __restrict__ rowM2, int* __restrict__ rowJ, int* __restrict__ redo_rows,
    Ctrl* __restrict__ ctrl, int64_t r0, const double* __restrict__ p, double kappa) {
  // redo_rows == nullptr: rows whose estimate failed are redone here, exactly,
  // by the whole CTA (the single-pass sweep, whose column step follows at once)
  __shared__ double sh[kRowThreads / 32];
  __shared__ float shf[kRowThreads / 32];
  __shared__ int shj[kRowThreads / 32];
  __shared__ float sSc[R], resT[R];
  __shared__ double resS[R];
  __shared__ int resJ[R];
  __shared__ int bad[R];
  if (threadIdx.x < R) {
    const int64_t i = r0 + threadIdx.x < n ? r0 + threadIdx.x : n - 1;
    const double M2 = rowM2[i];
    const double lo = M2 + dq[rowJ[i]], hi = M2 + ctrl->dmax2;
    sSc[threadIdx.x] = static_cast<float>(ceil(fmin(lo + 1.0, hi) * 256.0) * (1.0 / 256.0));
  }
  __syncthreads();
  // Inner loop on packed f32x2 arithmetic (FADD2 / FFMA2): the exponents are
  // bitwise those of the scalar form  t = fmaf(-c, kh, V - Sc) + fmaf(-c, kl, F)
  // at half the FP32 issue slots.  The argmax is tracked per thread as the
  // quad index only (one compare + select per quad); the column inside the
  // winning quad is resolved once at the end.
  // loop-carried state kept small (the kernel runs 4 CTAs/SM at 64
  // registers): the fp64 row sums live in shared memory, the rows are one
  // base pointer + 32-bit offsets
  float tm[R];
  int tq[R];       // column code of the running max: 4q (quad) or j (ragged tail)
  float2 fs2[R];   // fp32 partial sums, flushed to fp64 every 16 columns
  float2 nSc2[R];  // -(row shift), twice (packed operand)
  int rof[R];      // row r's offset from row r0, in elements / ldc
  float4 xr[R];
  __shared__ double sSS[R][kRowThreads];  // this thread's fp64 row sums
#pragma unroll
  for (int r = 0; r < R; ++r) {
    nSc2[r] = make_float2(-sSc[r], -sSc[r]);
    tm[r] = -FLT_MAX;
    tq[r] = 0;
    fs2[r] = make_float2(0.f, 0.f);
    sSS[r][threadIdx.x] = 0.0;
    rof[r] = static_cast<int>((r0 + r < n ? r0 + r : n - 1) - r0);
    xr[r] = OTF ? src.X[r0 + rof[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float* crow0 = OTF ? nullptr : src.C + r0 * src.ldc;
  const float2 nkh2 = make_float2(-kh, -kh), nkl2 = make_float2(-kl, -kl);
  const int64_t nq = m >> 2;
  const float4* Vq = reinterpret_cast<const float4*>(vq);
  const float4* Fq = reinterpret_cast<const float4*>(vq + mpad);
  const float4* Eq = reinterpret_cast<const float4*>(vq + 2 * mpad);  // 2^F (on the fly)
  int chunk = 0;
  for (int64_t q = threadIdx.x; q < nq; q += kRowThreads) {
    const float4 V = __ldg(Vq + q), F = __ldg(OTF ? Eq + q : Fq + q);
    YQ y4;
    load_y4<OTF>(src, q, y4);
    float4 c[R];
    if constexpr (!OTF && PF == 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        c[r] = ld_stream256(reinterpret_cast<const float4*>(crow0 + static_cast<int64_t>(rof[r]) * src.ldc) + q);
    } else if constexpr (!OTF) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        c[r] = ld_stream(reinterpret_cast<const float4*>(crow0 + static_cast<int64_t>(rof[r]) * src.ldc) + q);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) c[r] = cost_quad<OTF>(src, r0 + rof[r], q, xr[r], y4);
    }
    if constexpr (!OTF && PF >= 2) {
      const int64_t qp = q + static_cast<int64_t>(PF - 1) * kRowThreads;
      if (qp < nq) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          prefetch_l2(reinterpret_cast<const float4*>(crow0 + static_cast<int64_t>(rof[r]) * src.ldc) + qp);
      }
    }
    const float2 V01 = make_float2(V.x, V.y), V23 = make_float2(V.z, V.w);
    const float2 F01 = make_float2(F.x, F.y), F23 = make_float2(F.z, F.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 t01, t23;
      if constexpr (OTF)  // (F01, F23 hold 2^F here)
        quad_exponents_nf(c[r], V01, V23, nSc2[r], nkh2, nkl2, t01, t23);
      else
        quad_exponents(c[r], V01, V23, F01, F23, nSc2[r], nkh2, nkl2, t01, t23);
      const float mx = fmaxf(fmaxf(fmaxf(tm[r], t01.x), t01.y), fmaxf(t23.x, t23.y));
      tq[r] = mx > tm[r] ? static_cast<int>(4 * q) : tq[r];
      tm[r] = mx;
      if constexpr (OTF) {
        fs2[r] = __ffma2_rn(make_float2(ex2_approx(t01.x), ex2_approx(t01.y)), F01, fs2[r]);
        fs2[r] = __ffma2_rn(make_float2(ex2_approx(t23.x), ex2_approx(t23.y)), F23, fs2[r]);
      } else {
        const float2 e = __fadd2_rn(make_float2(ex2_approx(t01.x), ex2_approx(t23.x)),
                                    make_float2(ex2_approx(t01.y), ex2_approx(t23.y)));
        fs2[r] = __fadd2_rn(fs2[r], e);
      }
    }
    if (++chunk == 4) {  // fp32 partials flushed into fp64 every 16 elements
      chunk = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sSS[r][threadIdx.x] += static_cast<double>(fs2[r].x) + static_cast<double>(fs2[r].y);
        fs2[r] = make_float2(0.f, 0.f);
      }
    }
  }
  for (int64_t j = 4 * nq + threadIdx.x; j < m; j += kRowThreads) {  // ragged tail
    const float V = vq[j], F = vq[mpad + j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float c = cost_one<OTF>(src, r0 + rof[r], j);
      const float t = OTF ? fmaf(-c, kl, fmaf(-c, kh, V + nSc2[r].x))
                          : fmaf(-c, kh, V + nSc2[r].x) + fmaf(-c, kl, F);
      if (t > tm[r]) {
        tm[r] = t;
        tq[r] = static_cast<int>(j);
      }
      if constexpr (OTF)
        fs2[r].x = fmaf(ex2_approx(t), vq[2 * mpad + j], fs2[r].x);
      else
        fs2[r].x += ex2_approx(t);
    }
  }
  // one barrier for all R rows: each warp leaves its (max, argmax code, sum)
  // per row in smem; thread r then folds the 8 warps of row r in fixed order
  constexpr int kW = kRowThreads / 32;
  __shared__ float wT[R][kW];
  __shared__ int wJ[R][kW];
  __shared__ double wS[R][kW];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double sv = sSS[r][threadIdx.x] + (static_cast<double>(fs2[r].x) + static_cast<double>(fs2[r].y));
    float t = tm[r];
    int jj = tq[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t2 = __shfl_xor_sync(0xffffffffu, t, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, jj, o);
      if (t2 > t || (t2 == t && j2 < jj)) {
        t = t2;
        jj = j2;
      }
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
    }
    if ((threadIdx.x & 31) == 0) {
      wT[r][threadIdx.x >> 5] = t;
      wJ[r][threadIdx.x >> 5] = jj;
      wS[r][threadIdx.x >> 5] = sv;
    }
  }
  __syncthreads();
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    float T = -FLT_MAX;
    int J = 0;
    double S = 0.0;
#pragma unroll
    for (int k = 0; k < kW; ++k) {
      if (wT[r][k] > T || (wT[r][k] == T && wJ[r][k] < J)) {
        T = wT[r][k];
        J = wJ[r][k];
      }
      S += wS[r][k];
    }
    resT[r] = T;
    resS[r] = S;
    resJ[r] = J;
  }
  // (the same threads r < R finish the rows: no barrier until the CTA-wide redo)
  if (threadIdx.x < R) {  // column of the max inside the winning quad
    const int r = threadIdx.x;
    const int code = resJ[r];
    if (code < 4 * nq) {
      const int64_t q = code >> 2;
      const int64_t ir = r0 + r < n ? r0 + r : n - 1;  // (no register-array indexing by r)
      YQ y4;
      load_y4<OTF>(src, q, y4);
      const float4 xi = OTF ? src.X[ir] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 cq = cost_quad<OTF>(src, ir, q, xi, y4);
      const float4 V = __ldg(Vq + q), F = __ldg(Fq + q);
      const float nsc = -sSc[r];
      float2 t01, t23;
      if constexpr (OTF)
        quad_exponents_nf(cq, make_float2(V.x, V.y), make_float2(V.z, V.w), make_float2(nsc, nsc),
                          nkh2, nkl2, t01, t23);
      else
        quad_exponents(cq, make_float2(V.x, V.y), make_float2(V.z, V.w), make_float2(F.x, F.y),
                       make_float2(F.z, F.w), make_float2(nsc, nsc), nkh2, nkl2, t01, t23);
      const float T = resT[r];
      resJ[r] = code + (t01.x == T ? 0 : t01.y == T ? 1 : t23.x == T ? 2 : t23.y == T ? 3 : 0);
    }
  }
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    const int64_t i = r0 + r;
    if (i < n) {
      const float T = resT[r];
      bad[r] = 0;
      if (!(T >= -kRedoLo && T <= kRedoHi)) {  // estimate too loose (or NaN): exact redo
        const unsigned slot = atomicAdd(&ctrl->redo_count, 1u);
        if (redo_rows)
          redo_rows[slot] = static_cast<int>(i);
        else
          bad[r] = 1;
      } else {
        const double S = resS[r];
        const double sc = static_cast<double>(sSc[r]);
        const double M = sc * kLn2;
        const double ui = (loga[i] - M) - log(S);
        const double wi = a[i] / S;
        rowM[i] = M;
        rowS[i] = S;
        u[i] = ui;
        wrow[i] = wi;
        rowM2[i] = sc + static_cast<double>(T);
        rowJ[i] = resJ[r];
        aux[i] = make_float4(sSc[r], 0.0f, static_cast<float>(wi), 0.0f);
      }
    } else {
      bad[r] = 0;
    }
  }
  if (redo_rows == nullptr) {
    __syncthreads();
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      if (bad[r]) {  // uniform over the CTA
        const int64_t rows[1] = {r0 + r};
        const bool valid[1] = {true};
        row_exact_block<1, OTF>(rows, src, m, p, kappa, a, loga, rowM, rowS, u, wrow, aux, rowM2,
                                rowJ, valid);
      }
    }
  }
}

// Exact redo of the rows the single-pass kernel (fused.cu) listed as loose:
// list c (c < ncl, in order) holds bad_rows[c cap + k], k < bad_count[c].
__global__ void __launch_bounds__(kRowThreads)
k_sp_redo(const CostSrc src, int64_t n, int64_t m, const double* __restrict__ p, double kappa,
          const double* __restrict__ a, const double* __restrict__ loga,
          double* __restrict__ rowM, double* __restrict__ rowS, double* __restrict__ u,
          double* __restrict__ wrow, float4* __restrict__ aux, double* __restrict__ rowM2,
          int* __restrict__ rowJ, const int* __restrict__ bad_rows,
          const int* __restrict__ bad_count, int ncl, int64_t cap,
          const unsigned* __restrict__ total, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  if (*total == 0u) return;  // (the single pass's count of listed rows)
  for (int c = 0; c < ncl; ++c) {
    const int nb = bad_count[c];
    const int64_t base = cap * c;
    for (int k = blockIdx.x; k < nb; k += gridDim.x) {
      const int64_t rows[1] = {bad_rows[base + k]};
      const bool valid[1] = {true};
      row_exact_block<1, false>(rows, src, m, p, kappa, a, loga, rowM, rowS, u, wrow, aux, rowM2,
                                rowJ, valid);
      __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && nb > 0) atomicAdd(&ctrl->redo_count, static_cast<unsigned>(nb));
  }
}

// vq = quantised split of p * log2(e) (the row pass's column potential),
// refreshed whenever the host sets a new evaluation point.
__global__ void k_split_p(int64_t m, int64_t mpad, const double* __restrict__ p,
                          float* __restrict__ vq) {
  pdl_wait();
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    split_store(p[j] * kLog2e, vq, mpad, j);
}

__constant__ int c_online_first = 1;  // OTG_ONLINE_FIRST=0: fp64-argument first pass
__device__ __forceinline__ bool online_first_pass() { return c_online_first != 0; }

// fp32 storage, row statistics WITHOUT a shift estimate (first evaluation of
// a solve): the k_row_shift inner loop with a per-thread RUNNING shift s (a
// multiple of 2^-8, so V - s stays exact).  s starts at the thread's first
// quad's (rounded-up) max; when a quad exceeds s by more than 8 the thread's
// partial sums are rescaled by 2^-(delta) and s moves up (a handful of times
// per row), so ex2 never overflows and the dominant terms keep full fp32
// precision.  The CTA then folds the per-thread (s, sum, max) onto the
// largest s.  Same arithmetic per element as the shift pass (~2x faster than
// the fp64-argument row_exact_block it replaces on the first evaluation).
template <int R, bool OTF>
__device__ __forceinline__ void row_online_block(
    const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq, int64_t mpad,
    float kh, float kl,
    const double* __restrict__ a, const double* __restrict__ loga, double* __restrict__ rowM,
    double* __restrict__ rowS, double* __restrict__ u, double* __restrict__ wrow,
    float4* __restrict__ aux, double* __restrict__ rowM2, int* __restrict__ rowJ, int64_t r0) {
  __shared__ double sh[kRowThreads / 32];
  __shared__ float shf[kRowThreads / 32];
  __shared__ int shj[kRowThreads / 32];
  __shared__ float resS0[R], resT[R];
  __shared__ double resS[R];
  __shared__ int resJ[R];
  float s[R], tm[R];
  int tq[R];
  float2 fs2[R];
  __shared__ double sSS[R][kRowThreads];  // fp64 partial sums (registers stay free)
  int64_t rr[R];
  float4 xr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s[r] = -FLT_MAX;  // no column seen yet
    tm[r] = -FLT_MAX;
    tq[r] = 0;
    fs2[r] = make_float2(0.f, 0.f);
    sSS[r][threadIdx.x] = 0.0;
    rr[r] = r0 + r < n ? r0 + r : n - 1;
    xr[r] = OTF ? src.X[rr[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float2 nkh2 = make_float2(-kh, -kh), nkl2 = make_float2(-kl, -kl);
  const int64_t nq = m >> 2;
  const float4* Vq = reinterpret_cast<const float4*>(vq);
  const float4* Fq = reinterpret_cast<const float4*>(vq + mpad);
  {
    // common starting shift per row: the max over the CTA's first 4 x 256
    // columns (rounded up), so most threads never rescale
    float rm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rm[r] = -FLT_MAX;
    if (threadIdx.x < nq) {
      const int64_t q = threadIdx.x;
      const float4 V = __ldg(Vq + q), F = __ldg(Fq + q);
      YQ y4;
      load_y4<OTF>(src, q, y4);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float2 r01, r23;
        quad_exponents(cost_quad<OTF>(src, rr[r], q, xr[r], y4), make_float2(V.x, V.y),
                       make_float2(V.z, V.w), make_float2(F.x, F.y), make_float2(F.z, F.w),
                       make_float2(0.f, 0.f), nkh2, nkl2, r01, r23);
        rm[r] = fmaxf(fmaxf(r01.x, r01.y), fmaxf(r23.x, r23.y));
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float b = rm[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
      __syncthreads();
      if ((threadIdx.x & 31) == 0) shf[threadIdx.x >> 5] = b;
      __syncthreads();
      float B = -FLT_MAX;
#pragma unroll
      for (int k = 0; k < kRowThreads / 32; ++k) B = fmaxf(B, shf[k]);
      if (B > -FLT_MAX) s[r] = ceilf(B * 256.0f) * (1.0f / 256.0f);
    }
  }
  int chunk = 0;
  for (int64_t q = threadIdx.x; q < nq; q += kRowThreads) {
    const float4 V = __ldg(Vq + q), F = __ldg(Fq + q);
    YQ y4;
    load_y4<OTF>(src, q, y4);
    float4 c[R];
#pragma unroll
    for (int r = 0; r < R; ++r) c[r] = cost_quad<OTF>(src, rr[r], q, xr[r], y4);
    if constexpr (!OTF) {  // L2 prefetch 4 chunks ahead: the rescale branch keeps the
      const int64_t qp = q + 4 * kRowThreads;  // compiler from pipelining these loads
      if (qp < nq) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          prefetch_l2(reinterpret_cast<const float4*>(src.C + rr[r] * src.ldc) + qp);
      }
    }
    const float2 V01 = make_float2(V.x, V.y), V23 = make_float2(V.z, V.w);
    const float2 F01 = make_float2(F.x, F.y), F23 = make_float2(F.z, F.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 t01, t23;
      quad_exponents(c[r], V01, V23, F01, F23, make_float2(-s[r], -s[r]), nkh2, nkl2, t01, t23);
      float mx = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
      if (mx > 8.0f) {  // a max well above the running shift: move s up (rare)
        const float d = ceilf(mx * 256.0f) * (1.0f / 256.0f) + 16.0f;  // 16 of headroom
        s[r] += d;
        const float sc = ex2_approx(-d);
        fs2[r] = make_float2(fs2[r].x * sc, fs2[r].y * sc);
        sSS[r][threadIdx.x] *= exp2(-static_cast<double>(d));
        tm[r] -= d;
        quad_exponents(c[r], V01, V23, F01, F23, make_float2(-s[r], -s[r]), nkh2, nkl2, t01, t23);
        mx = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
      }
      tq[r] = mx > tm[r] ? static_cast<int>(4 * q) : tq[r];
      tm[r] = fmaxf(tm[r], mx);
      const float2 e = __fadd2_rn(make_float2(ex2_approx(t01.x), ex2_approx(t23.x)),
                                  make_float2(ex2_approx(t01.y), ex2_approx(t23.y)));
      fs2[r] = __fadd2_rn(fs2[r], e);
    }
    if (++chunk == 4) {
      chunk = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sSS[r][threadIdx.x] += static_cast<double>(fs2[r].x) + static_cast<double>(fs2[r].y);
        fs2[r] = make_float2(0.f, 0.f);
      }
    }
  }
  for (int64_t j = 4 * nq + threadIdx.x; j < m; j += kRowThreads) {  // ragged tail
    const float V = vq[j], F = vq[mpad + j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float c = cost_one<OTF>(src, rr[r], j);
      if (s[r] == -FLT_MAX) s[r] = ceilf((fmaf(-c, kh, V) + fmaf(-c, kl, F)) * 256.0f) * (1.0f / 256.0f);
      float t = fmaf(-c, kh, V - s[r]) + fmaf(-c, kl, F);
      if (t > 8.0f) {
        const float d = ceilf(t * 256.0f) * (1.0f / 256.0f);
        s[r] += d;
        const float sc = ex2_approx(-d);
        fs2[r] = make_float2(fs2[r].x * sc, fs2[r].y * sc);
        sSS[r][threadIdx.x] *= exp2(-static_cast<double>(d));
        tm[r] -= d;
        t = fmaf(-c, kh, V - s[r]) + fmaf(-c, kl, F);
      }
      if (t > tm[r]) {
        tm[r] = t;
        tq[r] = static_cast<int>(j);
      }
      fs2[r].x += ex2_approx(t);
    }
  }
  // fold the threads onto the CTA's largest running shift
#pragma unroll
  for (int r = 0; r < R; ++r) {
    sSS[r][threadIdx.x] += static_cast<double>(fs2[r].x) + static_cast<double>(fs2[r].y);
    float sb = s[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sb = fmaxf(sb, __shfl_xor_sync(0xffffffffu, sb, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) shf[threadIdx.x >> 5] = sb;
    __syncthreads();
    float S0 = -FLT_MAX;
#pragma unroll
    for (int k = 0; k < kRowThreads / 32; ++k) S0 = fmaxf(S0, shf[k]);
    const bool seen = s[r] != -FLT_MAX;
    const double part = seen ? sSS[r][threadIdx.x] * exp2(static_cast<double>(s[r] - S0)) : 0.0;
    float t = seen ? (s[r] - S0) + tm[r] : -FLT_MAX;  // max relative to S0
    int jj = tq[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t2 = __shfl_xor_sync(0xffffffffu, t, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, jj, o);
      if (t2 > t || (t2 == t && j2 < jj)) {
        t = t2;
        jj = j2;
      }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      shf[threadIdx.x >> 5] = t;
      shj[threadIdx.x >> 5] = jj;
    }
    __syncthreads();
    float T = -FLT_MAX;
    int J = 0;
#pragma unroll
    for (int k = 0; k < kRowThreads / 32; ++k)
      if (shf[k] > T || (shf[k] == T && shj[k] < J)) {
        T = shf[k];
        J = shj[k];
      }
    const double Ssum = block_sum<kRowThreads>(part, sh);
    if (threadIdx.x == 0) {
      resS0[r] = S0;
      resT[r] = T;
      resS[r] = Ssum;
      resJ[r] = J;
    }
  }
  __syncthreads();
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    const int64_t i = r0 + r;
    const int code = resJ[r];
    const float S0 = resS0[r];
    int J = code;
    if (code < 4 * nq) {  // column of the max inside the winning quad
      const int64_t q = code >> 2;
      const int64_t ir = i < n ? i : n - 1;
      YQ y4;
      load_y4<OTF>(src, q, y4);
      const float4 xi = OTF ? src.X[ir] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 cq = cost_quad<OTF>(src, ir, q, xi, y4);
      const float4 V = __ldg(Vq + q), F = __ldg(Fq + q);
      float2 t01, t23;
      quad_exponents(cq, make_float2(V.x, V.y), make_float2(V.z, V.w), make_float2(F.x, F.y),
                     make_float2(F.z, F.w), make_float2(-S0, -S0), nkh2, nkl2, t01, t23);
      const float em = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
      J = code + (t01.x == em ? 0 : t01.y == em ? 1 : t23.x == em ? 2 : 3);
    }
    if (i < n) {
      const double S = resS[r];
      const double sc = static_cast<double>(S0);
      const double M = sc * kLn2;
      const double wi = a[i] / S;
      rowM[i] = M;
      rowS[i] = S;
      u[i] = (loga[i] - M) - log(S);
      wrow[i] = wi;
      rowM2[i] = sc + static_cast<double>(resT[r]);
      rowJ[i] = J;
      aux[i] = make_float4(S0, 0.0f, static_cast<float>(wi), 0.0f);
    }
  }
}

// fp32 row pass kernels: the exact body on the first evaluation of a solve// fp32 row pass kernels: the exact body on the first evaluation of a solve
// (no previous point), the shift-estimate body after; each returns at once
// when its case does not apply.  (Kept as two kernels: one kernel holding both
// bodies needs 76 registers and drops the shift pass to 3 CTAs per SM.)
template <int R, bool OTF>
__global__ void __launch_bounds__(kRowThreads, (R == 4 && !OTF) ? OTG_EXACT_MINB : 1)
k_row_exact(const CostSrc src, int64_t n, int64_t m, const double* __restrict__ p, double kappa,
            const double* __restrict__ a, const double* __restrict__ loga,
            double* __restrict__ rowM, double* __restrict__ rowS, double* __restrict__ u,
            double* __restrict__ wrow, float4* __restrict__ aux, double* __restrict__ rowM2,
            int* __restrict__ rowJ, const Ctrl* __restrict__ ctrl, const float* __restrict__ vq,
            int64_t mpad) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || ctrl->shift_valid) return;
  // grid-stride over row blocks: the launch is a no-op in every evaluation but
  // the first of a solve, so it is sized to the resident CTAs, not to n / R
  for (int64_t blk = blockIdx.x; blk * R < n; blk += gridDim.x) {
    if (online_first_pass()) {
      const double k2 = kappa * kLog2e;
      const float kh = static_cast<float>(k2);
      const float kl = static_cast<float>(k2 - static_cast<double>(kh));
      row_online_block<R, OTF>(src, n, m, vq, mpad, kh, kl, a, loga, rowM, rowS, u, wrow, aux,
                               rowM2, rowJ, blk * R);
    } else {
      int64_t rows[R];
      bool valid[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t i = blk * R + r;
        valid[r] = i < n;
        rows[r] = valid[r] ? i : n - 1;
      }
      row_exact_block<R, OTF>(rows, src, m, p, kappa, a, loga, rowM, rowS, u, wrow, aux, rowM2,
                              rowJ, valid);
    }
    __syncthreads();  // (shared scratch of the block helpers)
  }
}

template <int R, bool OTF, int PF>
__global__ void __launch_bounds__(kRowThreads, (R == 4 && !OTF) ? OTG_ROW_MINB
                                               : (R == 8 && OTF) ? OTG_ROW_OTF_MINB : 1)
k_row_shift(const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq,
            const double* __restrict__ dq, int64_t mpad, float kh, float kl,
            const double* __restrict__ a, const double* __restrict__ loga,
            double* __restrict__ rowM, double* __restrict__ rowS, double* __restrict__ u,
            double* __restrict__ wrow, float4* __restrict__ aux, double* __restrict__ rowM2,
            int* __restrict__ rowJ, int* __restrict__ redo_rows, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  row_shift_block<R, OTF, PF>(src, n, m, vq, dq, mpad, kh, kl, a, loga, rowM, rowS, u, wrow, aux,
                              rowM2, rowJ, redo_rows, ctrl, static_cast<int64_t>(blockIdx.x) * R,
                              nullptr, 0.0);
}

// ------------------------------------------------------------- K1-OTF ----
// On-the-fly row pass, transposed (the column pass's layout): every thread
// owns kOtfRT rows -- their points in registers as packed row pairs -- and
// walks a column split whose (-y, V, 2^F) are staged in shared memory and
// read as broadcasts, so a column's loads serve kOtfRT rows and no
// cross-thread reduction sits in the inner loop.  Per element: cost 6, exponent
// 2 (V - s, then one FMA with the instance's exact fp32 kh), accumulate 1 FP32
// op (packed f32x2) + 1 ex2, no per-element max: each
// row keeps its heaviest 16-column block (largest fp32 block sum, compared at
// the fp64 flush); the finishing kernel folds the column splits in order and
// takes the largest exponent T_J of that block (recomputed bitwise) as the
// row's reference column.  The true max is within 4 of T_J (it lies in some
// block whose sum is at most 16 2^T_J), which the redo rule and the next
// shift estimate allow for; otherwise as row_shift_block.
constexpr int kOtfRT = 8;     // rows per thread (4 packed pairs)
constexpr int kOtfTJ = 256;   // columns per staged tile
constexpr int kOtfBlk = 16;   // columns per max block / fp64 flush
constexpr int kOtfUnroll = OTG_ROW_OTF_UNROLL;  // columns in flight per thread

struct RowPart {
  float t;   // largest 16-column block sum of the split (fp32, relative to the row shift)
  int jb;    // first column of that block
  double s;  // sum of 2^t 2^F over the split
};

constexpr double kOtfSlack = 4.0;  // log2(kOtfBlk): true max <= T_J + 4

// rowM2 = s + T_J may sit up to kOtfSlack below the row's max, so the upper
// bound carries the slack (for rows whose rowM2 is the exact max, as after
// k_row_exact / k_row_redo, it is merely loose).
__device__ __forceinline__ float row_shift_estimate(const double* __restrict__ rowM2,
                                                    const int* __restrict__ rowJ,
                                                    const double* __restrict__ dq, double dmax2,
                                                    int64_t i) {
  const double M2 = rowM2[i];
  const double lo = M2 + dq[rowJ[i]], hi = M2 + dmax2 + kOtfSlack;
  return static_cast<float>(ceil(fmin(lo + 1.0, hi) * 256.0) * (1.0 / 256.0));
}

template <bool CULL>
__global__ void __launch_bounds__(kRowThreads, OTG_ROW_OTF_MINB)
k_row_otf(const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq,
          const double* __restrict__ dq, int64_t mpad, float kh, float kl,
          const double* __restrict__ rowM2, const int* __restrict__ rowJ, int64_t cols_per_split,
          RowPart* __restrict__ rpart, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  constexpr int NP = kOtfRT / 2;
  __shared__ float4 sA[kOtfTJ];  // (-x, -x, -y, -y)
  __shared__ float4 sB[kOtfTJ];  // (-z, -z, V, V)
  __shared__ float2 sE[kOtfTJ];  // (2^F, 2^F)
  __shared__ double sSS[kOtfRT][kRowThreads];
  // rows of this thread: r-th = base + r * stride.  CULL: sorted positions,
  // each warp's 256 rows consecutive (spatially compact: one culling test
  // per warp and column block)
  const int64_t cbase = static_cast<int64_t>(blockIdx.x) * (kRowThreads * kOtfRT);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rbase = CULL ? cbase + warp * (32 * kOtfRT) + lane : cbase + threadIdx.x;
  constexpr int64_t rstride = CULL ? 32 : kRowThreads;
  auto row_of = [&](int64_t pos) -> int64_t {  // row index (original order) at position pos
    const int64_t q = min(pos, n - 1);
    return CULL ? static_cast<int64_t>(src.perm_r[q]) : q;
  };
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * cols_per_split;
  const int64_t j1 = min(j0 + cols_per_split, m);
  const double dmax2 = ctrl->dmax2;
  float2 X[NP], Y[NP], Z[NP], nS[NP], fs[NP];
  float tm[kOtfRT];  // heaviest block sum so far and the block's first column
  int tj[kOtfRT];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    const int64_t p0 = rbase + (2 * pp) * rstride, p1 = rbase + (2 * pp + 1) * rstride;
    const int64_t i0 = row_of(p0), i1 = row_of(p1);
    const float4 x0 = CULL ? src.Xs[min(p0, n - 1)] : src.X[i0];
    const float4 x1 = CULL ? src.Xs[min(p1, n - 1)] : src.X[i1];
    X[pp] = make_float2(x0.x, x1.x);
    Y[pp] = make_float2(x0.y, x1.y);
    Z[pp] = make_float2(x0.z, x1.z);
    nS[pp] = make_float2(-row_shift_estimate(rowM2, rowJ, dq, dmax2, i0),
                         -row_shift_estimate(rowM2, rowJ, dq, dmax2, i1));
    fs[pp] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int r = 0; r < kOtfRT; ++r) {
    tm[r] = -FLT_MAX;
    tj[r] = static_cast<int>(j0);
    sSS[r][threadIdx.x] = 0.0;
  }
  const float2 nkh2 = make_float2(-kh, -kh), nkl2 = make_float2(-kl, -kl);
  const float* Vp = vq;
  const float* Ep = vq + 2 * mpad;
  const float kcull = kh * kCullSlack;
  for (int64_t t0 = j0; t0 < j1; t0 += kOtfTJ) {
    __syncthreads();
    for (int k = threadIdx.x; k < kOtfTJ; k += kRowThreads) {
      const int64_t jp = t0 + k;  // (CULL: sorted position; coordinates stored sorted)
      if (jp < j1) {
        const int64_t j = CULL ? static_cast<int64_t>(src.perm_c[jp]) : jp;
        const float nx = src.Yn[jp], ny = src.Yn[src.ypad + jp], nz = src.Yn[2 * src.ypad + jp];
        const float V = Vp[j];
        sA[k] = make_float4(nx, nx, ny, ny);
        sB[k] = make_float4(nz, nz, V, V);
        const float E = Ep[j];
        sE[k] = make_float2(E, E);
      } else {  // padding: t = -inf, contributes 0, never the max
        sA[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        sB[k] = make_float4(0.f, 0.f, -INFINITY, -INFINITY);
        sE[k] = make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
    const int tn = static_cast<int>(min(static_cast<int64_t>(kOtfTJ), j1 - t0));
    for (int kb = 0; kb < tn; kb += kOtfBlk) {
      if constexpr (CULL) {
        if ((kb % kCullCB) == 0) {  // a culling block starts: does any row of the warp see it?
          const int64_t cbk = (t0 + kb) / kCullCB;
          const float4 lo = __ldg(src.cbox + 2 * cbk), hi = __ldg(src.cbox + 2 * cbk + 1);
          const float vmax = __ldg(src.cvmax + cbk);
          bool live = false;
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            const float d0 = box_d2(X[pp].x, Y[pp].x, Z[pp].x, lo, hi);
            const float d1 = box_d2(X[pp].y, Y[pp].y, Z[pp].y, lo, hi);
            live |= fmaf(-kcull, d0, vmax + nS[pp].x) >= kCullT;
            live |= fmaf(-kcull, d1, vmax + nS[pp].y) >= kCullT;
          }
          if (!__any_sync(0xffffffffu, live)) {
            kb += kCullCB - kOtfBlk;  // every exponent of the block is below -127
            continue;
          }
        }
      }
#pragma unroll kOtfUnroll
      for (int k = kb; k < kb + kOtfBlk; ++k) {
        const float4 A = sA[k], B = sB[k];
        const float2 E2 = sE[k];
        const float2 ax = make_float2(A.x, A.y), ay = make_float2(A.z, A.w);
        const float2 az = make_float2(B.x, B.y), V2 = make_float2(B.z, B.w);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          const float2 dx = __fadd2_rn(X[pp], ax), dy = __fadd2_rn(Y[pp], ay),
                       dz = __fadd2_rn(Z[pp], az);
          const float2 c = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
          const float2 t = __ffma2_rn(c, nkh2, __fadd2_rn(V2, nS[pp]));
          fs[pp] = __ffma2_rn(make_float2(ex2_approx(t.x), ex2_approx(t.y)), E2, fs[pp]);
        }
      }
      // block end: fp32 partials into fp64, the heaviest block remembered
      const int jb = static_cast<int>(t0 + kb);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        sSS[2 * pp][threadIdx.x] += otf_cvt(fs[pp].x);
        sSS[2 * pp + 1][threadIdx.x] += otf_cvt(fs[pp].y);
        if (fs[pp].x > tm[2 * pp]) {
          tm[2 * pp] = fs[pp].x;
          tj[2 * pp] = jb;
        }
        if (fs[pp].y > tm[2 * pp + 1]) {
          tm[2 * pp + 1] = fs[pp].y;
          tj[2 * pp + 1] = jb;
        }
        fs[pp] = make_float2(0.f, 0.f);
      }
    }
  }
  RowPart* dst = rpart + static_cast<int64_t>(blockIdx.y) * n;
#pragma unroll
  for (int r = 0; r < kOtfRT; ++r) {
    const int64_t pos = rbase + r * rstride;
    if (pos < n) {
      RowPart rp;
      rp.t = tm[r];
      rp.jb = tj[r];  // (CULL: sorted column position; k_row_otf_fin maps it)
      rp.s = sSS[r][threadIdx.x];
      dst[row_of(pos)] = rp;
    }
  }
}

// Fold the column splits of k_row_otf (split order: ties keep the lowest
// column), resolve the argmax column inside its 16-column block, then the
// row_shift_block epilogue (redo rule, u, w, shift, next estimate).
__global__ void __launch_bounds__(kRowThreads)
k_row_otf_fin(const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq,
              const double* __restrict__ dq, int64_t mpad, float kh, float kl,
              const double* __restrict__ a, const double* __restrict__ loga,
              double* __restrict__ rowM, double* __restrict__ rowS, double* __restrict__ u,
              double* __restrict__ wrow, float4* __restrict__ aux, double* __restrict__ rowM2,
              int* __restrict__ rowJ, int* __restrict__ redo_rows, const RowPart* __restrict__ rpart,
              int splits, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowThreads + threadIdx.x;
  if (i >= n) return;
  const float sc = row_shift_estimate(rowM2, rowJ, dq, ctrl->dmax2, i);
  float T = -FLT_MAX;
  int JB = 0;
  double S = 0.0;
  for (int k = 0; k < splits; ++k) {
    const RowPart rp = rpart[static_cast<int64_t>(k) * n + i];
    if (rp.t > T) {
      T = rp.t;
      JB = rp.jb;
    }
    S += rp.s;
  }
  // the reference column: the largest exponent of the heaviest block (first on ties)
  const float4 xi = src.X[i];
  int J = JB;
  float TJ = -FLT_MAX;
  for (int k = 0; k < kOtfBlk && JB + k < m; ++k) {
    const int64_t j = src.perm_c ? static_cast<int64_t>(src.perm_c[JB + k]) : JB + k;
    const float c = otf_sqeuclid(xi, src.Y[j]);
    const float t = fmaf(c, -kh, vq[j] + (-sc));
    if (t > TJ) {
      TJ = t;
      J = static_cast<int>(j);
    }
  }
  // the max lies in [T_J, T_J + 4]: exact redo unless it is within
  // [-kRedoLo, kRedoHi + 4] (and the sum finite and positive)
  if (!(TJ >= -kRedoLo && TJ <= kRedoHi && S > 0.0 && S < 1e300)) {
    const unsigned slot = atomicAdd(&ctrl->redo_count, 1u);
    redo_rows[slot] = static_cast<int>(i);
    return;
  }
  T = TJ;
  const double scd = static_cast<double>(sc);
  const double M = scd * kLn2;
  const double ui = (loga[i] - M) - log(S);
  const double wi = a[i] / S;
  rowM[i] = M;
  rowS[i] = S;
  u[i] = ui;
  wrow[i] = wi;
  rowM2[i] = scd + static_cast<double>(T);
  rowJ[i] = J;
  aux[i] = make_float4(sc, 0.0f, static_cast<float>(wi), 0.0f);
}

// Per-evaluation bounds of the culled on-the-fly sweeps: the largest column
// potential (base 2, hi part) of each 64-column sorted block, and the largest
// -M (negated row shift) of each 16-row sorted block.
__global__ void __launch_bounds__(256)
k_cull_cols(int64_t m, int64_t mpad, const float* __restrict__ vq, const int* __restrict__ perm_c,
            float* __restrict__ cvmax, float2* __restrict__ ves, const Ctrl* __restrict__ ctrl) {
  pdl_wait();
  if (ctrl->done) return;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b * kCullCB >= m) return;
  float v = -INFINITY;
  for (int k = lane; k < kCullCB; k += 32) {
    const int64_t s = b * kCullCB + k;
    if (s < m) {
      const int64_t j = perm_c[s];
      const float V = vq[j];
      v = fmaxf(v, V);
      if (ves) ves[s] = make_float2(V, vq[2 * mpad + j]);  // (V, 2^F) in sorted order
    }
  }
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) cvmax[b] = v;
}

__global__ void __launch_bounds__(256)
k_cull_rows(int64_t n, const float4* __restrict__ aux, const int* __restrict__ perm_r,
            float* __restrict__ rnegm, float4* __restrict__ auxs, const Ctrl* __restrict__ ctrl) {
  pdl_wait();
  if (ctrl->done) return;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * 16 + (threadIdx.x >> 4);
  const int l = threadIdx.x & 15;
  const int64_t s = b * kCullRB + l;
  float v = -INFINITY;
  if (s < n) {
    float4 ax = aux[perm_r[s]];
    v = -ax.x;
    if (auxs) {  // sorted copy for the column pass, weight pre-scaled w' = w 2^-mf
      ax.z = ax.y == 0.0f ? ax.z : ax.z * exp2f(-ax.y);
      auxs[s] = ax;
    }
  }
  for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (l == 0 && b * kCullRB < n) rnegm[b] = v;
}

// otg_cull_stats: the fraction of (warp tile x block) pairs the culled sweeps
// would visit at the handle's current state -- the same bound, per pair.
__global__ void k_cull_prep(int64_t n, int64_t m, const int* __restrict__ perm_r,
                            const int* __restrict__ perm_c, const double* __restrict__ rowM2,
                            const int* __restrict__ rowJ, const double* __restrict__ dq,
                            const double* __restrict__ p, const float* __restrict__ Yns,
                            int64_t ypad, const Ctrl* __restrict__ ctrl, float* __restrict__ nS,
                            float* __restrict__ Vc, float4* __restrict__ Ys) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) nS[t] = -row_shift_estimate(rowM2, rowJ, dq, ctrl->dmax2, perm_r[t]);
  if (t < m) {
    float hi, lo;
    split_q(p[perm_c[t]] * kLog2e, hi, lo);
    Vc[t] = hi;
    Ys[t] = make_float4(-Yns[t], -Yns[ypad + t], -Yns[2 * ypad + t], 0.f);
  }
}
__global__ void k_cull_stat(int64_t npts, const float4* __restrict__ pts,
                            const float* __restrict__ val, int tile, const float4* __restrict__ box,
                            const float* __restrict__ bnd, int64_t nblocks, float kcull,
                            unsigned long long* __restrict__ kept) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t groups = (npts + tile - 1) / tile;
  if (idx >= groups * nblocks) return;
  const int64_t g = idx / nblocks, b = idx % nblocks;
  const float4 lo = box[2 * b], hi = box[2 * b + 1];
  const float bb = bnd[b];
  bool live = false;
  for (int k = 0; k < tile && !live; ++k) {
    const int64_t s = g * tile + k;
    if (s >= npts) break;
    const float4 q = pts[s];
    live = fmaf(-kcull, box_d2(q.x, q.y, q.z, lo, hi), bb + val[s]) >= kCullT;
  }
  if (live) atomicAdd(kept, 1ull);
}


// ------------------------------------------------------------------ K2 ----
// fp64: partial c_j = sum_i exp(((-C'_ij) + p_j) - M_i) * w_i  (dual.cpp:36,41)
__global__ void __launch_bounds__(kColThreads)
k_col_precise(const double* __restrict__ C, int64_t ldc, int64_t m,
              const double* __restrict__ p, const double* __restrict__ rowM,
              const double* __restrict__ wrow, int64_t row_lo, int64_t row_hi,
              int64_t rows_per_split, double* __restrict__ part, int64_t mpad,
              const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kColThreads + threadIdx.x;
  const int64_t i0 = row_lo + static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t i1 = min(i0 + rows_per_split, row_hi);
  double acc = 0.0;
  if (j < m) {
    const double pj = p[j];
    // 4 rows' exponentials in flight, accumulated in the same row order (so
    // the sum is bitwise the one-row-at-a-time loop)
    int64_t i = i0;
    for (; i + 4 <= i1; i += 4) {
      double e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = exp(((-C[(i + k) * ldc + j]) + pj) - rowM[i + k]) * wrow[i + k];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += e[k];
    }
    for (; i < i1; ++i) acc += exp(((-C[i * ldc + j]) + pj) - rowM[i]) * wrow[i];
    part[static_cast<int64_t>(blockIdx.y) * mpad + j] = acc;
  }
}

// One row of a thread's 4 columns: A = Vc - Mc (exact: both multiples of
// 2^-8), g = fmaf(-c, kl, vf - mf), t = fmaf(-c, kh, A) + g, acc += w ex2(t).
__device__ __forceinline__ void col_quad_step(const float4& c, const float4& ax, float2 Vc01,
                                              float2 Vc23, float2 vf01, float2 vf23, float2 nkh2,
                                              float2 nkl2, float2& acc01, float2& acc23) {
  const float2 nM = make_float2(-ax.x, -ax.x), nm = make_float2(-ax.y, -ax.y);
  const float2 w2 = make_float2(ax.z, ax.z);
  const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
  const float2 t01 = __fadd2_rn(__ffma2_rn(c01, nkh2, __fadd2_rn(Vc01, nM)),
                                __ffma2_rn(c01, nkl2, __fadd2_rn(vf01, nm)));
  const float2 t23 = __fadd2_rn(__ffma2_rn(c23, nkh2, __fadd2_rn(Vc23, nM)),
                                __ffma2_rn(c23, nkl2, __fadd2_rn(vf23, nm)));
  acc01 = __ffma2_rn(w2, make_float2(ex2_approx(t01.x), ex2_approx(t01.y)), acc01);
  acc23 = __ffma2_rn(w2, make_float2(ex2_approx(t23.x), ex2_approx(t23.y)), acc23);
}

// On the fly: A = Vc - Mc (exact), t = fmaf(-c, kh, A) (the instance's
// log2(e)/eps IS the fp32 kh: ot.otf_epsilon), acc += w' ex2(t) with
// w' = w 2^-mf folded at staging and the column factor 2^vf applied once to
// the fp64 totals: three FP32 ops per element instead of six.
__device__ __forceinline__ void col_quad_step_nf(const float4& c, const float4& ax, float2 Vc01,
                                                 float2 Vc23, float2 nkh2, float2 nkl2,
                                                 float2& acc01, float2& acc23) {
  const float2 nM = make_float2(-ax.x, -ax.x);
  const float2 w2 = make_float2(ax.z, ax.z);
  const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
  const float2 t01 = __ffma2_rn(c01, nkh2, __fadd2_rn(Vc01, nM));
  const float2 t23 = __ffma2_rn(c23, nkh2, __fadd2_rn(Vc23, nM));
  acc01 = __ffma2_rn(w2, make_float2(ex2_approx(t01.x), ex2_approx(t01.y)), acc01);
  acc23 = __ffma2_rn(w2, make_float2(ex2_approx(t23.x), ex2_approx(t23.y)), acc23);
}

__device__ __forceinline__ void flush_acc(float2& acc01, float2& acc23, double* acc64) {
  acc64[0] += static_cast<double>(acc01.x);
  acc64[1] += static_cast<double>(acc01.y);
  acc64[2] += static_cast<double>(acc23.x);
  acc64[3] += static_cast<double>(acc23.y);
  acc01 = make_float2(0.f, 0.f);
  acc23 = make_float2(0.f, 0.f);
}

// fp32: thread owns 4 consecutive columns, loops over the split's rows.  The
// rows' shift / weight (aux) -- and, on the fly, the rows' points -- are
// staged in shared memory per 256-row tile and read as broadcasts.
// ---------------------------------------------- culled on-the-fly sweeps ----
// Warp-independent forms of k_row_otf / k_col_fast<true> for the Morton-
// ordered handle (P.cull): each warp tests a block with the point-to-box
// bound, stages only live blocks in its own shared-memory slice and never
// waits for the CTA's other warps (a CTA-wide tile barrier made every tile
// cost its busiest warp).  Per pair the arithmetic is that of the dense
// kernels; skipped blocks are exactly the ones whose every exponent is
// below -127, where ex2.approx.ftz returns +0.

// Rows: warp = 256 consecutive sorted rows (8 per lane, 4 packed pairs);
// blocks of kCullCB sorted columns, flushed / max-tracked per kOtfBlk.
#ifndef OTG_CULL_ROW_THREADS_PER_SM
#define OTG_CULL_ROW_THREADS_PER_SM 512  // culled row pass: resident threads per SM (768: 6.14 -> 512: 6.10 ms at cfg5)
#endif
__global__ void __launch_bounds__(kCullRowT, OTG_CULL_ROW_THREADS_PER_SM / kCullRowT)
k_row_otf_cull(const CostSrc src, int64_t n, int64_t m, const float* __restrict__ vq,
               const double* __restrict__ dq, int64_t mpad, float kh,
               const double* __restrict__ rowM2, const int* __restrict__ rowJ,
               int64_t cols_per_split, RowPart* __restrict__ rpart, const Ctrl* __restrict__ ctrl) {
  pdl_wait();
  if (ctrl->done || !ctrl->shift_valid) return;
  constexpr int kCRT = OTG_CULL_RT;
  constexpr int NP = kCRT / 2;
  constexpr int kW = kCullRowT / 32;
  __shared__ float4 sA[kW][kCullCB];  // (-x, -x, -y, -y)
  __shared__ float4 sB[kW][kCullCB];  // (-z, -z, V, V)
  __shared__ float2 sE[kW][kCullCB];  // (2^F, 2^F)
  __shared__ double sSS[kCRT][kCullRowT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rbase = static_cast<int64_t>(blockIdx.x) * (kCullRowT * kCRT) +
                        warp * (32 * kCRT) + lane;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * cols_per_split;
  const int64_t j1 = min(j0 + cols_per_split, m);
  const double dmax2 = ctrl->dmax2;
  float2 X[NP], Y[NP], Z[NP], nS[NP], fs[NP];
  float tm[kCRT];
  int tj[kCRT];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    const int64_t p0 = min(rbase + (2 * pp) * 32, n - 1), p1 = min(rbase + (2 * pp + 1) * 32, n - 1);
    const float4 x0 = src.Xs[p0], x1 = src.Xs[p1];
    X[pp] = make_float2(x0.x, x1.x);
    Y[pp] = make_float2(x0.y, x1.y);
    Z[pp] = make_float2(x0.z, x1.z);
    nS[pp] = make_float2(-row_shift_estimate(rowM2, rowJ, dq, dmax2, src.perm_r[p0]),
                         -row_shift_estimate(rowM2, rowJ, dq, dmax2, src.perm_r[p1]));
    fs[pp] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int r = 0; r < kCRT; ++r) {
    tm[r] = -FLT_MAX;
    tj[r] = static_cast<int>(j0);
    sSS[r][threadIdx.x] = 0.0;
  }
  const float2 nkh2 = make_float2(-kh, -kh);
  const float kcull = kh * kCullSlack;
  float4* wA = sA[warp];
  float4* wB = sB[warp];
  float2* wE = sE[warp];
  for (int64_t b0 = j0; b0 < j1; b0 += kCullCB) {
    const int64_t cbk = b0 / kCullCB;
    {
      const float4 lo = __ldg(src.cbox + 2 * cbk), hi = __ldg(src.cbox + 2 * cbk + 1);
      const float vmax = __ldg(src.cvmax + cbk);
      bool live = false;
      const float2 nk2 = make_float2(-kcull, -kcull), vm2 = make_float2(vmax, vmax);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const float2 bnd = __ffma2_rn(nk2, box_d2x2(X[pp], Y[pp], Z[pp], lo, hi),
                                      __fadd2_rn(vm2, nS[pp]));
        live |= fmaxf(bnd.x, bnd.y) >= kCullT;
      }
      if (src.skip && !__any_sync(0xffffffffu, live)) continue;  // every exponent below -127
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < kCullCB / 32; ++h) {  // stage the block: lane -> columns lane, lane + 32
      const int k = lane + 32 * h;
      const int64_t jp = b0 + k;
      if (jp < j1) {
        const float nx = src.Yn[jp], ny = src.Yn[src.ypad + jp], nz = src.Yn[2 * src.ypad + jp];
        const float2 ve = src.ves[jp];
        wA[k] = make_float4(nx, nx, ny, ny);
        wB[k] = make_float4(nz, nz, ve.x, ve.x);
        wE[k] = make_float2(ve.y, ve.y);
      } else {  // padding: t = -inf
        wA[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        wB[k] = make_float4(0.f, 0.f, -INFINITY, -INFINITY);
        wE[k] = make_float2(0.f, 0.f);
      }
    }
    __syncwarp();
    for (int kb = 0; kb < kCullCB && b0 + kb < j1; kb += kOtfBlk) {
#pragma unroll kOtfUnroll
      for (int k = kb; k < kb + kOtfBlk; ++k) {
        const float4 A = wA[k], B = wB[k];
        const float2 E2 = wE[k];
        const float2 ax = make_float2(A.x, A.y), ay = make_float2(A.z, A.w);
        const float2 az = make_float2(B.x, B.y), V2 = make_float2(B.z, B.w);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          const float2 dx = __fadd2_rn(X[pp], ax), dy = __fadd2_rn(Y[pp], ay),
                       dz = __fadd2_rn(Z[pp], az);
          const float2 c = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
          const float2 t = __ffma2_rn(c, nkh2, __fadd2_rn(V2, nS[pp]));
          fs[pp] = __ffma2_rn(make_float2(ex2_approx(t.x), ex2_approx(t.y)), E2, fs[pp]);
        }
      }
      const int jb = static_cast<int>(b0 + kb);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        sSS[2 * pp][threadIdx.x] += otf_cvt(fs[pp].x);
        sSS[2 * pp + 1][threadIdx.x] += otf_cvt(fs[pp].y);
        if (fs[pp].x > tm[2 * pp]) {
          tm[2 * pp] = fs[pp].x;
          tj[2 * pp] = jb;
        }
        if (fs[pp].y > tm[2 * pp + 1]) {
          tm[2 * pp + 1] = fs[pp].y;
          tj[2 * pp + 1] = jb;
        }
        fs[pp] = make_float2(0.f, 0.f);
      }
    }
  }
  RowPart* dst = rpart + static_cast<int64_t>(blockIdx.y) * n;
#pragma unroll
  for (int r = 0; r < kCRT; ++r) {
    const int64_t pos = rbase + r * 32;
    if (pos < n) {
      RowPart rp;
      rp.t = tm[r];
      rp.jb = tj[r];  // sorted column position (k_row_otf_fin maps it)
      rp.s = sSS[r][threadIdx.x];
      dst[src.perm_r[pos]] = rp;
    }
  }
}

// Columns: thread = 4 consecutive sorted columns, warp = 128; rows of the
// split in blocks of kCullRB sorted rows, staged per warp when live.
#ifndef OTG_CULL_COL_THREADS_PER_SM
#define OTG_CULL_COL_THREADS_PER_SM 1024  // culled column pass: resident threads per SM the registers allow (64 regs; 512: 6.25 -> 1024: 6.06 ms at cfg5)
#endif
__global__ void __launch_bounds__(kCullColT, OTG_CULL_COL_THREADS_PER_SM / kCullColT)
k_col_otf_cull(const CostSrc src, int64_t m, const double* __restrict__ p, float kh,
               const float4* __restrict__ aux, int64_t row_lo, int64_t row_hi,
               int64_t rows_per_split, double* __restrict__ part, int64_t mpad,
               const Ctrl* __restrict__ ctrl) {
  pdl_wait();
  if (ctrl->done) return;
  constexpr int NT = kCullColT, kW = NT / 32;
  __shared__ float4 sX[kW][kCullRB];
  __shared__ float4 sAx[kW][kCullRB];
  __shared__ double sAcc[4][NT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  const int64_t j0 = 4 * q;  // sorted column positions j0 .. j0 + 3
  const int64_t i0 = row_lo + static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t i1 = min(i0 + rows_per_split, row_hi);
  float Vc[4], vf[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double pj = (j0 + k < m) ? p[src.perm_c[j0 + k]] : 0.0;
    split_q(pj * kLog2e, Vc[k], vf[k]);
  }
  YQ y4;
  y4.x = y4.y = y4.z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j0 < m) load_y4<true>(src, q, y4);
  const float2 Vc01 = make_float2(Vc[0], Vc[1]), Vc23 = make_float2(Vc[2], Vc[3]);
  const float2 nkh2 = make_float2(-kh, -kh), nkl2 = make_float2(0.f, 0.f);
  float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
#pragma unroll
  for (int e = 0; e < 4; ++e) sAcc[e][threadIdx.x] = 0.0;
  const float kcull = kh * kCullSlack;
  const float yx[4] = {-y4.x.x, -y4.x.y, -y4.x.z, -y4.x.w};
  const float yy[4] = {-y4.y.x, -y4.y.y, -y4.y.z, -y4.y.w};
  const float yz[4] = {-y4.z.x, -y4.z.y, -y4.z.z, -y4.z.w};
  // (columns past m: V = 0 at the origin -- they may keep a block live, never wrong)
  float4* wX = sX[warp];
  float4* wAx = sAx[warp];
  for (int64_t r0 = i0; r0 < i1; r0 += kCullRB) {
    const int64_t rb = r0 / kCullRB;
    {
      const float4 lo = __ldg(src.rbox + 2 * rb), hi = __ldg(src.rbox + 2 * rb + 1);
      const float nm = __ldg(src.rnegm + rb);
      bool live = false;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        live |= fmaf(-kcull, box_d2(yx[e], yy[e], yz[e], lo, hi), Vc[e] + nm) >= kCullT;
      if (src.skip && !__any_sync(0xffffffffu, live)) continue;  // every exponent below -127
    }
    const int rn = static_cast<int>(min(static_cast<int64_t>(kCullRB), i1 - r0));
    __syncwarp();
    if (lane < kCullRB) {
      if (lane < rn) {
        const int64_t sp = r0 + lane;
        wX[lane] = src.Xs[sp];
        wAx[lane] = src.auxs[sp];  // (w' = w 2^-mf, sorted: k_cull_rows)
      } else {  // (never read: rn bounds the loop)
        wX[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        wAx[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    __syncwarp();
    if (rn == kCullRB) {
#pragma unroll
      for (int h = 0; h < kCullRB; h += kColUnroll) {
        float4 c[kColUnroll];
#pragma unroll
        for (int r = 0; r < kColUnroll; ++r) c[r] = cost_quad<true>(src, 0, q, wX[h + r], y4);
#pragma unroll
        for (int r = 0; r < kColUnroll; ++r)
          col_quad_step_nf(c[r], wAx[h + r], Vc01, Vc23, nkh2, nkl2, acc01, acc23);
      }
    } else {
      for (int r = 0; r < rn; ++r) {
        const float4 cv = cost_quad<true>(src, 0, q, wX[r], y4);
        col_quad_step_nf(cv, wAx[r], Vc01, Vc23, nkh2, nkl2, acc01, acc23);
      }
    }
    // fp32 partials into the fp64 totals once per block (kCullRB = kFlushRows rows)
    sAcc[0][threadIdx.x] += otf_cvt(acc01.x);
    sAcc[1][threadIdx.x] += otf_cvt(acc01.y);
    sAcc[2][threadIdx.x] += otf_cvt(acc23.x);
    sAcc[3][threadIdx.x] += otf_cvt(acc23.y);
    acc01 = make_float2(0.f, 0.f);
    acc23 = make_float2(0.f, 0.f);
  }
  double* dst = part + static_cast<int64_t>(blockIdx.y) * mpad;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (j0 + e < m) dst[src.perm_c[j0 + e]] = sAcc[e][threadIdx.x] * exp2(static_cast<double>(vf[e]));
}

template <bool OTF, int NT, bool CULL = false>
__global__ void __launch_bounds__(NT, (!OTF && NT == 256) ? OTG_COL_MINB
                                      : (OTF && NT == 256) ? OTG_COL_OTF_MINB : 1)
k_col_fast(const CostSrc src, int64_t m, const double* __restrict__ p, float kh, float kl,
           const float4* __restrict__ aux, int64_t row_lo, int64_t row_hi,
           int64_t rows_per_split, double* __restrict__ part, int64_t mpad,
           const Ctrl* __restrict__ ctrl, int exact_only) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // exact_only: the single-pass kernel (fused.cu) does the steady-state columns
  if (ctrl->done || (exact_only && ctrl->shift_valid)) return;
  __shared__ float4 sh_aux[kAuxTile];
  __shared__ float4 sh_x[OTF ? kAuxTile : 1];
  const int64_t q = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  const int64_t j0 = 4 * q;
  const int64_t i0 = row_lo + static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t i1 = min(i0 + rows_per_split, row_hi);
  float Vc[4], vf[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // (CULL: j0 + k is a sorted column position)
    const double pj = (j0 + k < m) ? p[CULL ? src.perm_c[j0 + k] : j0 + k] : 0.0;
    split_q(pj * kLog2e, Vc[k], vf[k]);
  }
  YQ y4;
  if (j0 < m) load_y4<OTF>(src, q, y4);
  // packed f32x2 form of  acc += w * ex2((Vc - Mc) - c kh + ((vf - mf) - c kl)):
  // bitwise the scalar expression, half the FP32 issue slots
  const float2 Vc01 = make_float2(Vc[0], Vc[1]), Vc23 = make_float2(Vc[2], Vc[3]);
  const float2 vf01 = make_float2(vf[0], vf[1]), vf23 = make_float2(vf[2], vf[3]);
  const float2 nkh2 = make_float2(-kh, -kh), nkl2 = make_float2(-kl, -kl);
  float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
  // the fp64 column totals live in shared memory (registers stay under the
  // 5-CTA/SM budget); flushed from the fp32 partials every kFlushRows rows
  __shared__ double sAcc[4][NT];
#pragma unroll
  for (int e = 0; e < 4; ++e) sAcc[e][threadIdx.x] = 0.0;
  auto flush = [&]() {
    sAcc[0][threadIdx.x] += OTF ? otf_cvt(acc01.x) : static_cast<double>(acc01.x);
    sAcc[1][threadIdx.x] += OTF ? otf_cvt(acc01.y) : static_cast<double>(acc01.y);
    sAcc[2][threadIdx.x] += OTF ? otf_cvt(acc23.x) : static_cast<double>(acc23.x);
    sAcc[3][threadIdx.x] += OTF ? otf_cvt(acc23.y) : static_cast<double>(acc23.y);
    acc01 = make_float2(0.f, 0.f);
    acc23 = make_float2(0.f, 0.f);
  };
  const bool active = j0 < m;
  const unsigned amask = __ballot_sync(0xffffffffu, active);
  const float kcull = kh * kCullSlack;
  for (int64_t t0 = i0; t0 < i1; t0 += kAuxTile) {
    const int64_t tn = min(static_cast<int64_t>(kAuxTile), i1 - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < tn; k += NT) {
      float4 ax = aux[CULL ? src.perm_r[t0 + k] : t0 + k];
      if (OTF) {
        sh_x[k] = CULL ? src.Xs[t0 + k] : src.X[t0 + k];
        ax.z = ax.y == 0.0f ? ax.z : ax.z * exp2f(-ax.y);  // w' = w 2^-mf
      }
      sh_aux[k] = ax;
    }
    __syncthreads();
    if (!active) continue;
    int k = 0;
    for (; k + kColUnroll <= tn; k += kColUnroll) {
      if constexpr (CULL) {
        if (((t0 + k) % kCullRB) == 0 && k + kCullRB <= tn) {
          // a culling block of rows starts: is any of the warp's columns live?
          const int64_t rb = (t0 + k) / kCullRB;
          const float4 lo = __ldg(src.rbox + 2 * rb), hi = __ldg(src.rbox + 2 * rb + 1);
          const float nm = __ldg(src.rnegm + rb);
          const float yx[4] = {y4.x.x, y4.x.y, y4.x.z, y4.x.w};
          const float yy[4] = {y4.y.x, y4.y.y, y4.y.z, y4.y.w};
          const float yz[4] = {y4.z.x, y4.z.y, y4.z.z, y4.z.w};
          bool live = false;
#pragma unroll
          for (int e = 0; e < 4; ++e)  // (y4 holds the negated coordinates)
            live |= fmaf(-kcull, box_d2(-yx[e], -yy[e], -yz[e], lo, hi), Vc[e] + nm) >= kCullT;
          if (!__any_sync(amask, live)) {
            k += kCullRB - kColUnroll;  // every exponent of the block is below -127
            continue;
          }
        }
      }
      float4 c[kColUnroll];
#pragma unroll
      for (int r = 0; r < kColUnroll; ++r)
        c[r] = cost_quad<OTF>(src, t0 + k + r, q, sh_x[OTF ? k + r : 0], y4);
#pragma unroll
      for (int r = 0; r < kColUnroll; ++r) {
        if constexpr (OTF)
          col_quad_step_nf(c[r], sh_aux[k + r], Vc01, Vc23, nkh2, nkl2, acc01, acc23);
        else
          col_quad_step(c[r], sh_aux[k + r], Vc01, Vc23, vf01, vf23, nkh2, nkl2, acc01, acc23);
      }
      if (((k + kColUnroll) % kFlushRows) == 0) flush();
    }
    for (; k < tn; ++k) {
      const float4 cv = cost_quad<OTF>(src, t0 + k, q, sh_x[OTF ? k : 0], y4);
      if constexpr (OTF)
        col_quad_step_nf(cv, sh_aux[k], Vc01, Vc23, nkh2, nkl2, acc01, acc23);
      else
        col_quad_step(cv, sh_aux[k], Vc01, Vc23, vf01, vf23, nkh2, nkl2, acc01, acc23);
    }
    flush();
  }
  if (active) {
    double* dst = part + static_cast<int64_t>(blockIdx.y) * mpad;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (CULL && j0 + e >= m) continue;
      const int64_t j = CULL ? static_cast<int64_t>(src.perm_c[j0 + e]) : j0 + e;
      dst[j] = OTF ? sAcc[e][threadIdx.x] * exp2(static_cast<double>(vf[e])) : sAcc[e][threadIdx.x];
    }
  }
}

// ----------------------------------------------------------------- E1a ----
// c_j = sum over shards of (sum over the shard's splits of the partials); the
// inner sum is what one rank holds, the outer sum stands in for the allreduce.
// Work unit `blk` of `nblk` also folds <u, a> over row slice blk into
// col[mpad + 1 + blk] (the sharded all-reduce covers col[0, mpad + 1 + nblk);
// finalize sums them).
__device__ __forceinline__ void merge_body(const double* __restrict__ part, int nshards, int splits,
                                           int64_t m, int64_t mpad, double* __restrict__ col,
                                           double* __restrict__ col_log,
                                           int* __restrict__ flag_idx, int* __restrict__ fb_cols,
                                           const double* __restrict__ u,
                                           const double* __restrict__ a, int64_t nrows,
                                           int do_merge, int flag, Ctrl* __restrict__ ctrl,
                                           int blk, int nblk, double* sh, int fused_rows,
                                           int ua_n) {
  // single-pass steady state: the cluster partials + the patch row
  if (fused_rows && ctrl->shift_valid) {
    nshards = 1;
    splits = fused_rows;
  }
  if (do_merge && blk < ua_n) {  // <u, a> over the local rows (for f): slice blk of ua_n
    const int64_t r0 = nrows * blk / ua_n, r1 = nrows * (blk + 1) / ua_n;
    double t = 0.0;
    for (int64_t k = r0 + threadIdx.x; k < r1; k += kEThreads) t += u[k] * a[k];
    t = block_sum<kEThreads>(t, sh);
    if (threadIdx.x == 0) col[mpad + 1 + blk] = t;
  }
  const double tiny = ctrl->tiny;
  // groups of 32 columns: warp w sums the splits k = w (mod 8) of the group
  // (coalesced 256-byte rows, 8 loads in flight per column), warp 0 folds
  // the 8 chains -- the same tree as one thread per column with 8 chains
  __shared__ double chain[kEThreads / 32][32];
  static_assert(kEThreads == 256, "8 chains = 8 warps");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t grp = blk; grp * 32 < m; grp += nblk) {
    const int64_t j = grp * 32 + lane;
    const bool in = j < m;
    double c = 0.0;
    if (do_merge) {
      for (int s = 0; s < nshards; ++s) {
        const double* src = part + static_cast<int64_t>(s) * splits * mpad + (in ? j : 0);
        double l = 0.0;
        if (in)
          for (int k = w; k < splits; k += 8) l += src[static_cast<int64_t>(k) * mpad];
        chain[w][lane] = l;
        __syncthreads();
        if (w == 0)
          c += ((chain[0][lane] + chain[1][lane]) + (chain[2][lane] + chain[3][lane])) +
               ((chain[4][lane] + chain[5][lane]) + (chain[6][lane] + chain[7][lane]));
        __syncthreads();
      }
      if (w == 0 && in) col[j] = c;
    } else if (w == 0 && in) {
      c = col[j];  // already merged (and all-reduced across ranks)
    }
    if (flag && w == 0 && in) {
      if (c >= tiny) {
        col_log[j] = log(c);
        flag_idx[j] = -1;
      } else {
        const unsigned slot = atomicAdd(&ctrl->fb_count, 1u);
        fb_cols[slot] = static_cast<int>(j);
        flag_idx[j] = static_cast<int>(slot);
      }
    }
  }
}

__global__ void __launch_bounds__(kEThreads)
k_merge(const double* __restrict__ part, int nshards, int splits, int64_t m, int64_t mpad,
        double* __restrict__ col, double* __restrict__ col_log, int* __restrict__ flag_idx,
        int* __restrict__ fb_cols, const double* __restrict__ u, const double* __restrict__ a,
        int64_t nrows, int do_merge, int flag, Ctrl* __restrict__ ctrl, int fused_rows,
        int ua_n, int patch_merged) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  if (patch_merged && ctrl->shift_valid) return;  // k_sp_patch_merge did this evaluation's merge
  __shared__ double sh[kEThreads / 32];
  merge_body(part, nshards, splits, m, mpad, col, col_log, flag_idx, fb_cols, u, a, nrows,
             do_merge, flag, ctrl, blockIdx.x, gridDim.x, sh, fused_rows, ua_n);
}

// ------------------------------------------------------------------ K5 ----
// Exact column log-sum-exp (dual.cpp:54-69) for flagged columns, split over
// row chunks: fb_part[f][chunk] = (max_i t_ij, sum_i exp(t_ij - max)).
// One pass per work item: every thread gathers kFbUnroll exponents with all
// loads in flight (the column is strided in memory, so the item is latency-
// bound, not bandwidth-bound), keeps an online (max, sum) and the CTA merges
// the per-thread pairs.  Same value as the two-pass LSE up to rounding.
template <bool PRECISE, bool OTF, int NT = kEThreads>
__device__ __forceinline__ void fallback_body(const double* __restrict__ C64, const CostSrc& src,
                                              int64_t ldc, int64_t n, double kappa,
                                              const double* __restrict__ u,
                                              const double* __restrict__ p,
                                              const int* __restrict__ fb_cols,
                                              double2* __restrict__ fb_part, unsigned nf, int blk,
                                              int nblk, double* sh) {
  const int64_t rpc = (n + kFbChunks - 1) / kFbChunks;
  const int64_t items = static_cast<int64_t>(nf) * kFbChunks;
  for (int64_t it = blk; it < items; it += nblk) {
    const int64_t f = it / kFbChunks, ch = it % kFbChunks;
    const int64_t j = fb_cols[f];
    const double vj = p[j];
    const int64_t i0 = ch * rpc, i1 = min(n, i0 + rpc);
    double top = -INFINITY, sum = 0.0;
    for (int64_t base = i0 + threadIdx.x; base < i1; base += NT * kFbUnroll) {
      double t[kFbUnroll];
#pragma unroll
      for (int k = 0; k < kFbUnroll; ++k) {
        const int64_t i = base + static_cast<int64_t>(k) * NT;
        if (i < i1) {
          t[k] = PRECISE ? (u[i] + vj) - C64[i * ldc + j]
                         : fma(-static_cast<double>(cost_one<OTF>(src, i, j)), kappa, u[i] + vj);
        } else {
          t[k] = -INFINITY;
        }
      }
      double mx = t[0];
#pragma unroll
      for (int k = 1; k < kFbUnroll; ++k) mx = fmax(mx, t[k]);
      if (mx > -INFINITY) {
        if (mx > top) {
          sum = (top > -INFINITY) ? sum * exp(top - mx) : 0.0;
          top = mx;
        }
#pragma unroll
        for (int k = 0; k < kFbUnroll; ++k) sum += exp(t[k] - top);
      }
    }
    const double T = block_max<NT>(top, sh);
    const double part = (top > -INFINITY) ? sum * exp(top - T) : 0.0;
    const double S = block_sum<NT>(part, sh);
    if (threadIdx.x == 0) fb_part[f * kFbChunks + ch] = make_double2(T, S);
  }
}

// Many flagged columns (the seed evaluation at v = 0 flags ~2% of them at
// cfg3): thread per flagged column instead of CTA per (column, chunk).  The
// list is sorted by column in shared memory first, so the 32 columns of a warp
// lie within a few KB of each row and its gathers hit few DRAM pages; each
// thread keeps its column's online (max, sum) over the chunk -- no block
// reduction.  Same (max, sum) per (column, chunk) as fallback_body up to the
// summation order.
constexpr int kFbSortMax = 4096;
template <bool PRECISE, bool OTF>
__device__ __forceinline__ void fallback_sorted_body(
    const double* __restrict__ C64, const CostSrc& src, int64_t ldc, int64_t n, double kappa,
    const double* __restrict__ u, const double* __restrict__ p, const int* __restrict__ fb_cols,
    double2* __restrict__ fb_part, unsigned nf, int2* skey /* shared, kFbSortMax */) {
  // skey: (column, slot), sorted by column
  int P2 = 1;
  while (P2 < static_cast<int>(nf)) P2 <<= 1;
  for (int k = threadIdx.x; k < P2; k += kEThreads)
    skey[k] = k < static_cast<int>(nf) ? make_int2(fb_cols[k], k) : make_int2(0x7fffffff, -1);
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {  // bitonic sort
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = threadIdx.x; k < P2 / 2; k += kEThreads) {
        const int lo = 2 * k - (k & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const int2 x = skey[lo], y = skey[hi];
        if ((x.x > y.x) == up) {
          skey[lo] = y;
          skey[hi] = x;
        }
      }
      __syncthreads();
    }
  }
  const int64_t rpc = (n + kFbChunks - 1) / kFbChunks;
  const int groups = (static_cast<int>(nf) + kEThreads - 1) / kEThreads;
  for (int it = blockIdx.x; it < groups * kFbChunks; it += gridDim.x) {
    const int g = it / kFbChunks, ch = it % kFbChunks;
    const int k = g * kEThreads + threadIdx.x;
    if (k >= static_cast<int>(nf)) continue;
    const int64_t j = skey[k].x;
    const int f = skey[k].y;
    const double vj = p[j];
    const int64_t i0 = ch * rpc, i1 = min(n, i0 + rpc);
    double top = -INFINITY, sum = 0.0;
    for (int64_t i = i0; i < i1; i += kFbUnroll) {
      double t[kFbUnroll];
#pragma unroll
      for (int e = 0; e < kFbUnroll; ++e) {
        const int64_t ii = i + e;
        t[e] = ii < i1 ? (PRECISE ? (u[ii] + vj) - C64[ii * ldc + j]
                                  : fma(-static_cast<double>(cost_one<OTF>(src, ii, j)), kappa,
                                        u[ii] + vj))
                       : -INFINITY;
      }
      double mx = t[0];
#pragma unroll
      for (int e = 1; e < kFbUnroll; ++e) mx = fmax(mx, t[e]);
      if (mx > -INFINITY) {
        if (mx > top) {
          sum = (top > -INFINITY) ? sum * exp(top - mx) : 0.0;
          top = mx;
        }
#pragma unroll
        for (int e = 0; e < kFbUnroll; ++e) sum += exp(t[e] - top);
      }
    }
    fb_part[static_cast<int64_t>(f) * kFbChunks + ch] = make_double2(top, sum);
  }
}

template <bool PRECISE, bool OTF>
__global__ void __launch_bounds__(kEThreads)
k_fallback(const double* __restrict__ C64, const CostSrc src, int64_t ldc, int64_t n,
           double kappa, const double* __restrict__ u, const double* __restrict__ p,
           const int* __restrict__ fb_cols, double2* __restrict__ fb_part,
           const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  const unsigned nf = ctrl->fb_count;
  if (nf == 0) return;
  if (nf >= 2 * kEThreads && nf <= kFbSortMax) {
    __shared__ int2 skey[kFbSortMax];
    fallback_sorted_body<PRECISE, OTF>(C64, src, ldc, n, kappa, u, p, fb_cols, fb_part, nf, skey);
    return;
  }
  __shared__ double sh[kEThreads / 32];
  fallback_body<PRECISE, OTF>(C64, src, ldc, n, kappa, u, p, fb_cols, fb_part, nf, blockIdx.x,
                              gridDim.x, sh);
}

// Sharded fallback: this rank's (top, sum) of each flagged column over its
// rows, laid out densely by column so every rank's buffers line up for the
// MAX / SUM all-reduces (the slot order of fb_cols is rank-local).
__global__ void __launch_bounds__(kEThreads)
k_fb_local(int64_t m, const int* __restrict__ flag_idx, const double2* __restrict__ fb_part,
           double* __restrict__ fbA, double* __restrict__ fbS, double* __restrict__ fbT,
           const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kEThreads + threadIdx.x;
  if (j >= m) return;
  const int slot = flag_idx[j];
  double top = -DBL_MAX, s = 0.0;
  if (slot >= 0) {
    for (int k = 0; k < kFbChunks; ++k) top = fmax(top, fb_part[slot * kFbChunks + k].x);
    for (int k = 0; k < kFbChunks; ++k) {
      const double2 fp = fb_part[slot * kFbChunks + k];
      if (fp.y > 0.0) s += fp.y * exp(fp.x - top);
    }
  }
  fbA[j] = top;
  fbT[j] = top;
  fbS[j] = s;
}

__global__ void __launch_bounds__(kEThreads)
k_fb_rescale(int64_t m, const int* __restrict__ flag_idx, const double* __restrict__ fbA,
             double* __restrict__ fbS, const double* __restrict__ fbT,
             const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kEThreads + threadIdx.x;
  if (j >= m || flag_idx[j] < 0) return;
  if (fbS[j] > 0.0) fbS[j] *= exp(fbT[j] - fbA[j]);
}

// Sharded chunk graphs: pause the chunk when this evaluation flagged columns
// (the flag set comes from the all-reduced sums, so every rank pauses at the
// same evaluation); the host finishes it eagerly (solver.cu resume).
__global__ void k_pause_if_flagged(Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (threadIdx.x == 0 && !ctrl->done && ctrl->fb_count > 0) ctrl->done = kPaused;
}

// --------------------------------------------------------------- control --
__device__ void push_trace(Ctrl* C, double* trace, long long iter, double viol, double f,
                           double mu, double alpha) {
  const long long row = C->trace_count % C->trace_cap;
  double* r = trace + row * kTraceCols;
  r[0] = static_cast<double>(iter);
  r[1] = 0.0;
  r[2] = viol;
  r[3] = viol;
  r[4] = f;
  r[5] = mu;
  r[6] = alpha;
  for (int k = 7; k < kTraceCols; ++k) r[k] = __longlong_as_double(0x7ff8000000000000LL);
  C->trace_row = row;
  C->trace_count += 1;
}

__device__ void push_boundary(Ctrl* C, double* bounds) {
  if (C->boundary_count < C->boundary_cap) {
    double* r = bounds + C->boundary_count * kBoundCols;
    r[0] = static_cast<double>(C->stage);
    r[1] = C->mu;
    r[2] = C->alpha_next;
    r[3] = static_cast<double>(C->total_inner);
    r[4] = __longlong_as_double(0x7ff8000000000000LL);  // energy: k_apply, with a reference
  }
  C->boundary_count += 1;
  C->boundary_pending = 1;
}

// Scalar control flow after one evaluation (one thread).  Mirrors
// sinkhorn.cpp:80-113, accel.cpp:176-197, 211-230, 245-301.
__device__ void control_step(Ctrl* C, double* trace, double* bounds, double gl, double f) {
  const long long ev = ++C->evaluations;
  C->mu_step = C->mu;  // the observed step's mu (a stage change below halves C->mu)
  const bool seed = ev == 1;
  C->grad_l1 = gl;
  C->f_value = f;
  C->trace_row = -1;
  C->stage_changed = 0;
  C->final_violation = gl;
  C->final_f = f;
  const bool rec = C->record_trace != 0;
  const long long stride = C->trace_stride;
  switch (C->mode) {
    case MODE_EVAL:
      C->done = 1;
      break;
    case MODE_SINKHORN: {
      const long long k = C->k;
      const bool done = gl < C->tol || k >= C->max_iters;
      if (rec && (k % stride == 0 || done)) push_trace(C, trace, k, gl, f, 0.0, 0.0);
      if (done) {
        C->converged = gl < C->tol;
        C->iterations = k;
        C->done = 1;
      } else {
        C->k = k + 1;
      }
      break;
    }
    case MODE_ACC: {
      const long long k = C->k;
      C->is_step = !seed;
      C->alpha_step = C->alpha_next;
      const bool done = gl < C->tol || k >= C->max_iters;
      if (rec && (k % stride == 0 || done)) push_trace(C, trace, k, gl, f, C->mu, C->alpha_step);
      if (done) {
        C->converged = gl < C->tol;
        C->iterations = k;
        C->done = 1;
      } else {
        C->k = k + 1;
      }
      break;
    }
    case MODE_ACC_RUN: {
      const long long k = C->k;
      C->is_step = !seed;
      C->alpha_step = C->alpha_next;
      const bool terminal = k == C->msteps;
      if (rec && (k % stride == 0 || terminal))
        push_trace(C, trace, k, gl, f, C->mu, C->alpha_step);
      if (terminal) {
        C->iterations = C->msteps;
        C->done = 1;
      } else {
        C->k = k + 1;
      }
      break;
    }
    case MODE_HOMOTOPY: {
      C->is_step = !seed;
      C->alpha_step = C->alpha_next;
      const long long cap = C->max_total_inner;
      if (seed) {
        const bool conv = gl < C->tol;
        C->converged = conv;
        if (rec) push_trace(C, trace, 0, gl, f, C->mu, C->alpha_step);
        if (conv) {
          C->done = 1;
        } else {
          C->stage = 0;
          C->outer_stages = 1;
          C->inner_i = 0;
          C->m_stage = C->m0;
          push_boundary(C, bounds);
        }
      } else {
        C->total_inner += 1;
        C->inner_i += 1;
        const bool conv = gl < C->tol;
        C->converged = conv;
        const bool terminal = conv || C->total_inner >= cap;
        if (rec && (C->total_inner % stride == 0 || terminal))
          push_trace(C, trace, C->total_inner, gl, f, C->mu, C->alpha_step);
        if (conv) {
          C->done = 1;
        } else {
          if (C->inner_i == C->m_stage) {
            if (C->stage + 1 < C->max_outer) {
              C->stage += 1;
              C->mu /= 2.0;
              C->alpha_next = sqrt(2.0 * C->mu);
              C->m_stage = static_cast<long long>(floor(sqrt(2.0) * static_cast<double>(C->m_stage))) + 1;
              C->inner_i = 0;
              C->outer_stages += 1;
              C->stage_changed = 1;
              push_boundary(C, bounds);
            } else {
              C->done = 1;
            }
          }
          if (!C->done && C->total_inner >= cap) {
            C->capped = 1;
            C->done = 1;
          }
        }
      }
      C->iterations = C->total_inner;
      break;
    }
    default:
      C->done = 1;
  }
  C->live_e2 = 1;
}

// ----------------------------------------------------------------- E1b ----
struct FinArgs {
  int64_t m, mpad;
  const double* p;
  const double* b;
  const double* logb;
  double* col;
  double* col_log;
  const int* flag_idx;
  const double2* fb_part;
  const double* fbA;
  const double* fbS;
  int sharded;
  int ua_slices;
  double* y;
  double* grad;
  double* e1_part;
  double* trace;
  double* bounds;
  // the exact column LSE of flagged columns, folded into k_finalize when the
  // handle is not sharded (fold_fb): K5's inputs
  int fold_fb;
  int storage;
  const double* C64;
  CostSrc src;
  int64_t ldc, nrows;
  double kappa;
  const double* u;
  const int* fb_cols;
  double2* fb_part_w;
};

// Per-column finalize of work unit blk of nblk; its partials -> e1_part[blk].
// One column (after the merge): the exact LSE of a flagged column from the
// fallback partials, grad, y and the column's share of the E1 sums.
struct E1Acc {
  double s_abs = 0.0, s_y = 0.0, s_pb = 0.0, mx_p = 0.0, bad = 0.0;
};
__device__ __forceinline__ void finalize_col(const FinArgs& A, int64_t j, int slot, E1Acc& e) {
  double c = A.col[j], cl;
  if (slot >= 0) {
    double top, s;
    if (A.sharded) {  // combined across ranks (k_fb_local / k_fb_rescale + all-reduces)
      top = A.fbA[j];
      s = A.fbS[j];
    } else {
      top = -INFINITY;
      for (int k = 0; k < kFbChunks; ++k) top = fmax(top, A.fb_part[slot * kFbChunks + k].x);
      s = 0.0;
      for (int k = 0; k < kFbChunks; ++k) {
        const double2 fp = A.fb_part[slot * kFbChunks + k];
        if (fp.y > 0.0) s += fp.y * exp(fp.x - top);
      }
    }
    cl = top + log(s);
    c = exp(cl);
    A.col[j] = c;
    A.col_log[j] = cl;
  } else {
    cl = A.col_log[j];
  }
  if (!isfinite(cl)) e.bad = 1.0;
  const double g = c - A.b[j];
  A.grad[j] = g;
  const double pj = A.p[j];
  const double yj = pj + (A.logb[j] - cl);
  A.y[j] = yj;
  e.s_abs += fabs(g);
  e.s_y += yj;
  e.s_pb += pj * A.b[j];
  e.mx_p = fmax(e.mx_p, fabs(pj));
}

template <int NT = kEThreads>
__device__ __forceinline__ void store_e1(const FinArgs& A, int part, E1Acc& e, double* shm) {
  double v[5] = {e.s_abs, e.s_y, e.s_pb, e.mx_p, e.bad};
  block_multi<NT, 3, 2>(v, shm);
  if (threadIdx.x == 0) {
    double* dst = A.e1_part + part * 8;
#pragma unroll
    for (int q = 0; q < 5; ++q) dst[q] = v[q];
  }
}

// The E1 partials are per group of 32 consecutive columns (group g =
// columns 32 g .. 32 g + 31, one warp, a fixed shuffle tree): k_finalize,
// k_merge_fin and k_sp_patch_merge all produce them identically, so every
// path sums the same partials in the same order.
__device__ __forceinline__ void store_e1_warp(const FinArgs& A, int64_t g, E1Acc& e) {
  const double s0 = warp_sum(e.s_abs), s1 = warp_sum(e.s_y), s2 = warp_sum(e.s_pb);
  const double m0 = warp_max(e.mx_p), m1 = warp_max(e.bad);
  if ((threadIdx.x & 31) == 0) {
    double* dst = A.e1_part + g * 8;
    dst[0] = s0;
    dst[1] = s1;
    dst[2] = s2;
    dst[3] = m0;
    dst[4] = m1;
  }
}

// Per-column finalize of the 32-column groups of warp slots blk x warps ..
// (stride nblk x warps); each group's partials -> e1_part[group].
// defer: flagged columns are left to the last CTA (their fallback partials
// are complete only once every CTA has run its share of the fallback).
template <int NT = kEThreads>
__device__ __forceinline__ void finalize_cols(const FinArgs& A, int blk, int nblk, double* shm,
                                              bool defer = false) {
  (void)shm;
  constexpr int W = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t G = e1_groups_of(A.m);
  for (int64_t g = static_cast<int64_t>(blk) * W + w; g < G; g += static_cast<int64_t>(nblk) * W) {
    E1Acc e;
    const int64_t j = g * 32 + lane;
    if (j < A.m) {
      const int slot = A.flag_idx[j];
      if (!(defer && slot >= 0)) finalize_col(A, j, slot, e);
    }
    store_e1_warp(A, g, e);
  }
}

template <int NT = kEThreads>
__device__ __forceinline__ void finalize_tail(const FinArgs& A, int nparts, double* sh,
                                              Ctrl* __restrict__ ctrl) {
  double gl = 0.0, sy = 0.0, pb = 0.0, mp = 0.0, bd = 0.0;
  for (int k = threadIdx.x; k < nparts; k += NT) {
    const volatile double* src = A.e1_part + k * 8;
    gl += src[0];
    sy += src[1];
    pb += src[2];
    mp = fmax(mp, src[3]);
    bd = fmax(bd, src[4]);
  }
  double ua = 0.0;  // <u, a> partials of the merge work units (col[mpad + 1 + k])
  for (int k = threadIdx.x; k < A.ua_slices; k += NT) ua += A.col[A.mpad + 1 + k];
  {
    double v[6] = {gl, sy, pb, ua, mp, bd};
    block_multi<NT, 4, 2>(v, sh);
    gl = v[0];
    sy = v[1];
    pb = v[2];
    ua = v[3];
    mp = v[4];
    bd = v[5];
  }
  if (threadIdx.x != 0) return;
  Ctrl* C = ctrl;
  C->e1_counter = 0;
  C->fb_total += C->fb_count;
  C->fb_count = 0;
  C->redo_total += C->redo_count;
  C->redo_count = 0;
  const double f = (1.0 - ua) - pb;
  C->mean_y = sy / static_cast<double>(A.m);
  C->max_v_inf = fmax(C->max_v_inf, mp);
  if (bd > 0.0) {  // check_col_log_finite (sinkhorn.cpp:20-25)
    C->error = OTG_E_DOMAIN;
    C->done = 1;
    C->live_e2 = 0;
    return;
  }
  control_step(C, A.trace, A.bounds, gl, f);
}

template <bool PRECISE, bool OTF, int NT = kEThreads>
__device__ __forceinline__ void fallback_all(const FinArgs& A, unsigned nf, double* sh,
                                             int2* skey) {
  if (skey && nf >= 2 * NT && nf <= kFbSortMax)
    fallback_sorted_body<PRECISE, OTF>(A.C64, A.src, A.ldc, A.nrows, A.kappa, A.u, A.p, A.fb_cols,
                                       A.fb_part_w, nf, skey);
  else
    fallback_body<PRECISE, OTF, NT>(A.C64, A.src, A.ldc, A.nrows, A.kappa, A.u, A.p, A.fb_cols,
                                    A.fb_part_w, nf, blockIdx.x, gridDim.x, sh);
}

__global__ void __launch_bounds__(kEThreads, 2)
k_finalize(const FinArgs A, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || ctrl->fin_done) return;  // (fin_done: k_sp_patch_merge finalized it)
  __shared__ double sh[kEThreads / 32 * 8];
  __shared__ bool last;
  // K5 folded in (unsharded): every CTA takes its share of the flagged
  // columns' exact LSE, the last CTA finalizes those columns
  // flagged columns are finalized by the last CTA in column order whether the
  // fallback ran here or (sharded) in k_fallback + the all-reduces, so the
  // two paths sum the E1 partials identically
  const unsigned nf = ctrl->fb_count;
  if (nf > 0 && A.fold_fb) {
#if OTG_FIN_SORTED_FB
    __shared__ int2 skey[kFbSortMax];
#else
    int2* skey = nullptr;  // (unsorted work items only: no 32 KB static buffer)
#endif
    if (A.storage == OTG_STORE_F64)
      fallback_all<true, false>(A, nf, sh, skey);
    else if (A.storage == OTG_STORE_ON_THE_FLY)
      fallback_all<false, true>(A, nf, sh, skey);
    else
      fallback_all<false, false>(A, nf, sh, skey);
  }
  finalize_cols(A, blockIdx.x, gridDim.x, sh, nf > 0);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&ctrl->e1_counter, 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  int parts = static_cast<int>(e1_groups_of(A.m));
  if (nf > 0) {  // the flagged columns, in COLUMN order (the list's slot order
                 // comes from atomics): one more partial, deterministic
    E1Acc e;
    for (int64_t j = threadIdx.x; j < A.m; j += kEThreads) {
      const int slot = A.flag_idx[j];
      if (slot >= 0) finalize_col(A, j, slot, e);
    }
    store_e1(A, parts, e, sh);
    __syncthreads();
    ++parts;
  }
  finalize_tail(A, parts, sh, ctrl);
}

// Unsharded, single-shard solver evaluations (inside the chunk graph): the
// merge of k_merge (one 32-column group per CTA, 8 warps over the splits,
// the same 8-chain tree), its underflow flags and <u, a> slice, then warp 0
// finalizes the group's unflagged columns into the group's E1 partial and
// the last CTA runs the control step -- unless a column was flagged (then
// k_finalize redoes the whole finalize with the exact column LSE).  Saves
// k_finalize's launch and last-CTA round trip (cfg1: latency-bound).
__global__ void __launch_bounds__(kEThreads)
k_merge_fin(const double* __restrict__ part, int splits, int64_t m, int64_t mpad,
            double* __restrict__ col, double* __restrict__ col_log, int* __restrict__ flag_idx,
            int* __restrict__ fb_cols, const double* __restrict__ u, const double* __restrict__ a,
            int64_t nrows, Ctrl* __restrict__ ctrl, int fused_rows, int ua_n, int patch_merged,
            const FinArgs F) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  if (patch_merged && ctrl->shift_valid) return;  // k_sp_patch_merge did this evaluation's merge
  if (fused_rows && ctrl->shift_valid) splits = fused_rows;
  __shared__ double sh[kEThreads / 32 * 8];
  __shared__ double chain[kEThreads / 32][32];
  __shared__ bool last;
  const int blk = blockIdx.x, nblk = gridDim.x;
  if (blk < ua_n) {  // <u, a> over row slice blk of ua_n (as merge_body)
    const int64_t r0 = nrows * blk / ua_n, r1 = nrows * (blk + 1) / ua_n;
    double t = 0.0;
    for (int64_t k = r0 + threadIdx.x; k < r1; k += kEThreads) t += u[k] * a[k];
    t = block_sum<kEThreads>(t, sh);
    if (threadIdx.x == 0) col[mpad + 1 + blk] = t;
  }
  const double tiny = ctrl->tiny;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t grp = blk; grp * 32 < m; grp += nblk) {
    const int64_t j = grp * 32 + lane;
    const bool in = j < m;
    double l = 0.0;
    if (in)
      for (int k = w; k < splits; k += 8) l += part[static_cast<int64_t>(k) * mpad + j];
    chain[w][lane] = l;
    __syncthreads();
    if (w == 0) {
      const double c = 0.0 + (((chain[0][lane] + chain[1][lane]) + (chain[2][lane] + chain[3][lane])) +
                              ((chain[4][lane] + chain[5][lane]) + (chain[6][lane] + chain[7][lane])));
      E1Acc e;
      if (in) {
        col[j] = c;
        if (c >= tiny) {
          col_log[j] = log(c);
          flag_idx[j] = -1;
          finalize_col(F, j, -1, e);
        } else {
          const unsigned slot = atomicAdd(&ctrl->fb_count, 1u);
          fb_cols[slot] = static_cast<int>(j);
          flag_idx[j] = static_cast<int>(slot);
        }
      }
      store_e1_warp(F, grp, e);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ctrl->e1_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (*reinterpret_cast<volatile unsigned*>(&ctrl->fb_count) != 0u) {
    // underflowed columns need the exact column LSE: pause the chunk (every
    // later kernel of it returns); the host finishes this evaluation eagerly
    // (k_finalize with the fallback, k_apply) and keeps replaying
    if (threadIdx.x == 0) {
      ctrl->e1_counter = 0;
      ctrl->done = kPaused;
    }
    return;
  }
  finalize_tail<kEThreads>(F, static_cast<int>(e1_groups_of(m)), sh, ctrl);
  if (threadIdx.x == 0) ctrl->fin_done = 1;
}

// ------------------------------------------------------------------ E2 ----


__device__ __forceinline__ double expm1_over_z(double z) {  // mirror.cpp:21-24
  if (fabs(z) < 1e-8) return 1.0 + z / 2.0 + z * z / 6.0;
  return expm1(z) / z;
}

struct AppArgs {
  int64_t m, mpad;
  const double* b;
  double* p;
  double* wacc;
  double* y;
  const double* grad;
  double* prev_grad;
  double* prev_x;
  double* prev_y;
  float* vq;
  double* dq;
  int fast;
  double* e2_part;
  double* trace;
  const double* vstar;  // ReferenceSolution v* (energy / radii), or unused
  double* bounds;
};

// The solver's vector update for work unit blk of nblk (accel.cpp:161-168,
// 279; stability sums of diag.cpp); partials -> e2_part[blk].  The control
// fields are read through a volatile view: inside the single-kernel
// epilogue they were written by another CTA before a grid barrier.
template <int NT = kEThreads>
__device__ __forceinline__ void apply_cols(const AppArgs& A, const Ctrl* ctrl_in, int blk, int nblk,
                                           double* sh) {
  const volatile Ctrl* ctrl = ctrl_in;
  const int mode = ctrl->mode;
  const bool done = ctrl->done != 0;
  const double mean = ctrl->mean_y;
  const bool step = ctrl->is_step != 0;
  const double al = ctrl->alpha_step, an = ctrl->alpha_next;
  const bool resc = ctrl->stage_changed && ctrl->rescale_w;
  const bool stab = ctrl->stability != 0 && mode >= MODE_ACC_RUN;
  const bool have_prev = ctrl->have_prev != 0;
  // energy / radii (accel.cpp:46-60): acc_solve, acc_run, homotopy with a reference
  const bool refq = ctrl->have_ref != 0 && mode >= MODE_ACC;
  const bool bpend = refq && ctrl->boundary_pending != 0;
  // the next point replaces p: record max_j (p_new - p_old) and the split of
  // p_new for the fp32 row pass's shift estimate (k_row_shift)
  const bool moves = !done && mode != MODE_EVAL;
  double c1 = 0.0, br = 0.0, c2 = 0.0, qq = 0.0, drift = 0.0, ginf = 0.0, dom = 0.0;
  double qe = 0.0, qx = 0.0, qy = 0.0, qb = 0.0, domr = 0.0;
  double dstep = -INFINITY;
  for (int64_t j = static_cast<int64_t>(blk) * NT + threadIdx.x; j < A.m;
       j += static_cast<int64_t>(nblk) * NT) {
    const double S = A.y[j] - mean;  // project_zero_sum (mirror.cpp:103-105)
    if (mode == MODE_EVAL) {
      A.y[j] = S;
      continue;
    }
    const double x = A.p[j];
    double pn = S;
    if (mode != MODE_SINKHORN) {
      double w = A.wacc[j];
      if (step) w = (w + (al * al - 2.0) * x + 2.0 * S) / (1.0 + al);  // accel.cpp:168
      if (stab) {
        const double yn = w / al;
        const double g1 = A.grad[j];
        if (have_prev) {
          const double g0 = A.prev_grad[j], bj = A.b[j];
          ginf = fmax(ginf, fabs(g0));
          const double r0 = g0 / bj, r1 = g1 / bj;
          if (r0 <= -1.0 || r1 <= -1.0) {
            dom = 1.0;
          } else {
            const double D0 = bj * expm1_over_z(log1p(r0));
            const double D1 = bj * expm1_over_z(log1p(r1));
            c1 += g0 * g0 * D1 / (D0 * D0);
            br += g0 - bj * log1p(r0);
            const double vk = A.prev_y[j] - A.prev_x[j], vk1 = yn - x;
            c2 += (D1 - D0) * (vk * vk);
            qq += D1 * (vk1 * vk1);
            drift = fmax(drift, fabs(D1 - D0));
          }
        }
        A.prev_grad[j] = g1;
        A.prev_x[j] = x;
        A.prev_y[j] = yn;
      }
      if (refq) {  // D(p(x)) at the evaluated point; y = w / alpha (accel.cpp:44)
        const double bj = A.b[j], r1 = A.grad[j] / bj, vs = A.vstar[j];
        const double yn = w / al, zy = yn - vs, zx = x - vs;
        if (r1 <= -1.0) {
          domr = 1.0;  // DomainViolation: the row keeps empty cells
        } else {
          const double D1 = bj * expm1_over_z(log1p(r1));
          qe += D1 * (zy * zy);
          qx += D1 * (zx * zx);
          if (bpend) {  // stage_energy after the stage change (accel.cpp:104-114)
            const double yb = (resc ? w * (an / al) : w) / an, zb = yb - vs;
            qb += D1 * (zb * zb);
          }
        }
        qy += zy * zy;
      }
      if (resc) w *= an / al;  // accel.cpp:279
      A.wacc[j] = w;
      pn = (w + S) / (1.0 + an);  // accel.cpp:161
    }
    if (moves) {
      A.p[j] = pn;
      dstep = fmax(dstep, pn - x);
      if (A.fast) {
        split_store(pn * kLog2e, A.vq, A.mpad, j);
        A.dq[j] = (pn - x) * kLog2e;
      }
    }
  }
  {  // (unused quantities stay 0 / -inf: reduced anyway, in one pass)
    double v[13] = {c1, br, c2, qq, qe, qx, qy, qb, drift, ginf, dom, dstep, domr};
    block_multi<NT, 8, 5>(v, sh);
    c1 = v[0];
    br = v[1];
    c2 = v[2];
    qq = v[3];
    qe = v[4];
    qx = v[5];
    qy = v[6];
    qb = v[7];
    drift = v[8];
    ginf = v[9];
    dom = v[10];
    dstep = v[11];
    domr = v[12];
  }
  if (threadIdx.x == 0) {
    double* dst = A.e2_part + blk * kE2;
    dst[8] = qe;
    dst[9] = qx;
    dst[10] = qy;
    dst[11] = qb;
    dst[12] = domr;
    dst[0] = c1;
    dst[1] = br;
    dst[2] = c2;
    dst[3] = qq;
    dst[4] = drift;
    dst[5] = ginf;
    dst[6] = dom;
    dst[7] = dstep;
  }
}

template <int NT = kEThreads>
__device__ __forceinline__ void apply_tail(const AppArgs& A, int nparts, double* sh,
                                           Ctrl* __restrict__ ctrl) {
  const volatile Ctrl* cv = ctrl;
  const int mode = cv->mode;
  const bool done = cv->done != 0;
  const bool stab = cv->stability != 0 && mode >= MODE_ACC_RUN;
  const bool have_prev = cv->have_prev != 0;
  const double al = cv->alpha_step;
  const bool moves = !done && mode != MODE_EVAL;
  const bool refq = cv->have_ref != 0 && mode >= MODE_ACC;
  double t[13] = {0, 0, 0, 0, 0, 0, 0, -INFINITY, 0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < nparts; k += NT) {
    const volatile double* src = A.e2_part + k * kE2;
    for (int q = 0; q < 4; ++q) t[q] += src[q];
    for (int q = 4; q < 8; ++q) t[q] = fmax(t[q], src[q]);
    if (refq) {
      for (int q = 8; q < 12; ++q) t[q] += src[q];
      t[12] = fmax(t[12], src[12]);
    }
  }
  {
    double v[13] = {t[0], t[1], t[2], t[3], t[8], t[9], t[10], t[11], t[4], t[5], t[6], t[7], t[12]};
    block_multi<NT, 8, 5>(v, sh);
    for (int q = 0; q < 4; ++q) t[q] = v[q];
    for (int q = 8; q < 12; ++q) t[q] = v[q - 4];
    for (int q = 4; q < 8; ++q) t[q] = v[q + 4];
    t[12] = v[12];
  }
  if (threadIdx.x != 0) return;
  Ctrl* C = ctrl;
  if (refq) {  // lyapunov_energy_from_parts (diag.cpp:76-88) + RadiusTracker
    const double f = C->f_value;
    if (C->f_star > f + 1e-9) {  // OtError in the reference: the solve fails
      C->error = OTG_E_OT;
      C->done = 1;
    } else if (t[12] == 0.0) {
      const double energy = (f - C->f_star) + (C->mu_step != 0.0 ? 0.5 * C->mu_step * t[8] : 0.0);
      const double rx = sqrt(t[9]), ry = sqrt(t[10]);
      C->rmax_x = fmax(C->rmax_x, rx);
      C->rmax_y = fmax(C->rmax_y, ry);
      if (C->trace_row >= 0) {
        double* r = A.trace + C->trace_row * kTraceCols;
        r[12] = energy;
        r[13] = rx;
        r[14] = ry;
      }
      if (C->boundary_pending && C->boundary_count <= C->boundary_cap)
        A.bounds[(C->boundary_count - 1) * kBoundCols + 4] =
            (f - C->f_star) + (C->mu != 0.0 ? 0.5 * C->mu * t[11] : 0.0);
    }
    C->boundary_pending = 0;
  }
  if (stab && have_prev) {
    double cells[5];
    bool valid = true;
    if (t[5] < kGradFloor) {  // diag.cpp:116-123: skipped, counts as held, not checked
      cells[0] = cells[1] = cells[2] = cells[3] = cells[4] = 0.0;
    } else if (t[6] > 0.0) {  // DomainViolation caught by the observer (accel.cpp:68)
      valid = false;
    } else {
      const double coef = (4.0 - al * al - 2.0 * sqrt(al)) / (2.0 * al * (1.0 + al) * (1.0 + al));
      cells[0] = t[0];
      cells[1] = coef * t[1];
      cells[2] = t[2];
      cells[3] = pow(al, 1.5) * t[3];
      cells[4] = t[4];
      C->cond_checked += 1;
      C->cond_held += (cells[0] < cells[1] && cells[2] < cells[3]) ? 1 : 0;
    }
    if (valid && C->trace_row >= 0) {
      double* r = A.trace + C->trace_row * kTraceCols;
      for (int q = 0; q < 5; ++q) r[7 + q] = cells[q];
    }
  }
  if (stab) C->have_prev = 1;
  if (moves && A.fast) {
    C->dmax2 = t[7] * kLog2e;
    C->shift_valid = isfinite(t[7]) ? 1 : 0;
  }
  C->e2_counter = 0;
  C->live_e2 = 0;
}

__global__ void __launch_bounds__(kEThreads, 2)
k_apply(const AppArgs A, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // (this evaluation's finalize is over: the next one starts unfinalized)
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctrl->fin_done) ctrl->fin_done = 0;
  if (!ctrl->live_e2) return;
  __shared__ double sh[kEThreads / 32 * 16];
  __shared__ bool last;
  apply_cols(A, ctrl, blockIdx.x, gridDim.x, sh);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&ctrl->e2_counter, 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  apply_tail(A, gridDim.x, sh, ctrl);
}


int e_grid(int64_t m) {
  const int64_t blocks = (m + kEThreads - 1) / kEThreads;
  return static_cast<int>(blocks < 296 ? blocks : 296);
}

}  // namespace

// ---------------------------------------------------------------- launch ---
// Rows per CTA of the fp32 row pass (tuning knob OTG_ROW_R = 1, 4 or 8).
int64_t rows_per_cta_fast(const Problem& P) {
  constexpr int env = OTG_ROW_R;  // (compile-time tuning: 0 = auto)
  // on the fly, 8 rows share each column quad's coordinate / potential loads
  // (cfg5-shaped 100000^2: 5.86 -> 5.38 ms per row pass); stored, 4 rows keep
  // 3 CTAs per SM (8 rows: 65536^2 2.90 -> 4.06 ms)
  const int64_t dflt = P.storage == OTG_STORE_ON_THE_FLY ? 8 : 4;
  const int64_t want = (env == 1 || env == 4 || env == 8) ? env : dflt;
  return P.n_local >= want ? want : 1;
}

// Resident CTAs of the fp32 column pass over the whole GPU.
static int64_t col_slots(const Problem& P) {
  const void* fn = nullptr;
  const bool otf = P.storage == OTG_STORE_ON_THE_FLY;
  switch (P.col_threads) {
    case 512: fn = otf ? (const void*)k_col_fast<true, 512> : (const void*)k_col_fast<false, 512>; break;
    case 256: fn = otf ? (const void*)k_col_fast<true, 256> : (const void*)k_col_fast<false, 256>; break;
    default: fn = otf ? (const void*)k_col_fast<true, 128> : (const void*)k_col_fast<false, 128>;
  }
  int occ = 0, sms = 0;
  OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, P.col_threads, 0));
  OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  return std::max<int64_t>(1, static_cast<int64_t>(occ) * sms);
}

void configure_sweeps(Problem& P) {
  const int online = OTG_ONLINE_FIRST;
  OTG_CUDA(cudaMemcpyToSymbol(c_online_first, &online, sizeof(int)));
  // column-pass split: ~24 CTAs per SM over the grid so the dynamic CTA
  // scheduler balances the 148 SMs (ncu: 640 CTAs = 0.48 waves was
  // latency-bound); partials cost splits * m * 8 B (< 1% of the sweep)
  constexpr int env_t = OTG_COL_T;  // (compile-time tuning: 0 = auto)
  constexpr int env_s = OTG_COL_SPLITS;  // (compile-time tuning: 0 = auto)
  // 256 threads x 4 columns = 4 KB of each cost row per CTA, ~9 CTAs per SM
  // in one wave (tools/col_sweep.py on B200: 2.77 ms = 95% of HBM at
  // 65536^2, vs 3.53 ms for 128-thread CTAs in 2.7 waves)
  P.col_threads = (env_t == 128 || env_t == 256 || env_t == 512) ? env_t : 256;
  const int64_t colblocks =
      P.storage == OTG_STORE_F64 ? (P.m + kColThreads - 1) / kColThreads
                                 : (P.m + 4 * P.col_threads - 1) / (4 * P.col_threads);
  const int64_t shard_rows = (P.n_local + P.vshards - 1) / P.vshards;
  // (<= 64 partial rows: the merge reads every split of every column, so past
  // that the merge costs more than the column grid gains -- cfg2, 8192^2:
  // 92 splits 8.38 K it/s, 64 splits 8.51 K it/s)
  // fp64 (precise exp, latency-bound): small problems need the splits for
  // parallelism -- cfg1, 1000^2: 8 column blocks x 16 splits of 63 rows left
  // half the SMs idle (20.8 us); >= 8 rows per split, <= 256 splits
  const int64_t max_splits =
      P.storage == OTG_STORE_F64
          ? std::max<int64_t>(1, std::min<int64_t>(256, (shard_rows + 7) / 8))
          : std::max<int64_t>(1, std::min<int64_t>(64, (shard_rows + 63) / 64));
  int64_t splits = 1;
  if (env_s > 0) {
    splits = env_s;
  } else if (P.storage == OTG_STORE_F64) {
    splits = (24 * 148 + colblocks - 1) / colblocks;
  } else {
    // fp32: the CTA count is a near-integer number of waves of the resident
    // slots (B200, 65536^2: 1.04 waves 4.19 ms, 1.38 w 3.27 ms, 2.08 w
    // 3.27 ms, 1.99 w 2.59 ms): maximise the fill of the last wave, <= 4 waves
    const int64_t slots = col_slots(P);
    double best = -1.0;
    for (int64_t S = 1; S <= max_splits; ++S) {
      const double waves = static_cast<double>(colblocks * S) / static_cast<double>(slots);
      if (waves > 4.0 && S > 1) break;
      const double fill = waves / std::ceil(waves);
      if (fill > best + 1e-3) {
        best = fill;
        splits = S;
      }
    }
  }
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, max_splits));
  // culled on-the-fly column pass: per-CTA work varies with the geometry, so
  // many more CTAs than slots let the scheduler balance them
  if (P.cull && P.storage == OTG_STORE_ON_THE_FLY && env_s <= 0)
    splits = std::max<int64_t>(1, std::min<int64_t>(OTG_CULL_COL_SPLITS, (shard_rows + 255) / 256));
  P.col_splits = static_cast<int>(splits);
  P.rows_per_split = (shard_rows + splits - 1) / splits;
  if (P.cull) P.rows_per_split = (P.rows_per_split + kCullRB - 1) / kCullRB * kCullRB;  // whole blocks
  // on the fly: the transposed row pass (OTG_ROW_OTF_T=0: row_shift_block).
  // Column splits give ~8 waves of the resident CTAs, >= 256 columns each.
  constexpr int env_rt = OTG_ROW_OTF_T;
  P.row_splits = 0;
  if (P.storage == OTG_STORE_ON_THE_FLY && env_rt != 0) {
    int occ = 0, sms = 0;
    OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_row_otf<true>, kRowThreads, 0));
    OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
    const int64_t rb = (P.n_local + kRowThreads * kOtfRT - 1) / (kRowThreads * kOtfRT);
    const int64_t slots = std::max<int64_t>(1, static_cast<int64_t>(occ) * sms);
    int64_t S = (OTG_CULL_ROW_WAVES * (P.cull ? 1 : 0) + 8 * (P.cull ? 0 : 1)) * slots / rb + 1;
    S = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(S, 128), (P.m + 255) / 256));
    int64_t cps = (P.m + S - 1) / S;
    cps = (cps + kOtfBlk - 1) / kOtfBlk * kOtfBlk;
    if (P.cull) cps = (cps + kCullCB - 1) / kCullCB * kCullCB;  // whole culling blocks
    P.row_cols_per_split = cps;
    P.row_splits = static_cast<int>((P.m + cps - 1) / cps);
  }
  P.e_blocks = e_grid(P.m);
}

static CostSrc cost_src(const Problem& P);
// Test hook (otg_debug_cull): 1 = culled sweeps (default), 0 = the same
// sorted sweeps visiting every block, -1 = handles created from now on keep
// the caller's order (no culling set up).
int& cull_mode() {
  static int mode = 1;
  return mode;
}

// the culled sweeps' view: sorted coordinates, orders, block boxes / bounds
static CostSrc cull_src(const Problem& P) {
  CostSrc s = cost_src(P);
  s.Yn = P.Yns;
  s.perm_r = P.perm_r;
  s.perm_c = P.perm_c;
  s.Xs = reinterpret_cast<const float4*>(P.Xs);
  s.cbox = reinterpret_cast<const float4*>(P.cbox);
  s.cvmax = P.cvmax;
  s.rbox = reinterpret_cast<const float4*>(P.rbox);
  s.rnegm = P.rnegm;
  s.skip = cull_mode() > 0 ? 1 : 0;
  s.ves = reinterpret_cast<const float2*>(P.ves);
  s.auxs = reinterpret_cast<const float4*>(P.auxs);
  return s;
}

static CostSrc cost_src(const Problem& P) {
  CostSrc s;
  s.C = P.C32;
  s.ldc = P.ldc;
  s.X = reinterpret_cast<const float4*>(P.X);
  s.Y = reinterpret_cast<const float4*>(P.Y);
  s.Yn = P.Yn;
  s.ypad = P.mpad;
  s.perm_r = nullptr;
  s.perm_c = nullptr;
  s.Xs = nullptr;
  s.cbox = s.rbox = nullptr;
  s.cvmax = s.rnegm = nullptr;
  s.skip = 0;
  s.ves = nullptr;
  s.auxs = nullptr;
  return s;
}

// threads per row of the fp64 row pass: one warp for short rows, four warps
// up to 16384 columns (cfg1, 1000^2: 2 rows per CTA, 500 CTAs, ~8 exps per
// thread instead of 31), the whole CTA beyond
static int precise_row_group(const Problem& P) {
  return P.m <= 256 ? 32 : P.m <= 16384 ? 128 : kRowThreads;
}

int64_t row_blocks(const Problem& P) {
  if (P.storage == OTG_STORE_F64) {
    const int G = precise_row_group(P);
    const int64_t rpb = kRowThreads / G;
    return (P.n_local + rpb - 1) / rpb;
  }
  const int64_t R = rows_per_cta_fast(P);
  return (P.n_local + R - 1) / R;
}


// Resident CTAs of a grid-stride kernel (capped at `blocks`).
template <typename K>
static unsigned resident_grid(const Problem& P, K kernel, int64_t blocks) {
  int sms = 0, occ = 0;
  OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kRowThreads, 0));
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(blocks, int64_t{sms} * std::max(occ, 1))));
}

void launch_row_pass(Problem& P) {
  const int64_t blocks = row_blocks(P);
  double* rowpart = P.e1_part + (e1_groups_of(P.m) + 1) * 8;  // scratch after the E1 partials
  if (P.storage == OTG_STORE_F64) {
    const int G = precise_row_group(P);
    if (G == 32)
      launch_k(k_row_precise<32>, blocks, kRowThreads, 0, P.stream, 
          P.C64, P.ldc, P.n_local, P.m, P.p, P.a, P.loga, P.rowM, P.rowS, P.u, P.wrow, rowpart,
          P.ctrl);
    else if (G == 128)
      launch_k(k_row_precise<128>, blocks, kRowThreads, 0, P.stream, 
          P.C64, P.ldc, P.n_local, P.m, P.p, P.a, P.loga, P.rowM, P.rowS, P.u, P.wrow, rowpart,
          P.ctrl);
    else
      launch_k(k_row_precise<kRowThreads>, blocks, kRowThreads, 0, P.stream, 
          P.C64, P.ldc, P.n_local, P.m, P.p, P.a, P.loga, P.rowM, P.rowS, P.u, P.wrow, rowpart,
          P.ctrl);
  } else {
    // exact kernel (first evaluation of a solve / one-shots), shift-estimate
    // kernel (steady state), exact redo of the rows the estimate missed; each
    // returns at once when its case does not apply
    const int64_t R = rows_per_cta_fast(P);
    const double k2 = P.kappa * kLog2e;
    const float kh = static_cast<float>(k2);
    const float kl = static_cast<float>(k2 - static_cast<double>(kh));
    const CostSrc src = cost_src(P);
    // L2 prefetch of the cost ahead of the loads (OTG_ROW_PF: 0 off, 1 =
    // L2::256B loads, 3 / 5 = prefetch 2 / 4 chunks ahead).  B200, 65536^2:
    // with the scalar inner loop 3.19 ms (off) -> 2.95 ms (3); with the packed
    // f32x2 loop both take ~2.92 ms (3 CTAs/SM either way), so it is off
    constexpr int row_pf_env = OTG_ROW_PF;  // (compile-time tuning: -1 = auto)
    // cfg2 (8192^2): 70.8 -> 65.7 us with the prefetch; cfg3: equal, so only
    // rows short enough for the per-CTA latency to show get it by default
    const int row_pf = row_pf_env >= 0 ? row_pf_env : (P.m <= 16384 ? 3 : 0);
#define OTG_SHIFT_ARGS                                                                        \
  src, P.n_local, P.m, P.vq, P.dq, P.mpad, kh, kl, P.a, P.loga, P.rowM, P.rowS, P.u, P.wrow,  \
      P.aux, P.rowM2, P.rowJ, P.redo_rows, P.ctrl
#define OTG_ROW(RR, OTF)                                                                      \
  launch_k(k_row_exact<RR, OTF>, resident_grid(P, k_row_exact<RR, OTF>, blocks), kRowThreads, 0,  \
           P.stream,                                                                          \
      src, P.n_local, P.m, P.p, P.kappa, P.a, P.loga, P.rowM, P.rowS, P.u, P.wrow, P.aux,     \
      P.rowM2, P.rowJ, P.ctrl, P.vq, P.mpad);                                                 \
  if (RR == 4 && !OTF && row_pf == 1)                                                         \
    launch_k(k_row_shift<RR, OTF, 1>, blocks, kRowThreads, 0, P.stream, OTG_SHIFT_ARGS);            \
  else if (RR == 4 && !OTF && row_pf == 3)                                                    \
    launch_k(k_row_shift<RR, OTF, 3>, blocks, kRowThreads, 0, P.stream, OTG_SHIFT_ARGS);            \
  else if (RR == 4 && !OTF && row_pf == 5)                                                    \
    launch_k(k_row_shift<RR, OTF, 5>, blocks, kRowThreads, 0, P.stream, OTG_SHIFT_ARGS);            \
  else                                                                                        \
    launch_k(k_row_shift<RR, OTF, 0>, blocks, kRowThreads, 0, P.stream, OTG_SHIFT_ARGS);            \
  launch_k(k_row_redo<OTF>, 296, kRowThreads, 0, P.stream, src, P.m, P.p, P.kappa, P.a, P.loga,     \
                                                     P.rowM, P.rowS, P.u, P.wrow, P.aux,      \
                                                     P.rowM2, P.rowJ, P.redo_rows, P.ctrl)
    const bool otf = P.storage == OTG_STORE_ON_THE_FLY;
    if (P.fused) {
      // exact first evaluation (two-pass), then the single-pass kernel (the
      // steady graph follows an evaluation: no exact-path kernel)
      if (!P.steady_capture)
        launch_k(k_row_exact<4, false>, resident_grid(P, k_row_exact<4, false>, blocks),
                 kRowThreads, 0, P.stream, src, P.n_local, P.m, P.p, P.kappa, P.a, P.loga, P.rowM,
                 P.rowS, P.u, P.wrow, P.aux, P.rowM2, P.rowJ, P.ctrl, P.vq, P.mpad);
      launch_fused(P, kh, kl);
    } else if (otf && P.row_splits > 0 && R == 8) {
      launch_k(k_row_exact<8, true>, resident_grid(P, k_row_exact<8, true>, blocks), kRowThreads, 0,
               P.stream, src, P.n_local, P.m, P.p, P.kappa, P.a, P.loga, P.rowM, P.rowS, P.u,
               P.wrow, P.aux, P.rowM2, P.rowJ, P.ctrl, P.vq, P.mpad);
      RowPart* rp = static_cast<RowPart*>(P.rpart);
      const dim3 g(static_cast<unsigned>((P.n_local + kRowThreads * kOtfRT - 1) / (kRowThreads * kOtfRT)),
                   static_cast<unsigned>(P.row_splits));
      CostSrc fsrc = src;
      if (P.cull) {
        launch_k(k_cull_cols, static_cast<unsigned>((P.m + 8 * kCullCB - 1) / (8 * kCullCB)), 256, 0,
                 P.stream, P.m, P.mpad, static_cast<const float*>(P.vq),
                 static_cast<const int*>(P.perm_c), P.cvmax, reinterpret_cast<float2*>(P.ves),
                 static_cast<const Ctrl*>(P.ctrl));
        const dim3 gc(static_cast<unsigned>((P.n_local + kCullRowT * OTG_CULL_RT - 1) / (kCullRowT * OTG_CULL_RT)),
                      static_cast<unsigned>(P.row_splits));
        launch_k(k_row_otf_cull, gc, kCullRowT, 0, P.stream, cull_src(P), P.n_local, P.m,
                 static_cast<const float*>(P.vq), static_cast<const double*>(P.dq), P.mpad, kh,
                 static_cast<const double*>(P.rowM2), static_cast<const int*>(P.rowJ),
                 P.row_cols_per_split, rp, static_cast<const Ctrl*>(P.ctrl));
        fsrc.perm_c = P.perm_c;  // (the heaviest block's columns, in sorted order)
      } else {
        launch_k(k_row_otf<false>, g, kRowThreads, 0, P.stream, src, P.n_local, P.m,
                 static_cast<const float*>(P.vq), static_cast<const double*>(P.dq), P.mpad, kh, kl,
                 static_cast<const double*>(P.rowM2), static_cast<const int*>(P.rowJ),
                 P.row_cols_per_split, rp, static_cast<const Ctrl*>(P.ctrl));
      }
      launch_k(k_row_otf_fin, static_cast<unsigned>((P.n_local + kRowThreads - 1) / kRowThreads),
               kRowThreads, 0, P.stream, fsrc, P.n_local, P.m, static_cast<const float*>(P.vq),
               static_cast<const double*>(P.dq), P.mpad, kh, kl, static_cast<const double*>(P.a),
               static_cast<const double*>(P.loga), P.rowM, P.rowS, P.u, P.wrow, P.aux, P.rowM2,
               P.rowJ, P.redo_rows, static_cast<const RowPart*>(rp), P.row_splits, P.ctrl);
      launch_k(k_row_redo<true>, 296, kRowThreads, 0, P.stream, src, P.m, P.p, P.kappa, P.a,
               P.loga, P.rowM, P.rowS, P.u, P.wrow, P.aux, P.rowM2, P.rowJ, P.redo_rows, P.ctrl);
    } else if (R == 8) {
      if (otf) { OTG_ROW(8, true); } else { OTG_ROW(8, false); }
    } else if (R == 4) {
      if (otf) { OTG_ROW(4, true); } else { OTG_ROW(4, false); }
    } else {
      if (otf) { OTG_ROW(1, true); } else { OTG_ROW(1, false); }
    }
#undef OTG_ROW
#undef OTG_SHIFT_ARGS
  }
  OTG_CUDA(cudaGetLastError());
}

void launch_col_pass(Problem& P) {
  const int64_t shard_rows = (P.n_local + P.vshards - 1) / P.vshards;
  const double k2 = P.kappa * kLog2e;
  const float kh = static_cast<float>(k2);
  const float kl = static_cast<float>(k2 - static_cast<double>(kh));
  if (P.fused && P.steady_capture) return;  // the single pass did the columns
  for (int s = 0; s < P.vshards; ++s) {
    const int64_t lo = s * shard_rows, hi = std::min(P.n_local, lo + shard_rows);
    double* part = P.part + static_cast<int64_t>(s) * P.col_splits * P.mpad;
    if (P.storage == OTG_STORE_F64) {
      dim3 grid(static_cast<unsigned>((P.m + kColThreads - 1) / kColThreads), P.col_splits);
      launch_k(k_col_precise, grid, kColThreads, 0, P.stream, P.C64, P.ldc, P.m, P.p, P.rowM, P.wrow,
                                                        lo, hi, P.rows_per_split, part, P.mpad,
                                                        P.ctrl);
    } else {
      const int NT = P.col_threads;
      dim3 grid(static_cast<unsigned>((P.m + 4 * NT - 1) / (4 * NT)), P.col_splits);
#define OTG_COL(OTF, T)                                                                      \
  launch_k(k_col_fast<OTF, T>, grid, T, 0, P.stream, cost_src(P), P.m, P.p, kh, kl, P.aux, lo, hi, \
                                               P.rows_per_split, part, P.mpad, P.ctrl, P.fused)
      const bool otf = P.storage == OTG_STORE_ON_THE_FLY;
      if (otf && P.cull && P.vshards == 1 && NT == 256) {
        // culled on-the-fly column pass (sorted rows / columns, exact skips)
        launch_k(k_cull_rows, static_cast<unsigned>((P.n_local + 16 * kCullRB - 1) / (16 * kCullRB)),
                 256, 0, P.stream, P.n_local, static_cast<const float4*>(P.aux),
                 static_cast<const int*>(P.perm_r), P.rnegm, reinterpret_cast<float4*>(P.auxs),
                 static_cast<const Ctrl*>(P.ctrl));
        const dim3 gcc(static_cast<unsigned>((P.m + 4 * kCullColT - 1) / (4 * kCullColT)), P.col_splits);
        launch_k(k_col_otf_cull, gcc, kCullColT, 0, P.stream, cull_src(P), P.m, P.p, kh, P.aux, lo, hi,
                 P.rows_per_split, part, P.mpad, P.ctrl);
      } else if (NT == 512) {
        if (otf) { OTG_COL(true, 512); } else { OTG_COL(false, 512); }
      } else if (NT == 256) {
        if (otf) { OTG_COL(true, 256); } else { OTG_COL(false, 256); }
      } else {
        if (otf) { OTG_COL(true, 128); } else { OTG_COL(false, 128); }
      }
#undef OTG_COL
    }
  }
  OTG_CUDA(cudaGetLastError());
}

void launch_split_p(Problem& P) {
  if (P.storage == OTG_STORE_F64) return;
  const unsigned g = static_cast<unsigned>(std::min<int64_t>((P.m + 255) / 256, 1184));
  launch_k(k_split_p, g, 256, 0, P.stream, P.m, P.mpad, P.p, P.vq);
}

void launch_sp_redo(Problem& P, const int* bad_rows, const int* bad_count, int ncl, int64_t cap) {
  launch_k(k_sp_redo, 148, kRowThreads, 0, P.stream, cost_src(P), P.n_local, P.m, P.p, P.kappa, P.a,
                                                P.loga, P.rowM, P.rowS, P.u, P.wrow, P.aux,
                                                P.rowM2, P.rowJ, bad_rows, bad_count, ncl, cap,
                                                static_cast<const unsigned*>(P.sp_cnt + 2), P.ctrl);
}

int64_t merge_blocks(const Problem& P);

// Unsharded single pass, steady state: column j's patch (the rows the pass
// listed as loose, in list order -- k_sp_patch's formula), then the merge of
// the H group rows + that patch row with merge_body's 8-chain tree (bitwise
// the k_merge result), the underflow flag and <u, a> slice blk: one kernel
// instead of k_sp_patch + k_merge.
__global__ void __launch_bounds__(kEThreads)
k_sp_patch_merge(const float* __restrict__ C, int64_t ldc, int64_t m, int64_t mpad,
                 const double* __restrict__ p, float kh, float kl, const float4* __restrict__ aux,
                 const int* __restrict__ bad_rows, const int* __restrict__ bad_count, int nlists,
                 int64_t cap, const unsigned* __restrict__ total, double* __restrict__ part, int H,
                 double* __restrict__ col, double* __restrict__ col_log, int* __restrict__ flag_idx,
                 int* __restrict__ fb_cols, const double* __restrict__ u,
                 const double* __restrict__ a, int64_t nrows, int ua_n, const FinArgs F,
                 int fin_fuse, Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  __shared__ double sh[kEThreads / 32 * 8];
  __shared__ bool last;
  const int blk = blockIdx.x;
  if (blk < ua_n) {  // <u, a> over row slice blk of ua_n (as merge_body)
    const int64_t r0 = nrows * blk / ua_n, r1 = nrows * (blk + 1) / ua_n;
    double t = 0.0;
    for (int64_t k = r0 + threadIdx.x; k < r1; k += kEThreads) t += u[k] * a[k];
    t = block_sum<kEThreads>(t, sh);
    if (threadIdx.x == 0) col[mpad + 1 + blk] = t;
  }
  const int64_t j = static_cast<int64_t>(blk) * kEThreads + threadIdx.x;
  E1Acc e;
  if (j < m) {
    double patch = 0.0;
    if (*total != 0u) {
      const double x2 = p[j] * kLog2e;
      const double h = rint(x2 * 256.0) * (1.0 / 256.0);
      const float Vc = static_cast<float>(h), vf = static_cast<float>(x2 - h);
      for (int c = 0; c < nlists; ++c) {
        const int nbad = bad_count[c];
        for (int q = 0; q < nbad; ++q) {
          const int64_t i = bad_rows[c * cap + q];
          const float4 ax = aux[i];
          const float cc = C[i * ldc + j];
          const float Aq = Vc - ax.x;
          const float gq = fmaf(-cc, kl, vf - ax.y);
          const float tt = fmaf(-cc, kh, Aq) + gq;
          patch += static_cast<double>(ax.z * ex2_approx(tt));
        }
      }
    }
    part[static_cast<int64_t>(H) * mpad + j] = patch;
    double l[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < H; ++k) l[k & 7] += part[static_cast<int64_t>(k) * mpad + j];
    l[H & 7] += patch;
    const double c = 0.0 + (((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7])));
    col[j] = c;
    if (c >= ctrl->tiny) {
      col_log[j] = log(c);
      flag_idx[j] = -1;
      // steady graph: finalize the column now (flagged columns wait for the
      // exact LSE: k_finalize then redoes the whole evaluation's finalize)
      if (fin_fuse) finalize_col(F, j, -1, e);
    } else {
      const unsigned slot = atomicAdd(&ctrl->fb_count, 1u);
      fb_cols[slot] = static_cast<int>(j);
      flag_idx[j] = static_cast<int>(slot);
    }
  }
  if (!fin_fuse) return;
  // the E1 partials of this CTA's 32-column groups (one per warp); the last
  // CTA runs the solver's control step unless a column was flagged (then
  // k_finalize does it all)
  store_e1_warp(F, static_cast<int64_t>(blk) * (kEThreads / 32) + (threadIdx.x >> 5), e);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ctrl->e1_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (*reinterpret_cast<volatile unsigned*>(&ctrl->fb_count) != 0u) {
    // underflowed columns need the exact column LSE: pause the chunk (every
    // later kernel of it returns); the host finishes this evaluation eagerly
    // (k_finalize with the fallback, k_apply) and keeps replaying
    if (threadIdx.x == 0) {
      ctrl->e1_counter = 0;
      ctrl->done = kPaused;
    }
    return;
  }
  finalize_tail<kEThreads>(F, static_cast<int>(e1_groups_of(m)), sh, ctrl);
  if (threadIdx.x == 0) ctrl->fin_done = 1;
}

static FinArgs fin_args(const Problem& P, int64_t ua_slices);

void launch_sp_patch_merge(Problem& P, float kh, float kl, int nlists) {
  const unsigned g = static_cast<unsigned>(merge_blocks(P));
  // the finalize folds in only in the steady graph, with k_finalize's own
  // column partition (one 256-column work unit per CTA)
  const int fin_fuse = P.capturing ? 1 : 0;
  launch_k(k_sp_patch_merge, g, kEThreads, 0, P.stream, static_cast<const float*>(P.C32), P.ldc,
           P.m, P.mpad, static_cast<const double*>(P.p), kh, kl,
           static_cast<const float4*>(P.aux), static_cast<const int*>(P.sp_bad_rows),
           static_cast<const int*>(P.sp_bad_count), nlists, P.sp_cap,
           static_cast<const unsigned*>(P.sp_cnt + 2), P.part, P.fused_clusters, P.col, P.col_log,
           P.flag_idx, P.fb_cols, static_cast<const double*>(P.u),
           static_cast<const double*>(P.a), P.n_local, static_cast<int>(merge_blocks(P)),
           fin_args(P, merge_blocks(P)), fin_fuse, P.ctrl);
}

int partial_rows(const Problem& P) { return P.vshards * P.col_splits; }

int64_t merge_blocks(const Problem& P) { return (P.m + kEThreads - 1) / kEThreads; }

// k_merge CTAs: 32 columns each (<u, a> slices: the first merge_blocks(P))
static unsigned merge_grid(const Problem& P) { return static_cast<unsigned>((P.m + 31) / 32); }

static FinArgs fin_args(const Problem& P, int64_t ua_slices);

static void launch_merge(Problem& P, bool merge, bool flag) {
  const unsigned blocks = merge_grid(P);
  const int shards = P.vshards;
  const int splits = P.col_splits;
  if (merge && flag && P.capturing && !P.sharded && P.vshards == 1) {
    launch_k(k_merge_fin, blocks, kEThreads, 0, P.stream, P.part, splits, P.m, P.mpad, P.col,
             P.col_log, P.flag_idx, P.fb_cols, static_cast<const double*>(P.u),
             static_cast<const double*>(P.a), P.n_local, P.ctrl,
             P.fused ? P.fused_clusters + 1 : 0, static_cast<int>(merge_blocks(P)),
             patch_merges(P) ? 1 : 0, fin_args(P, merge_blocks(P)));
    OTG_CUDA(cudaGetLastError());
    return;
  }
  launch_k(k_merge, blocks, kEThreads, 0, P.stream, P.part, shards, splits, P.m, P.mpad, P.col,
                                              P.col_log, P.flag_idx, P.fb_cols, P.u, P.a,
                                              P.n_local, merge ? 1 : 0, flag ? 1 : 0, P.ctrl,
                                              P.fused ? P.fused_clusters + 1 : 0,
                                              static_cast<int>(merge_blocks(P)),
                                              patch_merges(P) ? 1 : 0);
  OTG_CUDA(cudaGetLastError());
}

void launch_merge_nolog(Problem& P) { launch_merge(P, true, false); }

// Local merge (no flagging) into `dst` (the sharded all-reduce's send buffer).
static void launch_merge_into(Problem& P, double* dst) {
  launch_k(k_merge, merge_grid(P), kEThreads, 0, P.stream, P.part, P.vshards, P.col_splits,
           P.m, P.mpad, dst, P.col_log, P.flag_idx, P.fb_cols, P.u, P.a, P.n_local, 1, 0,
           P.ctrl, P.fused ? P.fused_clusters + 1 : 0, static_cast<int>(merge_blocks(P)), 0);
  OTG_CUDA(cudaGetLastError());
}

// Event records are "external" so that, under stream capture, they become
// event-record nodes of the chunk graph (timestamps readable after replay).
static void mark(Problem& P, cudaEvent_t e) {
  OTG_CUDA(cudaEventRecordWithFlags(e, P.stream, cudaEventRecordExternal));
}

// Both O(nm) passes: the fused single-HBM-pass kernel when the handle has one
// (fp32 storage, m <= 65536), else the row pass then the column pass.
void launch_sweeps(Problem& P, bool timed, cudaEvent_t* ev4) {
  if (timed) mark(P, ev4[0]);
  launch_row_pass(P);
  if (timed) mark(P, ev4[1]);
  if (timed) mark(P, ev4[2]);
  launch_col_pass(P);
  if (timed) mark(P, ev4[3]);
}

static FinArgs fin_args(const Problem& P, int64_t ua_slices) {
  FinArgs A;
  A.m = P.m;
  A.mpad = P.mpad;
  A.p = P.p;
  A.b = P.b;
  A.logb = P.logb;
  A.col = P.col;
  A.col_log = P.col_log;
  A.flag_idx = P.flag_idx;
  A.fb_part = P.fb_part;
  A.fbA = P.fbA;
  A.fbS = P.fbS;
  A.sharded = P.sharded;
  A.ua_slices = static_cast<int>(ua_slices);
  A.y = P.y;
  A.grad = P.grad;
  A.e1_part = P.e1_part;
  A.trace = P.trace;
  A.bounds = P.bounds;
  A.fold_fb = P.sharded ? 0 : 1;
  A.storage = P.storage;
  A.C64 = P.C64;
  A.src = cost_src(P);
  A.ldc = P.ldc;
  A.nrows = P.n_local;
  A.kappa = P.kappa;
  A.u = P.u;
  A.fb_cols = P.fb_cols;
  A.fb_part_w = P.fb_part;
  return A;
}

static AppArgs app_args(const Problem& P) {
  AppArgs A;
  A.m = P.m;
  A.mpad = P.mpad;
  A.b = P.b;
  A.p = P.p;
  A.wacc = P.wacc;
  A.y = P.y;
  A.grad = P.grad;
  A.prev_grad = P.prev_grad;
  A.prev_x = P.prev_x;
  A.prev_y = P.prev_y;
  A.vq = P.vq;
  A.dq = P.dq;
  A.fast = P.storage != OTG_STORE_F64;  // fp32 stored or on the fly: shift estimate
  A.e2_part = P.e2_part;
  A.trace = P.trace;
  A.vstar = P.vstar;
  A.bounds = P.bounds;
  return A;
}

// CTAs of the single-kernel epilogue (co-resident: <= one per SM), 0 = off.
void launch_eval(Problem& P, bool with_log, bool timed, cudaEvent_t* ev4) {
  P.apply_pending = 0;
  launch_sweeps(P, timed, ev4);
  if (P.sharded) {
    // local merge into `red`, then THE collective of the evaluation: one
    // out-of-place all-reduce of the m column sums + <u, a> slices into col
    // (re-running it on unchanged `red` rewrites identical bytes, which the
    // paused chunk below relies on); the underflow test needs the global
    // sums, so flagging follows the reduce and is identical on every rank
    launch_merge_into(P, P.red);
    comm_allreduce_sum(P, P.red, P.col, static_cast<size_t>(P.mpad + 1 + merge_blocks(P)));
    if (with_log) launch_merge(P, false, true);
    if (with_log && P.capturing) {
      // inside the chunk graph: an evaluation that flags columns pauses the
      // chunk (ctrl->done = kPaused; every later kernel of the chunk returns)
      // and the host runs its cross-rank exact-LSE exchange eagerly
      // (resume_paused_eval) -- the steady state has no second collective
      launch_k(k_pause_if_flagged, 1, 32, 0, P.stream, P.ctrl);
      launch_k(k_finalize, P.e_blocks, kEThreads, 0, P.stream, fin_args(P, merge_blocks(P)),
               P.ctrl);
      OTG_CUDA(cudaGetLastError());
      P.apply_pending = 1;
      return;
    }
  } else if (!(P.steady_capture && patch_merges(P))) {
    launch_merge(P, true, with_log);
  }
  if (!with_log) return;
  launch_fallback_and_finalize(P);
}

// The rest of an evaluation after the flagging merge: the exact column LSE
// of flagged columns (sharded: local (top, sum) per column, MAX then SUM
// all-reduce), then finalize.
void launch_fallback_and_finalize(Problem& P) {
  if (!P.sharded && P.capturing && P.vshards == 1) {
    // the merge kernel (k_merge_fin / k_sp_patch_merge) finalizes every
    // captured evaluation; one with underflowed columns pauses the chunk and
    // the host runs this function eagerly (P.capturing = 0) for it
    P.apply_pending = 1;
    return;
  }
  if (!P.sharded) {
    // K5 runs inside k_finalize (fin_args: fold_fb) -- no separate launch
    launch_k(k_finalize, P.e_blocks, kEThreads, 0, P.stream, fin_args(P, merge_blocks(P)), P.ctrl);
    OTG_CUDA(cudaGetLastError());
    P.apply_pending = 1;
    return;
  }
  if (P.storage == OTG_STORE_F64)
    launch_k(k_fallback<true, false>, 296, kEThreads, 0, P.stream, 
        P.C64, cost_src(P), P.ldc, P.n_local, P.kappa, P.u, P.p, P.fb_cols, P.fb_part, P.ctrl);
  else if (P.storage == OTG_STORE_ON_THE_FLY)
    launch_k(k_fallback<false, true>, 296, kEThreads, 0, P.stream, 
        nullptr, cost_src(P), P.ldc, P.n_local, P.kappa, P.u, P.p, P.fb_cols, P.fb_part, P.ctrl);
  else
    launch_k(k_fallback<false, false>, 296, kEThreads, 0, P.stream, 
        nullptr, cost_src(P), P.ldc, P.n_local, P.kappa, P.u, P.p, P.fb_cols, P.fb_part, P.ctrl);
  OTG_CUDA(cudaGetLastError());
  if (P.sharded) {
    // exact column LSE across ranks: local (top, sum) per flagged column,
    // MAX all-reduce of the tops, rescale, SUM all-reduce of the sums
    const unsigned g = static_cast<unsigned>((P.m + kEThreads - 1) / kEThreads);
    launch_k(k_fb_local, g, kEThreads, 0, P.stream, P.m, P.flag_idx, P.fb_part, P.fbA, P.fbS, P.fbT,
                                              P.ctrl);
    comm_allreduce_max(P, P.fbA, static_cast<size_t>(P.m));
    launch_k(k_fb_rescale, g, kEThreads, 0, P.stream, P.m, P.flag_idx, P.fbA, P.fbS, P.fbT, P.ctrl);
    comm_allreduce_sum(P, P.fbS, static_cast<size_t>(P.m));
    OTG_CUDA(cudaGetLastError());
  }
  launch_k(k_finalize, P.e_blocks, kEThreads, 0, P.stream, fin_args(P, merge_blocks(P)), P.ctrl);
  OTG_CUDA(cudaGetLastError());
  P.apply_pending = 1;
}

void launch_apply(Problem& P) {
  if (!P.apply_pending) return;  // done inside the single-kernel epilogue
  launch_k(k_apply, P.e_blocks, kEThreads, 0, P.stream, app_args(P), P.ctrl);
  OTG_CUDA(cudaGetLastError());
}

int64_t rowpart_len(const Problem& P) { return row_blocks(P); }

}  // namespace otg

extern "C" int otg_debug_cull(int mode) {
  const int prev = otg::cull_mode();
  otg::cull_mode() = mode;
  return prev;
}

extern "C" otg_status otg_cull_stats(otg_problem h, double out[2]) {
  using namespace otg;
  return guard([&] {
    if (!out) fail(OTG_E_DIMENSION, "out is NULL");
    if (!h) fail(OTG_E_DIMENSION, "NULL problem handle");
    Problem& P = h->P;
    OTG_CUDA(cudaSetDevice(P.device));
    out[0] = out[1] = -1.0;
    if (!P.cull) return;
    // (the bound reads the rows' last base-2 max and argmax column: zeroed at
    // allocation, so a never-evaluated handle gives a harmless statistic)
    const int64_t n = P.n_local, m = P.m;
    float *nS = nullptr, *Vc = nullptr;
    float4* Ys = nullptr;
    unsigned long long* kept = nullptr;
    OTG_CUDA(cudaMalloc(&nS, n * sizeof(float)));
    OTG_CUDA(cudaMalloc(&Vc, m * sizeof(float)));
    OTG_CUDA(cudaMalloc(&Ys, m * sizeof(float4)));
    OTG_CUDA(cudaMalloc(&kept, 2 * sizeof(unsigned long long)));
    OTG_CUDA(cudaMemsetAsync(kept, 0, 2 * sizeof(unsigned long long), P.stream));
    const int64_t big = std::max(n, m);
    k_cull_prep<<<static_cast<unsigned>((big + 255) / 256), 256, 0, P.stream>>>(
        n, m, P.perm_r, P.perm_c, static_cast<const double*>(P.rowM2),
        static_cast<const int*>(P.rowJ), static_cast<const double*>(P.dq), P.p, P.Yns, P.mpad,
        static_cast<const Ctrl*>(P.ctrl), nS, Vc, Ys);
    k_cull_cols<<<static_cast<unsigned>((m + 8 * kCullCB - 1) / (8 * kCullCB)), 256, 0, P.stream>>>(
        m, P.mpad, static_cast<const float*>(P.vq), P.perm_c, P.cvmax, nullptr,
        static_cast<const Ctrl*>(P.ctrl));
    k_cull_rows<<<static_cast<unsigned>((n + 16 * kCullRB - 1) / (16 * kCullRB)), 256, 0, P.stream>>>(
        n, static_cast<const float4*>(P.aux), P.perm_r, P.rnegm, nullptr,
        static_cast<const Ctrl*>(P.ctrl));
    const float kh = static_cast<float>(P.kappa * kLog2e);
    const float kcull = kh * kCullSlack;
    const int64_t rt = 32 * OTG_CULL_RT, cbn = (m + kCullCB - 1) / kCullCB;
    const int64_t rp = ((n + rt - 1) / rt) * cbn;
    k_cull_stat<<<static_cast<unsigned>((rp + 255) / 256), 256, 0, P.stream>>>(
        n, reinterpret_cast<const float4*>(P.Xs), nS, static_cast<int>(rt),
        reinterpret_cast<const float4*>(P.cbox), P.cvmax, cbn, kcull, kept);
    const int64_t ct = 128, rbn = (n + kCullRB - 1) / kCullRB;
    const int64_t cp = ((m + ct - 1) / ct) * rbn;
    k_cull_stat<<<static_cast<unsigned>((cp + 255) / 256), 256, 0, P.stream>>>(
        m, Ys, Vc, static_cast<int>(ct), reinterpret_cast<const float4*>(P.rbox), P.rnegm, rbn,
        kcull, kept + 1);
    unsigned long long hk[2] = {0, 0};
    OTG_CUDA(cudaMemcpyAsync(hk, kept, sizeof hk, cudaMemcpyDeviceToHost, P.stream));
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    cudaFree(nS);
    cudaFree(Vc);
    cudaFree(Ys);
    cudaFree(kept);
    out[0] = static_cast<double>(hk[0]) / static_cast<double>(rp);
    out[1] = static_cast<double>(hk[1]) / static_cast<double>(cp);
  });
}
