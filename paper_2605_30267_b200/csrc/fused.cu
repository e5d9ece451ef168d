// fused.cu — single-HBM-pass evaluation sweep for fp32 stored costs (sm_100a).
//
// One evaluation needs, per row i, the row statistics (max M_i, sum S_i of
// exp(p_j - C'_ij - M_i)) BEFORE the row can contribute w_i exp(...) to the
// column sums (dual.cpp:34-41).  A 65536-wide fp32 row is 256 KB, more than
// one SM's shared memory, so the two-pass kernels of sweep.cu read the cost
// twice.  Here a cluster of kCL = 8 CTAs (one per SM) holds a whole row on
// chip, each CTA a W = m/8 column slice, and the cost is read from HBM once:
//
//   TMA      cp.async.bulk of the CTA's 32 KB row slice into a 6-slot smem
//            ring (mbarrier complete_tx), 3 rows ahead of use
//   pass A   rough row max from the slot: fmaf(-C, kappa2_hi, Vc_j) (2 ops/elem)
//   pass B   exact exponents relative to the quantised cluster-wide max
//            (all-fp32 exact cancellation, see sweep.cu), MUFU ex2, row sum;
//            e_ij written back into the slot
//   column   acc_j += w_i e_ij in fp32, flushed to fp64 registers every 16
//            rows; the CTA owns its 8192 columns for its cluster's whole row
//            range, so column partials never leave the SM until the end
//   exchange per row one cluster barrier (arrive / wait split around the
//            column step): CTA partials of (row max, row sum) in smem, read by
//            every CTA over DSMEM (mapa + ld.shared::cluster)
//
// Rows are software-pipelined three deep: iteration k runs pass A on row k,
// pass B on row k-1 (its max arrived at the end of iteration k-1) and the
// column step on row k-2 (its sum arrived at the end of iteration k-1).
//
// Output: per-cluster column partials part[cluster][j] (merged by k_merge like
// the column-split partials of the two-pass path), u, rowM, rowS, wrow, and
// the per-cluster <u, a> partial.
#include <cuda_runtime.h>

#include <cfloat>

#include "common.cuh"

namespace otg {

namespace {

constexpr int kCL = 8;         // CTAs per cluster (one row across the cluster)
constexpr int kFT = 512;       // threads per CTA
constexpr int kFW = kFT / 32;  // warps per CTA
constexpr int kSlotsMax = 16;
constexpr int kSmemBudget = 227 * 1024 - 2048;  // bytes of row slots per CTA

constexpr int kXD = 4;  // exchange ring depth (2 suffice: see the flow argument below)

struct XMsg {  // one CTA's partials for one iteration, pushed by st.async
  uint32_t max_bits;
  uint32_t pad;
  uint64_t sum_bits;
};

struct FusedShared {
  uint64_t full[kSlotsMax];  // TMA completion barriers
  uint64_t xbar[kXD];        // exchange barriers (8 messages of 12 bytes each)
  XMsg xin[kXD][kCL];        // partials received from every CTA of the cluster
  float wmax[2][kFW];        // warp partial max of the pass-A row
  double wsum[2][kFW];       // warp partial sum of the pass-B row
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Remote smem store that completes `bytes` on the remote mbarrier (DSMEM push).
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(
                   raddr),
               "r"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_u64(uint32_t raddr, uint64_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "l"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void split_q(double x2, float& hi, float& lo) {
  const double h = rint(x2 * 256.0) * (1.0 / 256.0);
  hi = static_cast<float>(h);
  lo = static_cast<float>(x2 - h);
}

template <int QPT>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kFT, 1)
k_fused(const float* __restrict__ C, int64_t ldc, int64_t n, int64_t m, int W, int nslots,
        const double* __restrict__ p, float kh, float kl, const double* __restrict__ a,
        const double* __restrict__ loga, double* __restrict__ rowM, double* __restrict__ rowS,
        double* __restrict__ u, double* __restrict__ wrow, double* __restrict__ part,
        int64_t mpad, double* __restrict__ rowpart, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;  // uniform over the grid: no cluster barrier is skipped unevenly
  extern __shared__ __align__(128) unsigned char smem_raw[];
  FusedShared& S = *reinterpret_cast<FusedShared*>(smem_raw);
  float* slots = reinterpret_cast<float*>(smem_raw + ((sizeof(FusedShared) + 127) / 128) * 128);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int64_t cid = blockIdx.x / kCL, ncl = gridDim.x / kCL;
  const int64_t r0 = n * cid / ncl, r1 = n * (cid + 1) / ncl;
  const int R = static_cast<int>(r1 - r0);
  const int64_t col0 = static_cast<int64_t>(rank) * W;
  const uint32_t slot_bytes = static_cast<uint32_t>(W) * 4u;

  // column potentials of my quads, base-2, quantised split (pad columns -> -1e30)
  float Vc[QPT][4], vf[QPT][4];
  bool qvalid[QPT];
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    const int q = tid + k * kFT;
    qvalid[k] = 4 * q < W;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t j = col0 + 4 * q + e;
      if (qvalid[k] && j < m) {
        split_q(p[j] * kLog2e, Vc[k][e], vf[k][e]);
      } else {
        Vc[k][e] = -1e30f;
        vf[k][e] = 0.f;
      }
    }
  }
  float acc[QPT][4];
  double acc64[QPT][4];
#pragma unroll
  for (int k = 0; k < QPT; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[k][e] = 0.f;
      acc64[k][e] = 0.0;
    }

  if (tid == 0) {
    for (int s = 0; s < nslots; ++s) mbar_init(&S.full[s], 1);
    for (int s = 0; s < kXD; ++s) mbar_init(&S.xbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int pre = R < nslots ? R : nslots;
    for (int k = 0; k < pre; ++k) {
      mbar_expect_tx(&S.full[k], slot_bytes);
      bulk_load(slots + static_cast<size_t>(k) * W, C + (r0 + k) * ldc + col0, slot_bytes,
                &S.full[k]);
    }
  }
  __syncthreads();
  cluster_arrive();  // every CTA of the cluster is resident before any DSMEM access
  cluster_wait();

  // Pipeline with a one-iteration lag between publishing and consuming the
  // cluster partials, so the DSMEM exchange latency is hidden behind a whole
  // iteration of work.  Iteration k:
  //   pass A  row k      (rough max)                     -> publish max(k)
  //   pass B  row k-2    (needs max(k-2): received at the end of k-1)
  //                                                      -> publish sum(k-2)
  //   column  row k-4    (needs sum(k-4): received at the end of k-1)
  //   receive the messages of iteration k-1: max(k-1), sum(k-3)
  // Row r lives in slot r % nslots from its load until its column step at
  // iteration r + 4; the slot is refilled at iteration r + 5 with row
  // r + nslots (nslots >= 7 keeps 2 rows of prefetch in flight).
  float shiftB = 0.f;      // shift of row k-2 (pass B this iteration)
  float shiftH[4] = {0.f, 0.f, 0.f, 0.f};  // shift used for row r, by r & 3
  float wC = 0.f;          // w of row k-4 (column step this iteration)
  int flush = 0;
  double ua = 0.0;
  const int K = R + 4;

  for (int k = 0; k <= K; ++k) {
    // ---- pass A: rough max of row k ----
    float tmax = -FLT_MAX;
    if (k < R) {
      const int s = k % nslots;
      mbar_wait(&S.full[s], (k / nslots) & 1);
      const float4* slot = reinterpret_cast<const float4*>(slots + static_cast<size_t>(s) * W);
#pragma unroll
      for (int q = 0; q < QPT; ++q) {
        if (!qvalid[q]) continue;
        const float4 c = slot[tid + q * kFT];
        tmax = fmaxf(tmax, fmaxf(fmaxf(fmaf(-c.x, kh, Vc[q][0]), fmaf(-c.y, kh, Vc[q][1])),
                                 fmaxf(fmaf(-c.z, kh, Vc[q][2]), fmaf(-c.w, kh, Vc[q][3]))));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if (lane == 0) S.wmax[k & 1][warp] = tmax;

    // ---- pass B: exact exponents of row k-2 relative to its cluster max ----
    double bsum = 0.0;
    const int rb = k - 2;
    if (rb >= 0 && rb < R) {
      const int s = rb % nslots;
      float4* slot = reinterpret_cast<float4*>(slots + static_cast<size_t>(s) * W);
      float fs = 0.f;
#pragma unroll
      for (int q = 0; q < QPT; ++q) {
        if (!qvalid[q]) continue;
        const float4 c = slot[tid + q * kFT];
        const float cc[4] = {c.x, c.y, c.z, c.w};
        float ev[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float A = Vc[q][e] - shiftB;  // exact (multiples of 2^-8)
          const float g = fmaf(-cc[e], kl, vf[q][e]);
          const float t = fmaf(-cc[e], kh, A) + g;
          ev[e] = ex2_approx(t);
          fs += ev[e];
        }
        slot[tid + q * kFT] = make_float4(ev[0], ev[1], ev[2], ev[3]);
      }
      bsum = static_cast<double>(fs);
      shiftH[rb & 3] = shiftB;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    if (lane == 0) S.wsum[k & 1][warp] = bsum;
    __syncthreads();

    // ---- publish {max(k), sum(k-2)} to every CTA of the cluster ----
    // st.async pushes 12 bytes into slot k % kXD of each CTA and completes them
    // on that CTA's exchange mbarrier.  Flow control: a CTA reaches iteration
    // k + kXD only after receiving every message of iteration k + kXD - 2, so
    // all CTAs are past iteration k + 1, where slot k % kXD was consumed.
    const int xs = k % kXD;
    if (warp == 0 && k < K) {  // the last iteration only receives
      float cm = lane < kFW ? S.wmax[k & 1][lane] : -FLT_MAX;
      double cs = lane < kFW ? S.wsum[k & 1][lane] : 0.0;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        cs += __shfl_xor_sync(0xffffffffu, cs, o);
      }
      if (lane == 0) mbar_expect_tx(&S.xbar[xs], kCL * 12u);  // my arrival on slot xs
      if (lane < kCL) {
        uint32_t ra, rbar;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(ra)
                     : "r"(smem_u32(&S.xin[xs][rank])), "r"(static_cast<uint32_t>(lane)));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(rbar)
                     : "r"(smem_u32(&S.xbar[xs])), "r"(static_cast<uint32_t>(lane)));
        cm = __shfl_sync(0x000000ffu, cm, 0, 8);
        cs = __shfl_sync(0x000000ffu, cs, 0, 8);
        st_async_u32(ra, __float_as_uint(cm), rbar);
        st_async_u64(ra + 8, static_cast<uint64_t>(__double_as_longlong(cs)), rbar);
      }
      // refill the slot of row k-5 (its column step ran in iteration k-1 and every
      // thread passed the barrier above since) with row k-5+nslots
      const int kr = k - 5;
      if (lane == 0 && kr >= 0 && kr + nslots < R) {
        const int s = kr % nslots;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&S.full[s], slot_bytes);
        bulk_load(slots + static_cast<size_t>(s) * W, C + (r0 + kr + nslots) * ldc + col0,
                  slot_bytes, &S.full[s]);
      }
    }

    // ---- column step: row k-4 ----
    const int rc = k - 4;
    if (rc >= 0 && rc < R) {
      const int s = rc % nslots;
      const float4* slot = reinterpret_cast<const float4*>(slots + static_cast<size_t>(s) * W);
#pragma unroll
      for (int q = 0; q < QPT; ++q) {
        if (!qvalid[q]) continue;
        const float4 ev = slot[tid + q * kFT];
        acc[q][0] = fmaf(wC, ev.x, acc[q][0]);
        acc[q][1] = fmaf(wC, ev.y, acc[q][1]);
        acc[q][2] = fmaf(wC, ev.z, acc[q][2]);
        acc[q][3] = fmaf(wC, ev.w, acc[q][3]);
      }
      if (++flush == 16) {
        flush = 0;
#pragma unroll
        for (int q = 0; q < QPT; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc64[q][e] += static_cast<double>(acc[q][e]);
            acc[q][e] = 0.f;
          }
      }
    }

    // ---- receive iteration k-1: max(k-1), sum(k-3) ----
    if (k >= 1) {
      const int ps = (k - 1) % kXD;
      mbar_wait(&S.xbar[ps], ((k - 1) / kXD) & 1);
      float gmax = -FLT_MAX;
      double gsum = 0.0;
      if (lane < kCL) {
        gmax = __uint_as_float(S.xin[ps][lane].max_bits);
        gsum = __longlong_as_double(static_cast<long long>(S.xin[ps][lane].sum_bits));
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
        gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
      }
      gmax = __shfl_sync(0xffffffffu, gmax, 0);
      gsum = __shfl_sync(0xffffffffu, gsum, 0);
      if (k - 1 < R) shiftB = rintf(gmax * 256.f) * (1.f / 256.f);  // row k-1, pass B at k+1
      const int rs = k - 3;                                          // row whose sum arrived
      if (rs >= 0 && rs < R) {
        const int64_t i = r0 + rs;
        const double ai = a[i];
        const double wi = ai / gsum;
        wC = static_cast<float>(wi);  // column step of row k-3 at iteration k+1
        if (rank == 0 && tid == 0) {
          const double M = static_cast<double>(shiftH[rs & 3]) * kLn2;
          const double ui = (loga[i] - M) - log(gsum);
          rowM[i] = M;
          rowS[i] = gsum;
          u[i] = ui;
          wrow[i] = wi;
          ua += ui * ai;
        }
      }
    }
  }

  // column partials of this cluster's rows
#pragma unroll
  for (int q = 0; q < QPT; ++q) {
    if (!qvalid[q]) continue;
    const int64_t j = col0 + 4 * (tid + q * kFT);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j + e < m) part[cid * mpad + j + e] = acc64[q][e] + static_cast<double>(acc[q][e]);
  }
  if (rank == 0 && tid == 0) rowpart[cid] = ua;
  // every message addressed to this CTA was received (the last iteration's
  // receive); the barrier keeps all CTAs resident until their peers are too
  cluster_arrive();
  cluster_wait();
}

template <int QPT>
int fused_clusters(int smem) {
  static int cached = -1;
  static int cached_smem = -1;
  if (cached >= 0 && cached_smem == smem) return cached;
  OTG_CUDA(cudaFuncSetAttribute(k_fused<QPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCL * 148);
  cfg.blockDim = dim3(kFT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = kCL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  OTG_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k_fused<QPT>, &cfg));
  cached = ncl;
  cached_smem = smem;
  return ncl;
}

}  // namespace

// Decide whether the fused path applies and size it (called at handle setup).
bool fused_configure(Problem& P) {
  P.fused = 0;
  if (P.storage != OTG_STORE_F32 || P.vshards != 1) return false;
  // Opt-in (OTG_FUSED=1) until it beats the two-pass path: measured 10.5 ms per
  // evaluation at n = m = 65536 vs 8.5 ms (profiles/r01_fused_v2.md).
  const char* s = getenv("OTG_FUSED");
  if (!s || atoi(s) == 0) return false;
  const int64_t W = round_up((P.m + kCL - 1) / kCL, 4);
  if (W * kCL > P.ldc) return false;  // C rows must hold whole slices
  const int64_t quads = W / 4;
  int qpt = quads <= kFT ? 1 : quads <= 2 * kFT ? 2 : quads <= 4 * kFT ? 4 : 0;
  if (qpt == 0 || P.n_local < 64 || P.m < 1024) return false;
  const int64_t slot_bytes = W * 4;
  int nslots = static_cast<int>(std::min<int64_t>(kSlotsMax, kSmemBudget / slot_bytes));
  if (nslots < 7) return false;
  const int smem = static_cast<int>(((sizeof(FusedShared) + 127) / 128) * 128 + nslots * slot_bytes);
  int ncl = qpt == 1 ? fused_clusters<1>(smem) : qpt == 2 ? fused_clusters<2>(smem)
                                                           : fused_clusters<4>(smem);
  if (ncl < 1) return false;
  // at least ~64 rows per cluster so the 3-deep pipeline fill is amortised
  ncl = static_cast<int>(std::min<int64_t>(ncl, std::max<int64_t>(1, P.n_local / 64)));
  P.fused = 1;
  P.fused_qpt = qpt;
  P.fused_W = static_cast<int>(W);
  P.fused_slots = nslots;
  P.fused_smem = smem;
  P.fused_clusters = ncl;
  return true;
}

void launch_fused(Problem& P, double* rowpart) {
  const double k2 = P.kappa * kLog2e;
  const float kh = static_cast<float>(k2);
  const float kl = static_cast<float>(k2 - static_cast<double>(kh));
  const dim3 grid(kCL * P.fused_clusters), block(kFT);
#define OTG_FUSED_LAUNCH(Q)                                                                   \
  k_fused<Q><<<grid, block, P.fused_smem, P.stream>>>(                                        \
      P.C32, P.ldc, P.n_local, P.m, P.fused_W, P.fused_slots, P.p, kh, kl, P.a, P.loga, P.rowM, \
      P.rowS, P.u, P.wrow, P.part, P.mpad, rowpart, P.ctrl)
  if (P.fused_qpt == 1)
    OTG_FUSED_LAUNCH(1);
  else if (P.fused_qpt == 2)
    OTG_FUSED_LAUNCH(2);
  else
    OTG_FUSED_LAUNCH(4);
#undef OTG_FUSED_LAUNCH
  OTG_CUDA(cudaGetLastError());
}

}  // namespace otg
