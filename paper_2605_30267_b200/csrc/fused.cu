// fused.cu — single-HBM-pass evaluation sweep for fp32 stored costs (sm_100a).
//
// One evaluation needs, per row i, the row sum S_i BEFORE the row can add
// w_i = a_i / S_i times its exponentials to the column sums (dual.cpp:34-41).
// A 65536-wide fp32 row is 256 KB, more than one SM's shared memory, so the
// two-pass kernels of sweep.cu read the cost twice.  Here a cluster of kCL = 8
// CTAs (one per SM) holds a row on chip, each CTA a W <= 8192-column slice,
// and the cost is read from HBM once per evaluation:
//
//   loads          thread 0 keeps kPre rows ahead: cp.async.bulk of the CTA's
//                  row slice and the row's 32-byte record (shift estimate, a,
//                  log a; k_sp_prep) into a kSlots-deep smem ring, completing
//                  on full[s]; a slot is refilled once every thread has passed
//                  the barrier that follows its column step
//   stats (row k)  exponents against the row's shift ESTIMATE s_i (the
//                  previous evaluation's base-2 row max plus the potential's
//                  move, exactly as k_row_shift in sweep.cu), e = ex2(t)
//                  written back over the cost, partial (sum, max, argmax)
//   exchange       the CTA's partial goes to all 8 CTAs of the cluster with
//                  st.async (DSMEM push, completes on the receiver's mbarrier)
//   column (k-D)   D = kLag rows later the 8 partials of row k-D have arrived:
//                  S, max T, w = a / S; acc_j += w e_ij from smem; fp32
//                  accumulators flushed into fp64 registers every 16 rows
//
// No max pass: s_i is known before the row is read.  A row whose true max T
// relative to s_i falls outside [-2, 6] (the estimate was too loose) adds
// nothing here and is listed; k_sp_redo recomputes it exactly and k_sp_patch
// adds its columns (both cheap: such rows are rare).  The per-element work is
// the k_row_shift inner loop (packed f32x2) plus one LDS/FFMA2 for the column.
//
// Output: per-cluster column partials part[cluster][j] plus one patch row
// part[clusters][j] (summed by k_merge), u, rowM, rowS, wrow, rowM2, rowJ, aux.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace otg {

namespace {

constexpr int kCLMax = 16;                   // CTAs per cluster: 16 or 8 (row slices), or
                                             // 1 when a whole row fits one CTA (m <= 8192)
constexpr int kSW = 8;                       // stats warps
constexpr int kCW = 8;                       // column warps
constexpr int kST = kSW * 32;                // threads per role
constexpr int kCT = (kSW + kCW) * 32;        // threads per CTA
constexpr int kQPT = 8;                      // max float4 quads per thread and row (W <= 8192)
constexpr int kSlotsMax = 32;                // row-slice ring (runtime depth <= this)
constexpr int kLagMax = 7;                   // (kept for the configuration knob)
constexpr int kXD = 16;                      // exchange ring
constexpr float kRedoLo = 2.0f;              // same window as sweep.cu k_row_shift
constexpr float kRedoHi = 6.0f;
constexpr int kPatchThreads = 256;

struct Msg {  // one CTA's partial of one row (16 bytes, one st.async.v4)
  double sum;
  float max;
  int code;
};

struct RowRec {  // per-row inputs, bulk-copied with the row slice (32 bytes)
  float shift;     // quantised base-2 shift estimate (k_sp_prep)
  int pad;
  double a, loga;
  double pad2;
};

struct SpShared {
  uint64_t full[kSlotsMax];    // TMA -> stats warps
  uint64_t sdone[kSlotsMax];   // stats warps -> column warps (e in the slot, partials)
  uint64_t empty[kSlotsMax];   // column warps -> loader (slot free)
  uint64_t xbar[kXD];          // cluster partials of a row received
  Msg xin[kXD][kCLMax];
  RowRec rec[kSlotsMax];
  unsigned wkey[kSlotsMax][kSW];  // stats-warp partials of the row in each slot
  int wcode[kSlotsMax][kSW];
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
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// float <-> unsigned key with the same order (for redux.sync max / min)
__device__ __forceinline__ unsigned ordered_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
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

struct SpArgs {
  const RowRec* rec;
  const float* C;
  int64_t ldc, n, m, mpad;
  int W;
  const double* p;     // potentials (for the column split)
  const float* vq;     // split potential of the row pass (Vc[mpad], vf[mpad])
  const double* dq;
  float kh, kl;
  const double* a;
  const double* loga;
  double* rowM;
  double* rowS;
  double* u;
  double* wrow;
  float4* aux;
  double* rowM2;
  int* rowJ;
  double* part;
  int* bad_rows;       // per cluster: bad_rows[r0 + k], k < bad_count[cluster]
  int* bad_count;
  int nslots, lag;     // ring depth; column step `lag` rows after the stats
  long long* dbg;      // optional timeline (OTG_SP_TRACE): 8 stamps per row, CTA 0 thread 0
};

// Per-row record of the steady state: the quantised shift estimate
// s = ceil(min(M2 + dq_J + 1, M2 + dmax2) 256) / 256 (as k_row_shift), a, log a.
__global__ void __launch_bounds__(256)
k_sp_prep(int64_t n, const double* __restrict__ rowM2, const int* __restrict__ rowJ,
          const double* __restrict__ dq, const double* __restrict__ a,
          const double* __restrict__ loga, RowRec* __restrict__ rec,
          const Ctrl* __restrict__ ctrl, unsigned* __restrict__ epoch) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
  if (epoch != nullptr && blockIdx.x == 0 && threadIdx.x == 0) ++*epoch;  // (k_sp2 counters)
  const double dmax2 = ctrl->dmax2;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    const double M2 = rowM2[i];
    const double lo = M2 + dq[rowJ[i]], hi = M2 + dmax2;
    RowRec r;
    r.shift = static_cast<float>(ceil(fmin(lo + 1.0, hi) * 256.0) * (1.0 / 256.0));
    r.pad = 0;
    r.a = a[i];
    r.loga = loga[i];
    r.pad2 = 0.0;
    rec[i] = r;
  }
}

// Kahan step on packed pairs: acc += x with the running error in cmp
// (cmp holds the NEGATED lost low part: true sum = acc - cmp).
__device__ __forceinline__ void kahan2(float2& acc, float2& cmp, float2 x) {
  const float2 y = __fadd2_rn(x, make_float2(-cmp.x, -cmp.y));
  const float2 tt = __fadd2_rn(acc, y);
  cmp = __fadd2_rn(__fadd2_rn(tt, make_float2(-acc.x, -acc.y)), make_float2(-y.x, -y.y));
  acc = tt;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised: 8 stats warps stream the rows (exponentials against the
// row's shift estimate, written back into the slot, per-warp partials) and
// never wait on the cluster; 8 column warps publish each row's CTA partial to
// the cluster, wait for the 8 CTA partials, and fold w * e into the column
// sums.  Hand-offs are mbarriers (full / sdone / empty / xbar), so the stats of
// row k overlap the exchange and column step of earlier rows; the only
// throttle is the slot ring.
template <int CL, int QPT>
__global__ void __launch_bounds__(kCT, 1)
k_sp(const SpArgs A, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;  // uniform: written by earlier launches
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SpShared& S = *reinterpret_cast<SpShared*>(smem_raw);
  float* slots = reinterpret_cast<float*>(smem_raw + ((sizeof(SpShared) + 127) / 128) * 128);
  const int nslots = A.nslots;
  float* tsum = slots + static_cast<size_t>(nslots) * A.W;  // [nslots][kST] thread partials

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int64_t r0 = A.n * cid / ncl, r1 = A.n * (cid + 1) / ncl;
  const int R = static_cast<int>(r1 - r0);
  const int64_t col0 = static_cast<int64_t>(rank) * A.W;
  const uint32_t slot_bytes = static_cast<uint32_t>(A.W) * 4u;

  auto issue_load = [&](int r) {  // row r of this cluster -> slot r % nslots
    const int s = r % nslots;
    mbar_expect_tx(&S.full[s], slot_bytes + static_cast<uint32_t>(sizeof(RowRec)));
    bulk_load(slots + static_cast<size_t>(s) * A.W, A.C + (r0 + r) * A.ldc + col0, slot_bytes,
              &S.full[s]);
    bulk_load(&S.rec[s], A.rec + r0 + r, static_cast<uint32_t>(sizeof(RowRec)), &S.full[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < nslots; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.sdone[s], kSW);
      mbar_init(&S.empty[s], kCW);
    }
    for (int s = 0; s < kXD; ++s) mbar_init(&S.xbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int r = 0; r < nslots && r < R; ++r) issue_load(r);
  }
  __syncthreads();
  cluster_sync();  // every CTA's barriers exist before any DSMEM push

  const int t = warp < kSW ? tid : tid - kST;  // thread index within its role
  auto stamp = [&](int k, int e) {  // OTG_SP_TRACE timeline (CTA 0)
    if (A.dbg != nullptr && blockIdx.x == 0 && k < 256) A.dbg[k * 8 + e] = clock64();
  };
  bool qvalid[QPT];
#pragma unroll
  for (int q = 0; q < QPT; ++q) qvalid[q] = 4 * (t + q * kST) < A.W;

  if (warp < kSW) {
    // =============================================== stats warps ====
    float2 V01[QPT], V23[QPT], F01[QPT], F23[QPT];  // row-pass split of p
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      const int qq = t + q * kST;
      float v[4], f[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t j = col0 + 4 * qq + e;
        if (qvalid[q] && j < A.m) {
          v[e] = A.vq[j];
          f[e] = A.vq[A.mpad + j];
        } else {
          v[e] = -1e30f;  // padding columns: e = 0, never the max
          f[e] = 0.f;
        }
      }
      V01[q] = make_float2(v[0], v[1]);
      V23[q] = make_float2(v[2], v[3]);
      F01[q] = make_float2(f[0], f[1]);
      F23[q] = make_float2(f[2], f[3]);
    }
    const float2 nkh2 = make_float2(-A.kh, -A.kh), nkl2 = make_float2(-A.kl, -A.kl);
    for (int k = 0; k < R; ++k) {
      const int s = k % nslots;
      if (tid == 0) stamp(k, 0);
      mbar_wait(&S.full[s], (k / nslots) & 1);
      if (tid == 0) stamp(k, 1);
      const float sc = S.rec[s].shift;
      const float2 nSc2 = make_float2(-sc, -sc);
      float4* slot = reinterpret_cast<float4*>(slots + static_cast<size_t>(s) * A.W);
      // running max and the quad holding it; the column inside the quad is
      // resolved at the column step from the exponentials (ex2 is monotonic)
      float tm = -FLT_MAX;
      int code = 0x7fffffff;
      float2 fs = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < QPT; ++q) {
        if (!qvalid[q]) continue;
        const int qq = t + q * kST;
        const float4 c = slot[qq];
        const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
        const float2 t01 = __fadd2_rn(__ffma2_rn(c01, nkh2, __fadd2_rn(V01[q], nSc2)),
                                      __ffma2_rn(c01, nkl2, F01[q]));
        const float2 t23 = __fadd2_rn(__ffma2_rn(c23, nkh2, __fadd2_rn(V23[q], nSc2)),
                                      __ffma2_rn(c23, nkl2, F23[q]));
        const float mx = fmaxf(fmaxf(fmaxf(tm, t01.x), t01.y), fmaxf(t23.x, t23.y));
        code = mx > tm ? static_cast<int>(col0) + 4 * qq : code;
        tm = mx;
        const float4 ev = make_float4(ex2_approx(t01.x), ex2_approx(t01.y), ex2_approx(t23.x),
                                      ex2_approx(t23.y));
        slot[qq] = ev;
        fs = __fadd2_rn(fs, __fadd2_rn(make_float2(ev.x, ev.z), make_float2(ev.y, ev.w)));
      }
      // per-thread fp32 partial (<= 32 terms) -> smem; the publisher folds them
      tsum[s * kST + t] = fs.x + fs.y;
      const unsigned key = ordered_key(tm);
      const unsigned wkey = __reduce_max_sync(0xffffffffu, key);
      const unsigned wcode = __reduce_min_sync(
          0xffffffffu, key == wkey ? static_cast<unsigned>(code) : 0x7fffffffu);
      if (lane == 0) {
        S.wkey[s][warp] = wkey;
        S.wcode[s][warp] = static_cast<int>(wcode);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.sdone[s]);  // release: e and partials visible
      if (tid == 0) stamp(k, 2);
    }
  } else {
    // ============================================== column warps ====
    const int cw = warp - kSW;
    // compensated (Kahan) fp32 column sums: sum + running error per column,
    // 2 registers per column instead of an fp32 partial plus an fp64 total
    float2 acc01[QPT], acc23[QPT], cmp01[QPT], cmp23[QPT];
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      acc01[q] = make_float2(0.f, 0.f);
      acc23[q] = make_float2(0.f, 0.f);
      cmp01[q] = make_float2(0.f, 0.f);
      cmp23[q] = make_float2(0.f, 0.f);
    }
    int nbad = 0;
    const int lag = A.lag;
    for (int kk = 0; kk < R + lag; ++kk) {
      // ---- publish the CTA partial of row kk (rotating warp), `lag` rows
      // ahead of its column step so the exchange latency is hidden ----
      if (kk < R && cw == kk % kCW) {
        const int sp = kk % nslots, xp = kk % kXD;
        mbar_wait(&S.sdone[sp], (kk / nslots) & 1);
        if (lane == 0) stamp(kk, 3);
        double cs = 0.0;  // fixed order: lane l folds threads l, l + 32, ..., then a tree
#pragma unroll
        for (int w = 0; w < kSW; ++w) cs += static_cast<double>(tsum[sp * kST + w * 32 + lane]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
        const unsigned lk = lane < kSW ? S.wkey[sp][lane] : 0u;
        const unsigned ck = __reduce_max_sync(0xffffffffu, lk);
        const unsigned cc = __reduce_min_sync(
            0xffffffffu,
            (lane < kSW && lk == ck) ? static_cast<unsigned>(S.wcode[sp][lane]) : 0x7fffffffu);
        const float cm = key_to_float(ck);
        if (lane == 0) mbar_expect_tx(&S.xbar[xp], CL * 16u);
        cs = __shfl_sync(0xffffffffu, cs, 0);
        if (lane < CL) {
          uint32_t ra, rbar;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                       : "=r"(ra)
                       : "r"(smem_u32(&S.xin[xp][rank])), "r"(static_cast<uint32_t>(lane)));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                       : "=r"(rbar)
                       : "r"(smem_u32(&S.xbar[xp])), "r"(static_cast<uint32_t>(lane)));
          const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(cs));
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, "
              "%4}, [%5];" ::"r"(ra),
              "r"(static_cast<uint32_t>(sb)), "r"(static_cast<uint32_t>(sb >> 32)),
              "r"(__float_as_uint(cm)), "r"(cc), "r"(rbar)
              : "memory");
        }
        if (lane == 0) stamp(kk, 4);
      }
      const int k = kk - lag;
      if (k < 0) continue;
      const int s = k % nslots;
      const int xs = k % kXD;
      mbar_wait(&S.sdone[s], (k / nslots) & 1);  // (acquire: e values of row k)
      // ---- column step of row k: the 8 CTA partials ----
      mbar_wait(&S.xbar[xs], (k / kXD) & 1);
      if (cw == 0 && lane == 0) stamp(k, 5);
      double Ssum = 0.0;
      float T = -FLT_MAX;
      int J = 0x7fffffff;
#pragma unroll
      for (int c = 0; c < CL; ++c) {  // fixed order: every CTA gets the same S, T, J
        const Msg msg = S.xin[xs][c];
        Ssum += msg.sum;
        if (msg.max > T || (msg.max == T && msg.code < J)) {
          T = msg.max;
          J = msg.code;
        }
      }
      const float sc = S.rec[s].shift;
      const int64_t i = r0 + k;
      const float4* slot = reinterpret_cast<const float4*>(slots + static_cast<size_t>(s) * A.W);
      if (T >= -kRedoLo && T <= kRedoHi) {
        const double ai = S.rec[s].a;
        const float wf = static_cast<float>(ai) / static_cast<float>(Ssum);  // IEEE fp32
        const float2 w2 = make_float2(wf, wf);
#pragma unroll
        for (int q = 0; q < QPT; ++q) {
          if (!qvalid[q]) continue;
          const float4 ev = slot[t + q * kST];
          kahan2(acc01[q], cmp01[q], __ffma2_rn(w2, make_float2(ev.x, ev.y), make_float2(0.f, 0.f)));
          kahan2(acc23[q], cmp23[q], __ffma2_rn(w2, make_float2(ev.z, ev.w), make_float2(0.f, 0.f)));
        }
        // row outputs (k_row_shift's epilogue): one CTA per row, rotating
        if (static_cast<int>(rank) == (k & (CL - 1)) && cw == 1 && lane == 0) {
          const double scd = static_cast<double>(sc);
          const double M = scd * kLn2;
          A.rowM[i] = M;
          A.rowS[i] = Ssum;
          A.u[i] = (S.rec[s].loga - M) - log(Ssum);
          A.wrow[i] = ai / Ssum;
          A.rowM2[i] = scd + static_cast<double>(T);
          A.aux[i] = make_float4(sc, 0.0f, wf, 0.0f);
        }
        {  // argmax column: the thread owning the winning quad picks its largest e
          const int64_t off = static_cast<int64_t>(J) - col0;
          if (off >= 0 && off < A.W && static_cast<int>((off >> 2) % kST) == t) {
            const float4 ev = slot[off >> 2];
            const float em = fmaxf(fmaxf(ev.x, ev.y), fmaxf(ev.z, ev.w));
            A.rowJ[i] = J + (ev.x == em ? 0 : ev.y == em ? 1 : ev.z == em ? 2 : 3);
          }
        }
      } else if (rank == 0 && cw == 0 && lane == 0) {
        A.bad_rows[r0 + nbad] = static_cast<int>(i);  // in row order: deterministic patch
        ++nbad;
      }
      // slot free: refill with row k + nslots once all column warps are done
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
      if (cw == 0 && lane == 0) stamp(k, 6);
      if (cw == kCW - 1 && lane == 0 && k + nslots < R) {
        mbar_wait(&S.empty[s], (k / nslots) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_load(k + nslots);
        stamp(k, 7);
      }
    }
    // column partials of this cluster's rows
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      if (!qvalid[q]) continue;
      const int64_t j = col0 + 4 * (t + q * kST);
      const double v[4] = {static_cast<double>(acc01[q].x) - static_cast<double>(cmp01[q].x),
                           static_cast<double>(acc01[q].y) - static_cast<double>(cmp01[q].y),
                           static_cast<double>(acc23[q].x) - static_cast<double>(cmp23[q].x),
                           static_cast<double>(acc23[q].y) - static_cast<double>(cmp23[q].y)};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j + e < A.m) A.part[cid * A.mpad + j + e] = v[e];
    }
    if (rank == 0 && cw == 0 && lane == 0) A.bad_count[cid] = nbad;
  }
  // every message addressed to this CTA has been consumed (the column warps
  // waited for each); keep the cluster resident until all peers are done
  __syncthreads();
  cluster_sync();
}

__global__ void __launch_bounds__(kPatchThreads)
k_sp_patch(const float* __restrict__ C, int64_t ldc, int64_t m, const double* __restrict__ p,
           float kh, float kl, const float4* __restrict__ aux, const int* __restrict__ bad_rows,
           const int* __restrict__ bad_count, int64_t n, int ncl, double* __restrict__ out,
           const Ctrl* __restrict__ ctrl, const unsigned* __restrict__ bad_epoch,
           const unsigned* __restrict__ epoch) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // columns of the rows the stream kernel skipped: out[j] = sum over the
  // listed rows (cluster order, then row order) of w_i ex2(t_ij), with the
  // exact split shift k_row_redo wrote into aux -- the k_col_fast formula
  if (ctrl->done || !ctrl->shift_valid) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kPatchThreads + threadIdx.x;
  if (j >= m) return;
  if (bad_epoch != nullptr && *bad_epoch != *epoch) {  // k_sp2: no loose row this evaluation
    out[j] = 0.0;
    return;
  }
  float Vc, vf;
  split_q(p[j] * kLog2e, Vc, vf);
  double acc = 0.0;
  for (int c = 0; c < ncl; ++c) {
    const int64_t r0 = n * c / ncl;
    const int nb = bad_count[c];
    for (int k = 0; k < nb; ++k) {
      const int64_t i = bad_rows[r0 + k];
      const float4 ax = aux[i];
      const float cc = C[i * ldc + j];
      const float Aq = Vc - ax.x;
      const float g = fmaf(-cc, kl, vf - ax.y);
      const float t = fmaf(-cc, kh, Aq) + g;
      acc += static_cast<double>(ax.z * ex2_approx(t));
    }
  }
  out[j] = acc;
}

// ===========================================================================
// Variant 2 (OTG_FUSED=2): the single pass staged through the SM's own L1 and
// the L2 instead of a cluster's shared memory.
//
// CTA s (one per SM, persistent) owns column segment s of every row: quads
// [Q s / G, Q (s + 1) / G) of the Q = m / 4 column quads, <= 4 per lane.  Rows
// go in chunks of ~32; two warp groups of the CTA walk the chunks:
//
//   stats warps    chunk c: the segment's exponentials against the row's shift
//                  estimate (exactly the k_sp / k_row_shift formula), per-row
//                  segment partial (sum, max, first argmax) -> a ring in global
//                  memory; one arrival per CTA on cnt[c]; the LAST CTA to arrive
//                  folds the G partials of each row of the chunk (fixed order),
//                  writes the row outputs and w = a / S (0 for a loose row),
//                  lists the loose rows in row order, then publishes ready[c]
//   column warps   chunk c - lag (once ready[c] is published): the same
//                  exponentials again -- the segment rows are re-read from the
//                  L1 / L2 the stats warps just filled, not from HBM -- times w,
//                  into Kahan fp32 column sums held in registers for the whole
//                  evaluation (the segment's columns belong to this CTA alone)
//
// HBM sees the cost once; the cross-SM exchange is one counter and one flag per
// chunk.  Loose rows are redone exactly by k_sp_redo and patched by k_sp_patch
// (chunk lists, in row order).  Counters are monotone across evaluations: the
// evaluation's epoch is bumped by k_sp_prep.
constexpr int kPWS = 8;       // stats warps
constexpr int kPWC = 6;       // column warps
constexpr int kPT = (kPWS + kPWC + 2) * 32;  // + reducer + producer: 16 warps, 128 registers
constexpr int kSegQ = 112;    // quads per ring slot (1792 B): m <= 148 * 448
constexpr int kNA = 64;       // ring A slots (HBM -> smem, stats warps): 2 per producer lane
constexpr int kNB = 32;       // ring B slots (L2 -> smem, column warps): 1 per producer lane
constexpr int kPQ = 4;        // quads per lane: segment <= 128 quads (512 columns)
constexpr int kPRing = 16;    // chunk ring of the segment partials
constexpr int kPRowsMax = 64; // rows per chunk, upper bound

struct SegPart {  // one CTA's partial of one row (16 bytes)
  double sum;
  float tmax;
  int jmax;
};

struct PArgs {
  const RowRec* rec;
  const float* C;
  int64_t ldc, n, m, mpad;
  const float* vq;
  float kh, kl;
  double* rowM;
  double* rowS;
  double* u;
  double* wrow;
  float4* aux;
  double* rowM2;
  int* rowJ;
  double* part;          // row 0: the column sums (segments are disjoint)
  int* bad_rows;         // chunk c: bad_rows[r0(c) + k], k < bad_count[c]
  int* bad_count;
  unsigned* bad_epoch;   // = epoch when some row of this evaluation was loose
  int nchunks, lag, pf;  // (pf unused)
  int64_t lag_rows;      // ring A may run this many rows ahead of ring B
  long long* dbg;        // OTG_SP_TRACE: stuck-wait records
  SegPart* seg;          // [kPRing][kPRowsMax][G]
  float* lam;            // [n] fp32 w of the row, 0 for a loose row
  unsigned* cnt;         // [nchunks] arrivals (monotone)
  unsigned* ready;       // [nchunks] rows folded (monotone)
  const unsigned* epoch;
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// exponents of one quad against the row shift (k_sp's packed form)
__device__ __forceinline__ void quad_t(const float4 c, float2 V01, float2 V23, float2 F01,
                                       float2 F23, float2 nSc2, float2 nkh2, float2 nkl2,
                                       float2& t01, float2& t23) {
  const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
  t01 = __fadd2_rn(__ffma2_rn(c01, nkh2, __fadd2_rn(V01, nSc2)), __ffma2_rn(c01, nkl2, F01));
  t23 = __fadd2_rn(__ffma2_rn(c23, nkh2, __fadd2_rn(V23, nSc2)), __ffma2_rn(c23, nkl2, F23));
}

// A wait that outlived its spin budget: log who / what (OTG_SP_TRACE buffer,
// 8 words per record, word 0 of the buffer = record count) and trap.
__device__ __noinline__ void sp2_stuck(long long* dbg, long long tag, long long a, long long b,
                                       long long c, long long d) {
  if (dbg != nullptr) {
    const long long k = atomicAdd(reinterpret_cast<unsigned long long*>(dbg), 1ull);
    if (k < 200) {
      long long* r = dbg + 8 * (k + 1);
      r[0] = tag;
      r[1] = blockIdx.x;
      r[2] = threadIdx.x;
      r[3] = a;
      r[4] = b;
      r[5] = c;
      r[6] = d;
    }
    __threadfence_system();
    for (int k = 0; k < 2000; ++k) __nanosleep(1000000);  // let other stuck waits log too
  }
  __trap();
}


__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, long long* dbg,
                                              long long tag, long long row) {
  for (unsigned spin = 0; !mbar_test(bar, parity); ++spin) {
    __nanosleep(32);
    if (spin > (1u << 24)) sp2_stuck(dbg, tag, row, parity, 0, 0);
  }
}

// Row-segment rings in shared memory, both filled by cp.async.bulk from one
// producer thread: ring A from HBM for the stats warps (a slot is released as
// soon as its row's statistics are taken), ring B re-reading the same rows
// from L2 for the column warps.  Loads in flight per SM: up to kNA + kNB
// segments (~190 KB), which is what HBM latency x per-SM bandwidth asks for.
__global__ void __launch_bounds__(kPT, 1)
k_sp2(const PArgs A, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;  // uniform: written by earlier launches
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* ringA = reinterpret_cast<float4*>(smem_raw);             // [kNA][kSegQ]
  float4* ringB = ringA + kNA * kSegQ;                              // [kNB][kSegQ]
  uint64_t* fullA = reinterpret_cast<uint64_t*>(ringB + kNB * kSegQ);
  uint64_t* emptyA = fullA + kNA;
  uint64_t* fullB = emptyA + kNA;
  uint64_t* emptyB = fullB + kNB;
  double* red = reinterpret_cast<double*>(smem_raw);  // end: [kPWC][4 * kSegQ] (over ring A)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, sgi = blockIdx.x;
  const int64_t Q = (A.m + 3) / 4;
  const int64_t q0 = Q * sgi / G, q1 = Q * (sgi + 1) / G;
  const unsigned E = *A.epoch;
  const int nch = A.nchunks;
  const int64_t n = A.n;
  const uint32_t seg_bytes = static_cast<uint32_t>((q1 - q0) * 16);
  if (tid == 0) {
    for (int s = 0; s < kNA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < kNB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kPWS + kPWC + 1) {
    // =============================================== producer ====
    // lane l streams rows l, l + 32, ...: ring A slots l and l + 32, ring B
    // slot l, so the 32 lanes issue their copies side by side
    const float* base = A.C + 4 * q0;
    const int64_t lag_rows = A.lag_rows;
    int64_t ia = lane, ib = lane;
    for (unsigned spin = 0; ib < n;) {
      bool moved = false;
      // ring A: next row from HBM once its slot is free, at most lag_rows
      // ahead of ring B (the L2 must still hold a row when B re-reads it)
      if (ia < n && ia < ib + lag_rows) {
        const int s = static_cast<int>(ia % kNA);
        const int64_t use = ia / kNA;
        if (use == 0 || mbar_test(&emptyA[s], static_cast<uint32_t>((use - 1) & 1))) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs the LDS reads
          mbar_expect_tx(&fullA[s], seg_bytes);
          bulk_load(ringA + s * kSegQ, base + ia * A.ldc, seg_bytes, &fullA[s]);
          ia += 32;
          moved = true;
        }
      }
      // ring B: row ib again (an L2 hit) once the stats warps took row ib
      // (its A slot came back) and the B slot is free.  (Once this lane issued
      // row ib + kNA, row ib's slot had come back; before that the slot's
      // phase for row ib is unambiguous.)
      if (ib < ia) {
        const bool stats_done =
            ia > ib + kNA ||
            mbar_test(&emptyA[ib % kNA], static_cast<uint32_t>((ib / kNA) & 1));
        const int s = static_cast<int>(ib % kNB);
        const int64_t use = ib / kNB;
        if (stats_done &&
            (use == 0 || mbar_test(&emptyB[s], static_cast<uint32_t>((use - 1) & 1)))) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&fullB[s], seg_bytes);
          bulk_load(ringB + s * kSegQ, base + ib * A.ldc, seg_bytes, &fullB[s]);
          ib += 32;
          moved = true;
        }
      }
      if (!moved) {
        __nanosleep(20);
        if (++spin > (1u << 25)) sp2_stuck(A.dbg, 1, ia, ib, lag_rows, n);
      } else {
        spin = 0;
      }
    }
    return;
  }

  // this lane's quads and their split potentials (padding columns: e = 0)
  bool qv[kPQ];
  float2 V01[kPQ], V23[kPQ], F01[kPQ], F23[kPQ];
#pragma unroll
  for (int k = 0; k < kPQ; ++k) {
    const int64_t q = q0 + lane + 32 * k;
    qv[k] = q < q1;
    float v[4], f[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t j = 4 * q + e;
      const bool ok = qv[k] && j < A.m;
      v[e] = ok ? A.vq[j] : -1e30f;
      f[e] = ok ? A.vq[A.mpad + j] : 0.f;
    }
    V01[k] = make_float2(v[0], v[1]);
    V23[k] = make_float2(v[2], v[3]);
    F01[k] = make_float2(f[0], f[1]);
    F23[k] = make_float2(f[2], f[3]);
  }
  const float2 nkh2 = make_float2(-A.kh, -A.kh), nkl2 = make_float2(-A.kl, -A.kl);

  if (warp < kPWS) {
    // ================================================ stats warps ====
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = n * c / nch, r1 = n * (c + 1) / nch;
      SegPart* ring = A.seg + static_cast<int64_t>(c % kPRing) * kPRowsMax * G;
      for (int64_t i = r0 + ((warp - r0) % kPWS + kPWS) % kPWS; i < r1; i += kPWS) {
        const int s = static_cast<int>(i % kNA);
        mbar_wait_dbg(&fullA[s], static_cast<uint32_t>((i / kNA) & 1), A.dbg, 4, i);
        const float4* slot = ringA + s * kSegQ;
        float4 cv[kPQ];
#pragma unroll
        for (int k = 0; k < kPQ; ++k) cv[k] = qv[k] ? slot[lane + 32 * k] : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[s]);  // the slot's data is in registers
        const float sc = A.rec[i].shift;
        const float2 nSc2 = make_float2(-sc, -sc);
        float2 fs = make_float2(0.f, 0.f);
        float tm = -FLT_MAX;
        int tk = 0;
#pragma unroll
        for (int k = 0; k < kPQ; ++k) {
          if (!qv[k]) continue;
          float2 t01, t23;
          quad_t(cv[k], V01[k], V23[k], F01[k], F23[k], nSc2, nkh2, nkl2, t01, t23);
          const float mq = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
          tk = mq > tm ? k : tk;
          tm = fmaxf(tm, mq);
          fs = __fadd2_rn(fs, __fadd2_rn(make_float2(ex2_approx(t01.x), ex2_approx(t23.x)),
                                         make_float2(ex2_approx(t01.y), ex2_approx(t23.y))));
        }
        double ds = static_cast<double>(fs.x + fs.y);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
        const unsigned key = ordered_key(tm);
        const unsigned wkey = __reduce_max_sync(0xffffffffu, key);
        const int64_t myq = q0 + lane + 32 * tk;
        const unsigned wq = __reduce_min_sync(
            0xffffffffu, key == wkey ? static_cast<unsigned>(myq) : 0xffffffffu);
        if (key == wkey && static_cast<unsigned>(myq) == wq) {
          // first column of the winning quad whose exponent is the max
          float2 t01, t23;
          float4 cq = cv[0];
#pragma unroll
          for (int k = 1; k < kPQ; ++k) cq = tk == k ? cv[k] : cq;
          float2 a01 = V01[0], a23 = V23[0], b01 = F01[0], b23 = F23[0];
#pragma unroll
          for (int k = 1; k < kPQ; ++k) {
            a01 = tk == k ? V01[k] : a01;
            a23 = tk == k ? V23[k] : a23;
            b01 = tk == k ? F01[k] : b01;
            b23 = tk == k ? F23[k] : b23;
          }
          quad_t(cq, a01, a23, b01, b23, nSc2, nkh2, nkl2, t01, t23);
          const int e = t01.x == tm ? 0 : t01.y == tm ? 1 : t23.x == tm ? 2 : 3;
          SegPart sp;
          sp.sum = ds;
          sp.tmax = tm;
          sp.jmax = static_cast<int>(4 * myq + e);
          ring[(i - r0) * G + sgi] = sp;
        }
      }
      // one arrival per CTA (after all 8 warps' partials are written)
      named_bar(1, kPWS * 32);
      if (tid == 0) {
        __threadfence();
        atomicAdd(&A.cnt[c], 1u);
      }
    }
  } else if (warp == kPWS + kPWC) {
    // ============================================== reducer warp ====
    // row i is folded by CTA i mod G, so a chunk's rows are folded by 32
    // different SMs at once: one L2 round trip of latency per chunk
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = n * c / nch, r1 = n * (c + 1) / nch;
      int64_t i = r0 + ((sgi - r0) % G + G) % G;
      if (i >= r1) continue;
      if (lane == 0)
        for (unsigned spin = 0; ld_acquire(&A.cnt[c]) < E * static_cast<unsigned>(G); ++spin) {
          __nanosleep(32);
          if (spin > (1u << 24)) sp2_stuck(A.dbg, 2, c, ld_acquire(&A.cnt[c]), E, G);
        }
      __syncwarp();
      const SegPart* ring = A.seg + static_cast<int64_t>(c % kPRing) * kPRowsMax * G;
      for (; i < r1; i += G) {
        const SegPart* rp = ring + (i - r0) * G;
        double S = 0.0;
        unsigned bk = 0u;
        int bj = 0x7fffffff;
        double2 x[5];
#pragma unroll
        for (int h = 0; h < 5; ++h) {
          const int g = lane + 32 * h;
          x[h] = g < G ? __ldcg(reinterpret_cast<const double2*>(rp + g)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int h = 0; h < 5; ++h) {
          if (lane + 32 * h >= G) continue;
          const int2 y = *reinterpret_cast<const int2*>(&x[h].y);
          S += x[h].x;
          const unsigned kk = ordered_key(__int_as_float(y.x));
          if (kk > bk || (kk == bk && y.y < bj)) {
            bk = kk;
            bj = y.y;
          }
        }
        for (int g = lane + 160; g < G; g += 32) {  // (more than 160 SMs)
          const double2 xx = __ldcg(reinterpret_cast<const double2*>(rp + g));
          const int2 y = *reinterpret_cast<const int2*>(&xx.y);
          S += xx.x;
          const unsigned kk = ordered_key(__int_as_float(y.x));
          if (kk > bk || (kk == bk && y.y < bj)) {
            bk = kk;
            bj = y.y;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        const unsigned K = __reduce_max_sync(0xffffffffu, bk);
        const int J = static_cast<int>(__reduce_min_sync(
            0xffffffffu, bk == K ? static_cast<unsigned>(bj) : 0x7fffffffu));
        if (lane == 0) {
          const float T = key_to_float(K);
          if (T >= -kRedoLo && T <= kRedoHi) {
            const RowRec rr = A.rec[i];
            const float wf = static_cast<float>(rr.a) / static_cast<float>(S);  // IEEE fp32
            const double scd = static_cast<double>(rr.shift);
            const double M = scd * kLn2;
            A.lam[i] = wf;
            A.rowM[i] = M;
            A.rowS[i] = S;
            A.u[i] = (rr.loga - M) - log(S);
            A.wrow[i] = rr.a / S;
            A.rowM2[i] = scd + static_cast<double>(T);
            A.rowJ[i] = J;
            A.aux[i] = make_float4(rr.shift, 0.0f, wf, 0.0f);
          } else {
            A.lam[i] = 0.f;  // loose row: listed by k_sp2_list, redone, patched
            *A.bad_epoch = E;
          }
          __threadfence();
          atomicAdd(&A.ready[c], 1u);
        }
      }
    }
  } else {
    // =============================================== column warps ====
    const int cw = warp - kPWS;
    float2 acc01[kPQ], acc23[kPQ], cmp01[kPQ], cmp23[kPQ];
#pragma unroll
    for (int k = 0; k < kPQ; ++k) {
      acc01[k] = make_float2(0.f, 0.f);
      acc23[k] = make_float2(0.f, 0.f);
      cmp01[k] = make_float2(0.f, 0.f);
      cmp23[k] = make_float2(0.f, 0.f);
    }
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = n * c / nch, r1 = n * (c + 1) / nch;
      const unsigned want = E * static_cast<unsigned>(r1 - r0);  // rows folded (monotone)
      if (lane == 0)
        for (unsigned spin = 0; ld_acquire(&A.ready[c]) < want; ++spin) {
          __nanosleep(64);
          if (spin > (1u << 24)) sp2_stuck(A.dbg, 3, c, ld_acquire(&A.ready[c]), want, cw);
        }
      __syncwarp();
      for (int64_t i = r0 + ((cw - r0) % kPWC + kPWC) % kPWC; i < r1; i += kPWC) {
        const int s = static_cast<int>(i % kNB);
        const float w = __ldcg(A.lam + i);
        mbar_wait_dbg(&fullB[s], static_cast<uint32_t>((i / kNB) & 1), A.dbg, 5, i);
        const float4* slot = ringB + s * kSegQ;
        float4 cv[kPQ];
#pragma unroll
        for (int k = 0; k < kPQ; ++k) cv[k] = qv[k] ? slot[lane + 32 * k] : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyB[s]);
        if (w == 0.f) continue;  // loose row: k_sp_redo / k_sp_patch
        const float sc = A.rec[i].shift;
        const float2 nSc2 = make_float2(-sc, -sc), w2 = make_float2(w, w);
#pragma unroll
        for (int k = 0; k < kPQ; ++k) {
          if (!qv[k]) continue;
          float2 t01, t23;
          quad_t(cv[k], V01[k], V23[k], F01[k], F23[k], nSc2, nkh2, nkl2, t01, t23);
          const float2 e01 = make_float2(ex2_approx(t01.x), ex2_approx(t01.y));
          const float2 e23 = make_float2(ex2_approx(t23.x), ex2_approx(t23.y));
          kahan2(acc01[k], cmp01[k], __ffma2_rn(w2, e01, make_float2(0.f, 0.f)));
          kahan2(acc23[k], cmp23[k], __ffma2_rn(w2, e23, make_float2(0.f, 0.f)));
        }
      }
    }
    // column sums of the segment: the column warps' partials, fixed order.
    // Ring A is free: every row's B load waited for its A slot to come back.
    named_bar(2, kPWC * 32);
    constexpr int kSeg = 4 * kSegQ;
#pragma unroll
    for (int k = 0; k < kPQ; ++k) {
      if (!qv[k]) continue;
      const int cl = 4 * (lane + 32 * k);
      double* r = red + cw * kSeg + cl;
      r[0] = static_cast<double>(acc01[k].x) - static_cast<double>(cmp01[k].x);
      r[1] = static_cast<double>(acc01[k].y) - static_cast<double>(cmp01[k].y);
      r[2] = static_cast<double>(acc23[k].x) - static_cast<double>(cmp23[k].x);
      r[3] = static_cast<double>(acc23[k].y) - static_cast<double>(cmp23[k].y);
    }
    named_bar(2, kPWC * 32);
    const int64_t ncols = 4 * (q1 - q0);
    for (int cl = tid - kPWS * 32; cl < ncols; cl += kPWC * 32) {
      const int64_t j = 4 * q0 + cl;
      if (j >= A.m) continue;
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kPWC; ++w) v += red[w * kSeg + cl];
      A.part[j] = v;
    }
  }
}

// Loose rows of a k_sp2 evaluation (lam == 0), in row order, as one list
// (the k_sp_redo / k_sp_patch layout with a single list).  Rare: gated on
// bad_epoch, so the kernel returns at once on a clean evaluation.
__global__ void __launch_bounds__(1024)
k_sp2_list(int64_t n, const float* __restrict__ lam, int* __restrict__ bad_rows,
           int* __restrict__ bad_count, const unsigned* __restrict__ bad_epoch,
           const unsigned* __restrict__ epoch, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid || *bad_epoch != *epoch) return;
  __shared__ int wsum[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const bool bad = i < n && lam[i] == 0.f;
    const unsigned mask = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) wsum[warp] = __popc(mask);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (bad) bad_rows[off + __popc(mask & ((1u << lane) - 1u))] = static_cast<int>(i);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += wsum[w];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) bad_count[0] = base;
}

long long*& sp_trace_buf() {
  static long long* p = nullptr;
  return p;
}
long long*& sp_trace_host() {
  static long long* p = nullptr;
  return p;
}

cudaLaunchConfig_t sp_config(int CL, unsigned clusters, int smem, cudaStream_t stream,
                             cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * clusters);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr->id = cudaLaunchAttributeClusterDimension;
  attr->val.clusterDim.x = CL;
  attr->val.clusterDim.y = 1;
  attr->val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

using SpKernel = void (*)(const SpArgs, const Ctrl*);

SpKernel sp_kernel(int CL, int qpt) {
  if (CL == 1) return k_sp<1, kQPT>;
  if (CL == 8) return k_sp<8, kQPT>;
  return qpt <= 4 ? k_sp<16, 4> : k_sp<16, kQPT>;
}

int sp_clusters(int CL, int qpt, int smem) {
  SpKernel k = sp_kernel(CL, qpt);
  OTG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (CL > 8) OTG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchAttribute attr;
  cudaLaunchConfig_t cfg = sp_config(CL, 148, smem, nullptr, &attr);
  int ncl = 0;
  OTG_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
  return ncl;
}

}  // namespace

// Decide whether the single-pass path applies and size it (handle setup).
// Opt-in (OTG_FUSED=1): on B200 at n = m = 65536 it takes 6.4 ms per
// evaluation against 5.6 ms for the two-pass kernels -- the per-row chain
// (stats -> cluster exchange -> column step) costs ~2000 cycles of latency per
// row that the 16 warps do not hide (tools/sp_trace.py timeline,
// profiles/r01_single_pass.md).
// Variant 2: one persistent CTA per SM owning a <= 512-column segment.
static bool fused2_configure(Problem& P) {
  int sms = 0;
  OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  const int64_t Q = (P.m + 3) / 4;
  if ((Q + sms - 1) / sms > kSegQ) return false;  // segment wider than a ring slot
  if (Q < 16 * sms) return false;                     // under ~16 quads per CTA: two-pass
  const char* r_env = getenv("OTG_SP2_ROWS");
  const int rows = std::max(8, std::min(kPRowsMax / 2, r_env ? atoi(r_env) : 32));
  const int nch = static_cast<int>(P.n_local / rows);
  const char* l_env = getenv("OTG_SP2_LAG");
  const char* p_env = getenv("OTG_SP2_PF");
  const int lag = std::max(0, std::min(kPRing - 3, l_env ? atoi(l_env) : 6));
  if (nch < lag + 2) return false;
  const int smem = (kNA + kNB) * kSegQ * 16 + 2 * (kNA + kNB) * 8;
  OTG_CUDA(cudaFuncSetAttribute(k_sp2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sp2, kPT, smem));
  if (occ < 1) return false;
  P.fused = 1;
  P.fused_kind = 2;
  P.fused_clusters = 1;  // one partial row: the segments are disjoint
  P.fused_grid = sms;
  P.fused_chunks = nch;
  P.fused_lag = lag;
  P.fused_pf = p_env ? std::max(0, atoi(p_env)) : 0;
  P.fused_smem = smem;
  if (getenv("OTG_VERBOSE"))
    fprintf(stderr, "[otg] single-pass v2: grid=%d chunks=%d rows/chunk=%lld lag=%d pf=%d smem=%d\n",
            sms, nch, static_cast<long long>(P.n_local / nch), lag, P.fused_pf, smem);
  return true;
}

bool fused_configure(Problem& P) {
  P.fused = 0;
  if (P.storage != OTG_STORE_F32 || P.vshards != 1) return false;
  const char* s = getenv("OTG_FUSED");
  if (!s || atoi(s) == 0) return false;
  if (atoi(s) == 2) return fused2_configure(P);
  P.fused_kind = 1;
  const char* cl_env = getenv("OTG_SP_CL");
  const int CL = P.m <= 4 * kST * kQPT ? 1 : (cl_env && atoi(cl_env) == 8 ? 8 : kCLMax);
  const int64_t W = round_up((P.m + CL - 1) / CL, 4);
  if (W * CL > P.ldc) return false;           // C rows must hold whole slices
  if (W > 4 * kST * kQPT) return false;       // columns per CTA held in registers
  if (P.n_local < 16 * 8 || P.m < 1024) return false;
  const int qpt = W <= 4 * kST * 4 ? 4 : kQPT;
  const int64_t head = ((sizeof(SpShared) + 127) / 128) * 128;
  const int64_t budget = 220 * 1024 - head;
  const int nslots = static_cast<int>(std::min<int64_t>(kSlotsMax, budget / (W * 4 + kST * 4)));
  if (nslots < 5) return false;
  const char* lag_env = getenv("OTG_SP_LAG");
  int lag = lag_env ? atoi(lag_env) : 3;
  lag = std::max(0, std::min(std::min(lag, kLagMax), nslots - 2));
  const int smem = static_cast<int>(head + static_cast<int64_t>(nslots) * (W * 4 + kST * 4));
  int ncl = sp_clusters(CL, qpt, smem);
  if (getenv("OTG_VERBOSE"))
    fprintf(stderr, "[otg] single-pass: CL=%d W=%lld qpt=%d smem=%d slots=%d lag=%d clusters=%d\n",
            CL, static_cast<long long>(W), qpt, smem, nslots, lag, ncl);
  if (ncl < 1) return false;
  // at least ~16 rows per cluster so the pipeline fill is amortised
  ncl = static_cast<int>(std::min<int64_t>(ncl, std::max<int64_t>(1, P.n_local / 16)));
  P.fused = 1;
  P.fused_W = static_cast<int>(W);
  P.fused_smem = smem;
  P.fused_clusters = ncl;
  P.fused_slots = nslots;
  P.fused_qpt = lag;  // (column-step lag of the single-pass kernel)
  P.fused_cl = CL;
  P.fused_qpt4 = qpt;
  return true;
}

void fused_alloc(Problem& P) {
  if (!P.fused) return;
  if (P.fused_kind == 2) {
    if (getenv("OTG_SP_TRACE") && !sp_trace_buf()) {  // mapped host memory: readable after a trap
      OTG_CUDA(cudaHostAlloc(&sp_trace_host(), 256 * 8 * sizeof(long long), cudaHostAllocMapped));
      memset(sp_trace_host(), 0, 256 * 8 * sizeof(long long));
      OTG_CUDA(cudaHostGetDevicePointer(&sp_trace_buf(), sp_trace_host(), 0));
    }
    const int nch = P.fused_chunks;
    P.sp_rec = dalloc<double>(P, static_cast<size_t>(P.n_local) * (sizeof(RowRec) / 8));
    P.sp_bad_rows = dalloc<int>(P, P.n_local);
    P.sp_bad_count = dalloc<int>(P, nch);
    P.sp_seg = dalloc<SegPart>(P, static_cast<size_t>(kPRing) * kPRowsMax * P.fused_grid);
    P.sp_lam = dalloc<float>(P, P.n_local);
    P.sp_sync = dalloc<unsigned>(P, 2 * static_cast<size_t>(nch) + 2);
    OTG_CUDA(cudaMemsetAsync(P.sp_sync, 0, (2 * static_cast<size_t>(nch) + 2) * sizeof(unsigned),
                             P.stream));
    OTG_CUDA(cudaMemsetAsync(P.sp_bad_count, 0, nch * sizeof(int), P.stream));
    return;
  }
  if (getenv("OTG_SP_TRACE") && !sp_trace_buf())
    OTG_CUDA(cudaMalloc(&sp_trace_buf(), 256 * 8 * sizeof(long long)));
  P.sp_rec = dalloc<double>(P, static_cast<size_t>(P.n_local) * (sizeof(RowRec) / 8));
  P.sp_bad_rows = dalloc<int>(P, P.n_local);
  P.sp_bad_count = dalloc<int>(P, P.fused_clusters);
  OTG_CUDA(cudaMemsetAsync(P.sp_bad_count, 0, P.fused_clusters * sizeof(int), P.stream));
}

// Steady-state evaluation sweep (launched after the exact-path kernels, each
// of which returns at once when the other applies): single pass, redo of the
// loose rows, their column patch into partial row `fused_clusters`.
static void launch_fused2(Problem& P, float kh, float kl) {
  RowRec* rec = reinterpret_cast<RowRec*>(P.sp_rec);
  const int nch = P.fused_chunks;
  unsigned* epoch = P.sp_sync + 2 * nch;
  unsigned* bad_epoch = epoch + 1;
  launch_k(k_sp_prep, 296, 256, 0, P.stream, P.n_local, P.rowM2, P.rowJ, P.dq, P.a, P.loga, rec,
           static_cast<const Ctrl*>(P.ctrl), epoch);
  PArgs A;
  A.rec = rec;
  A.C = P.C32;
  A.ldc = P.ldc;
  A.n = P.n_local;
  A.m = P.m;
  A.mpad = P.mpad;
  A.vq = P.vq;
  A.kh = kh;
  A.kl = kl;
  A.rowM = P.rowM;
  A.rowS = P.rowS;
  A.u = P.u;
  A.wrow = P.wrow;
  A.aux = P.aux;
  A.rowM2 = P.rowM2;
  A.rowJ = P.rowJ;
  A.part = P.part;
  A.bad_rows = P.sp_bad_rows;
  A.bad_count = P.sp_bad_count;
  A.bad_epoch = bad_epoch;
  A.nchunks = nch;
  A.lag = P.fused_lag;
  A.pf = P.fused_pf;
  A.dbg = sp_trace_buf();
  A.lag_rows = std::max<int64_t>(static_cast<int64_t>(P.fused_lag) * (P.n_local / nch),
                                 std::max<int64_t>(kNA, P.n_local / nch + 1) + 1);
  A.seg = static_cast<SegPart*>(P.sp_seg);
  A.lam = P.sp_lam;
  A.cnt = P.sp_sync;
  A.ready = P.sp_sync + nch;
  A.epoch = epoch;
  launch_k(k_sp2, P.fused_grid, kPT, P.fused_smem, P.stream, A, static_cast<const Ctrl*>(P.ctrl));
  launch_k(k_sp2_list, 1, 1024, 0, P.stream, P.n_local, static_cast<const float*>(P.sp_lam),
           P.sp_bad_rows, P.sp_bad_count, static_cast<const unsigned*>(bad_epoch),
           static_cast<const unsigned*>(epoch), static_cast<const Ctrl*>(P.ctrl));
  launch_sp_redo(P, P.sp_bad_rows, P.sp_bad_count, 1, bad_epoch, epoch);
  const unsigned g = static_cast<unsigned>((P.m + kPatchThreads - 1) / kPatchThreads);
  launch_k(k_sp_patch, g, kPatchThreads, 0, P.stream, P.C32, P.ldc, P.m,
           static_cast<const double*>(P.p), kh, kl, static_cast<const float4*>(P.aux),
           static_cast<const int*>(P.sp_bad_rows), static_cast<const int*>(P.sp_bad_count),
           P.n_local, 1, P.part + P.mpad, static_cast<const Ctrl*>(P.ctrl),
           static_cast<const unsigned*>(bad_epoch), static_cast<const unsigned*>(epoch));
  OTG_CUDA(cudaGetLastError());
}

void launch_fused(Problem& P, float kh, float kl) {
  if (P.fused_kind == 2) {
    launch_fused2(P, kh, kl);
    return;
  }
  RowRec* rec = reinterpret_cast<RowRec*>(P.sp_rec);
  launch_k(k_sp_prep, 296, 256, 0, P.stream, P.n_local, P.rowM2, P.rowJ, P.dq, P.a, P.loga, rec,
                                       P.ctrl, static_cast<unsigned*>(nullptr));
  SpArgs A;
  A.rec = rec;
  A.C = P.C32;
  A.ldc = P.ldc;
  A.n = P.n_local;
  A.m = P.m;
  A.mpad = P.mpad;
  A.W = P.fused_W;
  A.p = P.p;
  A.vq = P.vq;
  A.dq = P.dq;
  A.kh = kh;
  A.kl = kl;
  A.a = P.a;
  A.loga = P.loga;
  A.rowM = P.rowM;
  A.rowS = P.rowS;
  A.u = P.u;
  A.wrow = P.wrow;
  A.aux = P.aux;
  A.rowM2 = P.rowM2;
  A.rowJ = P.rowJ;
  A.part = P.part;
  A.bad_rows = P.sp_bad_rows;
  A.bad_count = P.sp_bad_count;
  A.nslots = P.fused_slots;
  A.lag = P.fused_qpt;
  A.dbg = sp_trace_buf();
  cudaLaunchAttribute attr;
  cudaLaunchConfig_t cfg = sp_config(P.fused_cl, P.fused_clusters, P.fused_smem, P.stream, &attr);
  OTG_CUDA(cudaLaunchKernelEx(&cfg, sp_kernel(P.fused_cl, P.fused_qpt4), A,
                              static_cast<const Ctrl*>(P.ctrl)));
  launch_sp_redo(P, P.sp_bad_rows, P.sp_bad_count, P.fused_clusters);
  const unsigned g = static_cast<unsigned>((P.m + kPatchThreads - 1) / kPatchThreads);
  launch_k(k_sp_patch, g, kPatchThreads, 0, P.stream, 
      P.C32, P.ldc, P.m, P.p, kh, kl, P.aux, P.sp_bad_rows, P.sp_bad_count, P.n_local,
      P.fused_clusters, P.part + static_cast<int64_t>(P.fused_clusters) * P.mpad, P.ctrl,
      static_cast<const unsigned*>(nullptr), static_cast<const unsigned*>(nullptr));
  OTG_CUDA(cudaGetLastError());
}

}  // namespace otg

// Debug: copy the single-pass kernel's timeline (OTG_SP_TRACE) to the host.
extern "C" int otg_debug_sp_trace(long long* out, int count) {
  if (long long* h = otg::sp_trace_host()) {  // k_sp2 stuck-wait records (survive a trap)
    memcpy(out, h, static_cast<size_t>(count) * sizeof(long long));
    return 0;
  }
  long long* p = otg::sp_trace_buf();
  if (!p) return 1;
  if (cudaMemcpy(out, p, static_cast<size_t>(count) * sizeof(long long), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return 2;
  return 0;
}
