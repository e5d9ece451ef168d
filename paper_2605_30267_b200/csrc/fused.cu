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

#include "common.cuh"

namespace otg {

namespace {

constexpr int kCLMax = 8;                    // CTAs per cluster: 8 (row slices), or 1
                                             // when a whole row fits one CTA (m <= 8192)
constexpr int kSW = 8;                       // stats warps
constexpr int kCW = 8;                       // column warps
constexpr int kST = kSW * 32;                // threads per role
constexpr int kCT = (kSW + kCW) * 32;        // threads per CTA
constexpr int kQPT = 8;                      // float4 quads per thread and row (W <= 8192)
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
          const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done || !ctrl->shift_valid) return;
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
template <int CL>
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
  bool qvalid[kQPT];
#pragma unroll
  for (int q = 0; q < kQPT; ++q) qvalid[q] = 4 * (t + q * kST) < A.W;

  if (warp < kSW) {
    // =============================================== stats warps ====
    float2 V01[kQPT], V23[kQPT], F01[kQPT], F23[kQPT];  // row-pass split of p
#pragma unroll
    for (int q = 0; q < kQPT; ++q) {
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
      for (int q = 0; q < kQPT; ++q) {
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
    float2 acc01[kQPT], acc23[kQPT], cmp01[kQPT], cmp23[kQPT];
#pragma unroll
    for (int q = 0; q < kQPT; ++q) {
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
        for (int q = 0; q < kQPT; ++q) {
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
    for (int q = 0; q < kQPT; ++q) {
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
           const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // columns of the rows the stream kernel skipped: out[j] = sum over the
  // listed rows (cluster order, then row order) of w_i ex2(t_ij), with the
  // exact split shift k_row_redo wrote into aux -- the k_col_fast formula
  if (ctrl->done || !ctrl->shift_valid) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kPatchThreads + threadIdx.x;
  if (j >= m) return;
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

long long*& sp_trace_buf() {
  static long long* p = nullptr;
  return p;
}

template <int CL>
cudaLaunchConfig_t sp_config(unsigned clusters, int smem, cudaStream_t stream,
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

template <int CL>
int sp_clusters(int smem) {
  OTG_CUDA(cudaFuncSetAttribute(k_sp<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchAttribute attr;
  cudaLaunchConfig_t cfg = sp_config<CL>(148, smem, nullptr, &attr);
  int ncl = 0;
  OTG_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k_sp<CL>, &cfg));
  return ncl;
}

}  // namespace

// Decide whether the single-pass path applies and size it (handle setup).
// Opt-in (OTG_FUSED=1): on B200 at n = m = 65536 it takes 6.4 ms per
// evaluation against 5.6 ms for the two-pass kernels -- the per-row chain
// (stats -> cluster exchange -> column step) costs ~2000 cycles of latency per
// row that the 16 warps do not hide (tools/sp_trace.py timeline,
// profiles/r01_single_pass.md).
bool fused_configure(Problem& P) {
  P.fused = 0;
  if (P.storage != OTG_STORE_F32 || P.vshards != 1) return false;
  const char* s = getenv("OTG_FUSED");
  if (!s || atoi(s) == 0) return false;
  const int CL = P.m <= 4 * kST * kQPT ? 1 : kCLMax;  // whole rows per CTA when they fit
  const int64_t W = round_up((P.m + CL - 1) / CL, 4);
  if (W * CL > P.ldc) return false;           // C rows must hold whole slices
  if (W > 4 * kST * kQPT) return false;       // columns per CTA held in registers
  if (P.n_local < 16 * 8 || P.m < 1024) return false;
  const int64_t head = ((sizeof(SpShared) + 127) / 128) * 128;
  const int64_t budget = 220 * 1024 - head;
  const int nslots = static_cast<int>(std::min<int64_t>(kSlotsMax, budget / (W * 4 + kST * 4)));
  if (nslots < 5) return false;
  const char* lag_env = getenv("OTG_SP_LAG");
  int lag = lag_env ? atoi(lag_env) : 3;
  lag = std::max(0, std::min(std::min(lag, kLagMax), nslots - 2));
  const int smem = static_cast<int>(head + static_cast<int64_t>(nslots) * (W * 4 + kST * 4));
  int ncl = CL == 1 ? sp_clusters<1>(smem) : sp_clusters<kCLMax>(smem);
  if (getenv("OTG_VERBOSE"))
    fprintf(stderr, "[otg] single-pass: CL=%d W=%lld smem=%d slots=%d lag=%d clusters=%d\n",
            CL, static_cast<long long>(W), smem, nslots, lag, ncl);
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
  return true;
}

void fused_alloc(Problem& P) {
  if (!P.fused) return;
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
void launch_fused(Problem& P, float kh, float kl) {
  RowRec* rec = reinterpret_cast<RowRec*>(P.sp_rec);
  launch_k(k_sp_prep, 296, 256, 0, P.stream, P.n_local, P.rowM2, P.rowJ, P.dq, P.a, P.loga, rec,
                                       P.ctrl);
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
  if (P.fused_cl == 1) {
    cudaLaunchConfig_t cfg = sp_config<1>(P.fused_clusters, P.fused_smem, P.stream, &attr);
    OTG_CUDA(cudaLaunchKernelEx(&cfg, k_sp<1>, A, static_cast<const Ctrl*>(P.ctrl)));
  } else {
    cudaLaunchConfig_t cfg = sp_config<kCLMax>(P.fused_clusters, P.fused_smem, P.stream, &attr);
    OTG_CUDA(cudaLaunchKernelEx(&cfg, k_sp<kCLMax>, A, static_cast<const Ctrl*>(P.ctrl)));
  }
  launch_sp_redo(P, P.sp_bad_rows, P.sp_bad_count, P.fused_clusters);
  const unsigned g = static_cast<unsigned>((P.m + kPatchThreads - 1) / kPatchThreads);
  launch_k(k_sp_patch, g, kPatchThreads, 0, P.stream, 
      P.C32, P.ldc, P.m, P.p, kh, kl, P.aux, P.sp_bad_rows, P.sp_bad_count, P.n_local,
      P.fused_clusters, P.part + static_cast<int64_t>(P.fused_clusters) * P.mpad, P.ctrl);
  OTG_CUDA(cudaGetLastError());
}

}  // namespace otg

// Debug: copy the single-pass kernel's timeline (OTG_SP_TRACE) to the host.
extern "C" int otg_debug_sp_trace(long long* out, int count) {
  long long* p = otg::sp_trace_buf();
  if (!p) return 1;
  if (cudaMemcpy(out, p, static_cast<size_t>(count) * sizeof(long long), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return 2;
  return 0;
}
