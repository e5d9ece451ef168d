// fused.cu — single-HBM-pass evaluation sweep for fp32 stored costs (sm_100a).
//
// One evaluation needs, per row i, the row sum S_i BEFORE the row can add
// w_i = a_i / S_i times its exponentials to the column sums (dual.cpp:34-41).
// The two-pass kernels of sweep.cu therefore read the cost twice.  Here the
// cost is read from HBM ONCE per evaluation by a persistent, grid-wide
// software pipeline (one CTA per SM):
//
//   columns   the m columns are cut into `group` contiguous quad-aligned
//             slices, one per CTA of a group (cfg3: 148 slices of ~444
//             columns); H = #SMs / group groups stream disjoint row bands
//             (band b of 16 rows goes to group b mod H)
//   load      warp 0 streams each band's 16 row segments (cp.async.bulk,
//             1.7 KB each at cfg3) into a smem ring (mbarrier full / empty)
//   row warps (4) e_ij = ex2(t_ij) against the row's shift ESTIMATE s_i (the
//             previous evaluation's base-2 row max plus the potential's move,
//             exactly as k_row_shift), kept in TENSOR MEMORY (tcgen05.st,
//             8 band slots of 64 columns x 128 lanes = the SM's 256 KB): the
//             element is never re-read from HBM and its exponential is never
//             recomputed.  Per row: the slice's partial sum as a 2^-40
//             fixed-point integer and the (max, argmax) as one ordered 64-bit
//             key, reduced in the warp (redux.sync), across the 4 warps
//             (smem), then across the group's CTAs by red.global.add/max --
//             integer arithmetic, so the row sums are deterministic -- and a
//             release increment of the band's arrival counter
//   col warps (4) wait for the band's counter to reach `group` (acquire),
//             read S_i and the key, w_i = a_i / S_i, tcgen05.ld the band's
//             exponentials and fold w_i e_ij into the slice's column sums
//             (fp32 over the band's 16 rows, then fp64); the band's owner CTA
//             writes the row outputs (u, M, S, w, M2, J, aux) and lists loose
//             rows
//
// The only grid-wide dependency is per band (16 rows), with 8 bands of
// tensor-memory slack between a CTA's row and column warps, so the counter
// latency is hidden behind ~5 us of streaming.  A row whose true max T
// relative to s_i falls outside [-2, 6] (the estimate was too loose) adds
// nothing here and is listed; k_sp_redo recomputes it exactly and k_sp_patch
// adds its columns in list order (both cheap: such rows are rare).
//
// Output: per-group column sums part[g][j] (g < H) plus one patch row
// part[H][j], summed in order by k_merge; u, rowM, rowS, wrow, rowM2, rowJ, aux.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace otg {

namespace {

constexpr int kR = 16;                 // rows per band
constexpr int kRowWarps = 4;           // warps 1..4 (TMEM lane quarters 1, 2, 3, 0)
constexpr int kColWarps = 4;           // warps 5..8 (same quarters)
constexpr int kThreads = 32 * (1 + kRowWarps + kColWarps);
constexpr int kQMax = 32 * kRowWarps;  // quads (4 columns) per CTA slice, at most
constexpr int kTSlots = 8;             // tensor-memory band slots (64 columns each)
constexpr int kRingMax = 8;            // smem band ring depth, at most
constexpr float kRedoLo = 2.0f;        // same window as sweep.cu k_row_shift
constexpr float kRedoHi = 6.0f;
constexpr int kPatchThreads = 256;

struct RowRec {  // per-row inputs (32 bytes)
  float shift;   // quantised base-2 shift estimate (k_sp_prep)
  int pad;
  double a, loga;
  double pad2;
};

struct S1Args {
  const RowRec* rec;
  const float* C;
  int64_t ldc, n, m, mpad;
  const float* vq;  // split potential of the row pass (Vc[mpad], vf[mpad])
  float kh, kl;
  double* rowM;
  double* rowS;
  double* u;
  double* wrow;
  float4* aux;
  double* rowM2;
  int* rowJ;
  double* part;                 // H rows of mpad
  unsigned long long* sfix;     // [2][n] fixed-point row sums
  unsigned long long* tkey;     // [2][n] (max, argmax) keys
  unsigned* cnt;                // [2][bands] arrivals, then [0] parity, [1] finished CTAs
  int* bad_rows;                // per CTA: bad_rows[cta * cap + k], k < bad_count[cta]
  int* bad_count;
  int64_t cap;
  int64_t bands;
  int64_t quads;                // ceil(m / 4)
  int H, group;                 // groups, CTAs per group
  int nslots;                   // smem ring depth
  int fix;                      // fixed-point scale 2^fix
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded waits: a pipeline that cannot make progress (a broken co-residency
// assumption, a bug) traps after ~seconds instead of hanging the device.
constexpr unsigned kSpinLimit = 1u << 28;
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  unsigned spins = 0;
  while (!mbar_try(bar, parity))
    if (++spins > kSpinLimit) __trap();
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned ordered_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// x * 2^fix rounded to an integer (x >= 0; zero, denormal or NaN -> 0, huge
// values saturate), on the integer pipe (no F2I on the XU pipe that carries
// the exponentials).  Exact function of x: the row sums are deterministic.
__device__ __forceinline__ unsigned long long to_fix(float x, int fix) {
  const unsigned b = __float_as_uint(x);
  const int e = static_cast<int>((b >> 23) & 0xffu);
  if (e == 0 || (b >> 31)) return 0ull;
  const unsigned long long mant = (b & 0x7fffffu) | 0x800000u;
  const int sh = e - 150 + fix;
  if (sh >= 0) return sh > 38 ? (1ull << 62) : (mant << sh);
  if (sh < -24) return 0ull;
  return (mant + (1ull << (-sh - 1))) >> (-sh);
}

// Warp sum of a 63-bit value as three 21-bit limbs (each redux.sync sum of 32
// lanes stays below 2^26).
__device__ __forceinline__ unsigned long long warp_sum_fix(unsigned long long v) {
  const unsigned l0 = static_cast<unsigned>(v & 0x1fffffull);
  const unsigned l1 = static_cast<unsigned>((v >> 21) & 0x1fffffull);
  const unsigned l2 = static_cast<unsigned>(v >> 42);
  const unsigned s0 = __reduce_add_sync(0xffffffffu, l0);
  const unsigned s1 = __reduce_add_sync(0xffffffffu, l1);
  const unsigned s2 = __reduce_add_sync(0xffffffffu, l2);
  return static_cast<unsigned long long>(s0) + (static_cast<unsigned long long>(s1) << 21) +
         (static_cast<unsigned long long>(s2) << 42);
}

// ---- tensor memory (tcgen05) ------------------------------------------------
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
// the loaded registers are defined only after wait::ld: tie them to the wait
__device__ __forceinline__ void tmem_wait_ld16(unsigned (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct alignas(16) S1Shared {
  uint64_t full[kRingMax];     // band loaded (TMA -> row warps)
  uint64_t empty[kRingMax];    // band consumed (row warps -> loader)
  uint64_t tfull[kTSlots];     // exponentials in TMEM (row warps -> column warps)
  uint64_t tempty[kTSlots];    // TMEM slot read (column warps -> row warps)
  unsigned long long wsum[2][kRowWarps][kR];  // per-warp partials of the band's rows
  unsigned long long wkey[2][kRowWarps][kR];
  float shift[2][kR];
  uint32_t tmem_base;
  int nbad;
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

__global__ void __launch_bounds__(kThreads, 1)
k_sweep1(const S1Args A, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done || !ctrl->shift_valid) return;  // uniform: written by earlier launches
  const int active = A.H * A.group;
  if (static_cast<int>(blockIdx.x) >= active) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S1Shared& S = *reinterpret_cast<S1Shared*>(smem_raw);
  float4* ring = reinterpret_cast<float4*>(smem_raw + ((sizeof(S1Shared) + 127) / 128) * 128);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x / A.group, k = blockIdx.x % A.group;
  const int64_t q0 = A.quads * k / A.group, q1 = A.quads * (k + 1) / A.group;
  const int nq = static_cast<int>(q1 - q0);
  const int64_t nb = A.bands > g ? (A.bands - g + A.H - 1) / A.H : 0;  // this group's bands
  const unsigned par = A.cnt[2 * A.bands];                           // buffer parity of this launch
  unsigned long long* sfix = A.sfix + static_cast<int64_t>(par) * A.n;
  unsigned long long* tkey = A.tkey + static_cast<int64_t>(par) * A.n;
  unsigned* cnt = A.cnt + static_cast<int64_t>(par) * A.bands;
  const int nslots = A.nslots;
  const uint32_t slot_elems = static_cast<uint32_t>(kR * nq);  // float4 per ring slot

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nslots; ++s) {
        mbar_init(&S.full[s], 1);
        mbar_init(&S.empty[s], kRowWarps);
      }
      for (int s = 0; s < kTSlots; ++s) {
        mbar_init(&S.tfull[s], kRowWarps);
        mbar_init(&S.tempty[s], kColWarps);
      }
      S.nbad = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // the whole tensor memory of the SM: 512 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&S.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ loader --
    if (lane == 0) {
      for (int64_t t = 0; t < nb; ++t) {
        const int s = static_cast<int>(t % nslots);
        if (t >= nslots) {
          mbar_wait(&S.empty[s], static_cast<uint32_t>((t / nslots - 1) & 1));
          // the row warps' generic-proxy reads of the slot precede the async refill
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t i0 = (g + A.H * t) * kR;
        const int rv = static_cast<int>((A.n - i0 < kR ? A.n - i0 : kR));
        mbar_expect_tx(&S.full[s], static_cast<uint32_t>(rv * nq * 16));
        float4* dst = ring + static_cast<size_t>(s) * slot_elems;
        for (int r = 0; r < rv; ++r)
          bulk_load(dst + r * nq, A.C + (i0 + r) * A.ldc + 4 * q0, static_cast<uint32_t>(nq * 16),
                    &S.full[s]);
      }
    }
  } else if (warp <= kRowWarps) {
    // ---------------------------------------------------------- row warps --
    const int qi = (warp - 1) * 32 + lane;  // this thread's quad of the slice
    const bool qvalid = qi < nq;
    const int64_t j0 = 4 * (q0 + qi);
    const uint32_t taddr0 = tbase + ((static_cast<uint32_t>(warp & 3) * 32u) << 16);
    float V[4], F[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool ok = qvalid && j0 + e < A.m;
      V[e] = ok ? A.vq[j0 + e] : -INFINITY;  // padded columns: ex2(-inf) = 0, never the max
      F[e] = ok ? A.vq[A.mpad + j0 + e] : 0.0f;
    }
    const float2 V01 = make_float2(V[0], V[1]), V23 = make_float2(V[2], V[3]);
    const float2 F01 = make_float2(F[0], F[1]), F23 = make_float2(F[2], F[3]);
    const float2 nkh2 = make_float2(-A.kh, -A.kh), nkl2 = make_float2(-A.kl, -A.kl);
    // the column-offset terms of the exponent do not depend on the row
    for (int64_t t = 0; t < nb; ++t) {
      const int s = static_cast<int>(t % nslots);
      const int ts = static_cast<int>(t % kTSlots);
      const int64_t b = g + A.H * t;
      const int64_t i0 = b * kR;
      const int rv = static_cast<int>((A.n - i0 < kR ? A.n - i0 : kR));
      const int pb = static_cast<int>(t & 1);
      // row shifts of the band (lane r holds row r's)
      const float sh_l = lane < rv ? A.rec[i0 + lane].shift : 0.0f;
      if (t >= kTSlots) {
        mbar_wait(&S.tempty[ts], static_cast<uint32_t>((t / kTSlots - 1) & 1));
        tc_fence_after();
      }
      mbar_wait(&S.full[s], static_cast<uint32_t>((t / nslots) & 1));
      const float4* slot = ring + static_cast<size_t>(s) * slot_elems;
      unsigned long long fx[kR];
      unsigned hk[kR], jk[kR];
#pragma unroll
      for (int sub = 0; sub < kR / 4; ++sub) {
        float E[16];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int r = sub * 4 + rr;
          const float sc = __shfl_sync(0xffffffffu, sh_l, r);
          float e0 = 0.f, e1 = 0.f, e2 = 0.f, e3 = 0.f;
          unsigned hkey = 0u, jj = 0xffffffffu;
          float psum = 0.f;
          if (r < rv && qvalid) {
            const float4 c = slot[r * nq + qi];
            const float2 c01 = make_float2(c.x, c.y), c23 = make_float2(c.z, c.w);
            const float2 nS = make_float2(-sc, -sc);
            const float2 t01 = __fadd2_rn(__ffma2_rn(c01, nkh2, __fadd2_rn(V01, nS)),
                                          __ffma2_rn(c01, nkl2, F01));
            const float2 t23 = __fadd2_rn(__ffma2_rn(c23, nkh2, __fadd2_rn(V23, nS)),
                                          __ffma2_rn(c23, nkl2, F23));
            e0 = ex2_approx(t01.x);
            e1 = ex2_approx(t01.y);
            e2 = ex2_approx(t23.x);
            e3 = ex2_approx(t23.y);
            psum = (e0 + e1) + (e2 + e3);
            const float mx = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
            hkey = ordered_key(mx);
            jj = static_cast<unsigned>(j0) + (t01.x == mx ? 0u : t01.y == mx ? 1u : t23.x == mx ? 2u : 3u);
          }
          E[4 * rr + 0] = e0;
          E[4 * rr + 1] = e1;
          E[4 * rr + 2] = e2;
          E[4 * rr + 3] = e3;
          fx[r] = to_fix(psum, A.fix);
          hk[r] = hkey;
          jk[r] = jj;
        }
        tmem_st16(taddr0 + static_cast<uint32_t>(ts * 64 + sub * 16), E);
      }
      // the slot's cost rows are no longer needed
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
      // warp-level row partials: sum (fixed point) and (max, lowest argmax)
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const unsigned long long sw = warp_sum_fix(fx[r]);
        const unsigned hm = __reduce_max_sync(0xffffffffu, hk[r]);
        const unsigned jm = __reduce_min_sync(0xffffffffu, hk[r] == hm ? jk[r] : 0xffffffffu);
        if (lane == r) {
          S.wsum[pb][warp - 1][r] = sw;
          S.wkey[pb][warp - 1][r] =
              (static_cast<unsigned long long>(hm) << 32) | static_cast<unsigned long long>(~jm);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tfull[ts]);
      // CTA partial of the band's rows -> the group's global sums
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kRowWarps) : "memory");
      if (warp == 1) {
        if (lane < rv) {
          unsigned long long sm = 0ull, km = 0ull;
#pragma unroll
          for (int w = 0; w < kRowWarps; ++w) {
            sm += S.wsum[pb][w][lane];
            km = max(km, S.wkey[pb][w][lane]);
          }
          atomicAdd(sfix + i0 + lane, sm);
          atomicMax(tkey + i0 + lane, km);
          __threadfence();
        }
        __syncwarp();
        if (lane == 0) red_release_add(cnt + b, 1u);
      }
    }
  } else {
    // ------------------------------------------------------- column warps --
    const int cw = warp - 1 - kRowWarps;  // 0..3
    const int qi = cw * 32 + lane;
    const bool qvalid = qi < nq;
    const int64_t j0 = 4 * (q0 + qi);
    const uint32_t taddr0 = tbase + ((static_cast<uint32_t>(warp & 3) * 32u) << 16);
    const bool owner_warp = cw == 0;
    const double scale = ldexp(1.0, -A.fix);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int nbad = 0;
    for (int64_t t = 0; t < nb; ++t) {
      const int ts = static_cast<int>(t % kTSlots);
      const int64_t b = g + A.H * t;
      const int64_t i0 = b * kR;
      const int rv = static_cast<int>((A.n - i0 < kR ? A.n - i0 : kR));
      // the group's partials of this band have all arrived
      for (unsigned spins = 0; ld_acquire(cnt + b) < static_cast<unsigned>(A.group);) {
        __nanosleep(64);
        if (++spins > (kSpinLimit >> 4)) __trap();
      }
      float w_l = 0.f;
      bool bad_l = true;
      double S_l = 1.0;
      float T_l = 0.f;
      unsigned J_l = 0u;
      if (lane < rv) {
        const unsigned long long sx = ld_relaxed64(sfix + i0 + lane);
        const unsigned long long kk = ld_relaxed64(tkey + i0 + lane);
        T_l = key_to_float(static_cast<unsigned>(kk >> 32));
        J_l = ~static_cast<unsigned>(kk & 0xffffffffull);
        S_l = static_cast<double>(sx) * scale;
        bad_l = !(T_l >= -kRedoLo && T_l <= kRedoHi) || !(S_l > 0.0);
        const RowRec rc = A.rec[i0 + lane];
        const double wi = rc.a / S_l;
        w_l = static_cast<float>(wi);
        if (owner_warp && (b / A.H) % A.group == k) {  // this CTA owns the band's rows
          const int64_t i = i0 + lane;
          if (!bad_l) {
            const double sc = static_cast<double>(rc.shift);
            const double M = sc * kLn2;
            A.rowM[i] = M;
            A.rowS[i] = S_l;
            A.u[i] = (rc.loga - M) - log(S_l);
            A.wrow[i] = wi;
            A.rowM2[i] = sc + static_cast<double>(T_l);
            A.rowJ[i] = static_cast<int>(J_l);
            A.aux[i] = make_float4(rc.shift, 0.0f, w_l, 0.0f);
          }
          // zero the other parity's slots for the next launch
          A.sfix[static_cast<int64_t>(par ^ 1u) * A.n + i] = 0ull;
          A.tkey[static_cast<int64_t>(par ^ 1u) * A.n + i] = 0ull;
        }
      }
      if (owner_warp && (b / A.H) % A.group == k) {
        const unsigned bm = __ballot_sync(0xffffffffu, lane < rv && bad_l);
        if (lane < rv && bad_l)
          A.bad_rows[blockIdx.x * A.cap + nbad + __popc(bm & ((1u << lane) - 1u))] =
              static_cast<int>(i0 + lane);
        nbad += __popc(bm);
        if (lane == 0) A.cnt[static_cast<int64_t>(par ^ 1u) * A.bands + b] = 0u;
      }
      // the band's exponentials
      mbar_wait(&S.tfull[ts], static_cast<uint32_t>((t / kTSlots) & 1));
      tc_fence_after();
      float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
      for (int sub = 0; sub < kR / 4; ++sub) {
        unsigned E[16];
        tmem_ld16(taddr0 + static_cast<uint32_t>(ts * 64 + sub * 16), E);
        tmem_wait_ld16(E);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int r = sub * 4 + rr;
          const float wr = __shfl_sync(0xffffffffu, w_l, r);
          const bool br = __shfl_sync(0xffffffffu, bad_l ? 1 : 0, r) != 0;
          if (!br) {  // uniform over the warp (one row)
            const float2 w2 = make_float2(wr, wr);
            a01 = __ffma2_rn(make_float2(__uint_as_float(E[4 * rr]), __uint_as_float(E[4 * rr + 1])),
                             w2, a01);
            a23 = __ffma2_rn(make_float2(__uint_as_float(E[4 * rr + 2]),
                                         __uint_as_float(E[4 * rr + 3])),
                             w2, a23);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tempty[ts]);
      acc[0] += static_cast<double>(a01.x);
      acc[1] += static_cast<double>(a01.y);
      acc[2] += static_cast<double>(a23.x);
      acc[3] += static_cast<double>(a23.y);
    }
    if (qvalid) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j0 + e < A.m) A.part[static_cast<int64_t>(g) * A.mpad + j0 + e] = acc[e];
    }
    if (owner_warp && lane == 0) A.bad_count[blockIdx.x] = nbad;
  }
  // teardown: free the tensor memory, flip the buffer parity after the last CTA
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    if (lane == 0) {
      __threadfence();
      unsigned* fin = A.cnt + 2 * A.bands + 1;
      if (atomicAdd(fin, 1u) == static_cast<unsigned>(active - 1)) {
        *fin = 0u;
        A.cnt[2 * A.bands] = par ^ 1u;
        __threadfence();
      }
    }
  }
}

__global__ void __launch_bounds__(kPatchThreads)
k_sp_patch(const float* __restrict__ C, int64_t ldc, int64_t m, const double* __restrict__ p,
           float kh, float kl, const float4* __restrict__ aux, const int* __restrict__ bad_rows,
           const int* __restrict__ bad_count, int nlists, int64_t cap, double* __restrict__ out,
           const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // columns of the rows the single pass skipped: out[j] = sum over the listed
  // rows (list order, then row order) of w_i ex2(t_ij), with the exact split
  // shift k_sp_redo wrote into aux -- the k_col_fast formula
  if (ctrl->done || !ctrl->shift_valid) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kPatchThreads + threadIdx.x;
  if (j >= m) return;
  const double x2 = p[j] * kLog2e;
  const double h = rint(x2 * 256.0) * (1.0 / 256.0);
  const float Vc = static_cast<float>(h), vf = static_cast<float>(x2 - h);
  double acc = 0.0;
  for (int c = 0; c < nlists; ++c) {
    const int nbad = bad_count[c];
    for (int q = 0; q < nbad; ++q) {
      const int64_t i = bad_rows[c * cap + q];
      const float4 ax = aux[i];
      const float cc = C[i * ldc + j];
      const float Aq = Vc - ax.x;
      const float gq = fmaf(-cc, kl, vf - ax.y);
      const float t = fmaf(-cc, kh, Aq) + gq;
      acc += static_cast<double>(ax.z * ex2_approx(t));
    }
  }
  out[j] = acc;
}

}  // namespace

// Decide whether the single-pass path applies and size it (handle setup).
// fp32 stored cost, no virtual shards (they use the two-pass kernels),
// m <= 128 quads per SM over the whole GPU, and the handle did not ask for
// the two-pass kernels (otg_device_opts.sweep = 1: A/B and cross-checks).
bool fused_configure(Problem& P) {
  P.fused = 0;
  if (P.storage != OTG_STORE_F32 || P.vshards != 1 || P.two_pass) return false;
  int sms = 0;
  OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  const int64_t quads = (P.m + 3) / 4;
  const int64_t min_group = (quads + kQMax - 1) / kQMax;
  if (min_group > sms || P.m < 256 || P.n_local < 2 * kR) return false;
  const int H = static_cast<int>(std::max<int64_t>(1, sms / min_group));
  const int group = sms / H;
  const int64_t qmax = (quads + group - 1) / group;
  const int64_t head = ((sizeof(S1Shared) + 127) / 128) * 128;
  const int64_t slot = kR * qmax * 16;
  const int64_t budget = 220 * 1024 - head;
  const int nslots = static_cast<int>(std::min<int64_t>(kRingMax, budget / slot));
  if (nslots < 3) return false;
  const int smem = static_cast<int>(head + nslots * slot);
  OTG_CUDA(cudaFuncSetAttribute(k_sweep1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep1, kThreads, smem));
  if (occ < 1) return false;
  // fixed-point scale: a CTA's row partial is at most 64 x (columns per CTA)
  // (exponents <= 6 after the redo test), the group's sum 64 x m; keep 2^62 headroom
  int fix = 40;
  while (fix > 24 && std::ldexp(64.0 * static_cast<double>(P.m + 4 * kQMax), fix) >= std::ldexp(1.0, 61))
    --fix;
  P.fused = 1;
  P.fused_clusters = H;
  P.sp_group = group;
  P.fused_slots = nslots;
  P.fused_smem = smem;
  P.sp_fix = fix;
  P.sp_bands = (P.n_local + kR - 1) / kR;
  P.sp_cap = kR * ((P.sp_bands + static_cast<int64_t>(H) * group - 1) / (static_cast<int64_t>(H) * group) + 1);
  if (getenv("OTG_VERBOSE"))
    fprintf(stderr, "[otg] single-pass: groups=%d x %d CTAs, quads/CTA<=%lld, smem=%d, slots=%d, fix=%d\n",
            H, group, static_cast<long long>(qmax), smem, nslots, fix);
  return true;
}

void fused_alloc(Problem& P) {
  if (!P.fused) return;
  const int64_t n = P.n_local;
  P.sp_rec = dalloc<double>(P, static_cast<size_t>(n) * (sizeof(RowRec) / 8));
  const int ctas = P.fused_clusters * P.sp_group;
  P.sp_bad_rows = dalloc<int>(P, static_cast<size_t>(ctas) * P.sp_cap);
  P.sp_bad_count = dalloc<int>(P, ctas);
  P.sp_sums = dalloc<unsigned long long>(P, 4 * static_cast<size_t>(n));
  P.sp_cnt = dalloc<unsigned>(P, 2 * static_cast<size_t>(P.sp_bands) + 2);
  OTG_CUDA(cudaMemsetAsync(P.sp_bad_count, 0, ctas * sizeof(int), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.sp_sums, 0, 4 * static_cast<size_t>(n) * sizeof(unsigned long long),
                           P.stream));
  OTG_CUDA(cudaMemsetAsync(P.sp_cnt, 0, (2 * static_cast<size_t>(P.sp_bands) + 2) * sizeof(unsigned),
                           P.stream));
}

// Steady-state evaluation sweep (launched after the exact-path kernels, each
// of which returns at once when the other applies): single pass, redo of the
// loose rows, their column patch into partial row H.
void launch_fused(Problem& P, float kh, float kl) {
  RowRec* rec = reinterpret_cast<RowRec*>(P.sp_rec);
  launch_k(k_sp_prep, 296, 256, 0, P.stream, P.n_local, P.rowM2, P.rowJ, P.dq, P.a, P.loga, rec,
           P.ctrl);
  S1Args A;
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
  A.sfix = static_cast<unsigned long long*>(P.sp_sums);
  A.tkey = A.sfix + 2 * P.n_local;
  A.cnt = P.sp_cnt;
  A.bad_rows = P.sp_bad_rows;
  A.bad_count = P.sp_bad_count;
  A.cap = P.sp_cap;
  A.bands = P.sp_bands;
  A.quads = (P.m + 3) / 4;
  A.H = P.fused_clusters;
  A.group = P.sp_group;
  A.nslots = P.fused_slots;
  A.fix = P.sp_fix;
  const int ctas = P.fused_clusters * P.sp_group;
  // co-residency of the whole grid is required (grid-wide band counters):
  // a cooperative launch guarantees it or fails
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ctas));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = P.fused_smem;
  cfg.stream = P.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OTG_CUDA(cudaLaunchKernelEx(&cfg, k_sweep1, A, static_cast<const Ctrl*>(P.ctrl)));
  launch_sp_redo(P, P.sp_bad_rows, P.sp_bad_count, ctas, P.sp_cap);
  const unsigned g = static_cast<unsigned>((P.m + kPatchThreads - 1) / kPatchThreads);
  launch_k(k_sp_patch, g, kPatchThreads, 0, P.stream, P.C32, P.ldc, P.m, P.p, kh, kl, P.aux,
           P.sp_bad_rows, P.sp_bad_count, ctas, P.sp_cap,
           P.part + static_cast<int64_t>(P.fused_clusters) * P.mpad, P.ctrl);
  OTG_CUDA(cudaGetLastError());
}

}  // namespace otg
