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
//             recomputed.  Per row: the slice's partial sum as a 2^-28
//             fixed-point integer and the (max, argmax) as one ordered 64-bit
//             key, reduced in the warp (redux.sync) and across the 4 warps
//             (smem), then across the group's CTAs by ONE red.global.add per
//             row whose low 8 bits count the arriving CTAs (integer
//             arithmetic: deterministic row sums; the sum and its completeness
//             travel in the same word, so no fence or flag is needed) and a
//             red.global.max of the key (read only by the next evaluation's
//             k_sp_prep, after the kernel boundary)
//   col warps (4) poll the band's 16 sum words until the count reaches
//             `group`, w_i = a_i / S_i, tcgen05.ld the band's exponentials and
//             fold w_i e_ij into the slice's column sums (fp32 over the band's
//             16 rows, then fp64); the band's owner CTA writes the row outputs
//             (u, M, S, w, aux) and lists loose rows
//
// The only grid-wide dependency is per band (16 rows), with 8 bands of
// tensor-memory slack between a CTA's row and column warps, so the atomic
// latency is hidden behind ~5 us of streaming.  A row whose sum is outside
// [1/4, 2^20] (shift estimate too loose for the fixed-point range) adds
// nothing here and is listed; k_sp_redo recomputes it exactly and k_sp_patch
// adds its columns in list order (both cheap: such rows are rare).
//
// Output: per-group column sums part[g][j] (g < H) plus one patch row
// part[H][j], summed in order by k_merge; u, rowM, rowS, wrow, rowM2, rowJ, aux.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

#ifndef SP_EXPER
#define SP_EXPER 0  // (timing experiments only: 1 = no TMEM store, 2 = no ex2)
#endif

namespace otg {

namespace {

#ifndef SP_ROWS
#define SP_ROWS 16
#endif
constexpr int kR = SP_ROWS;            // rows per band
constexpr int kRowWarps = 8;           // warps 1..8: bands t = w-1 mod 8 (two per TMEM lane quarter)
constexpr int kColWarps = 4;           // warps 5..8: the same quarters and bands
#ifndef SP_UNROLL
#define SP_UNROLL 2
#endif
constexpr int kUnroll = SP_UNROLL;     // row pairs interleaved by the compiler
#ifndef SP_LOADERS
#define SP_LOADERS 0
#endif
// loader warps (bands t = l mod kLoaders); 0: no loader warp -- the second of
// a band's two row warps to finish with its ring slot issues the slot's next
// band (12 warps instead of 13: 3 per SMSP, so up to 168 registers each)
constexpr int kLoaders = SP_LOADERS;
constexpr int kThreads = 32 * (kLoaders + kRowWarps + kColWarps);
constexpr int kQPL = 4;                // quads (4 columns) per lane: a lane covers 16 columns
constexpr int kQMax = 32 * kQPL;       // quads per CTA slice, at most (one warp covers it)
constexpr int kTCols = kR * 4 * kQPL;  // tensor-memory columns of one band slot
constexpr int kTPerQ = 512 / kTCols;   // band slots per lane quarter
constexpr int kTSlots = 4 * kTPerQ;    // bands in tensor memory (t mod kTSlots)
constexpr int kRingMax = 16;           // smem band ring depth, at most
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
  unsigned long long* sfix;     // [2][n] fixed-point row sums << 8 | arrivals
  unsigned long long* tkey;     // [2][n] (max, argmax) keys
  unsigned* state;              // [0] buffer parity of the next launch, [1] finished CTAs
  int* bad_rows;                // per CTA: bad_rows[cta * cap + k], k < bad_count[cta]
  int* bad_count;
  int64_t cap;
  int W;                        // slice width (columns) per CTA; CTA k: [k W, (k+1) W) of m
  unsigned long long* dbg;      // optional timeline (otg_debug_sp_trace): [cta 0, last][8][band]                // ceil(m / 4)
  int H, group;                 // groups, CTAs per group
  int nslots;                   // smem ring depth
  int nch;                      // TMA box: {cw columns, nch chunks, 16 rows}, W = cw nch
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
// try_wait with a suspend-time hint: a waiting warp is parked (up to the
// hint) instead of spinning on issue slots the row warps of its SMSP need
#ifndef SP_SUSPEND_NS
#define SP_SUSPEND_NS 0  // try_wait suspend-time hint (0: the instruction's default)
#endif
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if SP_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(static_cast<unsigned>(SP_SUSPEND_NS))
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
#ifndef SP_BACKOFF_NS
#define SP_BACKOFF_NS 64  // sleep between failed mbarrier tests (spinning warps steal issue slots)
#endif
#ifndef SP_POLL_NS
#define SP_POLL_NS 128    // sleep between polls of a band's row-sum words
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  unsigned spins = 0;
  while (!mbar_try(bar, parity)) {
    if (SP_BACKOFF_NS > 0) __nanosleep(SP_BACKOFF_NS);
    if (++spins > (kSpinLimit >> 8)) __trap();
  }
}
// 3-D tensor copy (TMA) of box {cw, nch, 16} at (x, chunk, row); rows past
// the matrix are zero-filled (and still counted in the bytes)
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int x, int c,
                                            int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(c), "r"(y), "r"(smem_u32(bar))
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

constexpr int kFix = 28;  // fixed-point scale 2^kFix of the row sums
// Row keys carry the largest QUAD SUM of exponentials (and its quad) instead
// of the largest exponent: 1 FADD per quad instead of 3 FMNMX.  The next
// evaluation's shift estimate takes M2 = s + log2(quad sum), an upper bound on
// the row's base-2 max within +2 (the estimate's upper bound U = M2 + dmax2
// stays valid), and the quad -- which holds an element within 2 of the max --
// for the lower bound L (an actual element of the new row, as before).
#ifndef SP_QSUM
#define SP_QSUM 1
#endif
constexpr unsigned long long kFixSat = 1ull << 48;  // = 2^20 in real units: the loose-row bound
static_assert(kFix == 28, "band_rows scales by 268435456.0f = 2^28");

// Warp reduction of one row's lane partials: the fixed-point sum (values
// <= 2^48) as two 24-bit limbs through redux.sync (each 32-lane limb sum
// stays below 2^29; integer: deterministic), the max exponent key through
// redux.sync.max, and the argmax quad as the lowest lane holding the max.
__device__ __forceinline__ void warp_row(unsigned long long v, unsigned hkey,
                                         unsigned long long& sum, unsigned& hmax,
                                         unsigned& lane_of_max) {
  const unsigned lo = static_cast<unsigned>(v & 0xffffffull);
  const unsigned hi = static_cast<unsigned>(v >> 24);
  const unsigned slo = __reduce_add_sync(0xffffffffu, lo);
  const unsigned shi = __reduce_add_sync(0xffffffffu, hi);
  hmax = __reduce_max_sync(0xffffffffu, hkey);
  lane_of_max = static_cast<unsigned>(__ffs(__ballot_sync(0xffffffffu, hkey == hmax)) - 1);
  sum = (static_cast<unsigned long long>(shi) << 24) + slo;
}

// ---- tensor memory (tcgen05) ------------------------------------------------
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kDbgBands = 256;
__device__ __forceinline__ void stamp(const S1Args& A, int what, int64_t t) {
  if (A.dbg && t < kDbgBands && (blockIdx.x == 0 || blockIdx.x == A.H * A.group - 1))
    A.dbg[((blockIdx.x == 0 ? 0 : 1) * 12 + what) * kDbgBands + t] = gtimer();
}

struct alignas(16) S1Shared {
  uint64_t full[kRingMax];     // band loaded (TMA -> row warp)
  uint64_t empty[kRingMax];    // band consumed (row warp -> loader)
  uint64_t tfull[kTSlots];     // exponentials in TMEM (row warp -> column warp)
  uint64_t tempty[kTSlots];    // TMEM slot read (column warp -> row warp)
  int slot_band[kRingMax];     // band the loader last issued into each ring slot
  int rel[kRingMax];           // (no loader warp) row warps done with the slot's band
  uint32_t tmem_base;
};

// Per-row record of the steady state: the quantised shift estimate
// s = ceil(min(L + 1, U) 256) / 256 (as k_row_shift).  U = M2 + dmax2 bounds
// the new row max from above (M2: the previous evaluation's base-2 max).  The
// lower bound L is an actual element of the NEW row: the largest exponent,
// at the new potential, of the four columns of the previous argmax's quad
// (the old argmax column is one of them, so L >= its new exponent, the bound
// k_row_shift uses) -- one 16-byte read of C per row.  Rows the previous
// single pass finished (rowJ = -1) take M2 = s_prev + T and the quad from
// that pass's key (complete now: kernel boundary).
__global__ void __launch_bounds__(256)
k_sp_prep(int64_t n, int64_t m, const float* __restrict__ C, int64_t ldc,
          const float* __restrict__ vq, int64_t mpad, float kh, float kl,
          double* __restrict__ rowM2, int* __restrict__ rowJ, const double* __restrict__ a,
          const double* __restrict__ loga, RowRec* __restrict__ rec,
          const unsigned long long* __restrict__ tkey, unsigned* __restrict__ state,
          Ctrl* __restrict__ ctrl, int steady) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  if (ctrl->done) return;
  if (!ctrl->shift_valid) {
    // the steady graph has no exact-path kernels: an evaluation without shift
    // estimates there (a non-finite step) ends the solve with an error
    if (steady && blockIdx.x == 0 && threadIdx.x == 0) {
      ctrl->error = OTG_E_OT;
      ctrl->done = 1;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[2] = 0u;       // loose rows listed by this evaluation
    ctrl->fin_done = 0;  // (k_sp_patch_merge may finalize this evaluation)
  }
  const double dmax2 = ctrl->dmax2;
  const unsigned long long* prev = tkey + static_cast<int64_t>(state[0] ^ 1u) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    double M2;
    int J = rowJ[i];
    if (J == -1) {
      const unsigned long long kk = prev[i];
#if SP_QSUM
      const double qs = static_cast<double>(key_to_float(static_cast<unsigned>(kk >> 32)));
      M2 = static_cast<double>(rec[i].shift) + (qs > 0.0 ? log2(qs) : 0.0);
#else
      M2 = static_cast<double>(rec[i].shift) +
           static_cast<double>(key_to_float(static_cast<unsigned>(kk >> 32)));
#endif
      J = 4 * static_cast<int>(~static_cast<unsigned>(kk & 0xffffffffull));
      rowM2[i] = M2;
      rowJ[i] = J;
    } else {
      M2 = rowM2[i];
    }
    const int64_t j0 = 4 * (J / 4);
    const float4 c = *reinterpret_cast<const float4*>(C + i * ldc + j0);
    const float cc[4] = {c.x, c.y, c.z, c.w};
    float lo = -INFINITY;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j0 + e < m)
        lo = fmaxf(lo, fmaf(-cc[e], kh, vq[j0 + e]) + fmaf(-cc[e], kl, vq[mpad + j0 + e]));
    const double hi = M2 + dmax2;
    RowRec r;
    r.shift = static_cast<float>(ceil(fmin(static_cast<double>(lo) + 1.0, hi) * 256.0) * (1.0 / 256.0));
    r.pad = 0;
    r.a = a[i];
    r.loga = loga[i];
    r.pad2 = 0.0;
    rec[i] = r;
  }
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]),
      "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]),
      "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16f(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]),
        "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]),
        "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr)
      : "memory");
}

// K (1 or 2) rows of a band for one lane's 16 columns (quads lane + 32 kq) from the
// smem slot (row stride rs4 float4):
// exponents against each row's shift (bitwise the k_row_shift exponents,
// sweep.cu quad_exponents), ex2 into E (tensor memory order: row, quad, 4),
// the lane's fixed-point row partials (fp32 sum of its 16 elements) and the
// (max, argmax quad) of its elements.  FULL: both rows exist (no masking).
template <bool FULL, int K>
__device__ __forceinline__ void row_pair(const float4* __restrict__ slot,
                                         float sh_l, int r0, int rv, int rs4,
                                         const int (&off)[kQPL], const float (&V)[kQPL][4],
                                         const float (&F)[kQPL][4], float2 nkh2, float2 nkl2,
                                         float (&E)[16 * K], unsigned long long (&fxr)[K],
                                         unsigned (&hkr)[K], unsigned (&qbr)[K]) {
#pragma unroll
  for (int h = 0; h < K; ++h) {
    const int r = r0 + h;
    const bool live = FULL || r < rv;
    const int rr = FULL ? r : (live ? r : 0);
    const float sc = __shfl_sync(0xffffffffu, sh_l, rr);  // (lane r holds row r's shift)
    const float2 nS = make_float2(-sc, -sc);
    const float4* row = slot + rr * rs4;  // (rs4: float4 per slot row)
    float4 c[kQPL];
#pragma unroll
    for (int kq = 0; kq < kQPL; ++kq) c[kq] = row[off[kq]];
    float2 ps = make_float2(0.f, 0.f);
    float mq[kQPL];
#pragma unroll
    for (int kq = 0; kq < kQPL; ++kq) {
      const float2 c01 = make_float2(c[kq].x, c[kq].y), c23 = make_float2(c[kq].z, c[kq].w);
      const float2 t01 = __fadd2_rn(
          __ffma2_rn(c01, nkh2, __fadd2_rn(make_float2(V[kq][0], V[kq][1]), nS)),
          __ffma2_rn(c01, nkl2, make_float2(F[kq][0], F[kq][1])));
      const float2 t23 = __fadd2_rn(
          __ffma2_rn(c23, nkh2, __fadd2_rn(make_float2(V[kq][2], V[kq][3]), nS)),
          __ffma2_rn(c23, nkl2, make_float2(F[kq][2], F[kq][3])));
      float e0 = ex2_approx(t01.x), e1 = ex2_approx(t01.y);
      float e2 = ex2_approx(t23.x), e3 = ex2_approx(t23.y);
      if (!FULL && !live) e0 = e1 = e2 = e3 = 0.0f;
      E[16 * h + 4 * kq + 0] = e0;
      E[16 * h + 4 * kq + 1] = e1;
      E[16 * h + 4 * kq + 2] = e2;
      E[16 * h + 4 * kq + 3] = e3;
#if SP_QSUM
      const float2 s2 = __fadd2_rn(make_float2(e0, e1), make_float2(e2, e3));
      ps = __fadd2_rn(ps, s2);
      mq[kq] = s2.x + s2.y;  // the quad's sum: max element <= it <= 4 x max element
#else
      ps = __fadd2_rn(ps, __fadd2_rn(make_float2(e0, e1), make_float2(e2, e3)));
      mq[kq] = fmaxf(fmaxf(t01.x, t01.y), fmaxf(t23.x, t23.y));
#endif
    }
    // argmax quad: the lowest of equal maxima
    const float m01 = fmaxf(mq[0], mq[1]), m23 = fmaxf(mq[2], mq[3]);
    const unsigned q01 = mq[1] > mq[0] ? 1u : 0u, q23 = mq[3] > mq[2] ? 3u : 2u;
    const float mx = fmaxf(m01, m23);
    qbr[h] = m23 > m01 ? q23 : q01;
    // fixed-point partial of the lane's 16 elements (fp32, <= 16 terms):
    // x 2^kFix is exact, the conversion saturates, the clamp marks rows past
    // the range (redone exactly)
    const unsigned long long v = __float2ull_rn((ps.x + ps.y) * 268435456.0f);
    fxr[h] = v < kFixSat ? v : kFixSat;
    hkr[h] = (FULL || live) ? ordered_key(mx) : 0u;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
k_sweep1(const S1Args A, const __grid_constant__ CUtensorMap cmap, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done || !ctrl->shift_valid) return;  // uniform: written by earlier launches
  const int active = A.H * A.group;
  if (static_cast<int>(blockIdx.x) >= active) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S1Shared& S = *reinterpret_cast<S1Shared*>(smem_raw);
  float4* ring = reinterpret_cast<float4*>(smem_raw + ((sizeof(S1Shared) + 127) / 128) * 128);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x / A.group, k = blockIdx.x % A.group;
  const int64_t q0 = static_cast<int64_t>(k) * (A.W / 4);                  // first quad
  const int64_t wk = A.m - 4 * q0 < A.W ? A.m - 4 * q0 : A.W;
  const int nq = static_cast<int>((wk + 3) / 4);  // quads of the slice
  const int rs4 = A.W / 4;                                                  // float4 per slot row
  const int64_t bands = (A.n + kR - 1) / kR;
  const int64_t nb = bands > g ? (bands - g + A.H - 1) / A.H : 0;  // this group's bands
  const unsigned par = A.state[0];  // buffer parity of this launch
  unsigned long long* sfix = A.sfix + static_cast<int64_t>(par) * A.n;
  unsigned long long* tkey = A.tkey + static_cast<int64_t>(par) * A.n;
  const int nslots = A.nslots;
  // ring slot: one band's [16 rows][W columns] (one TMA box; rows past n and
  // columns past m are zero-filled / masked)
  const uint32_t slot_f4 = static_cast<uint32_t>(kR * rs4);
  const uint32_t slot_bytes = slot_f4 * 16u;
  auto band_row0 = [&](int64_t t) { return (g + A.H * t) * kR; };

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nslots; ++s) {
        mbar_init(&S.full[s], 1);
        mbar_init(&S.empty[s], 2);  // both half-band row warps
        S.slot_band[s] = -1;
        S.rel[s] = 0;
      }
      for (int s = 0; s < kTSlots; ++s) {
        mbar_init(&S.tfull[s], 2);  // both half-band row warps
        mbar_init(&S.tempty[s], 1);
      }
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
  // ONE tensor copy per band: the 3-D view {cw, chunks, rows} of the cost
  // puts the slice's [16][W] block in one box (copy-engine cost is per box)
  auto issue_band = [&](int64_t t, int s) {
    mbar_expect_tx(&S.full[s], slot_bytes);
    // (after the expect: a row warp that sees band t here waits on the right phase)
    *reinterpret_cast<volatile int*>(&S.slot_band[s]) = static_cast<int>(t);
    tma_load_3d(ring + s * slot_f4, &cmap, 0, k * A.nch, static_cast<int>(band_row0(t)),
                &S.full[s]);
    stamp(A, 0, t);
  };
  if (kLoaders == 0 && warp == 0 && lane == 0)
    for (int64_t t = 0; t < nb && t < nslots; ++t) issue_band(t, static_cast<int>(t));
  // band t: row warp (t mod 8) + 1, column warp t mod 4; TMEM lane quarter of
  // those warps, column slot (t / 4) mod kTPerQ; barriers indexed t mod kTSlots
  auto tmem_of = [&](int w, int64_t t) {
    return tbase + ((static_cast<uint32_t>(w & 3) * 32u) << 16) +
           static_cast<uint32_t>(((t >> 2) % kTPerQ) * kTCols);
  };

  if (warp < kLoaders) {
    // ----------------------------------------------------------- loaders --
    if (lane == 0) {
      for (int64_t t = warp; t < nb; t += kLoaders) {
        const int s = static_cast<int>(t % nslots);
        if (t >= nslots) {
          // the slot's previous band (another loader's) must have been issued
          // before its release can be waited on (parity aliasing, as below)
          for (unsigned spins = 0;
               *reinterpret_cast<volatile int*>(&S.slot_band[s]) != static_cast<int>(t - nslots);
               ++spins) {
            __nanosleep(32);
            if (spins > (kSpinLimit >> 4)) __trap();
          }
          mbar_wait(&S.empty[s], static_cast<uint32_t>((t / nslots - 1) & 1));
          // the row warp's generic-proxy reads of the slot precede the async refill
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        issue_band(t, s);
      }
    }
  } else if (warp < kLoaders + kRowWarps) {
    // ---------------------------------------------------------- row warps --
    // Warp w streams bands t = w-1 (mod 8) alone: lane L covers quads L, L+32,
    // L+64, L+96 of the slice (16 columns per row), so the per-row warp
    // reduction is amortised over 16 elements per lane; two row warps share
    // each SMSP (and TMEM lane quarter), so one's reductions and waits
    // overlap the other's exponentials.
    // warps w and w + 4 (same TMEM lane quarter) take the two halves of
    // the bands t = w mod 4, so a ring slot is held for half a band's work
    const int wq = (warp - kLoaders) % 4;      // bands t = wq mod 4
    const int hr = (kR / 2) * ((warp - kLoaders) / 4);  // first row of this warp's half
    bool qv[kQPL];
    float V[kQPL][4], F[kQPL][4];
#pragma unroll
    for (int kq = 0; kq < kQPL; ++kq) {
      const int qi = lane + 32 * kq;
      qv[kq] = qi < nq;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t j = 4 * (q0 + qi) + e;
        const bool ok = qv[kq] && j < A.m;
        V[kq][e] = ok ? A.vq[j] : -INFINITY;  // padded columns: ex2(-inf) = 0, never the max
        F[kq][e] = ok ? A.vq[A.mpad + j] : 0.0f;
      }
    }
    const float2 nkh2 = make_float2(-A.kh, -A.kh), nkl2 = make_float2(-A.kl, -A.kl);
    // this lane's quads in a slot row (absent quads read quad 0, V = -inf)
    int off[kQPL];
#pragma unroll
    for (int kq = 0; kq < kQPL; ++kq) off[kq] = qv[kq] ? lane + 32 * kq : 0;
    // row shifts of the warp's next band, loaded one band ahead (lane r: row r)
    auto shift_of = [&](int64_t t) {
      const int64_t i = band_row0(t) + lane;
      return (lane < kR && t < nb && i < A.n) ? A.rec[i].shift : 0.0f;
    };
    float sh_next = shift_of(wq);
    for (int64_t t = wq; t < nb; t += 4) {
      const int s = static_cast<int>(t % nslots);
      const int ts = static_cast<int>(t % kTSlots);
      const int64_t i0 = band_row0(t);
      const int rv = static_cast<int>(A.n - i0 < kR ? A.n - i0 : kR);
      const float sh_l = sh_next;
      sh_next = shift_of(t + 4);
      if (t >= kTSlots) {
        mbar_wait(&S.tempty[ts], static_cast<uint32_t>((t / kTSlots - 1) & 1));
        tc_fence_after();
      }
      if (lane == 0) stamp(A, 1, t);
      // several row warps share a ring slot: wait until the loader has moved
      // the slot to this band before waiting on its phase (an mbarrier parity
      // wait cannot tell a phase two ahead from the completed one)
      for (unsigned spins = 0;
           *reinterpret_cast<volatile int*>(&S.slot_band[s]) != static_cast<int>(t); ++spins) {
        __nanosleep(64);
        if (spins > (kSpinLimit >> 4)) __trap();
      }
      mbar_wait(&S.full[s], static_cast<uint32_t>((t / nslots) & 1));
      if (lane == 0) stamp(A, 2, t);
      const float4* slot = ring + s * slot_f4;
      const uint32_t taddr = tmem_of(warp, t);
      unsigned long long my_sum = 0ull, my_key = 0ull;  // lane r: row r's warp totals
      // this warp's rows hr .. hr + kR/2 - 1: pairs, then a single row when kR/2 is odd
      auto fold_rows = [&](auto kk, int r) {
        constexpr int K = decltype(kk)::value;
        float E[16 * K];
        unsigned long long fxr[K];
        unsigned hkr[K], qbr[K];
        // (rows past the matrix are zero-filled by the copy and have shift 0:
        // their values are finite and never used -- not published, weight 0)
        row_pair<true, K>(slot, sh_l, r, rv, rs4, off, V, F, nkh2, nkl2, E, fxr, hkr, qbr);
        if constexpr (K == 2)
          tmem_st32(taddr + static_cast<uint32_t>(r * 16), E);
        else
          tmem_st16f(taddr + static_cast<uint32_t>(r * 16), E);
        // warp totals of the rows (integer sums: deterministic)
#pragma unroll
        for (int h = 0; h < K; ++h) {
          unsigned long long sw;
          unsigned hm, lm;
          warp_row(fxr[h], hkr[h], sw, hm, lm);
          const unsigned qm = static_cast<unsigned>(q0) + lm +
                              32u * __shfl_sync(0xffffffffu, qbr[h], static_cast<int>(lm));
          if (lane == r + h) {
            my_sum = sw;
            // (max, quad) as one ordered word: ties resolve to the lower quad
            my_key = (static_cast<unsigned long long>(hm) << 32) | ~qm;
          }
        }
      };
#pragma unroll kUnroll
      for (int rr = 0; rr + 1 < kR / 2; rr += 2) fold_rows(std::integral_constant<int, 2>{}, hr + rr);
      if constexpr ((kR / 2) % 2 == 1) fold_rows(std::integral_constant<int, 1>{}, hr + kR / 2 - 1);
      // the slot's cost rows are no longer needed
      if (lane == 0) stamp(A, 7, t);
      __syncwarp();
      if (kLoaders > 0) {
        if (lane == 0) mbar_arrive(&S.empty[s]);
      } else if (lane == 0) {
        // the band's second row warp done with the slot refills it (band t + nslots)
        __threadfence_block();
        if (atomicAdd(&S.rel[s], 1) == 1) {
          __threadfence_block();
          S.rel[s] = 0;
          if (t + nslots < nb) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_band(t + nslots, s);
          }
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tfull[ts]);
      // this CTA's partial of the band's rows -> the group's global words:
      // (sum << 8) + one arrival (the sum clamped at 2^48: 255 arrivals cannot
      // carry out of the word) and the (max, quad) key
      if (lane >= hr && lane < hr + kR / 2 && lane < rv) {
        const unsigned long long sm = my_sum < kFixSat ? my_sum : kFixSat;
        atomicMax(tkey + i0 + lane, my_key);
        atomicAdd(sfix + i0 + lane, (sm << 8) + 1ull);
      }
      if (lane == 0) stamp(A, 3, t);
    }
  } else {
    // ------------------------------------------------------- column warps --
    // Column warp cw reads back what row warp cw + 1 wrote (same lane
    // quarter, bands t = cw mod 4) and folds w_i e_ij into its lanes' 16
    // columns; the four warps' partial column sums are added in warp order.
    const int cw = warp - kLoaders - kRowWarps;  // 0..3
    const int list = blockIdx.x * kColWarps + cw;  // this warp's loose-row list
    const double scale = ldexp(1.0, -kFix);
    double acc[4 * kQPL];
#pragma unroll
    for (int e = 0; e < 4 * kQPL; ++e) acc[e] = 0.0;
    int nbad = 0;
    // lanes 0..kR-1 hold row (lane) of the band this warp folds next; its sum
    // word is loaded one band (of this warp: 4 bands of the CTA) ahead
    auto row_of = [&](int64_t t) -> int64_t { return band_row0(t) + (lane % kR); };
    auto prefetch = [&](int64_t t, unsigned long long& sx, RowRec& rc) {
      const int64_t i = row_of(t);
      if (lane < kR && t < nb && i < A.n) {
        sx = ld_relaxed64(sfix + i);
        rc = A.rec[i];
      }
    };
    unsigned long long sx = 0ull;
    RowRec rc{};
    prefetch(cw, sx, rc);
    for (int64_t t = cw; t < nb; t += kColWarps) {
      const int ts = static_cast<int>(t % kTSlots);
      const uint32_t ph = static_cast<uint32_t>((t / kTSlots) & 1);
      const int64_t i = row_of(t);
      const bool present = lane < kR && i < A.n;
      // the group's partials of the band's rows have all arrived when the
      // arrival count in the low byte of each row's sum word reaches `group`
      for (unsigned spins = 0;; ++spins) {
        const bool done = !present || (sx & 0xffull) >= static_cast<unsigned long long>(A.group);
        if (__all_sync(0xffffffffu, done)) break;
        __nanosleep(SP_POLL_NS);
        if (!done) sx = ld_relaxed64(sfix + i);
        if (spins > (kSpinLimit >> 4)) __trap();
      }
      if (lane == 0) stamp(A, 4, t);
      // the band's weights (only w gates the fold; the owner's row outputs
      // are written after the tensor-memory slot is released)
      float w_l = 0.0f;
      bool bad = false;
      double Sv = 1.0, wi = 0.0;
      if (present) {
        Sv = static_cast<double>(sx >> 8) * scale;
        bad = !(Sv >= 0.25 && Sv < 1048576.0);  // outside the fixed-point range: redo
        wi = rc.a / Sv;
        w_l = bad ? 0.0f : static_cast<float>(wi);
      }
      const RowRec rc_t = rc;
      prefetch(t + kColWarps, sx, rc);
      // the band's exponentials (row warps of this lane quarter)
      mbar_wait(&S.tfull[ts], ph);
      tc_fence_after();
      if (lane == 0) stamp(A, 5, t);
      const uint32_t taddr = tmem_of(warp, t);
      float a32[4 * kQPL];
#pragma unroll
      for (int e = 0; e < 4 * kQPL; ++e) a32[e] = 0.0f;
#pragma unroll 2
      for (int rp = 0; rp < kR / 2; ++rp) {
        float E[32];
        tmem_ld32(taddr + static_cast<uint32_t>(rp * 32), E);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float wr = __shfl_sync(0xffffffffu, w_l, 2 * rp + h);
          if (wr != 0.0f) {  // uniform over the warp (one row); 0 = loose or absent row
            const float2 w2 = make_float2(wr, wr);
#pragma unroll
            for (int e = 0; e < 4 * kQPL; e += 2) {
              const float2 r2 = __ffma2_rn(make_float2(E[16 * h + e], E[16 * h + e + 1]), w2,
                                           make_float2(a32[e], a32[e + 1]));
              a32[e] = r2.x;
              a32[e + 1] = r2.y;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tempty[ts]);
      if (lane == 0) stamp(A, 6, t);
#pragma unroll
      for (int e = 0; e < 4 * kQPL; ++e) acc[e] += static_cast<double>(a32[e]);
      // owner: the row outputs of band t and its loose rows (in row order)
      const bool owner = (t % A.group) == k;  // band t's rows belong to CTA t mod group
      if (owner) {
        if (present) {
          if (!bad) {
            const double sc = static_cast<double>(rc_t.shift);
            const double M = sc * kLn2;
            A.rowM[i] = M;
            A.rowS[i] = Sv;
            A.u[i] = (rc_t.loga - M) - log(Sv);
            A.wrow[i] = wi;
            A.rowJ[i] = -1;  // base-2 max + argmax quad: from this pass's key (k_sp_prep)
            A.aux[i] = make_float4(rc_t.shift, 0.0f, w_l, 0.0f);
          }
          // zero the other parity's words for the next launch
          A.sfix[static_cast<int64_t>(par ^ 1u) * A.n + i] = 0ull;
          A.tkey[static_cast<int64_t>(par ^ 1u) * A.n + i] = 0ull;
        }
        const unsigned bm = __ballot_sync(0xffffffffu, present && bad);
        if (present && bad)
          A.bad_rows[list * A.cap + nbad + __popc(bm & ((1u << lane) - 1u))] = static_cast<int>(i);
        nbad += __popc(bm);
      }
    }
    if (lane == 0) A.bad_count[list] = nbad;
    if (lane == 0 && nbad) atomicAdd(A.state + 2, static_cast<unsigned>(nbad));
    // the four column warps' partials, summed in warp order (the ring is free:
    // every band has been folded once all four warps reach the barrier)
    double* red = reinterpret_cast<double*>(ring);
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kColWarps) : "memory");
#pragma unroll
    for (int e = 0; e < 4 * kQPL; ++e) red[(cw * 4 * kQPL + e) * 32 + lane] = acc[e];
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kColWarps) : "memory");
    if (cw == 0) {
#pragma unroll
      for (int kq = 0; kq < kQPL; ++kq) {
        const int qi = lane + 32 * kq;
        if (qi >= nq) continue;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t j = 4 * (q0 + qi) + e;
          if (j >= A.m) continue;
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < kColWarps; ++w) v += red[(w * 4 * kQPL + 4 * kq + e) * 32 + lane];
          A.part[static_cast<int64_t>(g) * A.mpad + j] = v;
        }
      }
    }
  }
  // teardown: free the tensor memory, flip the buffer parity after the last CTA
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    if (lane == 0) {
      __threadfence();
      unsigned* fin = A.state + 1;
      if (atomicAdd(fin, 1u) == static_cast<unsigned>(active - 1)) {
        *fin = 0u;
        A.state[0] = par ^ 1u;
        __threadfence();
      }
    }
  }
}

__global__ void __launch_bounds__(kPatchThreads)
k_sp_patch(const float* __restrict__ C, int64_t ldc, int64_t m, const double* __restrict__ p,
           float kh, float kl, const float4* __restrict__ aux, const int* __restrict__ bad_rows,
           const int* __restrict__ bad_count, int nlists, int64_t cap, double* __restrict__ out,
           const unsigned* __restrict__ total, const Ctrl* __restrict__ ctrl) {
  pdl_wait();  // programmatic dependent launch: after the previous kernel
  // columns of the rows the single pass skipped: out[j] = sum over the listed
  // rows (list order, then row order) of w_i ex2(t_ij), with the exact split
  // shift k_sp_redo wrote into aux -- the k_col_fast formula
  if (ctrl->done || !ctrl->shift_valid) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kPatchThreads + threadIdx.x;
  if (j >= m) return;
  if (*total == 0u) {  // no loose rows (the usual case): the patch row is zero
    out[j] = 0.0;
    return;
  }
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

unsigned long long*& sp_trace_buf() {
  static unsigned long long* p = nullptr;
  return p;
}

}  // namespace

// Column layout of the single pass for m columns on `sms` SMs: H groups of
// `group` CTAs; CTA k of a group owns columns [k W, (k+1) W) with W = cw nch
// (cw a multiple of 32, <= 256: one TMA box {cw, nch, 16} per band); W <=
// 512 (a warp's 32 lanes x 16 columns).  The cost's row stride is a multiple
// of cw, so the 3-D view {cw, ldc / cw, rows} of it is a plain tensor.
SpLayout sp_layout(int64_t m, int sms) {
  SpLayout L;
  const int64_t quads = (m + 3) / 4;
  const int64_t min_group = (quads + kQMax - 1) / kQMax;
  if (m < 256 || min_group > sms) return L;
  L.H = static_cast<int>(std::max<int64_t>(1, sms / min_group));
  const int64_t per = (m + sms / L.H - 1) / (sms / L.H);  // columns per CTA, at least
  L.nch = static_cast<int>((per + 255) / 256);
  L.cw = static_cast<int>(((per + L.nch - 1) / L.nch + 31) / 32 * 32);
  if (L.cw > 256) {
    ++L.nch;
    L.cw = static_cast<int>(((per + L.nch - 1) / L.nch + 31) / 32 * 32);
  }
  const int64_t W = static_cast<int64_t>(L.cw) * L.nch;
  if (W > 4 * kQMax) return L;
  L.group = static_cast<int>((m + W - 1) / W);
  L.ok = true;
  return L;
}

// Decide whether the single-pass path applies and size it (handle setup):
// fp32 stored cost, no virtual shards (they use the two-pass kernels), the
// layout exists and the handle did not ask for the two-pass kernels
// (otg_device_opts.sweep = 1: A/B and cross-checks).
bool fused_configure(Problem& P) {
  P.fused = 0;
  if (P.storage != OTG_STORE_F32 || P.vshards != 1 || P.two_pass) return false;
  int sms = 0;
  OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
  const SpLayout L = sp_layout(P.m, sms);
  // the grid-wide band pipeline needs a run of bands per group to pay for its
  // fill (B200, round-2 kernel, us per evaluation single / two-pass,
  // tools/sp_crossover.py: 2048 x 8192 (14 bands per group) 78 / 81, 4096 x
  // 8192 (28) 105 / 104, 8192^2 (57) 115 / 136, 8192 x 2048 67 / 89, 65536 x
  // 1024 126 / 416, 2048 x 65536 208 / 259, 65536^2 3400 / 5100)
  const int64_t bands_per_group = ((P.n_local + kR - 1) / kR + L.H - 1) / std::max(L.H, 1);
  if (!L.ok || P.ldc % L.cw != 0 || P.n_local < 2 * kR) return false;
  if (bands_per_group < 32 && !P.force_single_pass) return false;
  const int64_t W = static_cast<int64_t>(L.cw) * L.nch;
  const int64_t head = ((sizeof(S1Shared) + 127) / 128) * 128;
  const int64_t slot = kR * W * 4;
  const int64_t budget = 220 * 1024 - head;
  const int nslots = static_cast<int>(std::min<int64_t>(kRingMax, budget / slot));
  if (nslots < 3) return false;
  // (the ring also holds the column warps' final 4 x 16 x 32 fp64 partials)
  const int smem = static_cast<int>(
      head + std::max<int64_t>(nslots * slot, kColWarps * 4 * kQPL * 32 * sizeof(double)));
  // (per kernel, not per handle: the largest size any handle can ask for)
  OTG_CUDA(cudaFuncSetAttribute(k_sweep1, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  int occ = 0;
  OTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep1, kThreads, smem));
  if (occ < 1) return false;
  // the cost as a 3-D tensor {cw, ldc / cw, n_local} (strides cw, ldc floats):
  // one box {cw, nch, 16} is a band of a CTA's slice; rows past n_local are
  // zero-filled by the copy engine, columns past m are the row padding (zero)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  OTG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return false;
  const cuuint64_t gdim[3] = {static_cast<cuuint64_t>(L.cw), static_cast<cuuint64_t>(P.ldc / L.cw),
                              static_cast<cuuint64_t>(P.n_local)};
  const cuuint64_t gstride[2] = {static_cast<cuuint64_t>(L.cw) * sizeof(float),
                                 static_cast<cuuint64_t>(P.ldc) * sizeof(float)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(L.cw), static_cast<cuuint32_t>(L.nch),
                             static_cast<cuuint32_t>(kR)};
  const cuuint32_t estride[3] = {1, 1, 1};
  CUtensorMap* map = reinterpret_cast<CUtensorMap*>(P.sp_tmap);
  if (reinterpret_cast<EncodeFn>(fn)(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, P.C32, gdim, gstride,
                                     box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  P.sp_bw = L.cw;
  P.sp_nbox = L.nch;
  P.fused = 1;
  P.fused_clusters = L.H;
  P.sp_group = L.group;
  P.fused_slots = nslots;
  P.fused_smem = smem;
  P.sp_fix = kFix;
  const int64_t bands = (P.n_local + kR - 1) / kR;
  // loose-row lists: one per column warp of every CTA (owned bands t = k mod
  // group of the warp's bands t = cw mod 4), each in row order
  P.sp_cap = kR * ((bands + static_cast<int64_t>(L.H) * L.group - 1) /
                       (static_cast<int64_t>(L.H) * L.group) + 1);
  if (getenv("OTG_VERBOSE"))
    fprintf(stderr,
            "[otg] single-pass: %d groups x %d CTAs, slices of %lld columns (box %d x %d x %d), "
            "smem %d, ring %d\n",
            L.H, L.group, static_cast<long long>(W), L.cw, L.nch, kR, smem, nslots);
  return true;
}

// Row minima of the stored cost (one CTA per row, columns < m only): the
// zero point's row statistics.  M2 = -(min_j C_ij) kappa log2(e) + 1/64 is
// an upper bound on the base-2 row max at p = 0 (the fp32 exponents round
// within ~1e-4 of it) and argmin_j C_ij (lowest index of equal minima) is its
// argmax -- what k_sp_prep reads after an evaluation.
__global__ void __launch_bounds__(256)
k_zero_rowstats(const float* __restrict__ C, int64_t ldc, int64_t n, int64_t m, double k2,
                double* __restrict__ zM2, int* __restrict__ zJ) {
  __shared__ float sv[8];
  __shared__ int sj[8];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const float* row = C + i * ldc;
    float bv = INFINITY;
    int bj = 0;
    for (int64_t j = threadIdx.x; j < m; j += 256) {
      const float c = row[j];
      if (c < bv) {  // (ascending j per thread: the lowest index of equal minima)
        bv = c;
        bj = static_cast<int>(j);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov < bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      sv[threadIdx.x >> 5] = bv;
      sj[threadIdx.x >> 5] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w)
        if (sv[w] < bv || (sv[w] == bv && sj[w] < bj)) {
          bv = sv[w];
          bj = sj[w];
        }
      zM2[i] = -static_cast<double>(bv) * k2 + 1.0 / 64.0;
      zJ[i] = bj;
    }
    __syncthreads();
  }
}

void fused_alloc(Problem& P) {
  if (!P.fused) return;
  const int64_t n = P.n_local;
  P.sp_zM2 = dalloc<double>(P, n);
  P.sp_zJ = dalloc<int>(P, n);
  k_zero_rowstats<<<static_cast<unsigned>(std::min<int64_t>(n, 148 * 8)), 256, 0, P.stream>>>(
      static_cast<const float*>(P.C32), P.ldc, n, P.m, P.kappa * kLog2e, P.sp_zM2, P.sp_zJ);
  OTG_CUDA(cudaGetLastError());
  P.sp_rec = dalloc<double>(P, static_cast<size_t>(n) * (sizeof(RowRec) / 8));
  const int lists = P.fused_clusters * P.sp_group * kColWarps;
  P.sp_bad_rows = dalloc<int>(P, static_cast<size_t>(lists) * P.sp_cap);
  P.sp_bad_count = dalloc<int>(P, lists);
  P.sp_sums = dalloc<unsigned long long>(P, 4 * static_cast<size_t>(n));
  P.sp_cnt = dalloc<unsigned>(P, 4);
  OTG_CUDA(cudaMemsetAsync(P.sp_bad_count, 0, lists * sizeof(int), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.sp_sums, 0, 4 * static_cast<size_t>(n) * sizeof(unsigned long long),
                           P.stream));
  OTG_CUDA(cudaMemsetAsync(P.sp_cnt, 0, 4 * sizeof(unsigned), P.stream));
}

// Steady-state evaluation sweep (launched after the exact-path kernels, each
// of which returns at once when the other applies): single pass, redo of the
// loose rows, their column patch into partial row H.
void launch_fused(Problem& P, float kh, float kl) {
  RowRec* rec = reinterpret_cast<RowRec*>(P.sp_rec);
  unsigned long long* sums = static_cast<unsigned long long*>(P.sp_sums);
  launch_k(k_sp_prep, 296, 256, 0, P.stream, P.n_local, P.m, static_cast<const float*>(P.C32), P.ldc,
           static_cast<const float*>(P.vq), P.mpad, kh, kl, P.rowM2, P.rowJ, P.a, P.loga, rec,
           static_cast<const unsigned long long*>(sums + 2 * P.n_local),
           P.sp_cnt, P.ctrl, P.steady_capture);
  S1Args A;
  A.dbg = nullptr;
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
  A.sfix = sums;
  A.tkey = sums + 2 * P.n_local;
  A.state = P.sp_cnt;
  A.bad_rows = P.sp_bad_rows;
  A.bad_count = P.sp_bad_count;
  A.cap = P.sp_cap;
  A.H = P.fused_clusters;
  A.group = P.sp_group;
  A.nslots = P.fused_slots;
  A.W = P.sp_bw * P.sp_nbox;
  A.nch = P.sp_nbox;
  A.dbg = sp_trace_buf();
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
  OTG_CUDA(cudaLaunchKernelEx(&cfg, k_sweep1, A, *reinterpret_cast<const CUtensorMap*>(P.sp_tmap),
                              static_cast<const Ctrl*>(P.ctrl)));
  launch_sp_redo(P, P.sp_bad_rows, P.sp_bad_count, ctas * kColWarps, P.sp_cap);
  if (patch_merges(P)) {  // patch + merge + flags + <u, a> in one kernel
    launch_sp_patch_merge(P, kh, kl, ctas * kColWarps);
    OTG_CUDA(cudaGetLastError());
    return;
  }
  const unsigned g = static_cast<unsigned>((P.m + kPatchThreads - 1) / kPatchThreads);
  launch_k(k_sp_patch, g, kPatchThreads, 0, P.stream, P.C32, P.ldc, P.m, P.p, kh, kl, P.aux,
           P.sp_bad_rows, P.sp_bad_count, ctas * kColWarps, P.sp_cap,
           P.part + static_cast<int64_t>(P.fused_clusters) * P.mpad,
           static_cast<const unsigned*>(P.sp_cnt + 2), P.ctrl);
  OTG_CUDA(cudaGetLastError());
}

}  // namespace otg

// Debug timeline of the single-pass kernel (globaltimer ns; CTA 0 and the last
// CTA; per band: loader issue, row wait start / end, row publish, watcher
// window ready, column start / end).  enable != 0 allocates the buffer (later
// launches record), out != NULL copies 2 x 8 x 256 stamps out.
extern "C" int otg_debug_sp_trace(int enable, unsigned long long* out) {
  auto& p = otg::sp_trace_buf();
  const size_t bytes = 2 * 12 * otg::kDbgBands * sizeof(unsigned long long);
  if (enable && !p) {
    if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
    cudaMemset(p, 0, bytes);
  }
  if (out && p && cudaMemcpy(out, p, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  return 0;
}
