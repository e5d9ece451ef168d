// problem.cu — handle creation: validation (core.cpp:9-29), upload, the
// rescale fold (core.cpp:42-49), device cost materialisation
// (data.cpp:69-110), plan statistics over the implicit plan (core.cpp:59-79).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstring>

#include <cstdlib>

#include "common.cuh"

namespace otg {

void configure_sweeps(Problem& P);
int64_t row_blocks(const Problem& P);

namespace {

constexpr int kT = 256;
constexpr int kFbChunks = 32;
constexpr int64_t kTraceCap = 4096;
constexpr int64_t kBoundaryCap = 4096;

std::string fmt17(double x) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

// core.cpp:9-29 for the marginals (host side; cheap).
void validate_marginals(const double* a, int64_t n, const double* b, int64_t m) {
  if (n < 1 || m < 1) fail(OTG_E_DIMENSION, "empty marginal");
  if (!a || !b) fail(OTG_E_DIMENSION, "marginal pointer is NULL");
  const double* ms[2] = {a, b};
  const int64_t ls[2] = {n, m};
  for (int k = 0; k < 2; ++k) {
    double mn = ms[k][0], s = 0.0;
    for (int64_t j = 0; j < ls[k]; ++j) {
      mn = std::min(mn, ms[k][j]);
      s += ms[k][j];
    }
    if (!(mn > 0.0)) fail(OTG_E_INVALID_MARGINALS, "marginals must be strictly positive");
    if (std::abs(s - 1.0) > 1e-9)
      fail(OTG_E_INVALID_MARGINALS, "marginal sums to " + fmt17(s) + ", expected 1");
  }
}

void validate_eps(double eps) {
  if (!(eps > 0.0) || !std::isfinite(eps)) fail(OTG_E_OT, "epsilon must be positive and finite");
}

__global__ void k_log(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = log(x[i]);
}

__global__ void k_div_rows(double* __restrict__ C, int64_t ldc, int64_t n, int64_t m, double eps) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    C[i * ldc + j] = C[i * ldc + j] / eps;
}

// raw cost of one pair, fp64, left-to-right without contraction (data.cpp:75-77, 98-99)
// D > 0: the dimension as a compile-time constant (the same operations in the
// same order, unrolled); D = 0: runtime d
template <int D = 0>
__device__ __forceinline__ double raw_cost(const double* __restrict__ x,
                                           const double* __restrict__ y, int64_t d_rt, int cost) {
  const int64_t d = D > 0 ? D : d_rt;
  double s = 0.0;
  if (cost == OTG_COST_SQEUCLID) {
#pragma unroll
    for (int64_t k = 0; k < d; ++k) {
      const double diff = __dsub_rn(x[k], y[k]);
      s = __dadd_rn(s, __dmul_rn(diff, diff));
    }
    return s;
  }
#pragma unroll
  for (int64_t k = 0; k < d; ++k) s = __dadd_rn(s, __dmul_rn(x[k], y[k]));
  return __dadd_rn(-s, 1.0);
}

// pass 1: per-block (min, max) of the raw cost
template <int D>
__global__ void k_cost_minmax(const double* __restrict__ X, const double* __restrict__ Y,
                              int64_t n, int64_t m, int64_t d, int cost,
                              double2* __restrict__ out) {
  __shared__ double smn[kT], smx[kT];
  double mn = DBL_MAX, mx = -DBL_MAX;
  // rows over the grid, columns over the CTA (no index division per pair)
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < m; j += kT) {
      const double c = raw_cost<D>(X + i * d, Y + j * d, d, cost);
      mn = fmin(mn, c);
      mx = fmax(mx, c);
    }
  smn[threadIdx.x] = mn;
  smx[threadIdx.x] = mx;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
      smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = make_double2(smn[0], smx[0]);
}

// pass 2: normalise and store. norm: NONE, MAX (c / mx), MINMAX ((c-mn)/(mx-mn)),
// HALFRANGE (c / 2); then fp64 storage divides by eps (rescale), fp32 rounds.
template <typename T, int D>
__global__ void k_cost_store(const double* __restrict__ X, const double* __restrict__ Y,
                             int64_t n, int64_t m, int64_t d, int cost, int norm, double mn,
                             double mx, double eps_div, T* __restrict__ C, int64_t ldc) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < ldc;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (j >= m) {  // row padding: zero (no separate memset of the whole matrix)
      C[i * ldc + j] = static_cast<T>(0);
      continue;
    }
    double c = raw_cost<D>(X + i * d, Y + j * d, d, cost);
    if (norm == OTG_NORM_MAX) {
      if (mx > 0.0) c = c / mx;
    } else if (norm == OTG_NORM_MINMAX) {
      c = (mx - mn > 1e-15) ? (c - mn) / (mx - mn) : 0.0;
    } else if (norm == OTG_NORM_HALFRANGE) {
      c = c / 2.0;
    }
    if (eps_div != 1.0) c = c / eps_div;
    C[i * ldc + j] = static_cast<T>(c);
  }
}

__global__ void k_otf_rows(const float4* __restrict__ X, const float4* __restrict__ Y,
                           int64_t row0, int64_t nrows, int64_t m, float* __restrict__ out) {
  const int64_t i = blockIdx.x;
  if (i >= nrows) return;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x)
    out[i * m + j] = otf_sqeuclid(X[row0 + i], Y[j]);
}

}  // namespace

void problem_free(Problem& P) {
  void* ptrs[] = {P.C64, P.C32, P.X, P.Y, P.Yn, P.a, P.loga, P.b, P.logb, P.rowM, P.rowS, P.u,
                  P.wrow, P.aux, P.rowM2, P.rowJ, P.dq, P.redo_rows, P.vq, P.p, P.wacc, P.col,
                  P.col_log,
                  P.y, P.grad, P.prev_grad,
                  P.prev_x, P.prev_y, P.flag_idx, P.fb_cols, P.fb_part, P.part, P.e1_part,
                  P.e2_part, P.sp_rec, P.sp_bad_rows, P.sp_bad_count, P.ctrl, P.trace, P.vstar, P.bounds, P.fbA, P.fbS, P.fbT, P.red, P.sp_sums, P.sp_cnt,
                  P.perm_r, P.perm_c, P.Xs, P.Yns, P.cbox, P.rbox, P.cvmax, P.rnegm, P.ves, P.auxs,
                  P.sp_zM2, P.sp_zJ};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (P.ctrl_host) cudaFreeHost(P.ctrl_host);
  if (P.chunk_exec) cudaGraphExecDestroy(P.chunk_exec);
  if (P.chunk_exec_timed) cudaGraphExecDestroy(P.chunk_exec_timed);
  if (P.chunk_exec_steady) cudaGraphExecDestroy(P.chunk_exec_steady);
  for (cudaEvent_t e : P.chunk_events) cudaEventDestroy(e);
  if (P.nccl_comm) comm_destroy(P);
  if (P.stream) cudaStreamDestroy(P.stream);
  P = Problem{};
}

void problem_alloc_state(Problem& P) {
  configure_sweeps(P);
  fused_configure(P);
  const int64_t n = P.n_local, mp = P.mpad;
  P.rowM = dalloc<double>(P, n);
  P.rowS = dalloc<double>(P, n);
  P.u = dalloc<double>(P, n);
  P.wrow = dalloc<double>(P, n);
  P.aux = dalloc<float4>(P, n);
  P.rowM2 = dalloc<double>(P, n);
  P.rowJ = dalloc<int>(P, n);
  P.dq = dalloc<double>(P, mp);
  P.redo_rows = dalloc<int>(P, n);
  P.vq = dalloc<float>(P, 3 * mp);  // [V | F | 2^F]
  P.p = dalloc<double>(P, mp);
  P.wacc = dalloc<double>(P, mp);
  P.col = dalloc<double>(P, mp + 8 + std::max<int64_t>((P.m + 255) / 256, kEpiMaxGrid));  // + <u, a> slices
  P.col_log = dalloc<double>(P, mp);
  P.y = dalloc<double>(P, mp);
  P.grad = dalloc<double>(P, mp);
  P.prev_grad = dalloc<double>(P, mp);
  P.prev_x = dalloc<double>(P, mp);
  P.prev_y = dalloc<double>(P, mp);
  P.flag_idx = dalloc<int>(P, mp);
  P.fb_cols = dalloc<int>(P, mp);
  P.fb_part = dalloc<double2>(P, mp * kFbChunks);
  if (P.sharded) {
    P.red = dalloc<double>(P, mp + 8 + std::max<int64_t>((P.m + 255) / 256, kEpiMaxGrid));
    P.fbA = dalloc<double>(P, mp);
    P.fbS = dalloc<double>(P, mp);
    P.fbT = dalloc<double>(P, mp);
  }
  const size_t prow = std::max<size_t>(static_cast<size_t>(P.vshards) * P.col_splits,
                                       static_cast<size_t>(P.fused_clusters) + 1);
  P.part = dalloc<double>(P, prow * mp);
  if (P.row_splits > 0) P.rpart = dalloc<double2>(P, static_cast<int64_t>(P.row_splits) * n);
  P.e1_part = dalloc<double>(P, (e1_groups_of(P.m) + 1) * 8 + row_blocks(P) + 8);
  P.e2_part = dalloc<double>(P, P.e_blocks * 16);
  fused_alloc(P);
  P.ctrl = dalloc<Ctrl>(P, 1);
  P.trace = dalloc<double>(P, kTraceCap * kTraceCols);
  P.bounds = dalloc<double>(P, kBoundaryCap * kBoundCols);
  // the reference solution's v* (energy / radii): allocated with the handle --
  // the cached chunk graphs capture this pointer, so a later instrumented
  // solve on the same handle must find it at the same address
  P.vstar = dalloc<double>(P, P.mpad);
  OTG_CUDA(cudaMallocHost(&P.ctrl_host, sizeof(Ctrl)));
  OTG_CUDA(cudaMemsetAsync(P.p, 0, mp * sizeof(double), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.wacc, 0, mp * sizeof(double), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.part, 0, prow * mp * sizeof(double), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.ctrl, 0, sizeof(Ctrl), P.stream));
  std::memset(P.ctrl_host, 0, sizeof(Ctrl));
}

static void begin(Problem& P, int64_t n, int64_t m, const otg_device_opts* opts) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(OTG_E_UNSUPPORTED, "no CUDA device available (libotg has no CPU fallback)");
  P.device = (opts && opts->device >= 0) ? opts->device : 0;
  if (!opts || opts->device < 0) OTG_CUDA(cudaGetDevice(&P.device));
  OTG_CUDA(cudaSetDevice(P.device));
  P.n = n;
  P.m = m;
  P.n_local = n;
  P.row_begin = 0;
  // Sharded (NCCL) when world_size > 1, or when an id is given for a 1-rank
  // communicator (exercises the collective path on one GPU).
  if (opts && (opts->world_size > 1 || opts->nccl_unique_id || opts->allreduce)) {
    if (opts->world_size < 1 || opts->rank < 0 || opts->rank >= opts->world_size)
      fail(OTG_E_DIMENSION, "rank outside [0, world_size)");
    if (opts->row_begin < 0 || opts->row_end > n || opts->row_begin >= opts->row_end)
      fail(OTG_E_DIMENSION, "row shard [row_begin, row_end) outside [0, n)");
    if (!opts->nccl_unique_id && !opts->allreduce)
      fail(OTG_E_NCCL, "world_size > 1 needs nccl_unique_id or an allreduce callback");
    P.world = opts->world_size;
    P.rank = opts->rank;
    P.row_begin = opts->row_begin;
    P.n_local = opts->row_end - opts->row_begin;
    P.sharded = 1;
  }
  P.vshards = (opts && opts->virtual_shards > 1) ? opts->virtual_shards : 1;
  P.two_pass = (opts && opts->sweep == 1) ? 1 : 0;
  P.force_single_pass = (opts && opts->sweep == 2) ? 1 : 0;
  if (P.vshards > P.n_local) P.vshards = static_cast<int>(P.n_local);
  P.mpad = round_up(m, 4);
  // rows padded to 128-byte multiples (aligned 16-byte loads of any quad)
  P.ldc = round_up(m, 32);
  {  // a row stride the single-pass sweep's 3-D tensor view can use (fused.cu)
    int sms = 0;
    OTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device));
    const SpLayout L = sp_layout(m, sms);
    if (L.ok) P.ldc = round_up(m, L.cw);
  }
  OTG_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
}

static void upload_marginals(Problem& P, const double* a, const double* b) {
  const int64_t n = P.n_local, m = P.m;
  P.a = dalloc<double>(P, n);
  P.loga = dalloc<double>(P, n);
  P.b = dalloc<double>(P, P.mpad);
  P.logb = dalloc<double>(P, P.mpad);
  OTG_CUDA(cudaMemsetAsync(P.b, 0, P.mpad * sizeof(double), P.stream));
  OTG_CUDA(cudaMemsetAsync(P.logb, 0, P.mpad * sizeof(double), P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.a, a + P.row_begin, n * sizeof(double), cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.b, b, m * sizeof(double), cudaMemcpyHostToDevice, P.stream));
  k_log<<<(n + kT - 1) / kT, kT, 0, P.stream>>>(P.a, P.loga, n);
  k_log<<<(m + kT - 1) / kT, kT, 0, P.stream>>>(P.b, P.logb, m);
  OTG_CUDA(cudaGetLastError());
}

// Culled on-the-fly sweeps: Morton orders (10 bits per axis over the joint
// bounding box; ties by index) of the rows and the columns, the points in
// those orders and the static boxes of the culling blocks (64 sorted
// columns, 16 sorted rows).  Only the two steady-state on-the-fly sweep
// kernels visit rows / columns in these orders; every array the API sees
// stays in the caller's order.
int& cull_mode();  // sweep.cu (test hook otg_debug_cull)

static void setup_cull(Problem& P, const std::vector<float>& hx, const std::vector<float>& hy) {
  constexpr int64_t kCB = 64, kRB = 16;
  const int64_t n = P.n_local, m = P.m;
  if (!OTG_CULL || cull_mode() < 0 || n < 4096 || m < 4096) return;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) lo[k] = std::min(lo[k], hx[i * 4 + k]), hi[k] = std::max(hi[k], hx[i * 4 + k]);
  for (int64_t j = 0; j < m; ++j)
    for (int k = 0; k < 3; ++k) lo[k] = std::min(lo[k], hy[j * 4 + k]), hi[k] = std::max(hi[k], hy[j * 4 + k]);
  auto code = [&](const float* pt) {
    uint32_t c = 0;
    for (int k = 0; k < 3; ++k) {
      const double span = static_cast<double>(hi[k]) - lo[k];
      const uint32_t q = span > 0 ? static_cast<uint32_t>(std::min(
                                        1023.0, std::floor((pt[k] - lo[k]) / span * 1024.0)))
                                  : 0u;
      for (int b = 0; b < 10; ++b) c |= ((q >> b) & 1u) << (3 * b + k);
    }
    return c;
  };
  auto order = [&](const std::vector<float>& pts, int64_t cnt) {
    std::vector<std::pair<uint32_t, int>> key(cnt);
    for (int64_t t = 0; t < cnt; ++t) key[t] = {code(&pts[t * 4]), static_cast<int>(t)};
    std::sort(key.begin(), key.end());
    std::vector<int> perm(cnt);
    for (int64_t t = 0; t < cnt; ++t) perm[t] = key[t].second;
    return perm;
  };
  const std::vector<int> pr = order(hx, n), pc = order(hy, m);
  std::vector<float> xs(n * 4), yns(P.mpad * 3, 0.f);
  for (int64_t s = 0; s < n; ++s)
    for (int k = 0; k < 4; ++k) xs[s * 4 + k] = hx[pr[s] * 4 + k];
  for (int64_t s = 0; s < m; ++s)
    for (int k = 0; k < 3; ++k) yns[k * P.mpad + s] = -hy[pc[s] * 4 + k];
  auto boxes = [](const std::vector<float>& pts, const std::vector<int>& perm, int64_t cnt,
                  int64_t B) {
    const int64_t nb = (cnt + B - 1) / B;
    std::vector<float> bx(nb * 8, 0.f);
    for (int64_t b = 0; b < nb; ++b) {
      float l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t s = b * B; s < std::min(cnt, (b + 1) * B); ++s)
        for (int k = 0; k < 3; ++k) {
          const float v = pts[static_cast<int64_t>(perm[s]) * 4 + k];
          l[k] = std::min(l[k], v);
          h[k] = std::max(h[k], v);
        }
      for (int k = 0; k < 3; ++k) bx[b * 8 + k] = l[k], bx[b * 8 + 4 + k] = h[k];
    }
    return bx;
  };
  const std::vector<float> cb = boxes(hy, pc, m, kCB), rb = boxes(hx, pr, n, kRB);
  P.perm_r = dalloc<int>(P, n);
  P.perm_c = dalloc<int>(P, m);
  P.Xs = dalloc<float>(P, n * 4);
  P.Yns = dalloc<float>(P, P.mpad * 3);
  P.cbox = dalloc<float>(P, cb.size());
  P.rbox = dalloc<float>(P, rb.size());
  P.cvmax = dalloc<float>(P, cb.size() / 8);
  P.rnegm = dalloc<float>(P, rb.size() / 8);
  P.ves = dalloc<float>(P, 2 * m);
  P.auxs = dalloc<float>(P, 4 * n);
  OTG_CUDA(cudaMemcpyAsync(P.perm_r, pr.data(), n * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.perm_c, pc.data(), m * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.Xs, xs.data(), xs.size() * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.Yns, yns.data(), yns.size() * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.cbox, cb.data(), cb.size() * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaMemcpyAsync(P.rbox, rb.data(), rb.size() * 4, cudaMemcpyHostToDevice, P.stream));
  OTG_CUDA(cudaStreamSynchronize(P.stream));  // (host vectors go out of scope)
  P.cull = 1;
}

static void finish_create(Problem& P, const otg_device_opts* opts, otg_problem* out) {
  if (P.sharded) comm_init(P, opts);
  problem_alloc_state(P);
  OTG_CUDA(cudaStreamSynchronize(P.stream));
  auto* h = new otg_problem_s;
  h->P = P;
  *out = h;
}

}  // namespace otg

using namespace otg;

extern "C" {

otg_status otg_problem_create_dense(int64_t n, int64_t m, const double* a, const double* b,
                                    const void* C, otg_dtype dtype, int64_t ldc,
                                    double epsilon, const otg_device_opts* opts,
                                    otg_problem* out) {
  Problem P;
  const otg_status st = guard([&] {
    if (!out) fail(OTG_E_DIMENSION, "out handle pointer is NULL");
    *out = nullptr;
    validate_marginals(a, n, b, m);
    validate_eps(epsilon);
    if (!C) fail(OTG_E_DIMENSION, "cost pointer is NULL");
    if (dtype != OTG_F64 && dtype != OTG_F32) fail(OTG_E_OT, "unknown dtype");
    const int64_t src_ld = ldc > 0 ? ldc : m;
    if (src_ld < m) fail(OTG_E_DIMENSION, "ldc < m");
    begin(P, n, m, opts);
    const int64_t nl = P.n_local;
    // core.cpp:20 C.allFinite() on the rows this handle holds
    if (dtype == OTG_F64) {
      const double* Cd = static_cast<const double*>(C);
      for (int64_t i = 0; i < nl; ++i)
        for (int64_t j = 0; j < m; ++j)
          if (!std::isfinite(Cd[i * src_ld + j])) fail(OTG_E_OT, "cost matrix has non-finite entries");
    } else {
      const float* Cf = static_cast<const float*>(C);
      for (int64_t i = 0; i < nl; ++i)
        for (int64_t j = 0; j < m; ++j)
          if (!std::isfinite(Cf[i * src_ld + j])) fail(OTG_E_OT, "cost matrix has non-finite entries");
    }
    P.epsilon = epsilon;
    P.kappa = 1.0 / epsilon;
    upload_marginals(P, a, b);
    if (dtype == OTG_F64) {
      P.storage = OTG_STORE_F64;
      P.C64 = dalloc<double>(P, static_cast<size_t>(nl) * P.ldc);
      OTG_CUDA(cudaMemsetAsync(P.C64, 0, static_cast<size_t>(nl) * P.ldc * sizeof(double), P.stream));
      OTG_CUDA(cudaMemcpy2DAsync(P.C64, P.ldc * sizeof(double), static_cast<const double*>(C),
                                 src_ld * sizeof(double), m * sizeof(double), nl,
                                 cudaMemcpyHostToDevice, P.stream));
      if (epsilon != 1.0) {
        dim3 grid(static_cast<unsigned>(std::min<int64_t>((m + kT - 1) / kT, 64)),
                  static_cast<unsigned>(std::min<int64_t>(nl, 65535)));
        k_div_rows<<<grid, kT, 0, P.stream>>>(P.C64, P.ldc, nl, m, epsilon);
        OTG_CUDA(cudaGetLastError());
      }
    } else {
      P.storage = OTG_STORE_F32;
      P.C32 = dalloc<float>(P, static_cast<size_t>(nl) * P.ldc);
      OTG_CUDA(cudaMemsetAsync(P.C32, 0, static_cast<size_t>(nl) * P.ldc * sizeof(float), P.stream));
      OTG_CUDA(cudaMemcpy2DAsync(P.C32, P.ldc * sizeof(float), static_cast<const float*>(C),
                                 src_ld * sizeof(float), m * sizeof(float), nl,
                                 cudaMemcpyHostToDevice, P.stream));
    }
    finish_create(P, opts, out);
  });
  if (st != OTG_OK) problem_free(P);
  return st;
}

otg_status otg_problem_create_points(int64_t n, int64_t m, int64_t d, const double* a,
                                     const double* b, const double* x, const double* y,
                                     otg_cost cost, otg_norm norm, otg_storage storage,
                                     double epsilon, const otg_device_opts* opts,
                                     otg_problem* out) {
  Problem P;
  const otg_status st = guard([&] {
    if (!out) fail(OTG_E_DIMENSION, "out handle pointer is NULL");
    *out = nullptr;
    validate_marginals(a, n, b, m);
    validate_eps(epsilon);
    if (d < 1 || !x || !y) fail(OTG_E_DIMENSION, "point clouds need d >= 1 and data");
    if (cost != OTG_COST_SQEUCLID && cost != OTG_COST_COSINE) fail(OTG_E_OT, "unknown cost");
    if (storage == OTG_STORE_ON_THE_FLY &&
        (cost != OTG_COST_SQEUCLID || norm != OTG_NORM_NONE || d > 3))
      fail(OTG_E_UNSUPPORTED,
           "on-the-fly storage recomputes raw squared-Euclidean costs of d <= 3 points "
           "(cost SQEUCLID, norm NONE)");
    if (storage != OTG_STORE_F64 && storage != OTG_STORE_F32 && storage != OTG_STORE_ON_THE_FLY)
      fail(OTG_E_OT, "unknown storage");
    begin(P, n, m, opts);
    const int64_t nl = P.n_local;
    const double* xl = x;  // the caller's local rows (otg.h: x is n_local x d)
    for (int64_t t = 0; t < nl * d; ++t)
      if (!std::isfinite(xl[t])) fail(OTG_E_OT, "point coordinates must be finite");
    for (int64_t t = 0; t < m * d; ++t)
      if (!std::isfinite(y[t])) fail(OTG_E_OT, "point coordinates must be finite");
    if (storage == OTG_STORE_ON_THE_FLY) {
      // fp32 coordinates padded to float4; the cost is recomputed per tile in
      // the sweeps (sweep.cu: otf_cost) and never stored
      // The instance keeps the caller's epsilon (reported, and the unit of
      // the primal cost).  The sweeps scale the fp32 cost by ONE fp32 number
      // kh = fl32(log2(e) / epsilon) (a hi/lo pair would cost a second FMA
      // per pair on the FMA-bound on-the-fly path), so every device kernel
      // -- fast sweeps, exact fp64 passes, fallback, plan statistics --
      // uses the same internal scale kappa = kh / log2(e), within 2^-25
      // relative of 1 / epsilon: one consistent model whose solution differs
      // from the exact-epsilon one by O(2^-25) relative (parity against the
      // oracle at the TRUE epsilon: tests/test_gpu_otf.py, test_gpu_configs.py).
      P.storage = OTG_STORE_ON_THE_FLY;
      P.epsilon = epsilon;
      P.kappa = static_cast<double>(static_cast<float>(kLog2e / epsilon)) / kLog2e;
      upload_marginals(P, a, b);
      std::vector<float> hx(nl * 4, 0.f), hy(P.mpad * 4, 0.f);
      for (int64_t i = 0; i < nl; ++i)
        for (int64_t k = 0; k < d; ++k) hx[i * 4 + k] = static_cast<float>(xl[i * d + k]);
      for (int64_t j = 0; j < m; ++j)
        for (int64_t k = 0; k < d; ++k) hy[j * 4 + k] = static_cast<float>(y[j * d + k]);
      std::vector<float> hyn(P.mpad * 3, 0.f);  // negated SoA copy for the packed kernels
      for (int64_t j = 0; j < m; ++j)
        for (int64_t k = 0; k < d; ++k) hyn[k * P.mpad + j] = -hy[j * 4 + k];
      P.X = dalloc<float>(P, hx.size());
      P.Y = dalloc<float>(P, hy.size());
      P.Yn = dalloc<float>(P, hyn.size());
      OTG_CUDA(cudaMemcpyAsync(P.X, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice, P.stream));
      OTG_CUDA(cudaMemcpyAsync(P.Y, hy.data(), hy.size() * 4, cudaMemcpyHostToDevice, P.stream));
      OTG_CUDA(cudaMemcpyAsync(P.Yn, hyn.data(), hyn.size() * 4, cudaMemcpyHostToDevice,
                               P.stream));
      setup_cull(P, hx, hy);
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      finish_create(P, opts, out);
      return;
    }
    if (cost == OTG_COST_COSINE) {  // data.cpp:89-96 unit-row check
      for (int side = 0; side < 2; ++side) {
        const double* Z = side ? y : xl;
        const int64_t rows = side ? m : nl;
        for (int64_t i = 0; i < rows; ++i) {
          double s = 0.0;
          for (int64_t k = 0; k < d; ++k) s += Z[i * d + k] * Z[i * d + k];
          if (std::abs(std::sqrt(s) - 1.0) > 1e-6)
            fail(OTG_E_OT, "cosine cost expects unit rows");
        }
      }
    }
    P.epsilon = epsilon;
    P.kappa = 1.0 / epsilon;
    upload_marginals(P, a, b);
    double *dX = nullptr, *dY = nullptr;
    OTG_CUDA(cudaMalloc(&dX, nl * d * sizeof(double)));
    OTG_CUDA(cudaMalloc(&dY, m * d * sizeof(double)));
    OTG_CUDA(cudaMemcpyAsync(dX, xl, nl * d * sizeof(double), cudaMemcpyHostToDevice, P.stream));
    OTG_CUDA(cudaMemcpyAsync(dY, y, m * d * sizeof(double), cudaMemcpyHostToDevice, P.stream));
    double mn = 0.0, mx = 0.0;
    if (norm != OTG_NORM_NONE && norm != OTG_NORM_HALFRANGE) {
      const int blocks = 148 * 8;
      double2* part = nullptr;
      OTG_CUDA(cudaMalloc(&part, blocks * sizeof(double2)));
      if (d == 3)
        k_cost_minmax<3><<<blocks, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, part);
      else
        k_cost_minmax<0><<<blocks, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, part);
      OTG_CUDA(cudaGetLastError());
      std::vector<double2> hp(blocks);
      OTG_CUDA(cudaMemcpyAsync(hp.data(), part, blocks * sizeof(double2), cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      cudaFree(part);
      mn = DBL_MAX;
      mx = -DBL_MAX;
      for (auto& v : hp) {
        mn = std::min(mn, v.x);
        mx = std::max(mx, v.y);
      }
      if (P.sharded) {
        comm_init(P, opts);
        double buf[2] = {-mn, mx};
        double* dbuf = nullptr;
        OTG_CUDA(cudaMalloc(&dbuf, 2 * sizeof(double)));
        OTG_CUDA(cudaMemcpyAsync(dbuf, buf, sizeof buf, cudaMemcpyHostToDevice, P.stream));
        comm_allreduce_max(P, dbuf, 2);
        OTG_CUDA(cudaMemcpyAsync(buf, dbuf, sizeof buf, cudaMemcpyDeviceToHost, P.stream));
        OTG_CUDA(cudaStreamSynchronize(P.stream));
        cudaFree(dbuf);
        mn = -buf[0];
        mx = buf[1];
      }
    }
    P.raw_min = mn;
    P.raw_max = mx;
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((m + kT - 1) / kT, 64)),
              static_cast<unsigned>(std::min<int64_t>(nl, 65535)));
    if (storage == OTG_STORE_F64) {
      P.storage = OTG_STORE_F64;
      P.C64 = dalloc<double>(P, static_cast<size_t>(nl) * P.ldc);
      if (d == 3)
        k_cost_store<double, 3><<<grid, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, norm, mn, mx,
                                                           epsilon, P.C64, P.ldc);
      else
        k_cost_store<double, 0><<<grid, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, norm, mn, mx,
                                                           epsilon, P.C64, P.ldc);
    } else {
      P.storage = OTG_STORE_F32;
      P.C32 = dalloc<float>(P, static_cast<size_t>(nl) * P.ldc);
      if (d == 3)
        k_cost_store<float, 3><<<grid, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, norm, mn, mx,
                                                          1.0, P.C32, P.ldc);
      else
        k_cost_store<float, 0><<<grid, kT, 0, P.stream>>>(dX, dY, nl, m, d, cost, norm, mn, mx,
                                                          1.0, P.C32, P.ldc);
    }
    OTG_CUDA(cudaGetLastError());
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    cudaFree(dX);
    cudaFree(dY);
    if (P.sharded && P.nccl_comm) {
      // communicator already built for the normaliser; finish_create must not re-init
      problem_alloc_state(P);
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      auto* h = new otg_problem_s;
      h->P = P;
      *out = h;
      return;
    }
    finish_create(P, opts, out);
  });
  if (st != OTG_OK) problem_free(P);
  return st;
}

otg_status otg_problem_destroy(otg_problem h) {
  return guard([&] {
    if (!h) return;
    cudaSetDevice(h->P.device);
    cudaStreamSynchronize(h->P.stream);
    problem_free(h->P);
    delete h;
  });
}

otg_status otg_problem_info_get(otg_problem h, otg_problem_info* out) {
  return guard([&] {
    if (!h || !out) fail(OTG_E_DIMENSION, "NULL handle");
    const Problem& P = h->P;
    out->n = P.n;
    out->m = P.m;
    out->n_local = P.n_local;
    out->row_begin = P.row_begin;
    out->storage = P.storage;
    out->epsilon = P.epsilon;
    out->cost_raw_min = P.raw_min;
    out->cost_raw_max = P.raw_max;
    out->device_bytes = P.device_bytes;
    out->world_size = P.world;
    out->rank = P.rank;
    out->device = P.device;
    out->sweep_mode = P.storage == OTG_STORE_F64 ? 0 : (P.fused ? 2 : 1);
    out->sweep_clusters = P.fused_clusters;
    out->col_splits = P.col_splits;
  });
}

otg_status otg_problem_get_cost(otg_problem h, int64_t row0, int64_t nrows, void* outp) {
  return guard([&] {
    if (!h || !outp) fail(OTG_E_DIMENSION, "NULL argument");
    Problem& P = h->P;
    if (row0 < 0 || nrows < 0 || row0 + nrows > P.n_local) fail(OTG_E_DIMENSION, "row range");
    OTG_CUDA(cudaSetDevice(P.device));
    if (P.storage == OTG_STORE_F64) {
      // stored C' = C / eps: undo the fold for the caller (exact only up to
      // rounding; the parity tests use fp32 storage or eps = 1 with fp64)
      std::vector<double> tmp(static_cast<size_t>(nrows) * P.m);
      OTG_CUDA(cudaMemcpy2DAsync(tmp.data(), P.m * sizeof(double), P.C64 + row0 * P.ldc,
                                 P.ldc * sizeof(double), P.m * sizeof(double), nrows,
                                 cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      double* o = static_cast<double*>(outp);
      for (size_t k = 0; k < tmp.size(); ++k) o[k] = P.epsilon == 1.0 ? tmp[k] : tmp[k] * P.epsilon;
    } else if (P.storage == OTG_STORE_ON_THE_FLY) {  // evaluate the recomputed cost
      float* d = nullptr;
      OTG_CUDA(cudaMalloc(&d, std::max<int64_t>(nrows * P.m, 1) * sizeof(float)));
      k_otf_rows<<<static_cast<unsigned>(std::max<int64_t>(nrows, 1)), kT, 0, P.stream>>>(
          reinterpret_cast<const float4*>(P.X), reinterpret_cast<const float4*>(P.Y), row0,
          nrows, P.m, d);
      OTG_CUDA(cudaGetLastError());
      OTG_CUDA(cudaMemcpyAsync(outp, d, nrows * P.m * sizeof(float), cudaMemcpyDeviceToHost,
                               P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      cudaFree(d);
    } else {
      OTG_CUDA(cudaMemcpy2DAsync(outp, P.m * sizeof(float), P.C32 + row0 * P.ldc,
                                 P.ldc * sizeof(float), P.m * sizeof(float), nrows,
                                 cudaMemcpyDeviceToHost, P.stream));
      OTG_CUDA(cudaStreamSynchronize(P.stream));
    }
  });
}

}  // extern "C"
