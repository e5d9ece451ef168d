// L2 staging probe: can a stream read from HBM be re-read from L2 by a
// second consumer a chunk later, at what aggregate rate?  Standalone tool
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu).
//
// modes: 0 = HBM stream once (baseline), 1 = pipelined producer/consumer
// (producer warps read chunk c from HBM, consumer warps re-read chunk c - 1),
// 2 = L2-resident re-read rate (a small buffer read many times).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ float4 ld_hint(const float4* a, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_plain(const float4* a) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(a));
  return r;
}

// chunk = R rows of W floats, split into segments of SEG float4 per warp item

__global__ void __launch_bounds__(512, 1)
k_pipe(const float4* __restrict__ C, int64_t nchunks, int64_t chunk_f4, int hints, int lag,
       unsigned* done, unsigned* cdone, float* sink) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool prod = warp < 8;
  const unsigned nw = gridDim.x * 8;
  const unsigned gw = blockIdx.x * 8 + (warp % 8);
  const uint64_t pl = pol_last(), pf = pol_first();
  float acc = 0.f;
  for (int64_t c = 0; c < nchunks + 1; ++c) {
    if (prod) {
      if (c >= nchunks) break;
      if (c >= lag) {  // do not run more than `lag` chunks ahead of the consumers
        if (threadIdx.x == 0) while (*(volatile unsigned*)&cdone[c - lag] < gridDim.x) __nanosleep(64);
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      const float4* base = C + c * chunk_f4;
      const int64_t seg = ((chunk_f4 + nw - 1) / nw + 255) / 256 * 256;
      for (int64_t i0 = gw * seg; i0 < (gw + 1) * seg && i0 < chunk_f4; i0 += 256) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (hints & 1) ? ld_hint(base + i0 + k * 32 + lane, pl) : ld_plain(base + i0 + k * 32 + lane);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 0) { __threadfence(); atomicAdd(&done[c], 1u); }
    } else {
      if (c == 0) continue;
      const int64_t cc = c - 1;
      if (threadIdx.x == 256) while (*(volatile unsigned*)&done[cc] < gridDim.x) __nanosleep(32);
      asm volatile("bar.sync 2, 256;" ::: "memory");
      const float4* base = C + cc * chunk_f4;
      // consumers take the items in a different order (a column-slab owner would)
      const unsigned g2 = (hints & 2) ? gw : (gw * 7 + 3) % nw;
      const int64_t seg = ((chunk_f4 + nw - 1) / nw + 255) / 256 * 256;
      for (int64_t i0 = g2 * seg; i0 < (g2 + 1) * seg && i0 < chunk_f4; i0 += 256) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (hints & 1) ? ld_hint(base + i0 + k * 32 + lane, pf) : ld_plain(base + i0 + k * 32 + lane);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k].x * v[k].y + v[k].z * v[k].w;
      }
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (threadIdx.x == 256) { __threadfence(); atomicAdd(&cdone[cc], 1u); }
    }
  }
  if (acc == 123.456f) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 1)
k_stream(const float4* __restrict__ C, int64_t n_f4, int reps, float* sink) {
  float acc = 0.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_f4; i += stride) {
      float4 v = ld_plain(C + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 123.456f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t W = 65536;
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 16384;
  int dev_sms = 0;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n_f4 = rows * W / 4;
  float4* C;
  CK(cudaMalloc(&C, n_f4 * 16));
  CK(cudaMemset(C, 0, n_f4 * 16));
  float* sink; CK(cudaMalloc(&sink, 4));
  unsigned *done, *cdone;
  CK(cudaMalloc(&done, 1 << 20)); CK(cudaMalloc(&cdone, 1 << 20));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  const double bytes = static_cast<double>(n_f4) * 16;
  // mode 0: HBM stream
  for (int t = 0; t < 3; ++t) {
    CK(cudaEventRecord(a));
    k_stream<<<dev_sms, 512>>>(C, n_f4, 1, sink);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  }
  CK(cudaEventElapsedTime(&ms, a, b));
  std::printf("stream once: %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
  // mode 2: L2-resident re-read
  for (int64_t mb : {16, 32, 48, 64, 96}) {
    const int64_t sf4 = mb * (1 << 20) / 16;
    for (int t = 0; t < 3; ++t) {
      CK(cudaEventRecord(a));
      k_stream<<<dev_sms, 512>>>(C, sf4, 50, sink);
      CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    }
    CK(cudaEventElapsedTime(&ms, a, b));
    std::printf("L2 re-read %3lld MB x50: %.3f ms  %.1f GB/s\n", (long long)mb, ms, 50.0 * sf4 * 16 / ms / 1e6);
  }
  // mode 1: pipeline
  for (int hints : {0, 1, 3})
    for (int R : {8, 16, 32, 64, 128})
      for (int lag : {2, 3, 4, 6, 8}) {
        if (R * lag > 512) continue;
        const int64_t chunk_f4 = R * W / 4;
        const int64_t nch = n_f4 / chunk_f4;
        float best = 1e9;
        for (int t = 0; t < 3; ++t) {
          CK(cudaMemset(done, 0, 1 << 20)); CK(cudaMemset(cdone, 0, 1 << 20));
          CK(cudaEventRecord(a));
          k_pipe<<<dev_sms, 512>>>(C, nch, chunk_f4, hints, lag, done, cdone, sink);
          CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
          CK(cudaEventElapsedTime(&ms, a, b));
          if (ms < best) best = ms;
        }
        std::printf("pipe hints=%d R=%3d (%3lld MB) lag=%d: %.3f ms  HBM-eq %.1f GB/s (%.2fx stream-once time)\n",
                    hints, R, (long long)(chunk_f4 * 16 >> 20), lag, best, bytes / best / 1e6, 0.0);
      }
  CK(cudaGetLastError());
  return 0;
}
