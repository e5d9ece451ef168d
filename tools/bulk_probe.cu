// Streaming-rate probe for 1-D bulk-copy (cp.async.bulk) row rings on B200:
// each CTA streams whole rows (row = ROWB bytes) of a buffer through NSLOT
// smem slots, split into SPLIT copies per row; the consumer (all threads)
// touches one word per 16 bytes and releases the slot.  Prints GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/bulk_probe tools/bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(su32(bar)) : "memory");
}

__global__ void __launch_bounds__(512, 1) k_stream(const float4* __restrict__ A, int64_t rows, int rowb, int nslot,
                                                   int split, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  float4* ring = reinterpret_cast<float4*>(sm + 1024);
  const int tid = threadIdx.x, H = gridDim.x, c = blockIdx.x;
  const int nr = rows > c ? static_cast<int>((rows - c + H - 1) / H) : 0;
  const int r4 = rowb / 16;
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], blockDim.x / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < nr && k < nslot; ++k) {
      mb_expect(&full[k], rowb);
      for (int p = 0; p < split; ++p)
        bulk(ring + k * r4 + p * (r4 / split), A + (c + (int64_t)H * k) * r4 + p * (r4 / split), rowb / split, &full[k]);
    }
  }
  float acc = 0.f;
  int s = 0; uint32_t ph = 0;
  for (int k = 0; k < nr; ++k) {
    mb_wait(&full[s], ph);
    for (int q = tid; q < r4; q += blockDim.x) acc += ring[s * r4 + q].x;
    __syncwarp();
    if ((tid & 31) == 0) mb_arrive(&empty[s]);
    if (tid == 0 && k + nslot < nr) {
      mb_wait(&empty[s], ph);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mb_expect(&full[s], rowb);
      for (int p = 0; p < split; ++p)
        bulk(ring + s * r4 + p * (r4 / split), A + (c + (int64_t)H * (k + nslot)) * r4 + p * (r4 / split), rowb / split, &full[s]);
    }
    if (++s == nslot) { s = 0; ph ^= 1; }
  }
  if (acc == 12345.f) sink[0] = 1;
}

int main() {
  const int64_t total = 268435456;  // bytes (cfg2 fp32 cost)
  float4* A; unsigned long long* sink;
  cudaMalloc(&A, total); cudaMemset(A, 0, total); cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int rowbs[] = {16384, 32768};
  const int splits[] = {1, 2, 4, 8};
  for (int rowb : rowbs) for (int split : splits) for (int nslot : {3, 4, 6, 8, 12}) { if (nslot > 220 * 1024 / rowb) continue;
    const int64_t rows = total / rowb;
    const int smem = 1024 + nslot * rowb;
    for (int it = 0; it < 3; ++it) k_stream<<<sms, 512, smem>>>(A, rows, rowb, nslot, split, sink);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) k_stream<<<sms, 512, smem>>>(A, rows, rowb, nslot, split, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("row %6d B  split %d  slots %2d : %7.1f us  %7.1f GB/s %s\n", rowb, split, nslot, 1000 * ms / reps,
           total / (ms / reps * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
  }
  return 0;
}
