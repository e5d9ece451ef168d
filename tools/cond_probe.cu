// Microbenchmark: per-node cost of kernel nodes vs false IF conditional
// nodes inside a CUDA-graph WHILE loop (B200).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/cond_probe tools/cond_probe.cu && /tmp/cond_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void k_work(int* c, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(c, 1);
}
__global__ void k_noop(const int* c) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*c < 0) printf("x");
}
__global__ void k_set(cudaGraphConditionalHandle h, unsigned v) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, v);
}
// WHILE body tail: count iterations, stop after `iters`
__global__ void k_loop(cudaGraphConditionalHandle h, int* it, int iters) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int k = ++*it;
    cudaGraphSetConditional(h, k < iters ? 1u : 0u);
  }
}

static void launch(void (*k)(int*, int), cudaStream_t s, int* c, int g, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, c, 0);
}
template <typename... A>
static void launchx(void (*k)(A...), cudaStream_t s, int g, bool pdl, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// body variant: K work kernels per iteration, plus `nif` false IF nodes
// (each guarding a k_noop) or `nnoop` plain no-op kernels.
static int run(int K, int nif, int nnoop, int grid, bool pdl, int iters, cudaStream_t s, int* d) {
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hf = 0;
  if (nif > 0) CK(cudaGraphConditionalHandleCreate(&hf, getenv("HF_TOP") ? g : body, 0, 0));
  cudaStream_t s2;
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  if (nif > 0) launchx(k_set, s, 1, pdl, hf, 0u);
  for (int k = 0; k < K; ++k) {
    launch(k_work, s, d, grid, pdl);
    if (k < nif) {
      cudaStreamCaptureStatus st;
      const cudaGraphNode_t* deps;
      const cudaGraphEdgeData* ed;
      size_t nd;
      cudaGraph_t cg;
      CK(cudaStreamGetCaptureInfo_v3(s, &st, nullptr, &cg, &deps, &ed, &nd));
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hf;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      cudaGraphNode_t in;
      cudaError_t e1 = cudaGraphAddNode_v2(&in, cg, deps, ed, nd, &ip);
      if (e1 != cudaSuccess) {
        printf("AddNode_v2 (cg %s body, %zu deps, edge type %d): %s\n", cg == body ? "==" : "!=", nd,
               nd ? (int)ed[0].type : -1, cudaGetErrorString(e1));
        cudaGraph_t o;
        cudaStreamEndCapture(s, &o);
        return 1;
      }
      CK(cudaStreamUpdateCaptureDependencies(s, &in, 1, cudaStreamSetCaptureDependencies));
      cudaGraph_t ib = ip.conditional.phGraph_out[0];
      CK(cudaStreamBeginCaptureToGraph(s2, ib, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      launchx(k_noop, s2, grid, false, (const int*)d);
      cudaGraph_t o;
      CK(cudaStreamEndCapture(s2, &o));
    }
    if (k < nnoop) launchx(k_noop, s, grid, pdl, (const int*)d);
  }
  launchx(k_loop, s, 1, pdl, hw, d + 1, iters);
  cudaGraph_t o;
  CK(cudaStreamEndCapture(s, &o));
  cudaGraphExec_t ex;
  {
    cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
    if (e2 != cudaSuccess) {
      cudaGraphInstantiateParams ipm = {};
      e2 = cudaGraphInstantiateWithParams(&ex, g, &ipm);
      printf("instantiate: %s (result %d)\n", cudaGetErrorString(e2), (int)ipm.result_out);
      return 1;
    }
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemsetAsync(d, 0, 8, s));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(ex, s));
    CK(cudaEventRecord(b, s));
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int h[2];
    CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    if (rep == 2)
      printf("K=%d work kernels, %d false IF nodes, %d no-op kernels, grid %d, pdl %d: %.2f us / iteration (%d its)\n",
             K, nif, nnoop, grid, pdl ? 1 : 0, 1e3 * ms / iters, h[1]);
  }
  cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g);
  return 0;
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* d;
  CK(cudaMalloc(&d, 64));
  const int iters = 2000;
  for (int grid : {148, 1184}) {
    for (int pdl : {0, 1}) {
      run(6, 0, 0, grid, pdl, iters, s, d);
      run(6, 3, 0, grid, pdl, iters, s, d);
      run(6, 0, 3, grid, pdl, iters, s, d);
      run(9, 0, 0, grid, pdl, iters, s, d);
    }
  }
  return 0;
}
