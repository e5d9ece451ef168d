// comm.cpp — the collective of row-sharded handles (one rank per GPU): NCCL,
// or a caller-supplied host all-reduce (otg_device_opts.allreduce).
//
// libnccl is opened lazily with dlopen (soname libnccl.so.2): a process that
// already loaded torch's NCCL 2.28.9 gets that same copy, and single-GPU
// handles never touch NCCL at all.  The only collective on the hot path is
// the in-place fp64 SUM all-reduce of the m column partial sums (+ the local
// <u, a> partial) once per evaluation; it is issued on the
// handle's stream, so it is captured into the solver's chunk graph.
#include <dlfcn.h>
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace otg {
namespace {

typedef int nccl_result_t;
typedef struct {
  char internal[128];
} nccl_unique_id_t;
typedef void* nccl_comm_t;

struct NcclApi {
  void* lib = nullptr;
  nccl_result_t (*get_unique_id)(nccl_unique_id_t*) = nullptr;
  nccl_result_t (*init_rank)(nccl_comm_t*, int, nccl_unique_id_t, int) = nullptr;
  nccl_result_t (*destroy)(nccl_comm_t) = nullptr;
  nccl_result_t (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t,
                              cudaStream_t) = nullptr;
  const char* (*error_string)(nccl_result_t) = nullptr;
  nccl_result_t (*get_async_error)(nccl_comm_t, nccl_result_t*) = nullptr;
  nccl_result_t (*abort)(nccl_comm_t) = nullptr;
};

constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;
constexpr int kNcclMax = 2;

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.lib, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
    a.get_async_error =
        reinterpret_cast<decltype(a.get_async_error)>(dlsym(a.lib, "ncclCommGetAsyncError"));
    a.abort = reinterpret_cast<decltype(a.abort)>(dlsym(a.lib, "ncclCommAbort"));
  });
  if (!a.lib || !a.init_rank || !a.all_reduce)
    fail(OTG_E_NCCL, "libnccl.so.2 not loadable (import torch first, or add it to LD_LIBRARY_PATH)");
  return a;
}

void check(nccl_result_t r, const char* what) {
  if (r != 0) {
    const char* s = api().error_string ? api().error_string(r) : "?";
    fail(OTG_E_NCCL, std::string(what) + ": " + s);
  }
}


// Host all-reduce (otg_device_opts.allreduce): D2H into pinned staging, a
// host node calls the caller's reduction, H2D back.  All three are stream
// operations, so the sequence is captured into the chunk graph like the NCCL
// call.  A failing callback is recorded and raised at the next sync point.
struct HostArgs {
  otg_allreduce_fn fn;
  void* ctx;
  double* buf;
  int64_t count;
  int op;
  int* failed;
  bool own;  // buf is this call site's own pinned buffer (captured calls)
};

void CUDART_CB host_allreduce(void* raw) {
  auto* a = static_cast<HostArgs*>(raw);
  if (a->fn(a->buf, a->count, a->op, a->ctx) != 0) *a->failed = 1;
}

struct HostComm {
  std::vector<HostArgs*> captured;  // call sites baked into chunk graphs
  HostArgs eager{};                 // reused by eager calls (stream-ordered)
  int failed = 0;
};

void host_allreduce_enqueue(Problem& P, const double* send, double* recv, size_t count, int op) {
  auto* hc = static_cast<HostComm*>(P.nccl_comm);
  HostArgs* a = nullptr;
  if (P.capturing) {
    // a graph keeps its pointers: every captured call site owns its staging
    a = new HostArgs{P.ar_fn, P.ar_ctx, nullptr, static_cast<int64_t>(count), op, &hc->failed,
                     true};
    // (pinned allocation is not a stream operation: relax the capture mode for it)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    OTG_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
    const cudaError_t e = cudaMallocHost(&a->buf, count * sizeof(double));
    OTG_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
    OTG_CUDA(e);
    hc->captured.push_back(a);
  } else {
    if (count > P.ar_host_len) {
      OTG_CUDA(cudaStreamSynchronize(P.stream));
      if (P.ar_host) cudaFreeHost(P.ar_host);
      P.ar_host = nullptr;
      OTG_CUDA(cudaMallocHost(&P.ar_host, count * sizeof(double)));
      P.ar_host_len = count;
    }
    a = &hc->eager;
    OTG_CUDA(cudaStreamSynchronize(P.stream));  // the previous eager call's args are done
    *a = HostArgs{P.ar_fn, P.ar_ctx, P.ar_host, static_cast<int64_t>(count), op, &hc->failed,
                  false};
  }
  OTG_CUDA(cudaMemcpyAsync(a->buf, send, count * sizeof(double), cudaMemcpyDeviceToHost,
                           P.stream));
  OTG_CUDA(cudaLaunchHostFunc(P.stream, host_allreduce, a));
  OTG_CUDA(cudaMemcpyAsync(recv, a->buf, count * sizeof(double), cudaMemcpyHostToDevice,
                           P.stream));
}

}  // namespace

void comm_init(Problem& P, const otg_device_opts* opts) {
  if (P.nccl_comm) return;
  if (opts && opts->allreduce) {
    P.ar_fn = opts->allreduce;
    P.ar_ctx = opts->allreduce_ctx;
    P.nccl_comm = new HostComm;
    return;
  }
  if (!opts || !opts->nccl_unique_id)
    fail(OTG_E_NCCL, "a sharded handle needs nccl_unique_id or an allreduce callback");
  nccl_unique_id_t id;
  std::memcpy(id.internal, opts->nccl_unique_id, sizeof id.internal);
  nccl_comm_t comm = nullptr;
  check(api().init_rank(&comm, P.world, id, P.rank), "ncclCommInitRank");
  P.nccl_comm = comm;
}

void comm_destroy(Problem& P) {
  if (!P.nccl_comm) return;
  if (P.ar_fn) {
    auto* hc = static_cast<HostComm*>(P.nccl_comm);
    for (auto* a : hc->captured) {
      cudaFreeHost(a->buf);
      delete a;
    }
    delete hc;
    if (P.ar_host) cudaFreeHost(P.ar_host);
    P.ar_host = nullptr;
  } else {
    api().destroy(static_cast<nccl_comm_t>(P.nccl_comm));
  }
  P.nccl_comm = nullptr;
}

// Host-side wait for the handle's stream that keeps polling the NCCL
// communicator's asynchronous error state (a peer rank that died or a broken
// link leaves the all-reduce -- and a plain stream synchronize -- waiting
// forever): on an error the communicator is aborted, which releases the
// stream, and the call fails with OTG_E_NCCL.  Host-callback handles and
// unsharded handles just synchronize.
void comm_sync(Problem& P) {
  if (!P.sharded || P.ar_fn || !P.nccl_comm || !api().get_async_error) {
    OTG_CUDA(cudaStreamSynchronize(P.stream));
    return;
  }
  for (unsigned spins = 0;; ++spins) {
    const cudaError_t q = cudaStreamQuery(P.stream);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) OTG_CUDA(q);
    nccl_result_t r = 0;
    api().get_async_error(static_cast<nccl_comm_t>(P.nccl_comm), &r);
    if (r != 0 && r != 7 /* ncclInProgress */) {
      const char* s = api().error_string ? api().error_string(r) : "?";
      if (api().abort) api().abort(static_cast<nccl_comm_t>(P.nccl_comm));
      P.nccl_comm = nullptr;  // aborted: nothing left to destroy
      fail(OTG_E_NCCL, std::string("NCCL asynchronous error: ") + s);
    }
    if (spins > 64) usleep(20);  // (after a short spin: chunks are ~ms long)
  }
}

int comm_failed(Problem& P) {
  return (P.ar_fn && P.nccl_comm) ? static_cast<HostComm*>(P.nccl_comm)->failed : 0;
}

void comm_allreduce_sum(Problem& P, const double* send, double* recv, size_t count) {
  if (P.ar_fn) return host_allreduce_enqueue(P, send, recv, count, 0);
  check(api().all_reduce(send, recv, count, kNcclDouble, kNcclSum,
                         static_cast<nccl_comm_t>(P.nccl_comm), P.stream),
        "ncclAllReduce");
}

void comm_allreduce_max(Problem& P, const double* send, double* recv, size_t count) {
  if (P.ar_fn) return host_allreduce_enqueue(P, send, recv, count, 1);
  check(api().all_reduce(send, recv, count, kNcclDouble, kNcclMax,
                         static_cast<nccl_comm_t>(P.nccl_comm), P.stream),
        "ncclAllReduce");
}

}  // namespace otg

extern "C" otg_status otg_nccl_get_unique_id(void* out128) {
  return otg::guard([&] {
    if (!out128) otg::fail(OTG_E_DIMENSION, "NULL output");
    otg::nccl_unique_id_t id;
    otg::check(otg::api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, sizeof id.internal);
  });
}
