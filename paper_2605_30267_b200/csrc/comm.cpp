// comm.cpp — NCCL for row-sharded handles (one rank per GPU).
//
// libnccl is opened lazily with dlopen (soname libnccl.so.2): a process that
// already loaded torch's NCCL 2.28.9 gets that same copy, and single-GPU
// handles never touch NCCL at all.  The only collective on the hot path is
// the in-place fp64 SUM all-reduce of the m column partial sums (+ the local
// <u, a> partial) once per evaluation; it is issued on the
// handle's stream, so it is captured into the solver's chunk graph.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

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

}  // namespace

void comm_init(Problem& P, const void* unique_id) {
  if (P.nccl_comm) return;
  if (!unique_id) fail(OTG_E_NCCL, "world_size > 1 needs nccl_unique_id");
  nccl_unique_id_t id;
  std::memcpy(id.internal, unique_id, sizeof id.internal);
  nccl_comm_t comm = nullptr;
  check(api().init_rank(&comm, P.world, id, P.rank), "ncclCommInitRank");
  P.nccl_comm = comm;
}

void comm_destroy(Problem& P) {
  if (P.nccl_comm) api().destroy(static_cast<nccl_comm_t>(P.nccl_comm));
  P.nccl_comm = nullptr;
}

void comm_allreduce_sum(Problem& P, double* buf, size_t count) {
  check(api().all_reduce(buf, buf, count, kNcclDouble, kNcclSum,
                         static_cast<nccl_comm_t>(P.nccl_comm), P.stream),
        "ncclAllReduce");
}

void comm_allreduce_max(Problem& P, double* buf, size_t count) {
  check(api().all_reduce(buf, buf, count, kNcclDouble, kNcclMax,
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
