// capi.cpp — ABI-level helpers: thread-local last error, version, devices.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "common.cuh"

namespace otg {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
bool pdl_enabled() { return OTG_PDL != 0; }
}  // namespace otg

extern "C" {

const char* otg_last_error(void) { return otg::g_last_error.c_str(); }

int otg_abi_version(void) { return OTG_ABI_VERSION; }

otg_status otg_device_count(int* count) {
  return otg::guard([&] {
    if (!count) otg::fail(OTG_E_DIMENSION, "NULL output");
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    *count = e == cudaSuccess ? c : 0;
  });
}

}  // extern "C"
