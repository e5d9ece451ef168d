// batched.cu — placeholder, replaced by the one-CTA-per-problem kernel.
#include "common.cuh"
using namespace otg;
extern "C" {
otg_status otg_batch_create_dense(int64_t, const int32_t*, const int32_t*, const double*,
                                  const double*, const float*, double, const otg_device_opts*,
                                  otg_batch*) {
  return guard([] { fail(OTG_E_UNSUPPORTED, "batched path not built yet"); });
}
otg_status otg_batch_create_cosine(int64_t, const int32_t*, const int32_t*, int64_t,
                                   const double*, const double*, const float*, const float*,
                                   otg_norm, double, const otg_device_opts*, otg_batch*) {
  return guard([] { fail(OTG_E_UNSUPPORTED, "batched path not built yet"); });
}
otg_status otg_batch_destroy(otg_batch) { return OTG_OK; }
otg_status otg_batch_get_cost(otg_batch, float*) {
  return guard([] { fail(OTG_E_UNSUPPORTED, "batched path not built yet"); });
}
otg_status otg_batch_homotopy_solve(otg_batch, const otg_homotopy_config*, otg_batch_result*) {
  return guard([] { fail(OTG_E_UNSUPPORTED, "batched path not built yet"); });
}
}
