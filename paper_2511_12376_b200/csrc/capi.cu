// C-ABI housekeeping: version, error text, device info.
#include <cstring>

#include "runtime.cuh"

namespace bsnp {
static thread_local char g_last_error[512] = "";

void set_last_error(const char* what, cudaError_t e) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", what,
                cudaGetErrorString(e), cudaGetErrorName(e));
}
}  // namespace bsnp

extern "C" int bsnp_abi_version(void) { return BSNP_ABI_VERSION; }

extern "C" const char* bsnp_last_error(void) { return bsnp::g_last_error; }

extern "C" int bsnp_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return sms;
}
