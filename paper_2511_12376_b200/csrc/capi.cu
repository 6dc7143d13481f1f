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

// Page-lock an existing host range (e.g. a mapped staging region) for DMA.
// A failed registration (a disk-backed mapping) is cleared from this
// runtime's error state and reported as BSNP_E_CUDA.
extern "C" int bsnp_host_register(void* ptr, size_t bytes) {
  if (!ptr || !bytes) return BSNP_E_INVALID;
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    bsnp::set_last_error("cudaHostRegister", e);
    return BSNP_E_CUDA;
  }
  return BSNP_OK;
}

extern "C" int bsnp_host_unregister(void* ptr) {
  if (!ptr) return BSNP_E_INVALID;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    bsnp::set_last_error("cudaHostUnregister", e);
    return BSNP_E_CUDA;
  }
  return BSNP_OK;
}
