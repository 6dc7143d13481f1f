// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/bitsnap_b200.h"

namespace bsnp {

void set_last_error(const char* what, cudaError_t e);

inline int cuda_status(const char* what, cudaError_t e) {
  if (e == cudaSuccess) return BSNP_OK;
  set_last_error(what, e);
  return BSNP_E_CUDA;
}

// Check the launch that was just enqueued.
inline int launch_status(const char* what) { return cuda_status(what, cudaGetLastError()); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// SM count of the current device (queried once per device ordinal); *dev
// receives the ordinal
inline int device_sms(int* dev = nullptr) {
  static int cache[64] = {0};
  int d = 0;
  cudaGetDevice(&d);
  if (dev) *dev = d;
  if (d < 0 || d >= 64) return 1;
  if (!cache[d]) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    cache[d] = sms < 1 ? 1 : sms;
  }
  return cache[d];
}

// Launch with programmatic stream serialization: the kernel (which must
// start with pdl_enter, common.cuh) may be scheduled while its predecessor
// in the stream still runs its last wave, so a chain of dependent launches
// does not pay a full drain + launch gap per kernel.  BSNP_PDL=0 (read once)
// launches ordinarily.
inline bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("BSNP_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on != 0;
}

template <typename... KArgs, typename... Args>
int launch_pdl_smem(const char* what, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                    size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cuda_status(what, cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...));
}

template <typename... KArgs, typename... Args>
int launch_pdl(const char* what, void (*kernel)(KArgs...), dim3 grid, dim3 block,
               cudaStream_t s, Args... args) {
  return launch_pdl_smem(what, kernel, grid, block, 0, s, args...);
}

}  // namespace bsnp
