// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdio>
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

}  // namespace bsnp
