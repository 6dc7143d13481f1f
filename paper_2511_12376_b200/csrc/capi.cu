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

// ---------------------------------------------------------------------------
// checkpoint blob assembly: one CTA per 64 KiB chunk of a segment
namespace {
__global__ void __launch_bounds__(256)
    gather_segments_kernel(const bsnp_segment* __restrict__ segs,
                           const uint32_t* __restrict__ first, uint32_t nsegs,
                           uint8_t* __restrict__ blob) {
  __shared__ uint32_t s_seg;
  const uint32_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = nsegs;  // largest s with first[s] <= b
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (first[mid] <= b) lo = mid;
      else hi = mid;
    }
    s_seg = lo;
  }
  __syncthreads();
  const bsnp_segment sg = segs[s_seg];
  const uint64_t c0 = (uint64_t)(b - first[s_seg]) * BSNP_GATHER_CHUNK;
  if (c0 >= sg.len) return;
  const uint64_t len = sg.len - c0 < BSNP_GATHER_CHUNK ? sg.len - c0 : BSNP_GATHER_CHUNK;
  const uint8_t* src = static_cast<const uint8_t*>(sg.src) + c0;
  uint8_t* dst = blob + sg.dst_off + c0;
  const uint32_t n = (uint32_t)len;
  const uint32_t mis = (uint32_t)(((uintptr_t)src ^ (uintptr_t)dst) & 15);
  uint32_t head = 0;
  if (mis == 0) {
    head = (uint32_t)((16 - ((uintptr_t)dst & 15)) & 15);
    if (head > n) head = n;
    const uint32_t nv = (n - head) / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) d4[i] = s4[i];
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) dst[i] = src[i];
    for (uint32_t i = head + nv * 16 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  } else {
    // dst-aligned 32-bit words built from two aligned source words with a
    // funnel shift (the byte offset between source and destination is the
    // same for the whole segment)
    head = (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3);
    if (head > n) head = n;
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) dst[i] = src[i];
    const uint32_t nw = (n - head) / 4;
    const uint8_t* s0 = src + head;
    const uint32_t sh = (uint32_t)((uintptr_t)s0 & 3) * 8;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>((uintptr_t)s0 & ~(uintptr_t)3);
    uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
    if (sh == 0) {
      for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) dw[i] = sw[i];
    } else {
      // the last word pair may read up to 3 bytes past the segment's source
      // end; those bytes stay inside the 4-byte word holding its last byte
      for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x)
        dw[i] = __funnelshift_r(sw[i], sw[i + 1], sh);
    }
    for (uint32_t i = head + nw * 4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

// small results to page-locked host memory through the SMs' stores rather
// than a copy engine: the read-back does not queue behind bulk
// device-to-host copies on other streams
__global__ void __launch_bounds__(256)
    copy_sm_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (((((uintptr_t)src) | ((uintptr_t)dst)) & 15) == 0) {
    const uint64_t nv = n / 16;
    for (uint64_t i = t0; i < nv; i += stride)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (uint64_t i = nv * 16 + t0; i < n; i += stride) dst[i] = src[i];
  } else {
    for (uint64_t i = t0; i < n; i += stride) dst[i] = src[i];
  }
}
}  // namespace

extern "C" int bsnp_copy_sm(const void* src, void* dst, uint64_t n, void* stream) {
  if (n == 0) return BSNP_OK;
  if (!src || !dst) return BSNP_E_INVALID;
  const int sms = bsnp::device_sms();  // one CTA per SM at most: small blocks, latency-bound
  uint64_t grid = (n / 16 + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > (uint64_t)sms) grid = (uint64_t)sms;
  copy_sm_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n);
  return bsnp::launch_status("copy_sm_kernel");
}

extern "C" int bsnp_gather_segments(const bsnp_segment* segs, const uint32_t* first,
                                    uint32_t nsegs, uint32_t nchunks, uint8_t* blob,
                                    void* stream) {
  if (nsegs == 0 || nchunks == 0) return BSNP_OK;
  if (!segs || !first || !blob) return BSNP_E_INVALID;
  gather_segments_kernel<<<nchunks, 256, 0, (cudaStream_t)stream>>>(segs, first, nsegs, blob);
  return bsnp::launch_status("gather_segments_kernel");
}
