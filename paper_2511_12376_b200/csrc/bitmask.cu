// Bitmask delta codec for sm_100a.
//
// Replaces the reference's encode_delta / decode_delta
// (/root/reference/pkg/src/bitsnap/bitmask.py:94-140).  Both directions are a
// single streaming pass over HBM:
//
//   tile      = 8192 elements = 256 threads x 4 groups x 8 elements
//   group g   = 8 consecutive elements = one 16-byte vector per operand =
//               exactly one mask byte (byte g, LSB-first, bitmask.py:102)
//   thread t of a tile owns groups j*256 + t (j = 0..3), so every warp-wide
//   load is 512 contiguous bytes and every mask store 32 contiguous bytes.
//
// Payload positions (ascending element order, bitmask.py:103) come from a
// block scan of per-group popcounts (packed 4 x 16-bit in a u64) plus a
// decoupled look-back across tiles (common.cuh), so the data is read once.
#include "common.cuh"
#include "runtime.cuh"

namespace bsnp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kVec = 4;                     // groups (16B vectors) per thread
constexpr uint64_t kTile = kThreads * kVec * 8;  // elements per tile
static_assert(kVec * kWarps == 32, "tile scan maps (group, warp) onto one warp");

constexpr size_t kWsHeader = 256;  // u32 tile ticket (+ padding)

inline uint64_t num_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }

struct TileScan {
  uint64_t prefix;          // exclusive prefix of the tile (elements)
  uint32_t off[kVec];       // offset of this thread's group j within the tile
  uint64_t total;           // tile popcount
};

// Block-wide scan of the 4 per-thread group counts + cross-tile look-back.
// Order of groups inside a tile: j-major, then thread (= element order).
__device__ __forceinline__ void tile_scan(const uint32_t (&cnt)[kVec], uint64_t tile,
                                          uint64_t* tile_status, TileScan& out,
                                          uint64_t* s_warp, uint32_t (*s_off)[kWarps],
                                          uint64_t* s_prefix) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t packed = 0;
#pragma unroll
  for (int j = 0; j < kVec; ++j) packed |= (uint64_t)cnt[j] << (16 * j);
  const uint64_t inc = warp_inclusive_scan_u64(packed, lane);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int j = lane / kWarps, w = lane % kWarps;
    const uint32_t v = (uint32_t)(s_warp[w] >> (16 * j)) & 0xffffu;
    const uint32_t x = warp_inclusive_scan_u32(v, lane);
    s_off[j][w] = x - v;
    const uint32_t total = __shfl_sync(kFull, x, 31);
    const uint64_t excl = lookback_exclusive(tile_status, tile, total, lane);
    if (lane == 0) {
      s_prefix[0] = excl;
      s_prefix[1] = total;
    }
  }
  __syncthreads();
  const uint64_t ex = inc - packed;
  out.prefix = s_prefix[0];
  out.total = s_prefix[1];
#pragma unroll
  for (int j = 0; j < kVec; ++j)
    out.off[j] = s_off[j][warp] + ((uint32_t)(ex >> (16 * j)) & 0xffffu);
}

// ------------------------------------------------------------------ encode
template <bool kAligned>
__global__ void __launch_bounds__(kThreads)
    delta_encode_kernel(const uint16_t* __restrict__ base, const uint16_t* __restrict__ cur,
                        uint64_t n, uint8_t* __restrict__ mask, uint16_t* __restrict__ payload,
                        uint64_t payload_cap, bsnp_status* __restrict__ st,
                        uint32_t* __restrict__ ticket, uint64_t* __restrict__ tile_status,
                        uint64_t ntiles) {
  __shared__ uint64_t s_warp[kWarps];
  __shared__ uint32_t s_off[kVec][kWarps];
  __shared__ uint64_t s_prefix[2];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * kTile;

  uint4 cv[kVec];
  uint32_t bits[kVec], cnt[kVec];
  if (kAligned && t0 + kTile <= n) {
    uint4 bv[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const uint64_t e = t0 + (uint64_t)(j * kThreads + tid) * 8;
      bv[j] = ld_stream_v4(base + e);
      cv[j] = ld_stream_v4(cur + e);
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) bits[j] = diff8(bv[j], cv[j]);
  } else {
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const uint64_t e = t0 + (uint64_t)(j * kThreads + tid) * 8;
      uint4 b = make_uint4(0, 0, 0, 0), c = make_uint4(0, 0, 0, 0);
      for (uint32_t k = 0; k < 8; ++k) {
        if (e + k < n) {
          set_u16_lane(b, k, base[e + k]);
          set_u16_lane(c, k, cur[e + k]);
        }
      }
      cv[j] = c;
      bits[j] = diff8(b, c);
    }
  }
#pragma unroll
  for (int j = 0; j < kVec; ++j) cnt[j] = __popc(bits[j]);

  TileScan sc;
  tile_scan(cnt, tile, tile_status, sc, s_warp, s_off, s_prefix);
  if (tid == 0 && tile == ntiles - 1) st->count = sc.prefix + sc.total;

  // mask bytes: 32 contiguous bytes per warp store
  const uint64_t g0 = t0 / 8;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const uint64_t g = g0 + j * kThreads + tid;
    if (g * 8 < n) mask[g] = (uint8_t)bits[j];
  }
  // payload: changed values in element order
  bool overflow = false;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    uint32_t b = bits[j];
    uint64_t pos = sc.prefix + sc.off[j];
    while (b) {
      const uint32_t k = __ffs(b) - 1;
      b &= b - 1;
      if (pos < payload_cap) payload[pos] = (uint16_t)u16_lane(cv[j], k);
      else overflow = true;
      ++pos;
    }
  }
  if (overflow) atomicOr(&st->err_flags, BSNP_ERR_PAYLOAD_CAP);
}

// ------------------------------------------------------------------ decode
// Mask pre-check for in-place decode: popcount of mask[:n] and padding bits.
__global__ void __launch_bounds__(256)
    delta_mask_check_kernel(const uint8_t* __restrict__ mask, uint64_t n,
                            bsnp_status* __restrict__ st) {
  const uint64_t nbytes = (n + 7) / 8;
  uint64_t local = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbytes;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = mask[i];
    const uint64_t e0 = i * 8;
    if (e0 + 8 > n) {
      const uint32_t valid = (uint32_t)(n - e0);
      if (b >> valid) atomicOr(&st->err_flags, BSNP_ERR_PADDING);
      b &= (1u << valid) - 1u;
    }
    local += __popc(b);
  }
  local = warp_sum_u64(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd((unsigned long long*)&st->count, local);
}

__global__ void delta_check_finish_kernel(bsnp_status* st, uint64_t n_c) {
  if (st->count != n_c) st->err_flags |= BSNP_ERR_POPCOUNT;
}

template <bool kAligned, bool kInPlace>
__global__ void __launch_bounds__(kThreads)
    delta_decode_kernel(const uint16_t* base, const uint8_t* __restrict__ mask,
                        const uint16_t* __restrict__ payload, uint64_t n, uint64_t n_c,
                        uint16_t* out, bsnp_status* __restrict__ st,
                        uint32_t* __restrict__ ticket, uint64_t* __restrict__ tile_status,
                        uint64_t ntiles) {
  __shared__ uint64_t s_warp[kWarps];
  __shared__ uint32_t s_off[kVec][kWarps];
  __shared__ uint64_t s_prefix[2];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x;
  if (kInPlace) {
    // the pre-check kernel validated the whole mask; never touch base on error
    if (*(volatile uint32_t*)&st->err_flags) return;
  }
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * kTile;
  const bool full = t0 + kTile <= n;
  const uint64_t g0 = t0 / 8;

  uint32_t bits[kVec], cnt[kVec];
  bool pad_err = false;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const uint64_t g = g0 + j * kThreads + tid;
    uint32_t b = 0;
    if (full) {
      b = __ldg(mask + g);
    } else if (g * 8 < n) {
      b = __ldg(mask + g);
      if (g * 8 + 8 > n) {
        const uint32_t valid = (uint32_t)(n - g * 8);
        pad_err |= (b >> valid) != 0;
        b &= (1u << valid) - 1u;
      }
    }
    bits[j] = b;
    cnt[j] = __popc(b);
  }
  if (!kInPlace && pad_err) atomicOr(&st->err_flags, BSNP_ERR_PADDING);

  uint4 bv[kVec];
  if (!kInPlace && kAligned && full) {
#pragma unroll
    for (int j = 0; j < kVec; ++j)
      bv[j] = ld_stream_v4(base + t0 + (uint64_t)(j * kThreads + tid) * 8);
  }

  TileScan sc;
  tile_scan(cnt, tile, tile_status, sc, s_warp, s_off, s_prefix);
  if (!kInPlace && tid == 0 && tile == ntiles - 1) {
    const uint64_t pc = sc.prefix + sc.total;
    st->count = pc;
    if (pc != n_c) atomicOr(&st->err_flags, BSNP_ERR_POPCOUNT);
  }

#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const uint64_t e = t0 + (uint64_t)(j * kThreads + tid) * 8;
    uint32_t b = bits[j];
    uint64_t pos = sc.prefix + sc.off[j];
    if (kInPlace) {
      while (b) {
        const uint32_t k = __ffs(b) - 1;
        b &= b - 1;
        if (pos < n_c) out[e + k] = payload[pos];
        ++pos;
      }
    } else if (kAligned && full) {
      uint4 v = bv[j];
      while (b) {
        const uint32_t k = __ffs(b) - 1;
        b &= b - 1;
        if (pos < n_c) set_u16_lane(v, k, payload[pos]);
        ++pos;
      }
      st_stream_v4(out + e, v);
    } else {
      for (uint32_t k = 0; k < 8; ++k) {
        if (e + k >= n) break;
        uint16_t v = base[e + k];
        if ((b >> k) & 1u) {
          if (pos < n_c) v = payload[pos];
          ++pos;
        }
        out[e + k] = v;
      }
    }
  }
}

}  // namespace
}  // namespace bsnp

using namespace bsnp;

extern "C" size_t bsnp_delta_ws_bytes(uint64_t n) {
  return kWsHeader + 8 * (size_t)num_tiles(n);
}

extern "C" int bsnp_delta_encode(const uint16_t* base, const uint16_t* target, uint64_t n,
                                 uint8_t* mask, uint16_t* payload, uint64_t payload_cap,
                                 bsnp_status* status, void* ws, size_t ws_bytes,
                                 void* stream) {
  if (!status) return BSNP_E_INVALID;
  if (n && (!base || !target || !mask || !ws || (!payload && payload_cap)))
    return BSNP_E_INVALID;
  if (((uintptr_t)base | (uintptr_t)target | (uintptr_t)payload) & 1) return BSNP_E_ALIGN;
  const size_t need = bsnp_delta_ws_bytes(n);
  if (n && ws_bytes < need) return BSNP_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = cuda_status("memset(status)", cudaMemsetAsync(status, 0, sizeof(bsnp_status), s));
  if (rc || n == 0) return rc;
  rc = cuda_status("memset(ws)", cudaMemsetAsync(ws, 0, need, s));
  if (rc) return rc;
  const uint64_t nt = num_tiles(n);
  uint32_t* ticket = (uint32_t*)ws;
  uint64_t* tstat = (uint64_t*)((char*)ws + kWsHeader);
  const bool aligned = (((uintptr_t)base | (uintptr_t)target) & 15) == 0;
  if (aligned)
    delta_encode_kernel<true><<<(unsigned)nt, kThreads, 0, s>>>(
        base, target, n, mask, payload, payload_cap, status, ticket, tstat, nt);
  else
    delta_encode_kernel<false><<<(unsigned)nt, kThreads, 0, s>>>(
        base, target, n, mask, payload, payload_cap, status, ticket, tstat, nt);
  return launch_status("delta_encode_kernel");
}

extern "C" int bsnp_delta_decode(const uint16_t* base, const uint8_t* mask,
                                 const uint16_t* payload, uint64_t n, uint64_t n_c,
                                 uint16_t* out, bsnp_status* status, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (!status) return BSNP_E_INVALID;
  if (n && (!base || !mask || !out || !ws || (!payload && n_c))) return BSNP_E_INVALID;
  if (n_c > n) return BSNP_E_INVALID;
  if (((uintptr_t)base | (uintptr_t)out | (uintptr_t)payload) & 1) return BSNP_E_ALIGN;
  const size_t need = bsnp_delta_ws_bytes(n);
  if (n && ws_bytes < need) return BSNP_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = cuda_status("memset(status)", cudaMemsetAsync(status, 0, sizeof(bsnp_status), s));
  if (rc || n == 0) return rc;
  rc = cuda_status("memset(ws)", cudaMemsetAsync(ws, 0, need, s));
  if (rc) return rc;
  const uint64_t nt = num_tiles(n);
  uint32_t* ticket = (uint32_t*)ws;
  uint64_t* tstat = (uint64_t*)((char*)ws + kWsHeader);
  const bool in_place = (const void*)base == (const void*)out;
  const bool aligned = (((uintptr_t)base | (uintptr_t)out) & 15) == 0;
  if (in_place) {
    const uint64_t nbytes = (n + 7) / 8;
    unsigned grid = (unsigned)((nbytes + 255) / 256);
    const unsigned cap = 148u * 8u;
    if (grid > cap) grid = cap;
    delta_mask_check_kernel<<<grid, 256, 0, s>>>(mask, n, status);
    if ((rc = launch_status("delta_mask_check_kernel"))) return rc;
    delta_check_finish_kernel<<<1, 1, 0, s>>>(status, n_c);
    if ((rc = launch_status("delta_check_finish_kernel"))) return rc;
    delta_decode_kernel<false, true><<<(unsigned)nt, kThreads, 0, s>>>(
        base, mask, payload, n, n_c, out, status, ticket, tstat, nt);
  } else if (aligned) {
    delta_decode_kernel<true, false><<<(unsigned)nt, kThreads, 0, s>>>(
        base, mask, payload, n, n_c, out, status, ticket, tstat, nt);
  } else {
    delta_decode_kernel<false, false><<<(unsigned)nt, kThreads, 0, s>>>(
        base, mask, payload, n, n_c, out, status, ticket, tstat, nt);
  }
  return launch_status("delta_decode_kernel");
}
