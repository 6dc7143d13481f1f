// Shared device helpers for the BitSnap sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/bitsnap_b200.h"

namespace bsnp {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Memory access helpers
// ---------------------------------------------------------------------------

// Streaming 128-bit load: read-only path, no L1 allocation, 256B L2 prefetch.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Streaming 128-bit store (evict-first in L2: outputs are not re-read).
__device__ __forceinline__ void st_stream_v4(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may be scheduled while its
// predecessor in the stream still runs; pdl_enter() makes it wait for that
// predecessor's completion (and memory) before touching anything, then lets
// ITS dependent launch early.  A no-op for an ordinary launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 16-byte read-only load with an explicit L2 eviction policy (the plain
// ld_stream_f4 is evict-first in L2: no reuse across passes)
__device__ __forceinline__ float4 ld_hint_f4(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// global -> shared bulk copy; bytes multiple of 16, both addresses 16B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// ---------------------------------------------------------------------------
// Decoupled look-back over per-tile status words (single-pass prefix scan).
// Word layout: [63:62] flag (0 = not ready, 1 = tile aggregate, 2 = inclusive
// prefix), [61:0] value.  Flag and value live in one 64-bit word, so a
// relaxed single-copy-atomic store publishes both at once.
// Must be called by all 32 lanes of ONE warp; returns the exclusive prefix
// of `tile` (valid on every lane) and publishes tile's inclusive prefix.
// Forward progress: tiles are claimed in increasing order by resident CTAs
// (atomic ticket), so every predecessor is running or done.
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

#ifdef BSNP_LOOKBACK_STATS
__device__ unsigned long long g_lookback_stats[4];  // calls, windows, spins
#endif

// Publish a tile's aggregate (tile 0 publishes its inclusive prefix).
__device__ __forceinline__ void publish_aggregate(uint64_t* status, uint64_t tile,
                                                  uint64_t aggregate) {
  st_relaxed_u64(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | aggregate);
}

__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, uint64_t tile,
                                                       uint64_t aggregate, int lane,
                                                       bool publish_agg = true) {
  if (tile == 0) {
    if (lane == 0 && publish_agg) st_relaxed_u64(status, kFlagInc | aggregate);
    return 0;
  }
  if (lane == 0 && publish_agg) st_relaxed_u64(status + tile, kFlagAgg | aggregate);
  uint64_t excl = 0;
  int64_t top = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = top - lane;
    uint64_t s;
    uint32_t inc, relevant;
    while (true) {
      s = idx >= 0 ? ld_relaxed_u64(status + idx) : kFlagInc;
      const uint32_t flag = (uint32_t)(s >> 62);
      const uint32_t bad = __ballot_sync(kFull, flag == 0);
      inc = __ballot_sync(kFull, flag == 2);
      const int first = inc ? __ffs(inc) - 1 : 31;
      relevant = first == 31 ? kFull : ((2u << first) - 1u);
      if (!(bad & relevant)) break;
#ifdef BSNP_LOOKBACK_STATS
      if (lane == 0) atomicAdd(&g_lookback_stats[2], 1ull);
#endif
      __nanosleep(32);
    }
#ifdef BSNP_LOOKBACK_STATS
    if (lane == 0) atomicAdd(&g_lookback_stats[1], 1ull);
#endif
    const uint64_t v = (relevant >> lane) & 1u ? (s & kValMask) : 0;
    excl += warp_sum_u64(v);
    if (inc) break;
    top -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | (excl + aggregate));
#ifdef BSNP_LOOKBACK_STATS
  if (lane == 0) atomicAdd(&g_lookback_stats[0], 1ull);
#endif
  return excl;
}

// Wide look-back: each round trip inspects kW*32 predecessors (element
// distance d = k*32 + lane + 1 for k = 0..kW-1).  The tile's own aggregate must
// already be published (publish_aggregate).  Returns the exclusive prefix on
// every lane and publishes the inclusive prefix.
#ifndef BSNP_SPIN_NS
#define BSNP_SPIN_NS 512
#endif
template <int kW>
__device__ __forceinline__ uint64_t lookback_wide(uint64_t* status, uint64_t tile,
                                                  uint64_t aggregate, int lane) {
  if (tile == 0) return 0;
  uint64_t excl = 0;
  int64_t top = (int64_t)tile - 1;
  uint32_t backoff = BSNP_SPIN_NS;
  while (true) {
    uint64_t sv[kW];
    uint32_t incm[kW], badm[kW];
    int kf, lf;
    while (true) {
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        const int64_t idx = top - (k * 32 + lane);
        sv[k] = idx >= 0 ? ld_relaxed_u64(status + idx) : kFlagInc;
      }
      kf = kW;
      lf = 31;
#pragma unroll
      for (int k = kW - 1; k >= 0; --k) {
        const uint32_t fl = (uint32_t)(sv[k] >> 62);
        incm[k] = __ballot_sync(kFull, fl == 2);
        badm[k] = __ballot_sync(kFull, fl == 0);
        if (incm[k]) {
          kf = k;
          lf = __ffs(incm[k]) - 1;
        }
      }
      bool bad = false;
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        const uint32_t rel = k < kf ? kFull : (k == kf ? (lf == 31 ? kFull : ((2u << lf) - 1u)) : 0u);
        bad |= (badm[k] & rel) != 0;
      }
#ifdef BSNP_LOOKBACK_STATS
      if (bad && lane == 0) atomicAdd(&g_lookback_stats[2], 1ull);
#endif
      if (!bad) break;
      __nanosleep(backoff);  // exponential back-off keeps spinners off the hot L2 lines
      if (backoff < 4096) backoff *= 2;
    }
#ifdef BSNP_LOOKBACK_STATS
    if (lane == 0) atomicAdd(&g_lookback_stats[1], 1ull);
#endif
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < kW; ++k)
      if (k < kf || (k == kf && lane <= lf)) v += sv[k] & kValMask;
    excl += warp_sum_u64(v);
    if (kf < kW) break;
    top -= 32 * kW;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | (excl + aggregate));
#ifdef BSNP_LOOKBACK_STATS
  if (lane == 0) atomicAdd(&g_lookback_stats[0], 1ull);
#endif
  return excl;
}

// Warp inclusive scan of packed 16-bit counters (4 lanes of a u64).
__device__ __forceinline__ uint64_t warp_inclusive_scan_u64(uint64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_inclusive_scan_u32(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// Halfword k (0..7) of an 8 x u16 vector held in a uint4, k dynamic, no local memory.
__device__ __forceinline__ uint32_t u16_lane(const uint4& v, uint32_t k) {
  const uint32_t lo = (k & 2) ? v.y : v.x;
  const uint32_t hi = (k & 2) ? v.w : v.z;
  const uint32_t w = (k & 4) ? hi : lo;
  return (k & 1) ? (w >> 16) : (w & 0xffffu);
}

__device__ __forceinline__ void set_u16_lane(uint4& v, uint32_t k, uint32_t val) {
  const uint32_t sh = (k & 1) * 16;
  const uint32_t keep = ~(0xffffu << sh), ins = (val & 0xffffu) << sh;
  const uint32_t w = k >> 1;
  if (w == 0) v.x = (v.x & keep) | ins;
  else if (w == 1) v.y = (v.y & keep) | ins;
  else if (w == 2) v.z = (v.z & keep) | ins;
  else v.w = (v.w & keep) | ins;
}

// 8-bit change mask of two 8 x u16 vectors: bit k = halfword k differs.
__device__ __forceinline__ uint32_t diff8(const uint4& a, const uint4& b) {
  const uint32_t d0 = __vcmpne2(a.x, b.x), d1 = __vcmpne2(a.y, b.y);
  const uint32_t d2 = __vcmpne2(a.z, b.z), d3 = __vcmpne2(a.w, b.w);
  // each dK holds 0xffff per differing halfword; gather one bit per halfword
  const uint32_t p01 = __byte_perm(d0, d1, 0x6420);  // bytes: d0.lo d0.hi d1.lo d1.hi
  const uint32_t p23 = __byte_perm(d2, d3, 0x6420);
  const uint32_t lo = ((p01 & 0x01010101u) * 0x01020408u) >> 24;
  const uint32_t hi = ((p23 & 0x01010101u) * 0x01020408u) >> 24;
  return (lo & 0xfu) | ((hi & 0xfu) << 4);
}

}  // namespace bsnp
