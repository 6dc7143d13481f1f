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
#include <cstdlib>

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

// ===========================================================================
// TMA-pipelined persistent kernels (16B-aligned operands, full tiles).
// Thread 0 claims tile tickets and issues cp.async.bulk copies of the
// operands into shared-memory stages that complete on mbarriers, so loads of
// later tiles are in flight while earlier tiles are scanned and written.
// ===========================================================================
constexpr uint32_t kTileBytes = kTile * 2;                    // 16 KiB per u16 operand
constexpr uint32_t kMaskBytes = kTile / 8;                    // 1 KiB
constexpr uint32_t kEncStage = 2 * kTileBytes;                // base + cur
constexpr uint32_t kDecPayloadCap = kTileBytes + 32;          // aligned superset of a slice
constexpr uint32_t kDecStage = kTileBytes + kMaskBytes + kDecPayloadCap + 96;  // 128B multiple
static_assert(kDecStage % 128 == 0, "stage alignment");

// Packed-count scan of one tile inside the CTA (no look-back): returns this
// thread's offsets of its kVec groups relative to the tile start, and the
// tile total.  Two barriers.
__device__ __forceinline__ uint32_t tile_local_scan(const uint32_t (&cnt)[kVec],
                                                    uint32_t (&off)[kVec], uint64_t* s_warp,
                                                    uint32_t (*s_off)[kWarps]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t packed = 0;
#pragma unroll
  for (int j = 0; j < kVec; ++j) packed |= (uint64_t)cnt[j] << (16 * j);
  const uint64_t inc = warp_inclusive_scan_u64(packed, lane);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t total = 0;
  if (warp == 0) {
    const int j = lane / kWarps, w = lane % kWarps;
    const uint32_t v = (uint32_t)(s_warp[w] >> (16 * j)) & 0xffffu;
    const uint32_t x = warp_inclusive_scan_u32(v, lane);
    s_off[j][w] = x - v;
    total = __shfl_sync(kFull, x, 31);
  }
  __syncthreads();
  const uint64_t ex = inc - packed;
#pragma unroll
  for (int j = 0; j < kVec; ++j)
    off[j] = s_off[j][warp] + ((uint32_t)(ex >> (16 * j)) & 0xffffu);
  return total;
}

// Warp-specialized single-pass encode.  Roles per CTA:
//   workers (warps 0..7): per tile (claimed by ticket, operands streamed into
//       a shared-memory stage by cp.async.bulk), read the stage into registers
//       and release it at once (refill = bulk copies of the next claimed
//       tile), scan the change bits inside the CTA, publish the tile aggregate
//       for the decoupled look-back, write the mask bytes and compact the
//       tile's changed values into the shared-memory arena (or, when the
//       arena has no room for them right now, into the tile's global scratch
//       slot).  Workers never wait for a look-back.
//   look-back warps (8 .. 8 + kLB - 1): record q of the CTA (ring of kRing)
//       is served by warp 8 + q % kLB: decoupled look-back for the tile's
//       exclusive prefix, then - once staged - the compacted values go to
//       payload[prefix...] with 16-byte stores (funnel-shifted granules);
//       arena bytes are released in record order, a global slot's L2 lines
//       are discarded so that staging never reaches DRAM.  Two look-back
//       warps keep dense tiles' prefixes coming (the look-back is the serial
//       part: p = 25 %: 1.46 ms with one, 1.08 ms with two).
// mbarriers: full[s] (TMA bytes), rec_full[r]/rec_empty[r] (workers <->
// look-back warps), staged[r] (8 worker warps -> look-back warp).
#ifndef BSNP_LB_WIDTH
#define BSNP_LB_WIDTH 2  // look-back predecessors per lane per round trip
#endif
#ifndef BSNP_KLB
#define BSNP_KLB 2
#endif
constexpr int kLB = BSNP_KLB;  // look-back warps per CTA
constexpr int kRing = 16;
static_assert(kRing % kLB == 0, "ring slots map to look-back warps");
constexpr int kEncThreads = kThreads + 32 * kLB;
#ifndef BSNP_ENC_STAGES
#define BSNP_ENC_STAGES 2
#endif
constexpr int kEncStagesWS = BSNP_ENC_STAGES;  // TMA stages (base + cur tiles)
// compacted payloads of the tiles in flight wait for their prefix in a
// shared-memory arena (a byte ring, 16-byte granules) sized so three CTAs
// still fit an SM; a tile too dense for it (> ~56 % changed) is staged in its
// global scratch slot instead
#ifndef BSNP_ARENA
#define BSNP_ARENA 8192
#endif
constexpr uint32_t kArena = BSNP_ARENA;
static_assert(kArena % 16 == 0, "arena granules");
constexpr uint32_t kDenseTile = 0xffffffffu;  // record base: staged in global scratch
#ifndef BSNP_DENSE_COMPACT
#define BSNP_DENSE_COMPACT 1024  // p = 25 %: 1.038 -> 1.000 ms; 6.25 % tiles stay below
#endif
constexpr uint32_t kDenseCompact = BSNP_DENSE_COMPACT;  // tile changes -> unrolled compaction

__device__ __forceinline__ void mbar_arrive_release(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

__global__ void __launch_bounds__(kEncThreads)
    delta_encode_ws_kernel(const uint16_t* __restrict__ base, const uint16_t* __restrict__ cur,
                           uint64_t n, uint8_t* __restrict__ mask,
                           uint16_t* __restrict__ payload, uint64_t payload_cap,
                           uint16_t* __restrict__ scratch, bsnp_status* __restrict__ st,
                           uint32_t* __restrict__ ticket, uint64_t* __restrict__ tile_status,
                           uint64_t ntiles, uint32_t ring_slots) {
  pdl_enter();
  constexpr int kStages = kEncStagesWS;
  // global staging slot of record q / tile t: per tile (ring_slots == 0), or
  // a per-CTA ring of kRing slots (the workspace then does not grow with n)
  auto slot_of = [&](uint32_t q, uint64_t t) {
    return scratch + (ring_slots ? ((uint64_t)blockIdx.x * kRing + q % kRing) : t) * kTile;
  };
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full_bar[kStages];
  __shared__ uint64_t rec_full[kRing], rec_empty[kRing], staged[kRing];
  __shared__ uint32_t s_tile[kStages];
  __shared__ uint32_t r_tile[kRing], r_count[kRing], r_base[kRing];
  __shared__ uint64_t s_warp[2][kWarps];
  __shared__ volatile uint32_t s_tail;  // arena bytes released by the look-back warps
  __shared__ volatile uint32_t s_relq;  // next record whose arena bytes get released
  __shared__ uint32_t s_snap[2];        // s_tail as seen before a tile's scan barrier
  uint8_t* arena = smem + (size_t)kEncStagesWS * kEncStage;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t nfull = n / kTile;
  uint64_t pol = 0;
  auto refill = [&](int s, uint32_t t) {  // worker thread 0 only
    s_tile[s] = t;
    if (t < nfull) {
      uint8_t* dst = smem + (size_t)s * kEncStage;
      mbar_arrive_expect_tx(&full_bar[s], kEncStage);
      bulk_g2s(dst, base + (uint64_t)t * kTile, kTileBytes, &full_bar[s], pol);
      bulk_g2s(dst + kTileBytes, cur + (uint64_t)t * kTile, kTileBytes, &full_bar[s], pol);
    }
  };
  // ring producer (worker thread 0): record q -> slot q % kRing
  auto push_record = [&](uint32_t q, uint32_t tile, uint32_t count, uint32_t abase) {
    const int r = q % kRing;
    if (q >= kRing) mbar_wait(&rec_empty[r], ((q / kRing) - 1) & 1u);
    r_tile[r] = tile;
    r_count[r] = count;
    r_base[r] = abase;
    mbar_arrive_release(&rec_full[r]);
  };
  if (tid == 0) {
    s_tail = 0;
    s_relq = 0;
    pol = policy_evict_first();
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&rec_full[r], 1);
      mbar_init(&rec_empty[r], 1);
      mbar_init(&staged[r], kWarps);
    }
    fence_mbar_init();
    for (int s = 0; s < kStages; ++s) refill(s, atomicAdd(ticket, 1u));
  }
  __syncthreads();

  if (warp >= kWarps) {
    // --------------------------------------------------------- look-back warps
    const int w = warp - kWarps;
    for (uint32_t q = w;; q += kLB) {
      const int r = q % kRing;
      const uint32_t parity = (q / kRing) & 1u;
      mbar_wait(&rec_full[r], parity);
      const uint32_t tile = r_tile[r];
      const uint32_t c = r_count[r];
      if (tile >= ntiles) break;
      const uint64_t excl = lookback_wide<BSNP_LB_WIDTH>(tile_status, tile, c, lane);
      if (lane == 0 && tile == ntiles - 1) st->count = excl + c;
      mbar_wait(&staged[r], parity);  // workers wrote the arena / scratch slot
      const uint32_t abase = r_base[r];
      const uint16_t* src = slot_of(q, tile);
      const bool overflow = excl + c > payload_cap;
      const bool in_arena = abase != kDenseTile;
      const uint32_t b0 = in_arena ? abase % kArena : 0;
      // record source: byte ring of the arena, or the tile's global slot
      auto granule = [&](uint32_t o) {  // 16 bytes at source byte o (16-aligned)
        if (in_arena) return *reinterpret_cast<const uint4*>(arena + o);
        return __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(src) + o));
      };
      auto elem = [&](uint32_t i) -> uint16_t {
        if (in_arena) return reinterpret_cast<const uint16_t*>(arena)[(b0 >> 1) + i];
        return src[i];
      };
      if (!overflow) {
        // a head of single elements up to 16-byte alignment of the
        // destination, whole 16-byte vectors (two source granules
        // funnel-shifted), a tail of single elements
        uint16_t* dst = payload + excl;
        uint32_t h = (uint32_t)(((16 - ((uintptr_t)dst & 15)) & 15) >> 1);
        h = h < c ? h : c;
        if ((uint32_t)lane < h) dst[lane] = elem(lane);
        const uint32_t nv = (c - h) / 8;
        for (uint32_t v = lane; v < nv; v += 32) {
          const uint32_t o = b0 + 2 * h + 16 * v;  // first source byte
          const uint32_t g = o & ~15u;
          const uint4 lo = granule(g), hi = granule(g + 16);
          const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
          // output word k = source bytes (o & 15) + 4k .. + 3: shift the 8
          // words down by (o & 15) / 4 words in two select steps, then
          // funnel-shift by the remaining 0 or 2 bytes
          const uint32_t ws = (o & 15) >> 2, bs = (o & 3) * 8;
          uint32_t v2[6], v1[5], out[4];
#pragma unroll
          for (int i = 0; i < 6; ++i) v2[i] = (ws & 2) ? w[i + 2] : w[i];
#pragma unroll
          for (int i = 0; i < 5; ++i) v1[i] = (ws & 1) ? v2[i + 1] : v2[i];
#pragma unroll
          for (int k = 0; k < 4; ++k) out[k] = __funnelshift_r(v1[k], v1[k + 1], bs);
          *reinterpret_cast<uint4*>(dst + h + 8 * v) = make_uint4(out[0], out[1], out[2], out[3]);
        }
        const uint32_t t0e = h + 8 * nv;
        if ((uint32_t)lane < c - t0e) dst[t0e + lane] = elem(t0e + lane);
      } else {
        for (uint32_t i = lane; i < c; i += 32)
          if (excl + i < payload_cap) payload[excl + i] = elem(i);
        if (lane == 0) atomicOr(&st->err_flags, BSNP_ERR_PAYLOAD_CAP);
      }
      if (!in_arena) {
        __syncwarp();
        for (uint32_t i = lane * 64; i < c; i += 32 * 64) discard_l2_line(src + i);
      }
      __syncwarp();
      if (lane == 0) {
        // arena bytes are released in record order (the records of the look-
        // back warps interleave): wait for the predecessor's release
        while (s_relq != q) __nanosleep(32);
        if (in_arena) s_tail = abase + ((2 * c + 15) & ~15u);
        __threadfence_block();
        s_relq = q + 1;
        mbar_arrive_release(&rec_empty[r]);
      }
      __syncwarp();
    }
    return;
  }

  // ------------------------------------------------------------------ workers
  uint32_t arena_head = 0;  // arena bytes reserved so far (same in every warp)
  for (uint32_t q = 0;; ++q) {
    const int s = q % kStages;
    const uint32_t parity = (q / kStages) & 1u;
    const uint32_t tile = s_tile[s];
    if (tile >= ntiles) {
      // end of work: poison one record per look-back warp so each exits
      if (tid == 0)
        for (int k = 0; k < kLB; ++k) push_record(q + k, 0xffffffffu, 0, 0);
      break;
    }
    const uint64_t t0 = (uint64_t)tile * kTile;
    // claim the stage's next tile now; the atomic's latency overlaps the wait
    uint32_t next_t = 0;
    if (tid == 0) next_t = atomicAdd(ticket, 1u);
    uint4 cv[kVec];
    uint32_t bits[kVec], cnt[kVec];
    if (tile < nfull) {
      mbar_wait(&full_bar[s], parity);
      const uint4* sb = reinterpret_cast<const uint4*>(smem + (size_t)s * kEncStage);
      const uint4* sc = reinterpret_cast<const uint4*>(smem + (size_t)s * kEncStage + kTileBytes);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const uint4 b = sb[j * kThreads + tid];
        cv[j] = sc[j * kThreads + tid];
        bits[j] = diff8(b, cv[j]);
      }
    } else {  // the partial last tile: bounded global loads
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
    uint64_t packed = 0;
#pragma unroll
    for (int j = 0; j < kVec; ++j) packed |= (uint64_t)cnt[j] << (16 * j);
    const uint64_t inc = warp_inclusive_scan_u64(packed, lane);
    const int db = q & 1;  // double-buffered scan scratch: 2 barriers per tile
    if (lane == 31) s_warp[db][warp] = inc;
    if (tid == 0) s_snap[db] = s_tail;  // one view of the arena for every warp
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    // every worker holds its part of the tile in registers: release the stage
    if (tid == 0) refill(s, next_t);
    // every warp scans the 8 warp totals itself (lane = group j * 8 + warp w,
    // the tile's element order), so no second barrier waits on warp 0's
    // publish / record hand-off
    uint32_t woff[kVec], total;
    {
      const int j = lane / kWarps, w = lane % kWarps;
      const uint32_t v = (uint32_t)(s_warp[db][w] >> (16 * j)) & 0xffffu;
      const uint32_t x = warp_inclusive_scan_u32(v, lane);
#pragma unroll
      for (int jj = 0; jj < kVec; ++jj) woff[jj] = __shfl_sync(kFull, x - v, jj * kWarps + warp);
      total = __shfl_sync(kFull, x, 31);
    }
    // arena space of this tile: every warp runs the same reservation sequence
    // against the same snapshot of the released bytes, so all decide alike;
    // a tile that does not fit NOW goes to its global slot (never wait: a
    // blocked CTA would hold back the aggregates other CTAs look back on)
    const uint32_t abytes = (2 * total + 15) & ~15u;
    // records never straddle the ring's end (the remainder is skipped), so
    // neither the compaction nor the look-back warp's copy wraps per element
    uint32_t start = arena_head;
    if (start % kArena + abytes > kArena) start += kArena - start % kArena;
    const bool in_arena = start + abytes - s_snap[db] <= kArena;
    const uint32_t abase = in_arena ? start : kDenseTile;
    if (warp == 0 && lane == 0) {
      publish_aggregate(tile_status, tile, total);
      push_record(q, tile, total, abase);
    }
    const uint64_t ex = inc - packed;
    const uint64_t g0 = t0 / 8;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const uint64_t g = g0 + j * kThreads + tid;
      if (g * 8 < n) mask[g] = (uint8_t)bits[j];
    }
    if (in_arena) {
      arena_head = start + abytes;
      uint16_t* a16 = reinterpret_cast<uint16_t*>(arena);
      const uint32_t b0 = abase % kArena;
      if (total >= kDenseCompact) {
        // dense tile: every element slot unrolled and predicated (no
        // divergent per-lane loop that waits on the lane with most changes)
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          const uint32_t b = bits[j];
          const uint32_t o0 = b0 + 2 * (woff[j] + ((uint32_t)(ex >> (16 * j)) & 0xffffu));
          const uint32_t w4[4] = {cv[j].x, cv[j].y, cv[j].z, cv[j].w};
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if ((b >> k) & 1u) {
              const uint32_t o = o0 + 2 * __popc(b & ((1u << k) - 1u));
              a16[o >> 1] = (uint16_t)(w4[k >> 1] >> (16 * (k & 1)));
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          uint32_t b = bits[j];
          uint32_t o = b0 + 2 * (woff[j] + ((uint32_t)(ex >> (16 * j)) & 0xffffu));
          while (b) {
            const uint32_t k = __ffs(b) - 1;
            b &= b - 1;
            a16[o >> 1] = (uint16_t)u16_lane(cv[j], k);
            o += 2;
          }
        }
      }
    } else {
      // a ring slot is free once the look-back warp moved record q - kRing
      // out of it (per-tile slots are never reused)
      if (ring_slots && q >= kRing) mbar_wait(&rec_empty[q % kRing], ((q / kRing) - 1) & 1u);
      uint16_t* slot = slot_of(q, tile);
      // (an unrolled predicated variant of these 2-byte global stores was
      // slower at p = 25 %: 1.074 vs 1.000 ms)
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        uint32_t b = bits[j];
        uint32_t pos = woff[j] + ((uint32_t)(ex >> (16 * j)) & 0xffffu);
        while (b) {
          const uint32_t k = __ffs(b) - 1;
          b &= b - 1;
          slot[pos++] = (uint16_t)u16_lane(cv[j], k);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_release(&staged[q % kRing]);
  }
}

// Payload offsets of every decode tile from the mask alone (n/8 bytes), and
// the validation of padding bits and popcount == n_c (bitmask.py:128-135),
// in two look-back-free launches:
//   delta_count_kernel  one CTA per chunk of kChunkTiles tiles (all loads of
//                       a warp's tiles in flight at once): per-tile offsets
//                       inside the chunk (u32) and the chunk's total;
//   delta_scan_kernel   one CTA: the exclusive scan of the chunk totals (u64
//                       chunk bases, the total last), status->count and the
//                       popcount check.
// A tile's payload offset is then base[chunk] + local[tile] (TileOffsets;
// delta_materialize_kernel writes them out as u64 for the TMA decode).
// (A single pass chained by a decoupled look-back over 128-tile chunks took
// 38 us at 2^30: its 1024 CTAs needed two waves at 58 registers.)
constexpr int kChunkTiles = 32;  // 4 tiles per warp, one batch of loads
constexpr int kChunkShift = 5;
static_assert((1 << kChunkShift) == kChunkTiles, "chunk shift");
constexpr int kScanThreads = 1024;

struct TileOffsets {
  const uint64_t* base;   // [nchunks + 1]: exclusive chunk bases, then the total
  const uint32_t* local;  // [ntiles + 1]: offset of each tile inside its chunk
  uint64_t ntiles;
  // t <= ntiles (local[ntiles] makes at(ntiles) the total: branch-free)
  __device__ __forceinline__ uint64_t at(uint64_t t) const {
    return base[t >> kChunkShift] + local[t];
  }
};

__device__ __forceinline__ uint32_t tile_lane_count(const uint8_t* __restrict__ mask, uint64_t n,
                                                    uint64_t nbytes, uint64_t b0, bool& pad) {
  uint32_t c = 0;
  for (uint64_t i = b0; i < b0 + 32 && i < nbytes; ++i) {
    uint32_t v = mask[i];
    if (i == nbytes - 1 && (n & 7)) {
      const uint32_t valid = (uint32_t)(n & 7);
      pad |= (v >> valid) != 0;
      v &= (1u << valid) - 1u;
    }
    c += __popc(v);
  }
  return c;
}

__global__ void __launch_bounds__(kThreads)
    delta_count_kernel(const uint8_t* __restrict__ mask, uint64_t n,
                       uint32_t* __restrict__ local, uint32_t* __restrict__ ctot,
                       bsnp_status* __restrict__ st) {
  pdl_enter();
  constexpr int kPerWarp = kChunkTiles / kWarps;
  __shared__ uint32_t s_cnt[kChunkTiles];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t chunk = blockIdx.x;
  const uint64_t nbytes = (n + 7) / 8;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const bool vec = ((uintptr_t)mask & 15) == 0;
  bool pad = false;
  uint4 a[kPerWarp], b[kPerWarp];
  uint32_t full = 0;  // bit q: tile q is loaded whole
#pragma unroll
  for (int q = 0; q < kPerWarp; ++q) {
    const uint64_t t = chunk * kChunkTiles + warp * kPerWarp + q;
    const uint64_t b0 = t * kMaskBytes + (uint64_t)lane * 32;
    if (t < ntiles && vec && b0 + 32 < nbytes) {  // the last byte goes the slow way
      full |= 1u << q;
      a[q] = ld_stream_v4(mask + b0);
      b[q] = ld_stream_v4(mask + b0 + 16);
    } else {
      a[q] = b[q] = make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int q = 0; q < kPerWarp; ++q) {
    const int lt = warp * kPerWarp + q;
    const uint64_t t = chunk * kChunkTiles + lt;
    uint32_t c = 0;
    if ((full >> q) & 1u) {
      c = __popc(a[q].x) + __popc(a[q].y) + __popc(a[q].z) + __popc(a[q].w) +
          __popc(b[q].x) + __popc(b[q].y) + __popc(b[q].z) + __popc(b[q].w);
    } else if (t < ntiles) {
      c = tile_lane_count(mask, n, nbytes, t * kMaskBytes + (uint64_t)lane * 32, pad);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
    if (lane == 0) s_cnt[lt] = c;
  }
  if (pad) atomicOr(&st->err_flags, BSNP_ERR_PADDING);
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = s_cnt[lane];
    const uint32_t x = warp_inclusive_scan_u32(v, lane);
    const uint64_t t = chunk * kChunkTiles + lane;
    if (t <= ntiles) local[t] = x - v;  // [ntiles]: the chunk total (at(ntiles) = total)
    if (lane == 31) ctot[chunk] = x;
  }
}

// off[t] = base[chunk] + local[t] for t <= ntiles (the TMA decode's table)
__global__ void __launch_bounds__(kThreads)
    delta_materialize_kernel(const uint64_t* __restrict__ base, const uint32_t* __restrict__ local,
                             uint64_t ntiles, uint64_t* __restrict__ off) {
  pdl_enter();
  const uint64_t t = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (t <= ntiles) off[t] = base[t >> kChunkShift] + local[t];
}

__global__ void __launch_bounds__(kScanThreads)
    delta_scan_kernel(const uint32_t* __restrict__ ctot, uint64_t nchunks,
                      uint64_t* __restrict__ base, uint32_t* __restrict__ local, uint64_t ntiles,
                      bsnp_status* __restrict__ st, uint64_t n_c,
                      const uint64_t* __restrict__ nc_dev) {
  pdl_enter();
  __shared__ uint64_t s_warp[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t per = (nchunks + kScanThreads - 1) / kScanThreads;
  const uint64_t lo = (uint64_t)tid * per, hi = lo + per < nchunks ? lo + per : nchunks;
  uint64_t sum = 0;
  for (uint64_t i = lo; i < hi; ++i) sum += __ldg(ctot + i);
  uint64_t x = sum;  // inclusive scan over the CTA
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += o;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = s_warp[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t o = __shfl_up_sync(kFull, w, d);
      if (lane >= d) w += o;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  uint64_t run = x - sum + (warp ? s_warp[warp - 1] : 0);
  for (uint64_t i = lo; i < hi; ++i) {
    base[i] = run;
    run += __ldg(ctot + i);
  }
  if (tid == kScanThreads - 1) {
    const uint64_t total = s_warp[31];
    base[nchunks] = total;
    if ((ntiles & (kChunkTiles - 1)) == 0) local[ntiles] = 0;  // at(ntiles) = base[nchunks]
    st->count = total;
    if (total != (nc_dev ? *nc_dev : n_c)) atomicOr(&st->err_flags, BSNP_ERR_POPCOUNT);
  }
}

template <int kStages, bool kDense>
__global__ void __launch_bounds__(kThreads)
    delta_decode_tma_kernel(const uint16_t* base, const uint8_t* __restrict__ mask,
                            const uint16_t* __restrict__ payload, uint64_t n, uint64_t n_c_arg,
                            uint16_t* out, const uint64_t* __restrict__ offsets,
                            uint32_t* __restrict__ ticket,
                            const bsnp_status* __restrict__ st,
                            const uint64_t* __restrict__ nc_dev = nullptr) {
  pdl_enter();
  // in place (out == base, dense chain replay): every tile is read by TMA
  // into shared memory before its words are written, tiles are disjoint, and
  // a record the validation pass rejected leaves the base untouched
  if (st && *(volatile const uint32_t*)&st->err_flags) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full_bar[kStages];
  __shared__ uint32_t s_tile[kStages];
  __shared__ uint32_t s_shift[kStages];   // payload element shift in smem, or ~0u: global
  __shared__ uint64_t s_poff[kStages];
  __shared__ uint64_t s_warp[kWarps];
  __shared__ uint32_t s_off[kVec][kWarps];

  const int tid = threadIdx.x;
  // n_c from the device (the encode's status word: no host round trip) or
  // by value
  const uint64_t n_c = nc_dev ? min(*nc_dev, n) : n_c_arg;  // a device count is not trusted
  const uint64_t nfull = n / kTile;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uintptr_t p_lo = ((uintptr_t)payload + 15) & ~(uintptr_t)15;
  const uintptr_t p_hi = ((uintptr_t)(payload + n_c)) & ~(uintptr_t)15;
  uint64_t pol = 0;
  auto refill = [&](int s, uint32_t t, uint64_t off, uint64_t off_end) {  // thread 0 only
    s_tile[s] = t;
    if (t >= ntiles) return;
    const uint64_t cnt = off_end - off;
    s_poff[s] = off;
    if (t >= nfull) {
      s_shift[s] = ~0u;
      return;
    }
    uint8_t* dst = smem + (size_t)s * kDecStage;
    const uintptr_t a = (uintptr_t)(payload + off), b = (uintptr_t)(payload + off + cnt);
    const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (b + 15) & ~(uintptr_t)15;
    const bool bulk_p = cnt > 0 && a0 >= p_lo && a1 <= p_hi;
    s_shift[s] = bulk_p ? (uint32_t)((a - a0) / 2) : ~0u;
    mbar_arrive_expect_tx(&full_bar[s], kTileBytes + kMaskBytes + (bulk_p ? (uint32_t)(a1 - a0) : 0));
    bulk_g2s(dst, base + t * kTile, kTileBytes, &full_bar[s], pol);
    bulk_g2s(dst + kTileBytes, mask + t * kMaskBytes, kMaskBytes, &full_bar[s], pol);
    if (bulk_p)
      bulk_g2s(dst + kTileBytes + kMaskBytes, (const void*)a0, (uint32_t)(a1 - a0), &full_bar[s],
               pol);
  };
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < kStages; ++s) {
      const uint32_t t = atomicAdd(ticket, 1u);
      refill(s, t, t < ntiles ? offsets[t] : 0, t < ntiles ? offsets[t + 1] : 0);
    }
  }
  __syncthreads();

  for (uint32_t it = 0;; ++it) {
    const int s = it % kStages;
    const uint32_t parity = (it / kStages) & 1u;
    const uint64_t tile = s_tile[s];
    if (tile >= ntiles) break;
    // claim the refill tile and fetch its payload offsets off the critical path
    uint32_t next_t = 0;
    uint64_t next_a = 0, next_b = 0;
    if (tid == 0) {
      next_t = atomicAdd(ticket, 1u);
      if (next_t < ntiles) {
        next_a = offsets[next_t];
        next_b = offsets[next_t + 1];
      }
    }
    const uint64_t t0 = tile * kTile;
    const uint64_t poff = s_poff[s];
    const uint32_t shift = s_shift[s];
    const bool full = tile < nfull;
    const uint8_t* stage = smem + (size_t)s * kDecStage;
    uint4 bv[kVec];
    uint32_t bits[kVec], cnt[kVec], off[kVec];
    if (full) {
      mbar_wait(&full_bar[s], parity);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        bv[j] = reinterpret_cast<const uint4*>(stage)[j * kThreads + tid];
        bits[j] = stage[kTileBytes + j * kThreads + tid];
      }
    } else {
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const uint64_t g = t0 / 8 + j * kThreads + tid;
        const uint64_t e = g * 8;
        uint4 b = make_uint4(0, 0, 0, 0);
        uint32_t m = 0;
        if (e < n) {
          m = mask[g];
          const uint32_t valid = (uint32_t)(n - e < 8 ? n - e : 8);
          m &= (valid == 8) ? 0xffu : ((1u << valid) - 1u);
          for (uint32_t k = 0; k < valid; ++k) set_u16_lane(b, k, base[e + k]);
        }
        bv[j] = b;
        bits[j] = m;
      }
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) cnt[j] = __popc(bits[j]);
    tile_local_scan(cnt, off, s_warp, s_off);
    const uint16_t* sp = reinterpret_cast<const uint16_t*>(stage + kTileBytes + kMaskBytes);

#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      uint32_t b = bits[j];
      uint32_t r = off[j];
      uint4 v = bv[j];
      auto fetch = [&](uint32_t rr) -> uint32_t {
        const uint64_t pos = poff + rr;
        if (shift != ~0u) return sp[shift + rr];
        return pos < n_c ? payload[pos] : 0u;
      };
      if (kDense) {
        // dense records (n_c > n/32, chosen on the host): expand with static
        // lane indices instead of walking the set bits
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if ((b >> k) & 1u) {
            set_u16_lane(v, (uint32_t)k, fetch(r));
            ++r;
          }
        }
      } else {
        while (b) {
          const uint32_t k = __ffs(b) - 1;
          b &= b - 1;
          set_u16_lane(v, k, fetch(r));
          ++r;
        }
      }
      const uint64_t e = t0 + (uint64_t)(j * kThreads + tid) * 8;
      if (full) {
        st_stream_v4(out + e, v);
      } else {
        for (uint32_t k = 0; k < 8 && e + k < n; ++k) out[e + k] = (uint16_t)u16_lane(v, k);
      }
    }
    __syncthreads();  // every thread is done with stage s
    if (tid == 0) refill(s, next_t, next_a, next_b);
  }
}

// Apply with precomputed offsets, one CTA per tile (in-place chain replay and
// the path for operands that are not 16-byte aligned).  In place it touches
// only changed elements and never runs when validation raised a flag.
template <bool kInPlace>
__global__ void __launch_bounds__(kThreads)
    delta_apply_kernel(const uint16_t* base, const uint8_t* __restrict__ mask,
                       const uint16_t* __restrict__ payload, uint64_t n, uint64_t n_c,
                       uint16_t* out, const TileOffsets offsets,
                       const bsnp_status* __restrict__ st) {
  pdl_enter();
  __shared__ uint64_t s_warp[kWarps];
  __shared__ uint32_t s_off[kVec][kWarps];
  if (kInPlace && *(volatile const uint32_t*)&st->err_flags) return;
  const uint64_t tile = blockIdx.x;
  const uint64_t t0 = tile * kTile;
  uint32_t bits[kVec], cnt[kVec], off[kVec];
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const uint64_t g = t0 / 8 + j * kThreads + threadIdx.x;
    uint32_t m = 0;
    if (g * 8 < n) {
      m = __ldg(mask + g);
      if (g * 8 + 8 > n) m &= (1u << (uint32_t)(n - g * 8)) - 1u;
    }
    bits[j] = m;
    cnt[j] = __popc(m);
  }
  tile_local_scan(cnt, off, s_warp, s_off);
  const uint64_t poff = offsets.at(tile);
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const uint32_t b = bits[j];
    uint64_t pos = poff + off[j];
    const uint64_t e = t0 + (uint64_t)(j * kThreads + threadIdx.x) * 8;
    for (uint32_t k = 0; k < 8 && e + k < n; ++k) {
      if ((b >> k) & 1u) {
        if (pos < n_c) out[e + k] = payload[pos];
        ++pos;
      } else if (!kInPlace) {
        out[e + k] = base[e + k];
      }
    }
  }
}

// In-place apply for sparse records (chain replay at small change
// fractions): one WARP per tile, no CTA barriers.  Lane l owns the 256
// elements of mask bytes [32 l, 32 l + 32) of the tile (two 16-byte loads);
// a warp scan of the lane popcounts plus offsets[tile] gives every lane its
// payload position.  The tile's payload run is contiguous, so the warp
// stages it in shared memory with coalesced 4-byte loads (one round trip
// instead of a dependent 2-byte load per changed element), then each lane
// scatters its values; mask, offsets and short payload runs are fetched two
// / one tiles ahead (see the loop).  Runs after delta_count / delta_scan validated the
// mask (never when a flag is raised: a corrupt record leaves the base
// untouched).
constexpr uint32_t kApplyStage = 1024;  // staged payload elements per warp
#ifndef BSNP_DENSE_DIV
#define BSNP_DENSE_DIV 16  // in place: n_c > n / DIV streams whole tiles (TMA decode); 6.25 %: 0.667 sparse vs 0.697 ms dense
#endif
#ifndef BSNP_APPLY_CTAS_PER_SM
#define BSNP_APPLY_CTAS_PER_SM 32  // more, shorter CTAs balance better (p = 6.25 %: 0.652 -> 0.600 ms)
#endif
#ifndef BSNP_COOP_SCATTER
#define BSNP_COOP_SCATTER 1
#endif

__global__ void __launch_bounds__(kThreads)
    delta_apply_warp_kernel(const uint8_t* __restrict__ mask,
                            const uint16_t* __restrict__ payload, uint64_t n, uint64_t n_c,
                            uint16_t* out, const TileOffsets offsets,
                            const bsnp_status* __restrict__ st) {
  pdl_enter();
  __shared__ __align__(16) uint16_t stage[kWarps][kApplyStage + 8];
  if (*(volatile const uint32_t*)&st->err_flags) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t nbytes = (n + 7) / 8;
  const bool mvec = ((uintptr_t)mask & 15) == 0;
  uint16_t* sp = stage[warp];
  const uint64_t nfull = n / kTile;  // tiles whose every element is < n
  auto load_mask = [&](uint64_t tile, uint32_t (&w)[8]) {
    const uint64_t b0 = tile * kMaskBytes + 32 * (uint64_t)lane;
    if (mvec && tile < nfull) {  // the common case: no bits past n to clear
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(mask + b0));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(mask + b0 + 16));
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
      return;
    }
    if (mvec && b0 + 32 <= nbytes) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(mask + b0));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(mask + b0 + 16));
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t v = 0;
        for (uint32_t i = 0; i < 4; ++i) {
          const uint64_t bi = b0 + 4 * k + i;
          if (bi < nbytes) v |= (uint32_t)__ldg(mask + bi) << (8 * i);
        }
        w[k] = v;
      }
    }
    // bits past n (validated zero) are ignored
    const uint64_t e0 = b0 * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t ek = e0 + 32 * k;
      if (ek + 32 > n) w[k] &= ek >= n ? 0u : (0xffffffffu >> (32 - (uint32_t)(n - ek)));
    }
  };
  uint64_t tile = (uint64_t)blockIdx.x * kWarps + warp;
  const uint64_t step = (uint64_t)gridDim.x * kWarps;
  const bool pal = ((uintptr_t)payload & 3) == 0;
  // payload word i (u16 pair from the even element below the run start)
  auto pword = [&](uint64_t a0, uint32_t i) -> uint32_t {
    const uint64_t e = a0 + 2 * (uint64_t)i;
    if (pal && e + 1 < n_c) return __ldg(reinterpret_cast<const uint32_t*>(payload + e));
    return (uint32_t)__ldg(payload + e) | (e + 1 < n_c ? (uint32_t)__ldg(payload + e + 1) << 16 : 0u);
  };
  // a depth-2 software pipeline per warp: while tile t is applied, the mask
  // and offsets of tile t + 2 step and the (short-run) payload words of tile
  // t + step are in flight, so neither the mask load nor the offsets ->
  // payload dependency is on a tile's critical path
  constexpr uint32_t kPre = 2;  // prefetched payload words per lane (runs <= 64 words)
  struct Slot {
    uint32_t w[8];
    uint64_t off, end;
  };
  auto load_slot = [&](uint64_t t, Slot& x) {
    if (t < ntiles) {
      load_mask(t, x.w);
      x.off = offsets.at(t);
      x.end = offsets.at(t + 1);
    } else {
      x.off = x.end = 0;
    }
  };
  auto load_pre = [&](const Slot& x, uint64_t t, uint32_t (&pw)[kPre]) {
    const uint64_t a0 = x.off & ~1ull;
    const uint32_t nw = t < ntiles ? (uint32_t)((x.end - a0 + 1) / 2) : 0u;
#pragma unroll
    for (uint32_t q = 0; q < kPre; ++q) {
      const uint32_t i = lane + 32 * q;
      pw[q] = (nw <= 32 * kPre && i < nw) ? pword(a0, i) : 0u;
    }
  };
  Slot A, B;
  uint32_t pa[kPre], pb[kPre];
  load_slot(tile, A);
  load_slot(tile + step, B);
  load_pre(A, tile, pa);
  for (; tile < ntiles; tile += step) {
    Slot C;
    load_slot(tile + 2 * step, C);
    load_pre(B, tile + step, pb);
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) c += __popc(A.w[k]);
    const uint32_t inc = warp_inclusive_scan_u32(c, lane);
    const uint32_t total = (uint32_t)(A.end - A.off);
    const uint64_t a0 = A.off & ~1ull;
    const uint32_t nw = (uint32_t)((A.end - a0 + 1) / 2);
    const bool staged = total <= kApplyStage;
    if (nw <= 32 * kPre) {
#pragma unroll
      for (uint32_t q = 0; q < kPre; ++q)
        if (lane + 32 * q < nw) reinterpret_cast<uint32_t*>(sp)[lane + 32 * q] = pa[q];
      __syncwarp();
    } else if (staged) {
      // coalesced copy of payload[off, end) into the stage
      for (uint32_t i = lane; i < nw; i += 32) reinterpret_cast<uint32_t*>(sp)[i] = pword(a0, i);
      __syncwarp();
    }
    uint32_t r = inc - c;  // rank of this lane's first change in the tile
    uint16_t* op = out + tile * kTile + 256 * (uint64_t)lane;  // this lane's elements
    if (staged && BSNP_COOP_SCATTER) {
      // warp-cooperative scatter: lane l writes the changes of rank l, l +
      // 32, ... of the tile (not its own lane's), so the warp runs
      // ceil(total / 32) rounds instead of a loop per mask word paced by
      // its busiest lane.  Rank q's owner lane is the first whose inclusive
      // count exceeds q (binary search by shuffles); its 8 mask words come
      // over by shuffles and the q-th set bit is found word by word.
      const uint32_t ex = inc - c;
      const uint16_t* sr = sp + (uint32_t)(A.off & 1);
      uint16_t* tp = out + tile * kTile;
      for (uint32_t r0 = 0; r0 < total; r0 += 32) {
        const uint32_t q = r0 + lane;
        uint32_t L = 0;
#pragma unroll
        for (uint32_t st = 16; st > 0; st >>= 1)
          if (__shfl_sync(kFull, inc, L + st - 1) <= q) L += st;
        uint32_t lq = q - __shfl_sync(kFull, ex, L);  // rank inside lane L
        uint32_t word = 0, kk = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t wk = __shfl_sync(kFull, A.w[k], L);
          const uint32_t pc = __popc(wk);
          const bool here = kk == 0 && lq < pc;  // first word holding rank lq
          if (here) {
            word = wk;
            kk = (uint32_t)k + 1;
          } else if (kk == 0) {
            lq -= pc;
          }
        }
        if (q < total) {
          for (uint32_t i = 0; i < lq; ++i) word &= word - 1;
          const uint32_t j = __ffs(word) - 1;
          tp[256 * L + 32 * (kk - 1) + j] = sr[q];
        }
      }
    } else if (staged) {
      const uint16_t* sr = sp + (uint32_t)(A.off & 1) + r;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t b = A.w[k];
        while (b) {
          const uint32_t j = __ffs(b) - 1;
          b &= b - 1;
          op[32 * k + j] = *sr++;
        }
      }
    } else {
      const uint16_t* pr = payload + A.off + r;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t b = A.w[k];
        while (b) {
          const uint32_t j = __ffs(b) - 1;
          b &= b - 1;
          if (pr < payload + n_c) op[32 * k + j] = __ldg(pr);
          ++pr;
        }
      }
    }
    __syncwarp();  // the stage is reused by the next tile
    A = B;
    B = C;
#pragma unroll
    for (uint32_t q = 0; q < kPre; ++q) pa[q] = pb[q];
  }
}

// persistent grid size for a dynamic-smem kernel (attribute + occupancy
// query once per kernel, device and thread: they cost microseconds per call;
// the shared-memory attribute is per device)
template <typename K>
int persistent_grid(K kernel, size_t smem, uint64_t work_items, int threads = kThreads) {
  struct Entry {
    const void* fn;
    size_t smem;
    int threads;
    int dev;
    int blocks;
  };
  thread_local Entry cache[16];
  thread_local int used = 0;
  int dev = 0;
  const int sms = device_sms(&dev);
  int blocks = 0;
  for (int i = 0; i < used; ++i)
    if (cache[i].fn == (const void*)kernel && cache[i].smem == smem &&
        cache[i].threads == threads && cache[i].dev == dev)
      blocks = cache[i].blocks;
  if (!blocks) {
    int per_sm = 0;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    blocks = sms * (per_sm < 1 ? 1 : per_sm);
    if (used < 16) cache[used++] = Entry{(const void*)kernel, smem, threads, dev, blocks};
  }
  const uint64_t g = (uint64_t)blocks < work_items ? (uint64_t)blocks : work_items;
  return (int)(g ? g : 1);
}

constexpr int kDecStages = 2;
}  // namespace
}  // namespace bsnp

using namespace bsnp;

#ifdef BSNP_LOOKBACK_STATS
extern "C" int bsnpdbg_lookback_stats(unsigned long long* out4, int reset) {
  cudaMemcpyFromSymbol(out4, g_lookback_stats, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_lookback_stats, z, sizeof(z));
  }
  return 0;
}
#endif

static size_t enc_scratch_offset(uint64_t n) {
  return align_up(kWsHeader + 8 * (size_t)num_tiles(n), 256);
}

// + 32 bytes: the look-back warp's funnel-shifted copy reads up to two
// granules past a record that ends at the arena's end
static size_t enc_smem() { return (size_t)kEncStagesWS * kEncStage + kArena + 32; }

// global staging slots of tiles too dense for the arena: one per tile, or a
// ring of kRing per CTA when that is fewer (large tensors: 2^30 elements
// need 111 MiB instead of 2 GiB)
static uint64_t enc_slots(uint64_t n, uint32_t* ring) {
  const uint64_t nt = num_tiles(n);
  const uint64_t ring_slots =
      (uint64_t)persistent_grid(delta_encode_ws_kernel, enc_smem(), nt, kEncThreads) * kRing;
  if (ring) *ring = ring_slots < nt ? 1u : 0u;
  return ring_slots < nt ? ring_slots : nt;
}

extern "C" size_t bsnp_delta_encode_ws_bytes(uint64_t n) {
  // ticket | tile status words | payload staging slots | one granule the
  // vector copy may read past the last slot
  return enc_scratch_offset(n) + 2 * (size_t)enc_slots(n, nullptr) * kTile + 256;
}

// decode workspace: ticket header | chunk bases u64 [nchunks + 1] | tile
// offsets inside their chunk u32 [ntiles + 1] | chunk totals u32 [nchunks]
struct DecWs {
  uint32_t* ticket;
  uint64_t* base;
  uint32_t* local;
  uint32_t* ctot;
  uint64_t* off;
  uint64_t nchunks;
};
static DecWs dec_ws(void* ws, uint64_t n) {
  DecWs w;
  const uint64_t nt = num_tiles(n);
  w.nchunks = (nt + kChunkTiles - 1) / kChunkTiles;
  w.ticket = (uint32_t*)ws;
  w.base = (uint64_t*)((char*)ws + kWsHeader);
  w.local = (uint32_t*)(w.base + w.nchunks + 1);
  w.ctot = w.local + nt + 1;
  w.off = (uint64_t*)(((uintptr_t)(w.ctot + w.nchunks) + 7) & ~(uintptr_t)7);
  return w;
}

extern "C" size_t bsnp_delta_decode_ws_bytes(uint64_t n) {
  const uint64_t nt = num_tiles(n);
  const uint64_t nchunks = (nt + kChunkTiles - 1) / kChunkTiles;
  return kWsHeader + 8 * (size_t)(nchunks + 1) + 4 * (size_t)(nt + 1) + 4 * (size_t)nchunks + 8 +
         8 * (size_t)(nt + 1);
}

// zero a status block and a workspace prefix (both 8-byte aligned, sizes in
// u64 words) in a kernel instead of two memsets, so the codec kernel after it
// can follow by programmatic dependent launch
__global__ void __launch_bounds__(256)
    zero_words_kernel(uint64_t* __restrict__ a, uint64_t na, uint64_t* __restrict__ b,
                      uint64_t nb) {
  pdl_enter();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb; i += stride) {
    if (i < na) a[i] = 0;
    else b[i - na] = 0;
  }
}

static int zero_prefix(bsnp_status* status, void* ws, size_t ws_bytes, cudaStream_t s) {
  const uint64_t nb = ws_bytes / 8, nw = 2 + nb;
  const unsigned grid = (unsigned)std::min<uint64_t>((nw + 1023) / 1024, 1024);
  return launch_pdl("zero_words_kernel", zero_words_kernel, dim3(grid ? grid : 1), dim3(256), s,
                    (uint64_t*)status, (uint64_t)2, (uint64_t*)ws, nb);
}

// the offsets + validation launches of a decode (n > 0)
// materialize: also the u64 offsets array the TMA decode reads (measured:
// its refill reading base + local directly ran 0.84 instead of 0.71 ms)
static int launch_offsets(const uint8_t* mask, uint64_t n, uint64_t n_c, const uint64_t* nc_dev,
                          const DecWs& w, bsnp_status* status, cudaStream_t s, bool materialize) {
  int rc = launch_pdl("delta_count_kernel", delta_count_kernel, dim3((unsigned)w.nchunks),
                      dim3(kThreads), s, mask, n, w.local, w.ctot, status);
  if (rc) return rc;
  // the passes after the count follow it by programmatic dependent launch
  rc = launch_pdl("delta_scan_kernel", delta_scan_kernel, dim3(1), dim3(kScanThreads), s, w.ctot,
                  w.nchunks, w.base, w.local, num_tiles(n), status, n_c, nc_dev);
  if (rc || !materialize) return rc;
  return launch_pdl("delta_materialize_kernel", delta_materialize_kernel,
                    dim3((unsigned)((num_tiles(n) + kThreads) / kThreads)), dim3(kThreads), s,
                    w.base, w.local, num_tiles(n), w.off);
}

extern "C" int bsnp_delta_encode(const uint16_t* base, const uint16_t* target, uint64_t n,
                                 uint8_t* mask, uint16_t* payload, uint64_t payload_cap,
                                 bsnp_status* status, void* ws, size_t ws_bytes,
                                 void* stream) {
  if (!status) return BSNP_E_INVALID;
  if (n && (!base || !target || !mask || !ws || (!payload && payload_cap)))
    return BSNP_E_INVALID;
  if (((uintptr_t)base | (uintptr_t)target | (uintptr_t)payload) & 1) return BSNP_E_ALIGN;
  const size_t need = bsnp_delta_encode_ws_bytes(n);
  if (n && ws_bytes < need) return BSNP_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0)
    return cuda_status("memset(status)", cudaMemsetAsync(status, 0, sizeof(bsnp_status), s));
  const uint64_t nt = num_tiles(n);
  // status, ticket and tile status words zeroed by a kernel the encode
  // follows by programmatic dependent launch
  int rc = zero_prefix(status, ws, kWsHeader + 8 * nt, s);
  if (rc) return rc;
  uint32_t* ticket = (uint32_t*)ws;
  uint64_t* tstat = (uint64_t*)((char*)ws + kWsHeader);
  const bool aligned = (((uintptr_t)base | (uintptr_t)target) & 15) == 0;
  if (aligned) {
    const size_t smem = enc_smem();
    auto k = delta_encode_ws_kernel;
    const int grid = persistent_grid(k, smem, nt, kEncThreads);
    uint32_t ring = 0;
    enc_slots(n, &ring);
    uint16_t* scratch = (uint16_t*)((char*)ws + enc_scratch_offset(n));
    return launch_pdl_smem("delta_encode_ws_kernel", k, dim3(grid), dim3(kEncThreads), smem, s,
                           base, target, n, mask, payload, payload_cap, scratch, status, ticket,
                           tstat, nt, ring);
  } else {
    delta_encode_kernel<false><<<(unsigned)nt, kThreads, 0, s>>>(
        base, target, n, mask, payload, payload_cap, status, ticket, tstat, nt);
  }
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
  const size_t need = bsnp_delta_decode_ws_bytes(n);
  if (n && ws_bytes < need) return BSNP_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0)
    return cuda_status("memset(status)", cudaMemsetAsync(status, 0, sizeof(bsnp_status), s));
  const uint64_t nt = num_tiles(n);
  const DecWs w = dec_ws(ws, n);
  uint32_t* ticket2 = w.ticket + 32;
  const TileOffsets offsets{w.base, w.local, nt};
  int rc = zero_prefix(status, ws, kWsHeader, s);
  if (rc) return rc;
  const bool in_place = (const void*)base == (const void*)out;
  const bool aligned = (((uintptr_t)base | (uintptr_t)out | (uintptr_t)mask) & 15) == 0;
  const bool tma = aligned && (!in_place || n_c * BSNP_DENSE_DIV > n);
  // pass 1: payload offsets per tile + validation (reads n/8 bytes)
  if ((rc = launch_offsets(mask, n, n_c, nullptr, w, status, s, tma))) return rc;
  if (in_place && aligned && n_c * BSNP_DENSE_DIV > n) {
    // dense: streaming the whole tile beats touching the changed words
    // (p = 25 %: 0.77 vs 1.27 ms at 2^30)
    const size_t smem = (size_t)kDecStages * kDecStage;
    auto k = delta_decode_tma_kernel<kDecStages, true>;
    const int grid = persistent_grid(k, smem, nt);
    return launch_pdl_smem("delta_decode_tma_kernel", k, dim3(grid), dim3(kThreads), smem, s,
                           base, mask, payload, n, n_c, out, w.off, ticket2, status, nullptr);
  } else if (in_place) {
    const int sms = device_sms();
    // one warp per tile, a few tiles per warp
    const uint64_t warps = (nt + 3) / 4;
    const uint64_t want = (warps + kWarps - 1) / kWarps;
    const uint64_t cap = (uint64_t)sms * BSNP_APPLY_CTAS_PER_SM;
    const uint64_t grid = want < cap ? want : cap;
    return launch_pdl("delta_apply_warp_kernel", delta_apply_warp_kernel,
                      dim3((unsigned)(grid ? grid : 1)), dim3(kThreads), s, mask, payload, n,
                      n_c, out, offsets, status);
  } else if (aligned) {
    const size_t smem = (size_t)kDecStages * kDecStage;
    auto k = n_c * 32 > n ? delta_decode_tma_kernel<kDecStages, true>
                          : delta_decode_tma_kernel<kDecStages, false>;
    const int grid = persistent_grid(k, smem, nt);
    return launch_pdl_smem("delta_decode_tma_kernel", k, dim3(grid), dim3(kThreads), smem, s,
                           base, mask, payload, n, n_c, out, w.off, ticket2, nullptr, nullptr);
  }
  return launch_pdl("delta_apply_kernel", delta_apply_kernel<false>, dim3((unsigned)nt),
                    dim3(kThreads), s, base, mask, payload, n, n_c, out, offsets, status);
}

extern "C" int bsnp_delta_decode_dn(const uint16_t* base, const uint8_t* mask,
                                    const uint16_t* payload, uint64_t n, const uint64_t* n_c_dev,
                                    uint16_t* out, bsnp_status* status, void* ws,
                                    size_t ws_bytes, void* stream) {
  if (!status) return BSNP_E_INVALID;
  if (n && (!base || !mask || !out || !ws || !n_c_dev)) return BSNP_E_INVALID;
  if ((const void*)base == (const void*)out && n) return BSNP_E_INVALID;  // out of place only
  if (((uintptr_t)base | (uintptr_t)out | (uintptr_t)payload) & 1) return BSNP_E_ALIGN;
  const size_t need = bsnp_delta_decode_ws_bytes(n);
  if (n && ws_bytes < need) return BSNP_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0)
    return cuda_status("memset(status)", cudaMemsetAsync(status, 0, sizeof(bsnp_status), s));
  const uint64_t nt = num_tiles(n);
  const DecWs w = dec_ws(ws, n);
  uint32_t* ticket2 = w.ticket + 32;
  int rc = zero_prefix(status, ws, kWsHeader, s);
  if (rc) return rc;
  if ((rc = launch_offsets(mask, n, 0, n_c_dev, w, status, s, true))) return rc;
  const bool aligned = (((uintptr_t)base | (uintptr_t)out | (uintptr_t)mask) & 15) == 0;
  if (aligned) {
    // the sparse (bit-walk) expansion: n_c is not known on the host
    const size_t smem = (size_t)kDecStages * kDecStage;
    auto k = delta_decode_tma_kernel<kDecStages, false>;
    const int grid = persistent_grid(k, smem, nt);
    return launch_pdl_smem("delta_decode_tma_kernel", k, dim3(grid), dim3(kThreads), smem, s,
                           base, mask, payload, n, (uint64_t)0, out, w.off, ticket2, nullptr,
                           n_c_dev);
  }
  return BSNP_E_ALIGN;
}
