// Cluster quantizer for sm_100a.
//
// Replaces build_clusters / quantize / dequantize of the reference
// (/root/reference/pkg/src/bitsnap/quantizer.py:100-204) with bit-identical
// results:
//
//  * fit statistics: numpy computes mean and std of the float64-widened
//    tensor with pairwise summation (np.add.reduce over a contiguous vector,
//    numpy/_core/src/umath/loops_utils.h.src): a node of s > 128 elements
//    splits at 8*floor(s/16); a leaf of <= 128 elements is summed with 8
//    interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
//    plus a sequential tail; a node of < 8 elements sums sequentially from 0.
//    The kernels reproduce that tree exactly: a unit is cut into the 2^D
//    nodes of depth D (<= kTileMax elements each, one CTA per node), every
//    CTA evaluates its node's sub-tree in shared memory (a heap of <= 255
//    nodes: leaves by 4-lane groups, then level-wise combines), and one CTA
//    per unit combines the 2^D partials as a perfect binary tree.
//  * fit labels use the unrounded float64 boundaries; for a float32 value v,
//    B64 < v  <=>  RD_f32(B64) < v, so the comparison runs in float32.
//  * quantize codes: a float32 estimate of ceil(255 (v-b)/S - 0.5) is exact
//    whenever its argument is farther than 2^-12 from an integer (the
//    estimate's error is < 6.2e-5); the rare ambiguous
//    elements evaluate the reference's float64 expression.
//  * dequantize: a per-unit 16 x 256 LUT of f32(f64(j)/255 * S + b).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ndtri_table.cuh"
#include "runtime.cuh"

namespace bsnp {
namespace {

constexpr int kQThreads = 256;
constexpr uint32_t kTileMax = 8192;  // elements per tree tile (a depth-D node)
constexpr int kHeapDepth = 7;        // leaves of a <= kTileMax node lie at depth <= 7
constexpr int kHeap = 1 << (kHeapDepth + 1);
constexpr uint32_t kSmemFloats = kTileMax + (kTileMax / 128) * 8 + 32;
constexpr uint32_t kDqChunk = 65536;  // elements per dequantize CTA (one LUT build)
static_assert(kDqChunk == BSNP_DEQUANT_CHUNK, "header chunk size");
static_assert(sizeof(bsnp_cluster_table) == 256, "table layout is part of the C-ABI");

// shared-memory layout: 8 floats of padding per 128-float chunk so that the
// 4-lane leaf groups of a warp hit distinct banks
__device__ __forceinline__ uint32_t padded(uint32_t i) { return i + ((i >> 7) << 3); }

struct QPlan {
  uint64_t n, block;  // block = unit length (n for one unit)
  uint64_t last_len;
  uint64_t total_tiles;
  uint32_t nunits, m;
  uint32_t D_full, T_full;  // tree depth / tiles of a full unit
  uint32_t D_last, T_last;  // of the last unit (T_last may exceed T_full: numpy's
                            // splits of a slightly shorter length can leave a
                            // piece above kTileMax one level deeper)
  uint32_t D_max, T_max;    // max of the two: per-unit enumerations use T_max
  uint32_t C_full, C_last;  // dequantize chunks per unit
};

struct TileRef {
  uint32_t u, j, D;
  uint64_t len, ustart, off, size;
};

__device__ __forceinline__ TileRef locate(const QPlan& P, uint64_t tile) {
  TileRef r;
  const uint64_t full_tiles = (uint64_t)(P.nunits - 1) * P.T_full;
  if (tile < full_tiles) {
    r.u = (uint32_t)(tile >> P.D_full);  // T_full = 2^D_full
    r.j = (uint32_t)(tile & (P.T_full - 1));
    r.D = P.D_full;
    r.len = P.block;
  } else {
    r.u = P.nunits - 1;
    r.j = (uint32_t)(tile - full_tiles);
    r.D = P.D_last;
    r.len = P.last_len;
  }
  r.ustart = (uint64_t)r.u * P.block;
  if ((r.len & (r.len - 1)) == 0 && (r.len >> r.D) >= 16) {
    // power-of-two unit: numpy's splits are exact halves
    r.size = r.len >> r.D;
    r.off = (uint64_t)r.j * r.size;
    return r;
  }
  uint64_t off = 0, size = r.len;
  for (int b = (int)r.D - 1; b >= 0; --b) {
    const uint64_t L = 8 * (size / 16);
    if ((r.j >> b) & 1u) {
      off += L;
      size -= L;
    } else {
      size = L;
    }
  }
  r.off = off;
  r.size = size;
  return r;
}

// order-preserving float -> int key (for min / max through integer atomics)
__device__ __forceinline__ int fkey(float f) {
  const int b = __float_as_int(f);
  return b >= 0 ? b : b ^ 0x7fffffff;
}
__device__ __forceinline__ float fkey_inv(int k) {
  return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff);
}

// #(t[k] < v) over a sorted 16-slot table (unused slots hold +inf)
__device__ __forceinline__ uint32_t count_below(const float* t, float v) {
  uint32_t lo = 0;
  lo += (t[lo + 7] < v) ? 8u : 0u;
  lo += (t[lo + 3] < v) ? 4u : 0u;
  lo += (t[lo + 1] < v) ? 2u : 0u;
  lo += (t[lo] < v) ? 1u : 0u;
  return lo;
}

// Label lookup: #(bnd[k] < v) through a 64-bin uniform grid over
// [bnd[0], bnd[m-2]]; each bin holds at most one boundary (else ok = 0 and
// the 4-step binary search is used).  bin() is monotone in v and the table is
// built with the same bin(), so the result is exact.
struct LabelLut {
  float g0, ginv;
  uint32_t ok;
  uint32_t ent[64];  // count of boundaries in lower bins | in-bin boundary index << 8
  float bnd[16];     // +inf padded
};

__device__ __forceinline__ int lut_bin(float v, float g0, float ginv) {
  const int b = __float2int_rd(__fmul_rn(__fsub_rn(v, g0), ginv));
  return min(max(b, 0), 63);
}

__device__ __forceinline__ uint32_t lut_label(const LabelLut& L, float v) {
  const uint32_t e = L.ent[lut_bin(v, L.g0, L.ginv)];
  return (e & 0xffu) + (L.bnd[e >> 8] < v ? 1u : 0u);
}


// CTA-wide build of a label LUT (threads 0..63 build, all threads vote).
// L.bnd[] (+inf padded) must be visible to every thread before the call.
__device__ void lut_build_cta(LabelLut& L, int m) {
  const int b = threadIdx.x;
  const float g0 = L.bnd[0], g1 = L.bnd[m > 2 ? m - 2 : 0];
  const float ginv = __fdiv_rn(64.0f, __fsub_rn(g1, g0));
  const bool usable = m > 2 && g1 > g0 && isfinite(ginv) && ginv > 0.0f;
  uint32_t cnt = 0;
  if (b < 64) {
    uint32_t base = 0, kin = 15;
    for (int k = 0; k < m - 1; ++k) {
      const int bk = lut_bin(L.bnd[k], g0, ginv);
      if (bk < b) ++base;
      else if (bk == b) {
        kin = (uint32_t)k;
        ++cnt;
      }
    }
    L.ent[b] = base | (kin << 8);
  }
  const bool ok = __syncthreads_and(usable && cnt <= 1) != 0;
  if (b == 0) {
    L.g0 = g0;
    L.ginv = ginv;
    L.ok = ok ? 1u : 0u;
  }
  __syncthreads();
}

// Load elements [0, size) of a tile into padded shared memory.
__device__ __forceinline__ void load_tile(float* s, const float* src, uint32_t size,
                                          uint64_t pol) {
  if (((uintptr_t)src & 15) == 0) {
    const uint32_t nv = size / 4;
    for (uint32_t v = threadIdx.x; v < nv; v += blockDim.x) {
      const float4 x = ld_hint_f4(src + 4 * v, pol);
      *reinterpret_cast<float4*>(&s[padded(4 * v)]) = x;
    }
    for (uint32_t i = nv * 4 + threadIdx.x; i < size; i += blockDim.x) s[padded(i)] = src[i];
  } else {
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) s[padded(i)] = src[i];
  }
}

template <bool kVar>
__device__ __forceinline__ double widen(float x, double mu) {
  const double d = (double)x;
  if (!kVar) return d;
  const double c = __dsub_rn(d, mu);  // arr - arrmean
  return __dmul_rn(c, c);             // x * x
}

struct Heap {
  uint16_t off[kHeap];
  uint16_t size[kHeap];
  uint8_t kind[kHeap];  // 0 absent, 1 leaf, 2 internal
  double val[kHeap];
};

// numpy pairwise sum of values widen(s[0..size)) — the sub-tree of one node.
template <bool kVar>
__device__ double tree_sum(const float* s, uint32_t size, double mu, Heap& H) {
  const int tid = threadIdx.x;
  for (int h = tid; h < kHeap; h += blockDim.x) {
    if (h == 0) continue;
    const int d = 31 - __clz(h);
    const uint32_t j = (uint32_t)h - (1u << d);
    uint32_t off = 0, sz = size;
    bool present = true;
    for (int b = d - 1; b >= 0; --b) {
      if (sz <= 128) {
        present = false;
        break;
      }
      const uint32_t L = 8 * (sz / 16);
      if ((j >> b) & 1u) {
        off += L;
        sz -= L;
      } else {
        sz = L;
      }
    }
    H.kind[h] = !present ? 0 : (sz <= 128 ? 1 : 2);
    H.off[h] = (uint16_t)off;
    H.size[h] = (uint16_t)sz;
  }
  __syncthreads();
  // leaves: 4 lanes per leaf, lane q owns accumulators r[2q], r[2q+1]
  const int g = tid >> 2, q = tid & 3;
  const int ngroups = blockDim.x >> 2;
  const unsigned gm = 0xfu << ((tid & 31) & ~3);
  for (int base = 0; base < kHeap; base += ngroups) {
    const int h = base + g;
    if (h == 0 || h >= kHeap || H.kind[h] != 1) continue;
    const uint32_t off = H.off[h], sz = H.size[h];
    double res = 0.0;
    if (sz < 8) {
      if (q == 0)
        for (uint32_t i = 0; i < sz; ++i) res = __dadd_rn(res, widen<kVar>(s[padded(off + i)], mu));
    } else {
      const uint32_t body = sz - sz % 8;
      float2 p = *reinterpret_cast<const float2*>(&s[padded(off + 2 * q)]);
      double ra = widen<kVar>(p.x, mu), rb = widen<kVar>(p.y, mu);
      for (uint32_t i = 8; i < body; i += 8) {
        p = *reinterpret_cast<const float2*>(&s[padded(off + i + 2 * q)]);
        ra = __dadd_rn(ra, widen<kVar>(p.x, mu));
        rb = __dadd_rn(rb, widen<kVar>(p.y, mu));
      }
      double pr = __dadd_rn(ra, rb);
      pr = __dadd_rn(pr, __shfl_xor_sync(gm, pr, 1));
      pr = __dadd_rn(pr, __shfl_xor_sync(gm, pr, 2));
      res = pr;
      if (q == 0)
        for (uint32_t i = body; i < sz; ++i) res = __dadd_rn(res, widen<kVar>(s[padded(off + i)], mu));
    }
    if (q == 0) H.val[h] = res;
  }
  for (int d = kHeapDepth - 1; d >= 0; --d) {
    __syncthreads();
    for (int h = (1 << d) + tid; h < (2 << d); h += blockDim.x)
      if (H.kind[h] == 2) H.val[h] = __dadd_rn(H.val[2 * h], H.val[2 * h + 1]);
  }
  __syncthreads();
  return H.val[1];
}

// pass 1 / pass 2 of the fit: per-tile pairwise sums of x (kVar = false) or
// of (x - mean)^2 (kVar = true)
// perfect 8192-element tiles: 8 floats of padding per 1024 (8 leaves)
__device__ __forceinline__ uint32_t epad(uint32_t e) { return e + ((e >> 10) << 3); }

// The pairwise sum of one tree tile (a depth-D node); the result is valid in
// thread 0.  s / H are the tile's shared-memory staging and heap.
template <bool kVar>
__device__ __forceinline__ double tree_tile(const float* __restrict__ x, const QPlan& P,
                                            uint64_t tile, double m, float* s, Heap& H,
                                            uint64_t pol) {
  const TileRef r = locate(P, tile);
  const float* src = x + r.ustart + r.off;
  if (r.size == kTileMax && ((uintptr_t)src & 15) == 0) {
    // a perfect sub-tree: 64 leaves of 128.  8 lanes per leaf (lane j owns
    // numpy's accumulator r[j]); the 4 lane groups of a warp take leaves
    // w, w+8, w+16, w+24 (+32), which the padding puts on distinct banks.
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = i * kQThreads + tid;
      *reinterpret_cast<float4*>(&s[epad(4 * v)]) = ld_hint_f4(src + 4 * v, pol);
    }
    __syncthreads();
    const int j = lane & 7, q = lane >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int leaf = warp + 8 * q + 32 * h;
      const float* lp = s + 128 * leaf + 8 * (leaf >> 3) + j;
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = lp[8 * i];
      double acc = widen<kVar>(a[0], m);
#pragma unroll
      for (int i = 1; i < 16; ++i) acc = __dadd_rn(acc, widen<kVar>(a[i], m));
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 1));
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 2));
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 4));
      if (j == 0) H.val[leaf] = acc;
    }
    __syncthreads();
    double v = 0.0;
    if (warp == 0) {
      v = __dadd_rn(H.val[2 * lane], H.val[2 * lane + 1]);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, d));
    }
    return v;
  }
  load_tile(s, src, (uint32_t)r.size, pol);
  __syncthreads();
  return tree_sum<kVar>(s, (uint32_t)r.size, m, H);
}

template <bool kVar>
__global__ void __launch_bounds__(kQThreads)
    fit_tree_kernel(const float* __restrict__ x, QPlan P, const double* __restrict__ mu,
                    double* __restrict__ partials) {
  __shared__ __align__(16) float s[kSmemFloats];
  __shared__ Heap H;
  // the variance pass walks the tiles backwards: its first tiles are the
  // last ones the sum pass read, still in L2 (the labels pass then walks
  // forwards again, the codes pass backwards); only the codes pass, the
  // last reader of x, marks its lines evict-first
  const uint64_t tile = kVar ? P.total_tiles - 1 - blockIdx.x : blockIdx.x;
  const double m = kVar ? mu[locate(P, tile).u] : 0.0;
  const double v = tree_tile<kVar>(x, P, tile, m, s, H, policy_evict_normal());
  if (threadIdx.x == 0) partials[tile] = v;
}

// Sum of the 2^D partials of one unit as a perfect binary tree.
__device__ double combine_perfect(const double* p, uint32_t T, double* sv) {
  const int tid = threadIdx.x;
  const uint32_t lanes = T < (uint32_t)blockDim.x ? T : blockDim.x;
  if ((uint32_t)tid < lanes) {
    const uint32_t chunk = T / lanes;  // power of two
    const double* c = p + (uint64_t)tid * chunk;
    // left-to-right binary-counter reduction == perfect tree over the chunk
    double stk[20];
    uint32_t lvl[20];
    int top = 0;
    for (uint32_t i = 0; i < chunk; ++i) {
      double v = __ldcg(c + i);
      uint32_t l = 0;
      while (top > 0 && lvl[top - 1] == l) {
        v = __dadd_rn(stk[top - 1], v);
        --top;
        ++l;
      }
      stk[top] = v;
      lvl[top] = l;
      ++top;
    }
    sv[tid] = stk[0];
  }
  __syncthreads();
  for (uint32_t w = lanes / 2; w >= 1; w /= 2) {
    double a = 0.0;
    if ((uint32_t)tid < w) a = __dadd_rn(sv[2 * tid], sv[2 * tid + 1]);
    __syncthreads();
    if ((uint32_t)tid < w) sv[tid] = a;
    __syncthreads();
  }
  return sv[0];
}

__device__ __forceinline__ void unit_shape(const QPlan& P, uint32_t u, uint32_t& T,
                                           uint64_t& len) {
  const bool last = u == P.nunits - 1;
  T = last ? P.T_last : P.T_full;
  len = last ? P.last_len : P.block;
}

// Mean (kVar = false) or std + table header + fit thresholds (kVar = true) of
// unit u from its tile partials; CTA-wide (sv: kQThreads doubles of smem).
constexpr uint32_t kPreGroup = 1024;  // partials per pre-reduction CTA
constexpr int kPreShift = 10;

template <bool kVar>
__device__ __forceinline__ void combine_unit(const QPlan& P, uint32_t u,
                                             const double* partials, double* mu, float* fthr,
                                             bsnp_cluster_table* tables, double* sdv,
                                             double* sv, const double* partials2 = nullptr) {
  uint32_t T;
  uint64_t len;
  unit_shape(P, u, T, len);
  // with T > kPreGroup the partials were pre-reduced in groups of kPreGroup
  // (pre_combine_kernel): the same perfect tree, one level set at a time
  const int sh = T > kPreGroup ? kPreShift : 0;
  const uint32_t Tg = T >> sh;
  const double S = combine_perfect(sh ? partials2 + (uint64_t)u * (P.T_max >> kPreShift)
                                      : partials + (uint64_t)u * P.T_full,
                                   Tg, sv);
  if (threadIdx.x != 0) return;
  const double mean = __ddiv_rn(__dadd_rn(0.0, S), (double)len);  // np.mean
  bsnp_cluster_table& tb = tables[u];
  if (!kVar) {
    mu[u] = mean;
    return;
  }
  const double m0 = __ldcg(mu + u);
  const double var = __ddiv_rn(__dadd_rn(0.0, S), (double)len);
  const double sd = __dsqrt_rn(var);  // np.std, ddof = 0
  if (sdv) sdv[u] = sd;
  const int m = (int)P.m;
  tb.mean = __double2float_rn(m0);
  tb.std = __double2float_rn(sd);
  tb.m = (uint32_t)m;
  tb.flags = (isfinite(m0) && isfinite(sd)) ? 0u : BSNP_ERR_NONFINITE;
  for (int k = 0; k < 15; ++k) {
    if (k < m - 1) {
      const double b = __dadd_rn(m0, __dmul_rn(sd, kNdtri[m][k]));  // mu + sigma * ndtri
      tb.boundaries[k] = __double2float_rn(b);
      fthr[u * 16 + k] = __double2float_rd(b);  // fit labels compare against b exactly
    } else {
      tb.boundaries[k] = 0.0f;
      fthr[u * 16 + k] = __int_as_float(0x7f800000);
    }
  }
  fthr[u * 16 + 15] = __int_as_float(0x7f800000);
  for (int k = 0; k < 13; ++k) tb.reserved[k] = 0;
}

template <bool kVar>
__global__ void __launch_bounds__(kQThreads)
    fit_combine_kernel(QPlan P, const double* __restrict__ partials, double* __restrict__ mu,
                       float* __restrict__ fthr, bsnp_cluster_table* __restrict__ tables,
                       double* __restrict__ sdv = nullptr,
                       const double* __restrict__ partials2 = nullptr) {
  __shared__ double sv[kQThreads];
  combine_unit<kVar>(P, blockIdx.x, partials, mu, fthr, tables, sdv, sv, partials2);
}

// Units with more than kPreGroup tiles (per-tensor units above 2^23
// elements): each CTA folds kPreGroup consecutive tile partials - a perfect
// sub-tree of the unit's perfect tree - so the per-unit combine folds
// T / kPreGroup values instead of T (a 2^30-element unit: 181 -> ~10 us).
__global__ void __launch_bounds__(kQThreads)
    pre_combine_kernel(QPlan P, const double* __restrict__ partials,
                       double* __restrict__ partials2) {
  __shared__ double v[kPreGroup];
  const uint64_t g = blockIdx.x;  // group index over all units (T_max-strided)
  const uint64_t gpu = P.T_max >> kPreShift;  // group slots per unit
  const uint32_t u = (uint32_t)(g / gpu);
  const uint32_t T = u == P.nunits - 1 ? P.T_last : P.T_full;
  const uint64_t gi = g % gpu;
  if ((gi << kPreShift) >= T) return;  // units with fewer tiles
  const double* src = partials + (uint64_t)u * P.T_full + (gi << kPreShift);
  for (int i = threadIdx.x; i < (int)kPreGroup; i += kQThreads) v[i] = src[i];
  constexpr int kPer = kPreGroup / 2 / kQThreads;  // pairs per thread at the first level
  for (uint32_t w = kPreGroup / 2; w >= 1; w /= 2) {
    __syncthreads();
    double a[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t i = threadIdx.x + q * kQThreads;
      if (i < w) a[q] = __dadd_rn(v[2 * i], v[2 * i + 1]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t i = threadIdx.x + q * kQThreads;
      if (i < w) v[i] = a[q];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) partials2[g] = v[0];
}

template <bool kLut>
__device__ __forceinline__ uint32_t label_t(const LabelLut& L, float v) {
  return kLut ? lut_label(L, v) : count_below(L.bnd, v);
}

template <bool kLut>
__device__ __forceinline__ void minmax_loop(const LabelLut& L, const float* src, uint32_t size,
                                            int* mnrow, int* mxrow) {
  const uint32_t mn_base = smem_addr(mnrow), mx_base = smem_addr(mxrow);
  auto visit = [&](float v) {
    const uint32_t c = label_t<kLut>(L, v);
    const int k = fkey(v);
    // predicated reductions: no branch / reconvergence per element; the
    // read-compare filter keeps the (contended) atomics rare once extrema settle
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .s32 a, b;\n\t"
        "ld.shared.s32 a, [%0];\n\tld.shared.s32 b, [%1];\n\t"
        "setp.lt.s32 p, %2, a;\n\tsetp.gt.s32 q, %2, b;\n\t"
        "@p red.shared.min.s32 [%0], %2;\n\t@q red.shared.max.s32 [%1], %2;\n}" ::"r"(
            mn_base + 4 * c),
        "r"(mx_base + 4 * c), "r"(k)
        : "memory");
  };
  uint32_t done = 0;
  if (((uintptr_t)src & 15) == 0) {
    const uint32_t nv = size / 4;
    constexpr int kB = 4;  // vectors per thread in flight (a tile is 8 per thread)
    for (uint32_t i0 = threadIdx.x; i0 < nv; i0 += kB * kQThreads) {
      float4 vb[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b)
        if (i0 + b * kQThreads < nv) vb[b] = ld_stream_f4(src + 4 * (i0 + b * kQThreads));
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        if (i0 + b * kQThreads >= nv) break;
        visit(vb[b].x);
        visit(vb[b].y);
        visit(vb[b].z);
        visit(vb[b].w);
      }
    }
    done = nv * 4;
  }
  for (uint32_t i = done + threadIdx.x; i < size; i += kQThreads) visit(src[i]);
}

// pass 3 of the fit: per-tile, per-cluster min / max with fit-time labels
__global__ void __launch_bounds__(kQThreads)
    fit_minmax_kernel(const float* __restrict__ x, QPlan P, const float* __restrict__ fthr,
                      int* __restrict__ tile_mm, const uint32_t* __restrict__ need = nullptr) {
  pdl_enter();
  __shared__ LabelLut L;
  __shared__ int wmin[kQThreads / 32][16], wmax[kQThreads / 32][16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t full_tiles = (uint64_t)(P.nunits - 1) * P.T_full;
  // grid-stride over tiles: with `need`, only the units the threshold-window
  // pass left undecided are visited (a small grid skips the rest quickly)
  if (need && !need[P.nunits]) return;  // no unit needs the exact round
  for (uint64_t tile = blockIdx.x; tile < P.total_tiles; tile += gridDim.x) {
    if (need) {
      const uint32_t uu = tile < full_tiles ? (uint32_t)(tile >> P.D_full) : P.nunits - 1;
      if (!need[uu]) continue;
    }
    const TileRef r = locate(P, tile);
    __syncthreads();  // the previous tile's reads of L / wmin / wmax are done
    if (tid < 16) L.bnd[tid] = fthr[r.u * 16 + tid];
    if (lane < 16) {
      wmin[warp][lane] = 0x7fffffff;
      wmax[warp][lane] = (int)0x80000000;
    }
    __syncthreads();
    lut_build_cta(L, (int)P.m);
    const float* src = x + r.ustart + r.off;
    const uint32_t size = (uint32_t)r.size;
    if (L.ok) minmax_loop<true>(L, src, size, wmin[warp], wmax[warp]);
    else minmax_loop<false>(L, src, size, wmin[warp], wmax[warp]);
    __syncthreads();
    if (tid < 16) {
      int a = 0x7fffffff, b = (int)0x80000000;
      for (int w = 0; w < kQThreads / 32; ++w) {
        a = min(a, wmin[w][tid]);
        b = max(b, wmax[w][tid]);
      }
      tile_mm[tile * 32 + tid] = a;
      tile_mm[tile * 32 + 16 + tid] = b;
    }
  }
}

// scales / offsets per unit (quantizer.py:117-125)
__global__ void __launch_bounds__(kQThreads)
    fit_finalize_kernel(QPlan P, const int* __restrict__ tile_mm,
                        bsnp_cluster_table* __restrict__ tables,
                        const uint32_t* __restrict__ need = nullptr) {
  pdl_enter();
  __shared__ int rmin[8][16], rmax[8][16];
  const uint32_t u = blockIdx.x;
  if (need && (!need[P.nunits] || !need[u])) return;
  uint32_t T;
  uint64_t len;
  unit_shape(P, u, T, len);
  const int c = threadIdx.x & 15, row = threadIdx.x >> 4;  // 16 rows x 16 clusters
  int mn = 0x7fffffff, mx = (int)0x80000000;
  const int* base = tile_mm + (uint64_t)u * P.T_full * 32;
  for (uint32_t t = row; t < T; t += 16) {
    mn = min(mn, base[t * 32 + c]);
    mx = max(mx, base[t * 32 + 16 + c]);
  }
  // fold 16 rows -> 8 via shuffles inside the warp (rows r and r+1 share a warp)
  mn = min(mn, __shfl_down_sync(kFull, mn, 16));
  mx = max(mx, __shfl_down_sync(kFull, mx, 16));
  if ((threadIdx.x & 31) < 16) {
    rmin[threadIdx.x >> 5][c] = mn;
    rmax[threadIdx.x >> 5][c] = mx;
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    int a = rmin[0][c], b = rmax[0][c];
    for (int w = 1; w < 8; ++w) {
      a = min(a, rmin[w][c]);
      b = max(b, rmax[w][c]);
    }
    bsnp_cluster_table& tb = tables[u];
    float scale = 0.0f, offset = 0.0f;
    if ((uint32_t)c < P.m && a <= b) {
      const float lo = fkey_inv(a), hi = fkey_inv(b);
      scale = __double2float_rn(__dsub_rn((double)hi, (double)lo));
      offset = lo;
    }
    tb.scales[c] = scale;
    tb.offsets[c] = offset;
  }
}

// ----------------------------------------------------------------- quantize
struct QuantParams {
  float bnd[16];  // boundaries, +inf padded
  float off[16];  // cluster min
  float rcp[16];  // 255 / S (0 if S == 0, NaN if not finite -> exact path)
  float scl[16];  // S
  uint32_t last;  // m - 1: numpy's searchsorted sorts NaN after every boundary
};

__device__ __forceinline__ void load_quant_params(const bsnp_cluster_table& tb, QuantParams& Q) {
  const int t = threadIdx.x;
  if (t < 16) {
    const uint32_t m = tb.m;
    Q.bnd[t] = ((uint32_t)t < m - 1) ? tb.boundaries[t] : __int_as_float(0x7f800000);
    const float S = tb.scales[t];
    Q.scl[t] = S;
    Q.off[t] = tb.offsets[t];
    float rc = 0.0f;
    if (S > 0.0f) {
      rc = __fdiv_rn(255.0f, S);
      if (!isfinite(rc)) rc = __int_as_float(0x7fffffff);
    }
    Q.rcp[t] = rc;
    if (t == 0) Q.last = m - 1;
  }
}

// exact code of quantizer.py:174-182 in float64 (the slow path)
__device__ __noinline__ uint32_t exact_code(float v, float b, float S) {
  double xn = 0.0;
  if (S > 0.0f) xn = __ddiv_rn(__dsub_rn((double)v, (double)b), (double)S);
  xn = fmin(fmax(xn, 0.0), 1.0);
  const double y = __dsub_rn(__dmul_rn(xn, 255.0), 0.5);
  double c = ceil(y);
  c = fmin(fmax(c, 0.0), 255.0);
  return (uint32_t)c;
}

__device__ __forceinline__ uint32_t quant_one(const QuantParams& Q, float v, uint32_t& label) {
  const uint32_t c = isnan(v) ? Q.last : count_below(Q.bnd, v);
  label = c;
  const float b = Q.off[c];
  const float t = __fsub_rn(__fmul_rn(__fsub_rn(v, b), Q.rcp[c]), 0.5f);
  // the float32 estimate t is within 6.2e-5 of 255(v-b)/S - 0.5
  const bool amb = isnan(t) || fabsf(__fsub_rn(t, rintf(t))) <= 0.000244140625f;
  if (__builtin_expect(amb, 0)) return exact_code(v, b, Q.scl[c]);
  int e = __float2int_ru(t);
  e = e < 0 ? 0 : (e > 255 ? 255 : e);
  return (uint32_t)e;
}

// code of one element from its cluster parameters; `amb` is set when the
// float32 estimate is not provably exact (then exact_code decides)
__device__ __forceinline__ uint32_t code_estimate(float v, float b, float rc, bool& amb) {
  const float tt = __fsub_rn(__fmul_rn(__fsub_rn(v, b), rc), 0.5f);
  amb |= !(fabsf(__fsub_rn(tt, rintf(tt))) > 0.000244140625f);  // also NaN
  return (uint32_t)min(max(__float2int_ru(tt), 0), 255);
}

template <bool kLut>
__device__ __forceinline__ void quant_loop(const LabelLut& L, const QuantParams& Q,
                                           const float2* qp, const float* src, uint8_t* cdst,
                                           uint8_t* ldst, uint32_t nv) {
  constexpr int kB = 4;  // vectors per thread in flight (the loop was load-latency bound)
  for (uint32_t i0 = threadIdx.x; i0 < nv; i0 += kB * kQThreads) {
    float4 vb[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b)
      if (i0 + b * kQThreads < nv) vb[b] = ld_stream_f4(src + 4 * (i0 + b * kQThreads));
#pragma unroll
    for (int b = 0; b < kB; ++b) {
    const uint32_t i = i0 + b * kQThreads;
    if (i >= nv) break;
    const float4 v4 = vb[b];
    const float v[4] = {v4.x, v4.y, v4.z, v4.w};
    uint32_t c[4], code[4];
    bool amb = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) c[e] = label_t<kLut>(L, v[e]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 bp = qp[c[e]];
      code[e] = code_estimate(v[e], bp.x, bp.y, amb);
    }
    if (__builtin_expect(amb, 0)) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bool a1 = false;
        code_estimate(v[e], qp[c[e]].x, qp[c[e]].y, a1);
        if (a1) {
          if (isnan(v[e])) c[e] = Q.last;
          code[e] = exact_code(v[e], Q.off[c[e]], Q.scl[c[e]]);
        }
      }
    }
    *reinterpret_cast<uint32_t*>(cdst + 4 * i) =
        code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
    *reinterpret_cast<uint16_t*>(ldst + 2 * i) =
        (uint16_t)(c[0] | (c[1] << 4) | (c[2] << 8) | (c[3] << 12));
    }
  }
}

__global__ void __launch_bounds__(kQThreads)
    quantize_kernel(const float* __restrict__ x, QPlan P,
                    const bsnp_cluster_table* __restrict__ tables, uint8_t* __restrict__ labels,
                    uint8_t* __restrict__ codes) {
  __shared__ QuantParams Q;
  __shared__ LabelLut L;
  __shared__ float2 qp[16];
  // one CTA per kDqChunk-element chunk of a unit (one parameter / LUT setup
  // per 64 Ki elements)
  const uint64_t full_chunks = (uint64_t)(P.nunits - 1) * P.C_full;
  uint32_t u;
  uint64_t c0, ulen;
  if (blockIdx.x < full_chunks) {
    u = (uint32_t)(blockIdx.x / P.C_full);
    c0 = (blockIdx.x % P.C_full) * kDqChunk;
    ulen = P.block;
  } else {
    u = P.nunits - 1;
    c0 = (blockIdx.x - full_chunks) * kDqChunk;
    ulen = P.last_len;
  }
  load_quant_params(tables[u], Q);
  __syncthreads();
  if (threadIdx.x < 16) {
    L.bnd[threadIdx.x] = Q.bnd[threadIdx.x];
    qp[threadIdx.x] = make_float2(Q.off[threadIdx.x], Q.rcp[threadIdx.x]);
  }
  __syncthreads();
  lut_build_cta(L, (int)tables[u].m);
  const uint64_t ustart = (uint64_t)u * P.block;
  const float* src = x + ustart + c0;
  uint8_t* cdst = codes + ustart + c0;
  uint8_t* ldst = labels + (uint64_t)u * (P.block / 2) + c0 / 2;
  const uint32_t size = (uint32_t)((c0 + kDqChunk < ulen ? c0 + kDqChunk : ulen) - c0);
  const bool vec = (((uintptr_t)src & 15) | ((uintptr_t)cdst & 3) | ((uintptr_t)ldst & 1)) == 0;
  const uint32_t nv = vec ? size / 4 : 0;
  if (L.ok) quant_loop<true>(L, Q, qp, src, cdst, ldst, nv);
  else quant_loop<false>(L, Q, qp, src, cdst, ldst, nv);
  // tail (and unaligned tiles): element pairs through the reference-exact path
  for (uint32_t p = nv * 2 + threadIdx.x; 2 * p < size; p += blockDim.x) {
    uint32_t la, lb = 0;
    cdst[2 * p] = (uint8_t)quant_one(Q, src[2 * p], la);
    if (2 * p + 1 < size) cdst[2 * p + 1] = (uint8_t)quant_one(Q, src[2 * p + 1], lb);
    ldst[p] = (uint8_t)(la | (lb << 4));
  }
}

// ------------------------------------------------------- one-tile units
// A unit of at most kTileMax elements (biases, norms: 2/3 of a GPT-2
// checkpoint's optimizer tensors) in ONE CTA: x stays in shared memory
// through the pairwise mean and variance trees, the table, the fit-label
// min/max and the codes - one launch instead of the tiled path's ten.
// Same primitives, so the same bits.
__global__ void __launch_bounds__(kQThreads)
    tiny_encode_kernel(const float* __restrict__ x, uint32_t n, int m,
                       bsnp_cluster_table* __restrict__ tbl, uint8_t* __restrict__ labels,
                       uint8_t* __restrict__ codes) {
  __shared__ __align__(16) float s[kSmemFloats];
  __shared__ Heap H;
  __shared__ QuantParams Q;
  __shared__ float F[16];
  __shared__ int cmin[16], cmax[16];
  __shared__ double s_mu, s_sd;
  const int tid = threadIdx.x;
  load_tile(s, x, n, policy_evict_first());
  if (tid < 16) {
    cmin[tid] = 0x7fffffff;
    cmax[tid] = (int)0x80000000;
  }
  __syncthreads();
  const double sum = tree_sum<false>(s, n, 0.0, H);
  if (tid == 0) s_mu = __ddiv_rn(__dadd_rn(0.0, sum), (double)n);  // np.mean
  __syncthreads();
  const double mu = s_mu;
  const double sq = tree_sum<true>(s, n, mu, H);
  if (tid == 0) s_sd = __dsqrt_rn(__ddiv_rn(__dadd_rn(0.0, sq), (double)n));  // np.std
  __syncthreads();
  const double sd = s_sd;
  if (tid < 16) {
    float f = __int_as_float(0x7f800000), b32 = f;
    if (tid < m - 1) {
      const double b = __dadd_rn(mu, __dmul_rn(sd, kNdtri[m][tid]));
      f = __double2float_rd(b);   // fit labels compare against b exactly
      b32 = __double2float_rn(b);
    }
    F[tid] = f;
    Q.bnd[tid] = b32;
  }
  __syncthreads();
  // fit labels (#(B64_k < v) == #(F_k < v)) and per-cluster extremes
  for (uint32_t i = tid; i < n; i += kQThreads) {
    const float v = s[padded(i)];
    const uint32_t c = count_below(F, v);
    const int k = fkey(v);
    atomicMin(&cmin[c], k);
    atomicMax(&cmax[c], k);
  }
  __syncthreads();
  if (tid < 16) {
    float scale = 0.0f, offset = 0.0f;
    if (tid < m && cmin[tid] <= cmax[tid]) {
      const float lo = fkey_inv(cmin[tid]), hi = fkey_inv(cmax[tid]);
      scale = __double2float_rn(__dsub_rn((double)hi, (double)lo));
      offset = lo;
    }
    Q.off[tid] = offset;
    Q.scl[tid] = scale;
    float rc = 0.0f;
    if (scale > 0.0f) {
      rc = __fdiv_rn(255.0f, scale);
      if (!isfinite(rc)) rc = __int_as_float(0x7fffffff);
    }
    Q.rcp[tid] = rc;
    if (tid == 0) Q.last = (uint32_t)m - 1;
    tbl->scales[tid] = scale;
    tbl->offsets[tid] = offset;
    if (tid < 15) tbl->boundaries[tid] = tid < m - 1 ? Q.bnd[tid] : 0.0f;
    if (tid < 13) tbl->reserved[tid] = 0;
    if (tid == 0) {
      tbl->mean = __double2float_rn(mu);
      tbl->std = __double2float_rn(sd);
      tbl->m = (uint32_t)m;
      tbl->flags = (isfinite(mu) && isfinite(sd)) ? 0u : BSNP_ERR_NONFINITE;
    }
  }
  __syncthreads();
  // quantize labels (vs the f32 boundaries) and codes, a label byte per pair
  for (uint32_t p = tid; 2 * p < n; p += kQThreads) {
    uint32_t la, lb = 0;
    codes[2 * p] = (uint8_t)quant_one(Q, s[padded(2 * p)], la);
    if (2 * p + 1 < n) codes[2 * p + 1] = (uint8_t)quant_one(Q, s[padded(2 * p + 1)], lb);
    labels[p] = (uint8_t)(la | (lb << 4));
  }
}

// --------------------------------------------------------------- dequantize
// One CTA's chunk [c0, c1) of a unit: LUT from the unit's table, then
// out = lut[label][code]; the unit's largest label goes to st.
__device__ __forceinline__ void dequant_chunk(const uint8_t* __restrict__ ls,
                                              const uint8_t* __restrict__ cs,
                                              float* __restrict__ o, uint64_t c0, uint64_t c1,
                                              const bsnp_cluster_table& tb, bsnp_status* st,
                                              float* lut, uint32_t* s_maxlab) {
  const uint32_t m = tb.m;
  if (threadIdx.x == 0) *s_maxlab = 0;
  for (uint32_t i = threadIdx.x; i < 16 * 256; i += blockDim.x) {
    const uint32_t c = i >> 8, j = i & 255;
    // restored = (qmap(code) * S + b).astype(float32)   (quantizer.py:199-201)
    lut[i] = c < m ? __double2float_rn(__dadd_rn(__dmul_rn(kQmap[j], (double)tb.scales[c]),
                                                 (double)tb.offsets[c]))
                   : 0.0f;
  }
  __syncthreads();
  uint32_t maxlab = 0;
  const bool vec = ((((uintptr_t)(cs + c0)) & 7) | (((uintptr_t)(ls + c0 / 2)) & 3) |
                    (((uintptr_t)(o + c0)) & 15)) == 0;
  uint64_t e = c0;
  if (vec) {
    const uint32_t nv = (uint32_t)((c1 - c0) / 8);
    constexpr int kB = 4;  // 8-element groups per thread with loads in flight
    for (uint32_t i0 = threadIdx.x; i0 < nv; i0 += kB * kQThreads) {
      uint2 cc[kB];
      uint32_t ll[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint32_t i = i0 + b * kQThreads;
        if (i < nv) {
          const uint64_t e0 = c0 + 8ull * i;
          cc[b] = __ldg(reinterpret_cast<const uint2*>(cs + e0));
          ll[b] = __ldg(reinterpret_cast<const uint32_t*>(ls + e0 / 2));
        }
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint32_t i = i0 + b * kQThreads;
        if (i >= nv) break;
        const uint64_t e0 = c0 + 8ull * i;
        float r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t lab = (ll[b] >> (4 * k)) & 15u;
          const uint32_t code = ((k < 4 ? cc[b].x : cc[b].y) >> (8 * (k & 3))) & 255u;
          maxlab = lab > maxlab ? lab : maxlab;
          r[k] = lut[lab * 256 + code];
        }
        *reinterpret_cast<float4*>(o + e0) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<float4*>(o + e0 + 4) = make_float4(r[4], r[5], r[6], r[7]);
      }
    }
    e = c0 + (uint64_t)nv * 8;
  }
  for (uint64_t i = e + threadIdx.x; i < c1; i += blockDim.x) {
    const uint32_t lab = (ls[i / 2] >> (4 * (i & 1))) & 15u;
    maxlab = lab > maxlab ? lab : maxlab;
    o[i] = lut[lab * 256 + cs[i]];
  }
  // the reference raises with the largest label of the tensor (quantizer.py:196-197)
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) maxlab = max(maxlab, __shfl_xor_sync(kFull, maxlab, d));
  if ((threadIdx.x & 31) == 0 && maxlab) atomicMax(s_maxlab, maxlab);
  __syncthreads();
  if (threadIdx.x == 0 && *s_maxlab) {
    atomicMax((unsigned long long*)&st->count, (unsigned long long)*s_maxlab);
    if (*s_maxlab >= m) atomicOr(&st->err_flags, BSNP_ERR_LABEL);
  }
}

// the dequantize status blocks zeroed by a kernel (not a memset node) so the
// dequantize can follow the previous kernel by programmatic dependent launch
__global__ void __launch_bounds__(256)
    dq_zero_status_kernel(bsnp_status* __restrict__ st, uint32_t count) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    st[i] = bsnp_status{0, 0, 0};
}

__global__ void __launch_bounds__(kQThreads)
    dequantize_kernel(const uint8_t* __restrict__ labels, const uint8_t* __restrict__ codes,
                      QPlan P, const bsnp_cluster_table* __restrict__ tables,
                      float* __restrict__ out, bsnp_status* __restrict__ st) {
  pdl_enter();
  __shared__ float lut[16 * 256];
  __shared__ uint32_t s_maxlab;
  // chunk -> (unit, element range)
  const uint64_t cidx = blockIdx.x;
  const uint64_t full_chunks = (uint64_t)(P.nunits - 1) * P.C_full;
  uint32_t u;
  uint64_t c0, len;
  if (cidx < full_chunks) {
    u = (uint32_t)(cidx / P.C_full);
    c0 = (cidx % P.C_full) * kDqChunk;
    len = P.block;
  } else {
    u = P.nunits - 1;
    c0 = (cidx - full_chunks) * kDqChunk;
    len = P.last_len;
  }
  const uint64_t c1 = c0 + kDqChunk < len ? c0 + kDqChunk : len;
  const uint64_t ustart = (uint64_t)u * P.block;
  dequant_chunk(labels + (uint64_t)u * (P.block / 2), codes + ustart, out + ustart, c0, c1,
                tables[u], st, lut, &s_maxlab);
}

// many per-tensor records, one launch: CTA -> (item, chunk) through first[]
__global__ void __launch_bounds__(kQThreads)
    dequantize_batch_kernel(const bsnp_dequant_item* __restrict__ items,
                            const uint32_t* __restrict__ first, uint32_t nitems,
                            bsnp_status* __restrict__ st) {
  pdl_enter();
  __shared__ float lut[16 * 256];
  __shared__ uint32_t s_maxlab, s_item;
  const uint32_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = nitems;  // largest i with first[i] <= b
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (first[mid] <= b) lo = mid;
      else hi = mid;
    }
    s_item = lo;
  }
  __syncthreads();
  const uint32_t i = s_item;
  const bsnp_dequant_item it = items[i];
  const uint64_t c0 = (uint64_t)(b - first[i]) * kDqChunk;
  if (c0 >= it.n) return;
  const uint64_t c1 = c0 + kDqChunk < it.n ? c0 + kDqChunk : it.n;
  dequant_chunk(it.labels, it.codes, it.out, c0, c1, *it.table, st + i, lut, &s_maxlab);
}

// ------------------------------------------------------- precision report
// sum (o-r)^2, sum |o-r|/|o| over |o| > 1e-12, count of such o (float64).
// Deterministic: part p of kPrecParts reduces the contiguous range
// [p n / P, (p + 1) n / P) - each thread a strided subsequence in order, then
// a fixed shuffle / shared-memory tree - and one CTA folds the P partials in
// a fixed tree.  No atomics: the same bits on every run and every GPU.
constexpr int kPrecParts = 1024;

__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sm) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(kFull, a, d);
    b += __shfl_xor_sync(kFull, b, d);
    c += __shfl_xor_sync(kFull, c, d);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    sm[3 * warp] = a;
    sm[3 * warp + 1] = b;
    sm[3 * warp + 2] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = b = c = 0.0;
    for (int w = 0; w < nw; ++w) {
      a += sm[3 * w];
      b += sm[3 * w + 1];
      c += sm[3 * w + 2];
    }
  }
}

__global__ void __launch_bounds__(kQThreads)
    precision_kernel(const float* __restrict__ o, const float* __restrict__ r, uint64_t n,
                     double* __restrict__ parts) {
  __shared__ double sm[3 * kQThreads / 32];
  const uint64_t p = blockIdx.x;
  const uint64_t lo = p * n / kPrecParts, hi = (p + 1) * n / kPrecParts;
  double sse = 0.0, rel = 0.0, cnt = 0.0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double a = (double)o[i], b = (double)r[i];
    const double e = a - b;
    sse += e * e;
    if (fabs(a) > 1e-12) {
      rel += fabs(e) / fabs(a);
      cnt += 1.0;
    }
  }
  block_sum3(sse, rel, cnt, sm);
  if (threadIdx.x == 0) {
    parts[3 * p] = sse;
    parts[3 * p + 1] = rel;
    parts[3 * p + 2] = cnt;
  }
}

__global__ void __launch_bounds__(kQThreads)
    precision_final_kernel(const double* __restrict__ parts, double* __restrict__ acc) {
  __shared__ double sm[3 * kQThreads / 32];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int p = threadIdx.x; p < kPrecParts; p += blockDim.x) {
    a += parts[3 * p];
    b += parts[3 * p + 1];
    c += parts[3 * p + 2];
  }
  block_sum3(a, b, c, sm);
  if (threadIdx.x == 0) {
    acc[0] = a;
    acc[1] = b;
    acc[2] = c;
  }
}

#include "quant_window.cuh"
#include "quant_stats.cuh"

// ---------------------------------------------------------------- host plan
uint32_t tree_depth(uint64_t len) {
  std::vector<uint64_t> sizes{len};
  uint32_t d = 0;
  while (*std::max_element(sizes.begin(), sizes.end()) > kTileMax) {
    std::vector<uint64_t> next;
    for (uint64_t s : sizes) {
      const uint64_t L = 8 * (s / 16);
      next.push_back(L);
      next.push_back(s - L);
    }
    std::sort(next.begin(), next.end());
    next.erase(std::unique(next.begin(), next.end()), next.end());
    sizes.swap(next);
    ++d;
  }
  return d;
}

bool make_plan(uint64_t n, uint64_t block, int m, QPlan& P) {
  if (n == 0) return false;
  if (block != 0 && (block % 8) != 0) return false;
  const uint64_t b = (block == 0 || block >= n) ? n : block;
  P.n = n;
  P.block = b;
  P.nunits = (uint32_t)((n + b - 1) / b);
  P.last_len = n - (uint64_t)(P.nunits - 1) * b;
  P.m = (uint32_t)m;
  P.D_full = tree_depth(b);
  P.T_full = 1u << P.D_full;
  P.D_last = tree_depth(P.last_len);
  P.T_last = 1u << P.D_last;
  P.D_max = P.D_full > P.D_last ? P.D_full : P.D_last;
  P.T_max = 1u << P.D_max;
  P.total_tiles = (uint64_t)(P.nunits - 1) * P.T_full + P.T_last;
  P.C_full = (uint32_t)((b + kDqChunk - 1) / kDqChunk);
  P.C_last = (uint32_t)((P.last_len + kDqChunk - 1) / kDqChunk);
  return true;
}

struct UGrid;
struct QWs {
  double* partials;  // total_tiles
  double* partials2; // nunits * (T_max / kPreGroup): pre-reduced partials (T > kPreGroup)
  double* mu;        // nunits
  float* fthr;       // nunits * 16
  int* tile_mm;      // total_tiles * 32
  double* sd;        // nunits
  UGrid* ug;         // nunits
  uint32_t* need;    // nunits + 1: exact min/max round needed (per unit, any)
  double* partials_q;   // total_tiles: sum (x - c)^2 per tile (quant_stats.cuh)
  double* partials2_q;  // as partials2
  uint32_t* list;       // 1 + nunits: units needing numpy's exact variance tree
  size_t bytes;
};

QWs carve(const QPlan& P, void* ws) {
  QWs w;
  char* p = (char*)ws;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* r = p + o;
    o = align_up(o + bytes, 256);
    return r;
  };
  w.partials = (double*)take(8 * P.total_tiles);
  w.partials2 = (double*)take(8 * (size_t)P.nunits * (P.T_max >> kPreShift) + 8);
  w.mu = (double*)take(8 * (size_t)P.nunits);
  w.fthr = (float*)take(64 * (size_t)P.nunits);
  w.tile_mm = (int*)take(128 * P.total_tiles);
  w.sd = (double*)take(8 * (size_t)P.nunits);
  w.ug = (UGrid*)take(kUGridBytes * (size_t)P.nunits);
  w.need = (uint32_t*)take(4 * ((size_t)P.nunits + 1));
  w.partials_q = (double*)take(8 * P.total_tiles);
  w.partials2_q = (double*)take(8 * (size_t)P.nunits * (P.T_max >> kPreShift) + 8);
  w.list = (uint32_t*)take(4 * ((size_t)P.nunits + 1));
  w.bytes = o;
  return w;
}

// the per-unit combine, pre-reducing groups of kPreGroup partials for units
// with more tiles
template <bool kVar>
int launch_combine(const QPlan& P, bsnp_cluster_table* tables, const QWs& w, cudaStream_t s) {
  int rc;
  const double* p2 = nullptr;
  if (P.T_max > kPreGroup) {
    pre_combine_kernel<<<(unsigned)(P.nunits * (P.T_max >> kPreShift)), kQThreads, 0, s>>>(
        P, w.partials, w.partials2);
    if ((rc = launch_status("pre_combine_kernel"))) return rc;
    p2 = w.partials2;
  }
  fit_combine_kernel<kVar><<<P.nunits, kQThreads, 0, s>>>(P, w.partials, w.mu, w.fthr, tables,
                                                          kVar ? w.sd : nullptr, p2);
  return launch_status(kVar ? "fit_combine_kernel<std>" : "fit_combine_kernel<mean>");
}

int run_fit(const float* x, const QPlan& P, bsnp_cluster_table* tables, const QWs& w,
            cudaStream_t s) {
  int rc;
  const unsigned tiles = (unsigned)P.total_tiles;
  fit_tree_kernel<false><<<tiles, kQThreads, 0, s>>>(x, P, w.mu, w.partials);
  if ((rc = launch_status("fit_tree_kernel<sum>"))) return rc;
  if ((rc = launch_combine<false>(P, tables, w, s))) return rc;
  fit_tree_kernel<true><<<tiles, kQThreads, 0, s>>>(x, P, w.mu, w.partials);
  if ((rc = launch_status("fit_tree_kernel<var>"))) return rc;
  if ((rc = launch_combine<true>(P, tables, w, s))) return rc;
  fit_minmax_kernel<<<tiles, kQThreads, 0, s>>>(x, P, w.fthr, w.tile_mm);
  if ((rc = launch_status("fit_minmax_kernel"))) return rc;
  fit_finalize_kernel<<<P.nunits, kQThreads, 0, s>>>(P, w.tile_mm, tables);
  return launch_status("fit_finalize_kernel");
}

// Encode (labels != nullptr) or fit only: the threshold-window tiled path
// (quant_window.cuh); BSNP_WINDOW=0 selects the four-pass kernels (mean
// tree, variance tree, per-element min/max, quantize) — a second exact
// implementation the tests compare with (read per call so a test can switch)
bool window_enabled() {
  const char* e = getenv("BSNP_WINDOW");
  return !(e && atoi(e) == 0);
}

// BSNP_VAR_EXACT=1: every unit takes numpy's variance tree (tests of the
// fallback path; read per call so a test can switch it)
int var_exact_forced() {
  const char* e = getenv("BSNP_VAR_EXACT");
  return e && atoi(e) != 0;
}

int run_window(const float* x, const QPlan& P, bsnp_cluster_table* tables, uint8_t* labels,
               uint8_t* codes, const QWs& w, cudaStream_t s) {
  int rc;
  const unsigned tiles = (unsigned)P.total_tiles;
  const dim3 T(kQThreads);
  // one read of x for mean and sigma (quant_stats.cuh); numpy's variance
  // tree only for the units whose sigma interval does not decide the tables.
  // The first kernel waits for the stream as usual; the rest follow it by
  // programmatic dependent launch.
  fit_sum_kernel<<<tiles, kQThreads, 0, s>>>(x, P, w.partials, w.partials_q, w.list);
  if ((rc = launch_status("fit_sum_kernel"))) return rc;
  if (P.T_max > kPreGroup &&
      (rc = launch_pdl("pre_combine2_kernel", pre_combine2_kernel,
                       dim3((unsigned)(2 * P.nunits * (P.T_max >> kPreShift))), T, s, P,
                       w.partials, w.partials_q, w.partials2, w.partials2_q)))
    return rc;
  // statistics + the bin grid of every unit the sigma interval decides; the
  // listed units get numpy's variance tree and their grid afterwards
  if ((rc = launch_pdl("fit_stats_kernel", fit_stats_kernel, dim3(P.nunits), T, s, x, P,
                       w.partials, w.partials_q, w.partials2, w.partials2_q, w.mu, w.fthr,
                       tables, w.sd, w.list, var_exact_forced(), w.ug, w.need + P.nunits)))
    return rc;
  const unsigned fb_grid = (unsigned)std::min<uint64_t>(tiles, 2 * (uint64_t)device_sms());
  if ((rc = launch_pdl("fit_var_fallback_kernel", fit_var_fallback_kernel, dim3(fb_grid), T, s,
                       x, P, w.mu, w.list, w.partials)))
    return rc;
  if ((rc = launch_pdl("fit_var_combine_kernel", fit_var_combine_kernel,
                       dim3(std::min(P.nunits, 256u)), T, s, P, w.partials, w.list, w.mu,
                       w.fthr, tables, w.sd, w.ug)))
    return rc;
  const unsigned chunks = (unsigned)((uint64_t)(P.nunits - 1) * P.C_full + P.C_last);
  if ((rc = launch_pdl("fit_label_kernel", fit_label_kernel, dim3(chunks), T, s, x, P, w.ug,
                       labels)))
    return rc;
  if ((rc = launch_pdl("fit_decide_kernel", fit_decide_kernel, dim3(P.nunits), dim3(32), s, P,
                       w.ug, tables, w.need)))
    return rc;
  // exact per-element min/max, only for the units the window left undecided
  if ((rc = launch_pdl("fit_minmax_kernel", fit_minmax_kernel, dim3(std::min(tiles, 4096u)), T,
                       s, x, P, w.fthr, w.tile_mm, w.need)))
    return rc;
  if ((rc = launch_pdl("fit_finalize_kernel", fit_finalize_kernel, dim3(P.nunits), T, s, P,
                       w.tile_mm, tables, w.need)))
    return rc;
  if (!labels) return BSNP_OK;
  return launch_pdl("quantize_codes_kernel", quantize_codes_kernel, dim3(chunks), T, s, x, P,
                    tables, labels, codes);
}

}  // namespace
}  // namespace bsnp

using namespace bsnp;


extern "C" size_t bsnp_cluster_ws_bytes(uint64_t n, uint64_t block) {
  QPlan P;
  if (!make_plan(n ? n : 1, block, 16, P)) return 0;
  return carve(P, nullptr).bytes;
}

static int cluster_run(const float* x, uint64_t n, uint64_t block, int m,
                       bsnp_cluster_table* tables, uint8_t* labels, uint8_t* codes, void* ws,
                       size_t ws_bytes, cudaStream_t s) {
  if (labels && n <= kTileMax && (block == 0 || block >= n) && window_enabled()) {
    tiny_encode_kernel<<<1, kQThreads, 0, s>>>(x, (uint32_t)n, m, tables, labels, codes);
    return launch_status("tiny_encode_kernel");
  }
  QPlan P;
  if (!make_plan(n, block, m, P)) return BSNP_E_INVALID;
  const QWs w = carve(P, ws);
  if (ws_bytes < w.bytes) return BSNP_E_WORKSPACE;
  if (window_enabled()) return run_window(x, P, tables, labels, codes, w, s);
  int rc = run_fit(x, P, tables, w, s);
  if (rc || !labels) return rc;
  quantize_kernel<<<(unsigned)((uint64_t)(P.nunits - 1) * P.C_full + P.C_last), kQThreads, 0,
                    s>>>(x, P, tables, labels, codes);
  return launch_status("quantize_kernel");
}

extern "C" int bsnp_cluster_fit(const float* x, uint64_t n, uint64_t block, int m,
                                bsnp_cluster_table* tables, void* ws, size_t ws_bytes,
                                void* stream) {
  QPlan P;
  if (!x || !tables || !ws || m < 2 || m > 16 || !make_plan(n, block, m, P))
    return BSNP_E_INVALID;
  if (((uintptr_t)x & 3) || ((uintptr_t)tables & 15)) return BSNP_E_ALIGN;
  if (ws_bytes < carve(P, nullptr).bytes) return BSNP_E_WORKSPACE;
  return cluster_run(x, n, block, m, tables, nullptr, nullptr, ws, ws_bytes,
                     (cudaStream_t)stream);
}

extern "C" int bsnp_cluster_quantize(const float* x, uint64_t n, uint64_t block,
                                     const bsnp_cluster_table* tables, uint8_t* labels,
                                     uint8_t* codes, void* ws, size_t ws_bytes, void* stream) {
  QPlan P;
  if (!x || !tables || !labels || !codes || !make_plan(n, block, 16, P)) return BSNP_E_INVALID;
  if (((uintptr_t)x & 3) || ((uintptr_t)tables & 15)) return BSNP_E_ALIGN;
  (void)ws;
  (void)ws_bytes;
  quantize_kernel<<<(unsigned)((uint64_t)(P.nunits - 1) * P.C_full + P.C_last), kQThreads, 0,
                    (cudaStream_t)stream>>>(x, P, tables, labels, codes);
  return launch_status("quantize_kernel");
}

extern "C" int bsnp_cluster_encode(const float* x, uint64_t n, uint64_t block, int m,
                                   bsnp_cluster_table* tables, uint8_t* labels, uint8_t* codes,
                                   void* ws, size_t ws_bytes, void* stream) {
  QPlan P;
  if (!x || !tables || !labels || !codes || !ws || m < 2 || m > 16 || !make_plan(n, block, m, P))
    return BSNP_E_INVALID;
  if (((uintptr_t)x & 3) || ((uintptr_t)tables & 15)) return BSNP_E_ALIGN;
  if (ws_bytes < carve(P, nullptr).bytes) return BSNP_E_WORKSPACE;
  return cluster_run(x, n, block, m, tables, labels, codes, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int bsnp_cluster_dequantize(const uint8_t* labels, const uint8_t* codes, uint64_t n,
                                       uint64_t block, const bsnp_cluster_table* tables,
                                       float* out, bsnp_status* status, void* ws,
                                       size_t ws_bytes, void* stream) {
  QPlan P;
  if (!labels || !codes || !tables || !out || !status || !make_plan(n, block, 16, P))
    return BSNP_E_INVALID;
  if (((uintptr_t)out & 3) || ((uintptr_t)tables & 15)) return BSNP_E_ALIGN;
  (void)ws;
  (void)ws_bytes;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = launch_pdl("dq_zero_status_kernel", dq_zero_status_kernel, dim3(1), dim3(256), s,
                      status, 1u);
  if (rc) return rc;
  const uint64_t chunks = (uint64_t)(P.nunits - 1) * P.C_full + P.C_last;
  return launch_pdl("dequantize_kernel", dequantize_kernel, dim3((unsigned)chunks),
                    dim3(kQThreads), s, labels, codes, P, tables, out, status);
}

extern "C" int bsnp_cluster_dequantize_batch(const bsnp_dequant_item* items,
                                             const uint32_t* first, uint32_t nitems,
                                             uint32_t nchunks, bsnp_status* status,
                                             void* stream) {
  if (nitems == 0) return BSNP_OK;
  if (!items || !first || !status) return BSNP_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = cuda_status("memset(status)",
                       cudaMemsetAsync(status, 0, (size_t)nitems * sizeof(bsnp_status), s));
  if (rc || nchunks == 0) return rc;
  dequantize_batch_kernel<<<nchunks, kQThreads, 0, s>>>(items, first, nitems, status);
  return launch_status("dequantize_batch_kernel");
}

extern "C" size_t bsnp_precision_ws_bytes(void) { return 3 * sizeof(double) * kPrecParts; }

extern "C" int bsnp_precision_report(const float* original, const float* restored, uint64_t n,
                                     double* acc3, void* ws, size_t ws_bytes, void* stream) {
  if (!acc3 || (n && (!original || !restored || !ws))) return BSNP_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0)
    return cuda_status("memset(acc)", cudaMemsetAsync(acc3, 0, 3 * sizeof(double), s));
  if (ws_bytes < bsnp_precision_ws_bytes()) return BSNP_E_WORKSPACE;
  double* parts = (double*)ws;
  precision_kernel<<<kPrecParts, kQThreads, 0, s>>>(original, restored, n, parts);
  int rc = launch_status("precision_kernel");
  if (rc) return rc;
  precision_final_kernel<<<1, kQThreads, 0, s>>>(parts, acc3);
  return launch_status("precision_final_kernel");
}
