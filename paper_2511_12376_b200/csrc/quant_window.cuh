// Tiled cluster encoder, threshold-window variant (included by quant.cu
// inside its anonymous namespace; the default encode path).
//
// The fit's per-cluster min/max pass and the quantize pass of the tiled
// kernels are replaced by:
//
//   grid_unit         (per unit)  bin grid over mu +- 2 sd, a 16384-bin label
//                                 LUT and the threshold window delta (built
//                                 by fit_stats_kernel, quant_stats.cuh, or
//                                 after the exact variance tree)
//   fit_label_kernel  (per tile)  quantize labels (written out: they are the
//                                 final label stream) + unit extremes +
//                                 candidates within delta of the fit
//                                 thresholds F_k next to each element's label
//   fit_decide_kernel (per unit)  scales / offsets when every F_k has a
//                                 candidate on both sides; else the unit is
//                                 marked for the exact min/max round
//   quantize_codes_kernel (tile)  codes from x and the written labels
//
// Why the candidates are exact: with fit thresholds F_k = RD_f32(B64_k), the
// minimum of cluster c > 0 is succ(F_{c-1}) = the smallest element > F_{c-1},
// the maximum of cluster c < m-1 is pred(F_c) = the largest element <= F_c,
// and cluster 0's minimum / cluster m-1's maximum are the unit's extremes.
// An element v with quantize label c (B32_{c-1} < v <= B32_c, B32 = RN(B64))
// is a candidate for F_{c-1} and F_c when |v - F| < delta.  If a candidate
// lo <= F_k exists, every element in (lo, F_k] has label k and lies within
// delta, so it is a candidate too: lo is pred(F_k).  Likewise for succ
// (elements in (F_k, hi) have label k+1, or equal B32_k > F_k with label k).
// delta = 160 sd / n: for dense data pred/succ are ~sd/(n pdf) away (<= 8.3
// sd / n for every threshold of m <= 16 on Gaussian data), so a missing side
// only costs the exact round of that unit; one-sided heavy-tailed data
// (Adam-v) has thresholds in thinner tails, where 160 instead of 80 sd / n
// halves the units sent to the exact round (C2 Adam-v: 2.57 -> 2.48 ms).
// LUT byte: bits 0-3 L = #quantize boundaries in lower bins; bit 7: boundary L
// lies in this bin (label = L + (v > B32[L])); bit 6: kLutN below.
constexpr uint32_t kLutB = 0x80u;

// order-preserving float -> u32 (0 is below every non-NaN key)
__device__ __forceinline__ uint32_t ukey(float f) {
  const uint32_t b = __float_as_uint(f);
  return b ^ (uint32_t)(((int)b >> 31) | (int)0x80000000);
}
__device__ __forceinline__ float ukey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// ceil to u8 with saturation (the reference's clip(ceil(..), 0, 255))
__device__ __forceinline__ uint32_t ceil_u8(float t) {
  uint32_t r;
  asm("cvt.rpi.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(t));
  return r;
}

#ifndef BSNP_WDELTA
#define BSNP_WDELTA 160
#endif
constexpr uint32_t kWDeltaNum = BSNP_WDELTA;
constexpr int kWBins = 16384;           // label LUT bins over mu +- 2 sd
constexpr uint32_t kLutN = 0x40u;       // LUT bit: the bin meets some [F_k - delta, F_k + delta]

__device__ __forceinline__ uint32_t w_bin(float v, float gi, float c0) {
  return min(__float2uint_rd(__fmaf_rn(v, gi, c0)), (uint32_t)kWBins - 1);
}

struct UGrid {
  float c0, gi, delta;
  uint32_t mode;          // bit 0: exact round (grid unusable); bit 1: labels by comparisons
  uint32_t gmax, gmin_c;  // unit extremes: max ukey, ~(min ukey)
  uint32_t pad[2];
  float F[16];            // fit thresholds RD_f32(B64), +inf padded
  float B32[16];          // quantize boundaries RN_f32(B64), +inf padded
  uint32_t lo[16];        // max ukey of candidates <= F_k; 0 = none
  uint32_t hi_c[16];      // ~(min ukey of candidates > F_k); 0 = none
  uint8_t lut[kWBins];
};
constexpr size_t kUGridBytes = sizeof(UGrid);
static_assert(sizeof(UGrid) % 16 == 0, "UGrid alignment");

struct GridSmem {
  __align__(16) uint8_t lut[kWBins];
  int binB[16], nlo[16], nhi[16];
  float s_gi, s_c0, s_delta;
  uint32_t s_mode;
};

// CTA-wide: the bin grid, label LUT and threshold window of unit u
__device__ __forceinline__ void grid_unit(const QPlan& P, uint32_t u, double m0, double sd,
                                          UGrid* ug, GridSmem& g) {
  uint8_t* lut = g.lut;
  int *binB = g.binB, *nlo = g.nlo, *nhi = g.nhi;
  float &s_gi = g.s_gi, &s_c0 = g.s_c0, &s_delta = g.s_delta;
  uint32_t& s_mode = g.s_mode;
  const int tid = threadIdx.x, m = (int)P.m;
  UGrid& G = ug[u];
  uint32_t T;
  uint64_t len;
  unit_shape(P, u, T, len);
  if (tid == 0) {
    const float r0 = __double2float_rn(__dsub_rn(m0, __dmul_rn(2.0, sd)));
    const float wd = __double2float_rn(__dmul_rn(4.0, sd));
    const float gi = __fdiv_rn((float)kWBins, wd);
    const float c0 = -__fmul_rn(r0, gi);
    const bool ok = isfinite(r0) && isfinite(gi) && gi > 0.0f && isfinite(c0) &&
                    isfinite(m0) && isfinite(sd);
    s_gi = gi;
    s_c0 = c0;
    s_mode = ok ? 0u : 3u;
    G.gi = gi;
    G.c0 = c0;
    s_delta = __double2float_ru(__ddiv_rn(__dmul_rn((double)kWDeltaNum, sd), (double)len));
    G.gmax = 0;
    G.gmin_c = 0;
  }
  __syncthreads();
  float f = __int_as_float(0x7f800000), r = f;
  if (tid < 16) {
    if (tid < m - 1) {
      const double b64 = __dadd_rn(m0, __dmul_rn(sd, kNdtri[m][tid]));
      f = __double2float_rd(b64);
      r = __double2float_rn(b64);
      // a window narrower than a few f32 spacings at F would miss pred/succ
      // of large units (2^30 elements: 160 sd / n is below one ulp of F)
      const float af = fabsf(f);
      if (isfinite(af)) atomicMax(reinterpret_cast<int*>(&s_delta),
                                  __float_as_int(4.0f * (nextafterf(af, INFINITY) - af)));
    }
    G.F[tid] = f;
    G.B32[tid] = r;
    G.lo[tid] = 0;
    G.hi_c[tid] = 0;
  }
  __syncthreads();
  if (tid == 0) G.delta = s_delta;
  if (tid < 16) {
    binB[tid] = tid < m - 1 ? (int)w_bin(r, s_gi, s_c0) : 0x3fffffff;
    // bins meeting the window around F_k (monotone bins: |v - F| < delta
    // implies bin(F - delta) <= bin(v) <= bin(F + delta))
    nlo[tid] = tid < m - 1 ? (int)w_bin(__fsub_rd(f, s_delta), s_gi, s_c0) : 0x3fffffff;
    nhi[tid] = tid < m - 1 ? (int)w_bin(__fadd_ru(f, s_delta), s_gi, s_c0) : -1;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t mode = s_mode;
    for (int k = 1; k < m - 1; ++k)
      if (binB[k] == binB[k - 1]) mode |= 2u;  // two boundaries in one bin
    s_mode = mode;
    G.mode = mode;
  }
  // thread t: bins [64t, 64t + 64): L = #boundaries in lower bins, kLutB
  constexpr int kPer = kWBins / kQThreads;
  const int b0 = kPer * tid;
  int cnt = 0;
  for (int k = 0; k < m - 1; ++k) cnt += binB[k] < b0;
  for (int q = 0; q < kPer; q += 4) {
    uint32_t w = 0;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int bb = b0 + q + qq;
      while (cnt < m - 1 && binB[cnt] < bb) ++cnt;
      uint32_t e = (uint32_t)cnt;
      if (cnt < m - 1 && binB[cnt] == bb) e |= kLutB;
      w |= e << (8 * qq);
    }
    *reinterpret_cast<uint32_t*>(&lut[b0 + q]) = w;
  }
  __syncthreads();
  // threshold windows (disjoint for any usable grid; overlaps only set a bit
  // twice)
  for (int k = 0; k < m - 1; ++k)
    for (int bb = nlo[k] + tid; bb <= nhi[k]; bb += kQThreads) lut[bb] |= (uint8_t)kLutN;
  __syncthreads();
  for (int i = tid; i < kWBins / 16; i += kQThreads)
    reinterpret_cast<uint4*>(G.lut)[i] = reinterpret_cast<const uint4*>(lut)[i];
}

// elementwise passes run over kDqChunk-element chunks of each unit (the
// dequantize partition), not the pairwise-tree tiles
struct ChunkRef {
  uint32_t u;
  uint64_t c0, len, ustart;
};
__device__ __forceinline__ ChunkRef chunk_of(const QPlan& P, uint64_t cidx) {
  ChunkRef r;
  const uint64_t full_chunks = (uint64_t)(P.nunits - 1) * P.C_full;
  uint64_t ulen;
  if (cidx < full_chunks) {
    r.u = (uint32_t)(cidx / P.C_full);
    r.c0 = (cidx % P.C_full) * kDqChunk;
    ulen = P.block;
  } else {
    r.u = P.nunits - 1;
    r.c0 = (cidx - full_chunks) * kDqChunk;
    ulen = P.last_len;
  }
  r.len = (r.c0 + kDqChunk < ulen ? r.c0 + kDqChunk : ulen) - r.c0;
  r.ustart = (uint64_t)r.u * P.block;
  return r;
}

struct WSmem {
  __align__(16) uint8_t lut[kWBins];
  float F[16], B32[16];
  float2 FF[16];  // (F[c-1], F[c]) around quantize cluster c
  uint32_t lo[16], hi_c[16];
  float wmin[kQThreads / 32], wmax[kQThreads / 32];
  float gi, c0, delta;
  uint32_t mode;
};

__device__ __forceinline__ uint32_t w_label(const WSmem& S, float v, bool cmp) {
  if (cmp) return count_below(S.B32, v);
  const uint32_t le = S.lut[w_bin(v, S.gi, S.c0)];
  const uint32_t L = le & 15u;
  return L + ((le >> 7) & (v > S.B32[L] ? 1u : 0u));
}

// label + "maybe within delta of a fit threshold" from one LUT byte
template <bool kCmp>
__device__ __forceinline__ uint32_t w_label_n(const WSmem& S, float v, uint32_t& near) {
  const uint32_t le = S.lut[w_bin(v, S.gi, S.c0)];
  near |= le;
  if (kCmp) return count_below(S.B32, v);
  const uint32_t L = le & 15u;
  return L + ((le >> 7) & (v > S.B32[L] ? 1u : 0u));
}

__device__ __forceinline__ bool w_near(const WSmem& S, float v, uint32_t c) {
  const float2 ff = S.FF[c];
  return fminf(__fsub_rn(v, ff.x), __fsub_rn(ff.y, v)) < S.delta;
}

__device__ __forceinline__ void w_candidates(WSmem& S, float v, uint32_t c, int m) {
  const uint32_t key = ukey(v);
  for (int d = 0; d < 2; ++d) {
    const int k = (int)c - 1 + d;
    if (k < 0 || k >= m - 1) continue;
    const float f = S.F[k];
    if (!(fabsf(__fsub_rn(v, f)) < S.delta)) continue;
    const bool below = v <= f;
    atomicMax(below ? &S.lo[k] : &S.hi_c[k], below ? key : ~key);
  }
}

// labels of 4 consecutive elements (nibbles of the returned u16) + their
// threshold-window candidates and extremes.  LUT path: the 4 LUT bytes are
// merged into one word (label in the low nibble, flags in bits 6-7 of each
// byte), so the common case is one test and a nibble pack.
template <bool kCmp>
__device__ __forceinline__ uint32_t w_label4(WSmem& S, const float (&v)[4], float gi, float c0,
                                             int m, float& vmin, float& vmax) {
  vmin = fmin3(vmin, fminf(v[0], v[1]), fminf(v[2], v[3]));
  vmax = fmax3(vmax, fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
  if (kCmp) {  // two quantize boundaries share a bin: binary search
    uint32_t c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      c[q] = count_below(S.B32, v[q]);
      if ((S.lut[w_bin(v[q], gi, c0)] & kLutN) && w_near(S, v[q], c[q]))
        w_candidates(S, v[q], c[q], m);
    }
    return c[0] | (c[1] << 4) | (c[2] << 8) | (c[3] << 12);
  }
  const uint32_t e0 = S.lut[w_bin(v[0], gi, c0)], e1 = S.lut[w_bin(v[1], gi, c0)];
  const uint32_t e2 = S.lut[w_bin(v[2], gi, c0)], e3 = S.lut[w_bin(v[3], gi, c0)];
  uint32_t le = __byte_perm(__byte_perm(e0, e1, 0x0040), __byte_perm(e2, e3, 0x0040), 0x5410);
  uint32_t spec = le & 0xc0c0c0c0u;
  if (__builtin_expect(spec != 0, 0)) {
    // rare (~0.3 % of elements): a quantize boundary inside the bin, or a
    // fit threshold near; each lane walks only its own flagged bytes
    do {
      const int q = (__ffs(spec) - 1) >> 3;
      spec &= ~(0xffu << (8 * q));
      const uint32_t leq = (le >> (8 * q)) & 0xffu;
      const float vq = q == 0 ? v[0] : q == 1 ? v[1] : q == 2 ? v[2] : v[3];
      uint32_t cq = leq & 15u;
      if ((leq & kLutB) && vq > S.B32[cq]) {
        ++cq;
        le += 1u << (8 * q);  // the label nibble stays below 16 (cq < m - 1)
      }
      if ((leq & kLutN) && w_near(S, vq, cq)) w_candidates(S, vq, cq, m);
    } while (spec);
  }
  // nibble-pack the 4 labels: c0 | c1 << 4 | c2 << 8 | c3 << 12
  uint32_t x = le & 0x0f0f0f0fu;
  x = (x | (x >> 4)) & 0x00ff00ffu;
  return (x | (x >> 8)) & 0xffffu;
}

template <bool kCmp>
__device__ __forceinline__ void w_label_loop(WSmem& S, const float* src, uint32_t size,
                                             uint8_t* lab, int m, float& vmin, float& vmax,
                                             uint64_t pol) {
  const int tid = threadIdx.x;
  const bool vec = ((((uintptr_t)src) & 15) | (((uintptr_t)lab) & 1)) == 0;
  const uint32_t nv = vec ? size / 4 : 0;
  const float gi = S.gi, c0 = S.c0;
  constexpr int kB = 4;  // vectors per thread in flight
  for (uint32_t i0 = tid; i0 < nv; i0 += kB * kQThreads) {
    float4 v4[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint32_t i = i0 + b * kQThreads;
      if (i < nv) v4[b] = ld_hint_f4(src + 4 * i, pol);
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint32_t i = i0 + b * kQThreads;
      if (i >= nv) break;
      const float v[4] = {v4[b].x, v4[b].y, v4[b].z, v4[b].w};
      const uint32_t w = w_label4<kCmp>(S, v, gi, c0, m, vmin, vmax);
      if (lab) *reinterpret_cast<uint16_t*>(lab + 2 * i) = (uint16_t)w;
    }
  }
  // tail (and unaligned tiles): element pairs (one label byte each)
  for (uint32_t p = 2 * nv + tid; 2 * p < size; p += kQThreads) {
    uint32_t byte = 0;
    for (uint32_t q = 0; q < 2 && 2 * p + q < size; ++q) {
      const float v = src[2 * p + q];
      const uint32_t c = w_label(S, v, kCmp);
      vmin = fminf(vmin, v);
      vmax = fmaxf(vmax, v);
      if (w_near(S, v, c)) w_candidates(S, v, c, m);
      byte |= c << (4 * q);
    }
    if (lab) lab[p] = (uint8_t)byte;
  }
}

// CTA-wide: labels + threshold-window candidates + extremes of one chunk
// (the unit's grid is read with L2 loads: it may come from another CTA of the
// same launch in the pipelined encoder)
__device__ __forceinline__ void label_chunk(const float* __restrict__ x, const QPlan& P,
                                            const ChunkRef& r, UGrid* ug, uint8_t* labels,
                                            WSmem& S, uint64_t pol) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, m = (int)P.m;
  UGrid& G = ug[r.u];
  for (int i = tid; i < kWBins / 16; i += kQThreads)
    reinterpret_cast<uint4*>(S.lut)[i] = __ldcg(reinterpret_cast<const uint4*>(G.lut) + i);
  if (tid < 16) {
    const float f = __ldcg(G.F + tid);
    S.F[tid] = f;
    S.B32[tid] = __ldcg(G.B32 + tid);
    S.FF[tid] = make_float2(tid > 0 ? __ldcg(G.F + tid - 1) : __int_as_float(0xff800000), f);
    S.lo[tid] = 0;
    S.hi_c[tid] = 0;
  }
  if (tid == 0) {
    S.gi = __ldcg(&G.gi);
    S.c0 = __ldcg(&G.c0);
    S.delta = __ldcg(&G.delta);
    S.mode = __ldcg(&G.mode);
  }
  __syncthreads();
  const float* src = x + r.ustart + r.c0;
  uint8_t* lab = labels ? labels + (uint64_t)r.u * (P.block / 2) + r.c0 / 2 : nullptr;
  float vmin = __int_as_float(0x7f800000), vmax = __int_as_float(0xff800000);
  if (S.mode & 2u) w_label_loop<true>(S, src, (uint32_t)r.len, lab, m, vmin, vmax, pol);
  else w_label_loop<false>(S, src, (uint32_t)r.len, lab, m, vmin, vmax, pol);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    vmin = fminf(vmin, __shfl_xor_sync(kFull, vmin, d));
    vmax = fmaxf(vmax, __shfl_xor_sync(kFull, vmax, d));
  }
  if (lane == 0) {
    S.wmin[warp] = vmin;
    S.wmax[warp] = vmax;
  }
  __syncthreads();
  if (tid < m - 1) {
    if (S.lo[tid]) atomicMax(&G.lo[tid], S.lo[tid]);
    if (S.hi_c[tid]) atomicMax(&G.hi_c[tid], S.hi_c[tid]);
  }
  if (tid == 0) {
    float a = S.wmin[0], b = S.wmax[0];
    for (int w = 1; w < kQThreads / 32; ++w) {
      a = fminf(a, S.wmin[w]);
      b = fmaxf(b, S.wmax[w]);
    }
    atomicMax(&G.gmax, ukey(b));
    atomicMax(&G.gmin_c, ~ukey(a));
  }
}

__global__ void __launch_bounds__(kQThreads)
    fit_label_kernel(const float* __restrict__ x, QPlan P, UGrid* __restrict__ ug,
                     uint8_t* __restrict__ labels) {
  pdl_enter();
  __shared__ __align__(16) WSmem S;
  label_chunk(x, P, chunk_of(P, blockIdx.x), ug, labels, S, policy_evict_normal());
}

// one warp per unit: extremes from the candidates, or mark the exact round;
// returns ok (warp-uniform).
//
// Per fit threshold F_k (lane k): pred = the largest element <= F_k, succ =
// the smallest element > F_k (ukeys, 0 = none).  With the unit extremes
// gmin / gmax known exactly: F_k < gmin has no pred and succ = gmin; F_k >=
// gmax has pred = gmax and no succ (thresholds outside the data, e.g. the
// lower tail of a one-sided Adam v); otherwise both exist and the window
// candidates must hold them (else the exact round).  Cluster c then has min =
// succ(F_{c-1}) (gmin for c = 0) and max = pred(F_c) (gmax for c = m-1), and
// is empty (scale = offset = 0, quantizer.py:117-125) when those fall outside
// (F_{c-1}, F_c].  A constant unit (gmin == gmax) is decided directly.
__device__ __forceinline__ bool decide_unit(const QPlan& P, uint32_t u, const UGrid* ug,
                                            bsnp_cluster_table* tables, uint32_t* need) {
  const int lane = threadIdx.x & 31, m = (int)P.m;
  const UGrid& G = ug[u];
  bsnp_cluster_table& tb = tables[u];
  const uint32_t kgmin = ~__ldcg(&G.gmin_c), kgmax = __ldcg(&G.gmax);
  const float gmin = ukey_inv(kgmin), gmax = ukey_inv(kgmax);
  const bool finite = kgmax != 0 && isfinite(gmin) && isfinite(gmax);
  bool ok = finite && (!(__ldcg(&G.mode) & 1u) || kgmin == kgmax);
  const float inf = __int_as_float(0x7f800000);
  const float f = lane < m - 1 ? __ldcg(G.F + lane) : inf;
  uint32_t pk = 0, sk = 0;
  if (lane < m - 1) {
    if (f < gmin) {
      sk = kgmin;
    } else if (f >= gmax) {
      pk = kgmax;
    } else {
      pk = __ldcg(G.lo + lane);
      const uint32_t hc = __ldcg(G.hi_c + lane);
      sk = hc ? ~hc : 0u;
      ok = ok && pk != 0 && sk != 0;
    }
  }
  ok = __all_sync(kFull, ok);
  const uint32_t sk_prev = __shfl_up_sync(kFull, sk, 1);
  const float f_prev = __shfl_up_sync(kFull, f, 1);
  if (lane == 0) {
    need[u] = ok ? 0u : 1u;
    if (!ok) atomicOr(need + P.nunits, 1u);  // need[nunits]: any unit
  }
  if (!ok || lane >= 16) return ok;
  const int c = lane;
  float scale = 0.0f, offset = 0.0f;
  if (c < m) {
    const float lo_f = c == 0 ? -inf : f_prev;  // cluster c is (lo_f, hi_f]
    const float hi_f = c == m - 1 ? inf : f;
    const uint32_t kmin = c == 0 ? kgmin : sk_prev;
    const uint32_t kmax = c == m - 1 ? kgmax : pk;
    if (kmin && kmax) {
      const float a = ukey_inv(kmin), b = ukey_inv(kmax);
      if (a <= hi_f && b > lo_f) {
        scale = __double2float_rn(__dsub_rn((double)b, (double)a));
        offset = a;
      }
    }
  }
  tb.scales[c] = scale;
  tb.offsets[c] = offset;
  return ok;
}

__global__ void __launch_bounds__(32)
    fit_decide_kernel(QPlan P, const UGrid* __restrict__ ug,
                      bsnp_cluster_table* __restrict__ tables, uint32_t* __restrict__ need) {
  pdl_enter();
  decide_unit(P, blockIdx.x, ug, tables, need);
}

// codes of one chunk from x and its written labels (quantizer.py:174-182).
// Labels are only read here: a NaN element keeps the label of stage C (its
// unit is non-finite and the host raises QuantizerError).
struct CodesSmem {
  float2 qp[16];
  float qs[16];
};

// CTA-wide: codes of one chunk (tables and labels read with L2 loads, see
// label_chunk)
__device__ __forceinline__ void codes_chunk(const float* __restrict__ x, const QPlan& P,
                                            const ChunkRef& r, const bsnp_cluster_table* tables,
                                            const uint8_t* labels, uint8_t* codes,
                                            CodesSmem& cs, uint64_t pol) {
  float2* qp = cs.qp;
  float* qs = cs.qs;
  const int tid = threadIdx.x;
  const bsnp_cluster_table& tb = tables[r.u];
  bool finite_rc = true;
  if (tid < 16) {
    const float S_ = __ldcg(tb.scales + tid);
    float rc = 0.0f;
    if (S_ > 0.0f) {
      rc = __fdiv_rn(255.0f, S_);
      if (!isfinite(rc)) {
        rc = __int_as_float(0x7fffffff);
        finite_rc = false;
      }
    }
    qp[tid] = make_float2(__ldcg(tb.offsets + tid), rc);
    qs[tid] = S_;
  }
  // every 255/S finite (all but subnormal-width clusters): the fixed-point
  // fast path below
  const bool fast = __syncthreads_and(finite_rc) != 0;
  const float* src = x + r.ustart + r.c0;
  uint8_t* cdst = codes + r.ustart + r.c0;
  const uint8_t* lab = labels + (uint64_t)r.u * (P.block / 2) + r.c0 / 2;
  const uint32_t size = (uint32_t)r.len;
  const bool vec = ((((uintptr_t)src) & 15) | (((uintptr_t)cdst) & 3) | (((uintptr_t)lab) & 1)) == 0;
  const uint32_t nv = vec ? size / 4 : 0;
  constexpr int kB = 4;  // vectors per thread in flight
  if (fast) {
    // T = RN(RN(v - b) * rc + 3071.5) lies within 1.53e-4 of
    // 255 (v - b) / S + 3071.5 (relative error of d * rc <= 2^-23 + 2^-48 on
    // |z| <= 257, plus half an ulp, 2^-13, of T in [2^11, 2^12)); once T is
    // clamped to [3071 + 2^-12, 3327 - 2^-12], (bits(T) - bits(3071) >> 12)
    // is the code ceil(255 x - 0.5) clipped to [0, 255] unless T is an
    // integer (its 12 fraction bits are 0: within 1.53e-4 < 2^-12 of a code
    // boundary), when the reference's float64 expression decides.  The
    // reference's own float64 roundings are ~1e-13 from the exact value, far
    // inside the 2^-12 - 1.53e-4 margin.  NaN T (a NaN element) clamps to
    // code 0 as exact_code does.
    constexpr float kK = 3071.5f, kLo = 3071.000244140625f, kHi = 3326.999755859375f;
    constexpr uint32_t kBase = 0x453FF000u;  // bits(3071.0f)
    for (uint32_t i0 = tid; i0 < nv; i0 += kB * kQThreads) {
      float4 v4[kB];
      uint32_t lw[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint32_t i = i0 + b * kQThreads;
        if (i < nv) {
          v4[b] = ld_hint_f4(src + 4 * i, pol);
          lw[b] = __ldcg(reinterpret_cast<const unsigned short*>(lab) + i);
        }
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint32_t i = i0 + b * kQThreads;
        if (i >= nv) break;
        const float v[4] = {v4[b].x, v4[b].y, v4[b].z, v4[b].w};
        uint32_t c[4], fmin = 0xfffu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 bp = qp[(lw[b] >> (4 * q)) & 15u];
          const float t = __fmaf_rn(__fsub_rn(v[q], bp.x), bp.y, kK);
          const uint32_t u = __float_as_uint(fminf(fmaxf(t, kLo), kHi));
          c[q] = (u - kBase) >> 12;
          fmin = min(fmin, u & 0xfffu);
        }
        if (__builtin_expect(fmin == 0, 0)) {
          // some T is an integer: those elements take the exact path
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t k = (lw[b] >> (4 * q)) & 15u;
            const float t = __fmaf_rn(__fsub_rn(v[q], qp[k].x), qp[k].y, kK);
            if ((__float_as_uint(fminf(fmaxf(t, kLo), kHi)) & 0xfffu) == 0)
              c[q] = exact_code(v[q], qp[k].x, qs[k]);
          }
        }
        *reinterpret_cast<uint32_t*>(cdst + 4 * i) =
            __byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410);
      }
    }
  }
  for (uint32_t i0 = tid; !fast && i0 < nv; i0 += kB * kQThreads) {
    float4 v4[kB];
    uint32_t lw[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint32_t i = i0 + b * kQThreads;
      if (i < nv) {
        v4[b] = ld_hint_f4(src + 4 * i, pol);
        lw[b] = __ldcg(reinterpret_cast<const unsigned short*>(lab) + i);
      }
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint32_t i = i0 + b * kQThreads;
      if (i >= nv) break;
      const float v[4] = {v4[b].x, v4[b].y, v4[b].z, v4[b].w};
      uint32_t code[4];
      bool amb = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 bp = qp[(lw[b] >> (4 * q)) & 15u];
        // within 6.2e-5 of 255(v-b)/S - 0.5: exact unless flagged ambiguous;
        // the saturation is the reference's clip (labels vs RN boundaries can
        // put v just outside the [b, b+S] of the fit's RD thresholds)
        const float tt = __fsub_rn(__fmul_rn(__fsub_rn(v[q], bp.x), bp.y), 0.5f);
        amb |= !(fabsf(__fsub_rn(tt, rintf(tt))) > 0.000244140625f);  // also NaN
        code[q] = ceil_u8(tt);
      }
      if (__builtin_expect(amb, 0)) {
        for (int q = 0; q < 4; ++q) {
          const uint32_t c = (lw[b] >> (4 * q)) & 15u;
          bool a1 = false;
          code_estimate(v[q], qp[c].x, qp[c].y, a1);
          if (a1) code[q] = exact_code(v[q], qp[c].x, qs[c]);
        }
      }
      *reinterpret_cast<uint32_t*>(cdst + 4 * i) =
          code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
    }
  }
  for (uint32_t p = 2 * nv + tid; 2 * p < size; p += kQThreads) {
    const uint32_t byte = __ldcg(lab + p);
    for (uint32_t q = 0; q < 2 && 2 * p + q < size; ++q) {
      const float v = src[2 * p + q];
      const uint32_t c = (byte >> (4 * q)) & 15u;
      bool a1 = false;
      uint32_t code = code_estimate(v, qp[c].x, qp[c].y, a1);
      if (a1) code = exact_code(v, qp[c].x, qs[c]);
      cdst[2 * p + q] = (uint8_t)code;
    }
  }
}

__global__ void __launch_bounds__(kQThreads)
    quantize_codes_kernel(const float* __restrict__ x, QPlan P,
                          const bsnp_cluster_table* __restrict__ tables,
                          const uint8_t* __restrict__ labels, uint8_t* __restrict__ codes) {
  pdl_enter();
  __shared__ CodesSmem cs;
  const uint64_t nch = (uint64_t)(P.nunits - 1) * P.C_full + P.C_last;
  codes_chunk(x, P, chunk_of(P, nch - 1 - blockIdx.x), tables, labels, codes, cs,
              policy_evict_first());
}
