// Fit statistics in ONE read of x (included by quant.cu inside its anonymous
// namespace; the default encode path).
//
// numpy's std (quantizer.py:113) is a second pairwise sum, of (x - mean)^2,
// and mean is only known once the first sum is complete: read literally, the
// fit reads x twice before the labels.  But sigma only ever reaches the
// outputs through float32 roundings — table.std = f32(sigma), the quantize
// boundaries B32_k = RN_f32(mu + sigma z_k) and the fit thresholds F_k =
// RD_f32(mu + sigma z_k) (quantizer.py:113-135) — and every one of them is a
// monotone function of sigma.  So:
//
//   fit_sum_kernel     per tree tile: numpy's exact pairwise sum of x (as
//                      before) AND D2 = sum (x - c)^2 in float64, c = the
//                      unit's first element (any summation order);
//   fit_stats_kernel   per unit: the exact mean mu from the pairwise tree;
//                      a rigorous interval [T_lo, T_hi] for numpy's pairwise
//                      sum of fl(fl(x - mu)^2) from D2 (directed rounding,
//                      error bounds of both summations below), hence
//                      [sigma_lo, sigma_hi]; if every f32 output is the same
//                      at both ends it is the same for numpy's sigma, and the
//                      unit's header is written from sigma_lo;
//   otherwise (probability ~1e-5 per unit) the unit goes on a list, and
//   fit_var_fallback_kernel + fit_var_combine_kernel compute numpy's exact
//   variance tree for the listed units only (x read again for those units).
//
// Bounds (u = 2^-53): our D2 is a sum of at most 44 sequential / shuffle /
// warp steps inside a tile and a perfect tree of <= 2^17 tile partials, each
// term (x - c)^2 rounded twice: |D2~ - D2| <= 128 u D2~.  numpy's pairwise
// sum has depth <= 26 inside a 128-element leaf plus <= 23 levels above it,
// each term fl(fl(x - mu)^2) within 3u: |T_np - T| <= 64 u T, and the same
// tree gives |S_np - S| <= 64 u sum|x|, sum|x| <= sqrt(n D2) + n|c|.  With
// m* = S / n (exact mean): T = D2 - n (m* - c)^2 + n (m* - mu)^2.

constexpr double kU = 1.1102230246251565e-16;  // 2^-53

// per-tile: exact pairwise sum of x (thread 0's return) and D2 (in *q)
__device__ __forceinline__ double sum_tile_q(const float* __restrict__ x, const QPlan& P,
                                             uint64_t tile, float* s, Heap& H, double* sw,
                                             double& q_out, uint64_t pol) {
  const TileRef r = locate(P, tile);
  const float* src = x + r.ustart + r.off;
  const double c = (double)__ldg(x + r.ustart);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double q = 0.0;
  double v = 0.0;
  if (r.size == kTileMax && ((uintptr_t)src & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t vv = i * kQThreads + tid;
      *reinterpret_cast<float4*>(&s[epad(4 * vv)]) = ld_hint_f4(src + 4 * vv, pol);
    }
    __syncthreads();
    const int j = lane & 7, qq = lane >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int leaf = warp + 8 * qq + 32 * h;
      const float* lp = s + 128 * leaf + 8 * (leaf >> 3) + j;
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = lp[8 * i];
      double acc = (double)a[0];
#pragma unroll
      for (int i = 1; i < 16; ++i) acc = __dadd_rn(acc, (double)a[i]);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double d = __dsub_rn((double)a[i], c);
        q = __fma_rn(d, d, q);
      }
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 1));
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 2));
      acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, 4));
      if (j == 0) H.val[leaf] = acc;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) q = __dadd_rn(q, __shfl_xor_sync(kFull, q, d));
    if (lane == 0) sw[warp] = q;
    __syncthreads();
    if (warp == 0) {
      v = __dadd_rn(H.val[2 * lane], H.val[2 * lane + 1]);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, d));
    }
  } else {
    load_tile(s, src, (uint32_t)r.size, pol);
    __syncthreads();
    for (uint32_t i = tid; i < r.size; i += kQThreads) {
      const double d = __dsub_rn((double)s[padded(i)], c);
      q = __fma_rn(d, d, q);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) q = __dadd_rn(q, __shfl_xor_sync(kFull, q, d));
    if (lane == 0) sw[warp] = q;
    v = tree_sum<false>(s, (uint32_t)r.size, 0.0, H);  // syncs: sw[] visible after
  }
  double qt = 0.0;
  if (tid == 0)
    for (int w = 0; w < kQThreads / 32; ++w) qt = __dadd_rn(qt, sw[w]);
  q_out = qt;
  return v;
}

// ws.list: [0] = count of units needing numpy's exact variance, then the units
__global__ void __launch_bounds__(kQThreads)
    fit_sum_kernel(const float* __restrict__ x, QPlan P, double* __restrict__ partials,
                   double* __restrict__ partials_q, uint32_t* __restrict__ list) {
  pdl_enter();
  __shared__ __align__(16) float s[kSmemFloats];
  __shared__ Heap H;
  __shared__ double sw[kQThreads / 32];
  const uint64_t tile = blockIdx.x;
  if (tile == 0 && threadIdx.x == 0) list[0] = 0;
  double q;
  const double v = sum_tile_q(x, P, tile, s, H, sw, q, policy_evict_normal());
  if (threadIdx.x == 0) {
    partials[tile] = v;
    partials_q[tile] = q;
  }
}

// groups of kPreGroup partials of units above kPreGroup tiles: the sum as a
// perfect tree (numpy's), D2 in the same tree (any order would do)
__global__ void __launch_bounds__(kQThreads)
    pre_combine2_kernel(QPlan P, const double* __restrict__ partials,
                        const double* __restrict__ partials_q, double* __restrict__ partials2,
                        double* __restrict__ partials2_q) {
  pdl_enter();
  __shared__ double v[kPreGroup];
  const uint64_t g = blockIdx.x >> 1;
  const bool isq = blockIdx.x & 1;
  const uint64_t gpu = P.T_max >> kPreShift;  // group slots per unit
  const uint32_t u = (uint32_t)(g / gpu);
  const uint32_t T = u == P.nunits - 1 ? P.T_last : P.T_full;
  const uint64_t gi = g % gpu;
  if ((gi << kPreShift) >= T) return;
  const double* src = (isq ? partials_q : partials) + (uint64_t)u * P.T_full + (gi << kPreShift);
  for (int i = threadIdx.x; i < (int)kPreGroup; i += kQThreads) v[i] = src[i];
  constexpr int kPer = kPreGroup / 2 / kQThreads;
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
  if (threadIdx.x == 0) (isq ? partials2_q : partials2)[g] = v[0];
}

// f32 outputs of sigma (the table's std, B32_k, F_k) as numpy computes them
struct SigmaOut {
  float std_, b32[15], f[15];
};
__device__ __forceinline__ void sigma_outputs(double mu, double sd, int m, SigmaOut& o) {
  o.std_ = __double2float_rn(sd);
  for (int k = 0; k < 15; ++k) {
    if (k < m - 1) {
      const double b = __dadd_rn(mu, __dmul_rn(sd, kNdtri[m][k]));  // mu + sigma * ndtri
      o.b32[k] = __double2float_rn(b);
      o.f[k] = __double2float_rd(b);
    } else {
      o.b32[k] = 0.0f;
      o.f[k] = 0.0f;
    }
  }
}

// table header + fit thresholds of unit u from (mu, sd) (thread-local)
__device__ __forceinline__ void write_header(const QPlan& P, uint32_t u, double m0, double sd,
                                             float* fthr, bsnp_cluster_table* tables,
                                             double* sdv) {
  const int m = (int)P.m;
  bsnp_cluster_table& tb = tables[u];
  sdv[u] = sd;
  tb.mean = __double2float_rn(m0);
  tb.std = __double2float_rn(sd);
  tb.m = (uint32_t)m;
  tb.flags = (isfinite(m0) && isfinite(sd)) ? 0u : BSNP_ERR_NONFINITE;
  for (int k = 0; k < 15; ++k) {
    if (k < m - 1) {
      const double b = __dadd_rn(m0, __dmul_rn(sd, kNdtri[m][k]));
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

// The interval of numpy's sigma from the exact pairwise sum S, our D2 and the
// shift c; returns true when every f32 output is determined (sd = sigma_lo).
__device__ bool sigma_from_d2(double S, double D2, double c, double len, double mu, int m,
                              double& sd) {
  if (!(isfinite(S) && isfinite(D2) && isfinite(mu))) return false;
  const double eq = __dmul_ru(D2, 128.0 * kU);
  const double d2lo = fmax(__dsub_rd(D2, eq), 0.0), d2hi = __dadd_ru(D2, eq);
  const double absb = __dadd_ru(__dsqrt_ru(__dmul_ru(len, d2hi)), __dmul_ru(len, fabs(c)));
  const double e2 = __dmul_ru(absb, 64.0 * kU);
  const double mlo = __ddiv_rd(__dsub_rd(S, e2), len), mhi = __ddiv_ru(__dadd_ru(S, e2), len);
  const double dlo = __dsub_rd(mlo, c), dhi = __dsub_ru(mhi, c);
  const double admax = fmax(fabs(dlo), fabs(dhi));
  const double admin = (dlo <= 0.0 && dhi >= 0.0) ? 0.0 : fmin(fabs(dlo), fabs(dhi));
  const double elo = __dsub_rd(mlo, mu), ehi = __dsub_ru(mhi, mu);
  const double aemax = fmax(fabs(elo), fabs(ehi));
  // T = D2 - n (m* - c)^2 + n (m* - mu)^2
  double tlo = __dsub_rd(d2lo, __dmul_ru(len, __dmul_ru(admax, admax)));
  double thi = __dadd_ru(__dsub_ru(d2hi, __dmul_rd(len, __dmul_rd(admin, admin))),
                         __dmul_ru(len, __dmul_ru(aemax, aemax)));
  tlo = fmax(tlo, 0.0);
  // numpy's own rounding of the same T
  tlo = __dmul_rd(tlo, 1.0 - 64.0 * kU);
  thi = __dmul_ru(thi, 1.0 + 64.0 * kU);
  if (!(thi >= tlo) || !isfinite(thi)) return false;
  const double sdlo = __dsqrt_rn(__ddiv_rn(tlo, len));  // np.std: sqrt(T / n)
  const double sdhi = __dsqrt_rn(__ddiv_rn(thi, len));
  sd = sdlo;
  if (sdlo == sdhi) return true;
  SigmaOut a, b;
  sigma_outputs(mu, sdlo, m, a);
  sigma_outputs(mu, sdhi, m, b);
  bool same = __float_as_uint(a.std_) == __float_as_uint(b.std_);
  for (int k = 0; k < 15; ++k)
    same = same && __float_as_uint(a.b32[k]) == __float_as_uint(b.b32[k]) &&
           __float_as_uint(a.f[k]) == __float_as_uint(b.f[k]);
  return same;
}

// per unit: exact mean; sigma from the D2 interval, or the unit is listed
__global__ void __launch_bounds__(kQThreads)
    fit_stats_kernel(const float* __restrict__ x, QPlan P, const double* __restrict__ partials,
                     const double* __restrict__ partials_q, const double* __restrict__ partials2,
                     const double* __restrict__ partials2_q, double* __restrict__ mu,
                     float* __restrict__ fthr, bsnp_cluster_table* __restrict__ tables,
                     double* __restrict__ sdv, uint32_t* __restrict__ list, int force_exact,
                     UGrid* __restrict__ ug, uint32_t* __restrict__ any_need) {
  pdl_enter();
  __shared__ double sv[kQThreads];
  __shared__ GridSmem g;
  __shared__ double s_mean, s_sd;
  __shared__ uint32_t s_ok;
  const uint32_t u = blockIdx.x;
  // the "some unit needs the exact min/max round" word, set by fit_decide
  if (u == 0 && threadIdx.x == 0) *any_need = 0;
  uint32_t T;
  uint64_t len;
  unit_shape(P, u, T, len);
  const int sh = T > kPreGroup ? kPreShift : 0;
  const uint64_t first = sh ? (uint64_t)u * (P.T_max >> kPreShift) : (uint64_t)u * P.T_full;
  const double S = combine_perfect((sh ? partials2 : partials) + first, T >> sh, sv);
  __syncthreads();
  const double D2 = combine_perfect((sh ? partials2_q : partials_q) + first, T >> sh, sv);
  if (threadIdx.x == 0) {
    const double ld = (double)len;
    const double mean = __ddiv_rn(__dadd_rn(0.0, S), ld);  // np.mean
    mu[u] = mean;
    double sd;
    const double c = (double)x[(uint64_t)u * P.block];
    uint32_t ok = 1;
    if (!force_exact && sigma_from_d2(S, D2, c, ld, mean, (int)P.m, sd)) {
      write_header(P, u, mean, sd, fthr, tables, sdv);
    } else if (!isfinite(mean)) {
      // NaN / Inf in the unit: the host raises; any sd will do
      sd = mean;
      write_header(P, u, mean, sd, fthr, tables, sdv);
    } else {
      const uint32_t i = atomicAdd(list, 1u);
      list[1 + i] = u;
      ok = 0;
    }
    s_mean = mean;
    s_sd = sd;
    s_ok = ok;
  }
  __syncthreads();
  if (s_ok) grid_unit(P, u, s_mean, s_sd, ug, g);
}

// numpy's variance tree for the listed units only (grid-stride over their
// tiles; a launch with an empty list returns at once)
__global__ void __launch_bounds__(kQThreads)
    fit_var_fallback_kernel(const float* __restrict__ x, QPlan P, const double* __restrict__ mu,
                            const uint32_t* __restrict__ list, double* __restrict__ partials) {
  pdl_enter();
  __shared__ __align__(16) float s[kSmemFloats];
  __shared__ Heap H;
  const uint32_t cnt = __ldcg(list);
  for (uint64_t item = blockIdx.x;; item += gridDim.x) {
    // T_max tile slots per listed unit (the last unit may have more tiles
    // than a full one)
    const uint64_t i = item >> P.D_max, j = item & (P.T_max - 1);
    if (i >= cnt) break;
    const uint32_t u = __ldcg(list + 1 + i);
    const uint32_t T = u == P.nunits - 1 ? P.T_last : P.T_full;
    if (j >= T) continue;
    const uint64_t tile = (uint64_t)u * P.T_full + j;
    const double v = tree_tile<true>(x, P, tile, mu[u], s, H, policy_evict_first());
    if (threadIdx.x == 0) partials[tile] = v;
    __syncthreads();  // s / H are reused by the next item
  }
}

__global__ void __launch_bounds__(kQThreads)
    fit_var_combine_kernel(QPlan P, const double* __restrict__ partials,
                           const uint32_t* __restrict__ list, const double* __restrict__ mu,
                           float* __restrict__ fthr, bsnp_cluster_table* __restrict__ tables,
                           double* __restrict__ sdv, UGrid* __restrict__ ug) {
  pdl_enter();
  __shared__ double sv[kQThreads];
  __shared__ GridSmem g;
  __shared__ double s_sd;
  const uint32_t cnt = __ldcg(list);
  for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const uint32_t u = __ldcg(list + 1 + i);
    uint32_t T;
    uint64_t len;
    unit_shape(P, u, T, len);
    __syncthreads();
    const double S = combine_perfect(partials + (uint64_t)u * P.T_full, T, sv);
    if (threadIdx.x == 0) {
      const double sd = __dsqrt_rn(__ddiv_rn(__dadd_rn(0.0, S), (double)len));  // np.std
      write_header(P, u, mu[u], sd, fthr, tables, sdv);
      s_sd = sd;
    }
    __syncthreads();
    grid_unit(P, u, mu[u], s_sd, ug, g);  // the unit's bin grid (fit_stats skipped it)
  }
}
