// build.cuh — per-cell device functions of the cost-table builders, shared
// by the standalone launch (tables.cu) and the fused plan kernel (fused.cuh).
//   K2 node_cost_cell: compute_cost + sync_cost (cost.hpp:60-94)
//   K1 xfer_cell:      transfer_profile seconds (cost.hpp:103-131)
#pragma once

#include "tables.hpp"

#include "parplan/geometry.hpp"

namespace pp {
namespace geo = parplan::geo;

constexpr int kBuildThreads = 128;

__device__ inline void node_cost_cell(const BuildArgs &a, int64_t gi) {
  // layer with cat_off <= gi < cat_off + count (binary search)
  int lo = 0, hi = a.nl - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.layers[mid].cat_off <= gi)
      lo = mid;
    else
      hi = mid - 1;
  }
  const LayerDev &L = a.layers[lo];
  const int32_t *c32 = a.cfg + 4 * gi;
  const int64_t c[4] = {c32[0], c32[1], c32[2], c32[3]};
  const int64_t total = c[0] * c[1] * c[2] * c[3];
  // compute_cost (cost.hpp:60-72)
  const int64_t flops = geo::layer_flops(L.kind, L.params, L.shape, L.in_shape);
  double tc = 0.0;
  if (flops != 0) {
    double slowest = a.rates[0];
    for (int64_t p = 1; p < total; ++p) slowest = fmin(slowest, a.rates[p]);
    tc = geo::compute_seconds(flops, total, slowest);
  }
  // sync_cost (cost.hpp:79-94): sequential sum, reference order
  const double P = geo::parameter_bytes(L.kind, L.params, L.shape, L.in_shape);
  double ts = 0.0;
  if (P != 0.0 && total / c[1] != 1) {
    const double shard = P / static_cast<double>(c[1]);
    for (int64_t p = 1; p < total; ++p) ts = ts + 2.0 * shard / a.bw[p * a.D + 0];
  }
  a.compute[gi] = tc;
  a.sync[gi] = ts;
  a.node[gi] = tc + ts;
}

// One (c_src, c_dst) cell.  Coordinates are int32 (tensor extents < 2^31,
// checked on the host); volumes are int64.  Destination partitions q are
// walked with an odometer over their per-dimension digits (W fastest), so
// no division sits in the q loop except the O(1) piece lookups.
// dim_stats (geometry.hpp) with the two divisions by the piece size done as a
// float multiply by a per-cell reciprocal plus one exact correction (valid
// for coordinates < 2^22; the host checks tensor extents before choosing it).
__device__ __forceinline__ int div_fast(int a, int P, float rcp) {
  int x = __float2int_rz(__int2float_rn(a) * rcp);
  if (x * P > a) --x;
  else if ((x + 1) * P <= a) ++x;
  return x;
}

__device__ __forceinline__ geo::DimStats<int> dim_stats_fast(int a, int b, int P, float rcp) {
  geo::DimStats<int> s{0, 0, 0, false};
  if (b <= a) return s;
  const int x0 = div_fast(a, P, rcp), x1 = div_fast(b - 1, P, rcp);
  if (x0 == x1) {
    s.best = b - a, s.arg = x0, s.unique = true, s.second = 0;
    return s;
  }
  const int o0 = (x0 + 1) * P - a, o1 = b - x1 * P;
  if (x1 == x0 + 1) {
    if (o0 == o1) {
      s.best = s.second = o0, s.unique = false;
    } else {
      s.unique = true;
      s.best = o0 > o1 ? o0 : o1;
      s.second = o0 > o1 ? o1 : o0;
      s.arg = o0 > o1 ? x0 : x1;
    }
    return s;
  }
  const int full = (x1 - x0 - 1) + (o0 == P) + (o1 == P);
  s.best = P;
  if (full >= 2) {
    s.second = P, s.unique = false;
  } else {
    s.unique = true, s.arg = x0 + 1, s.second = o0 > o1 ? o0 : o1;
  }
  return s;
}

// Uniform bandwidth (the common case): seconds = RN(4 * maxvol / bw) with
// maxvol = max over destination partitions q (non-empty need) of
// max_{p != q} vol(owned(p) ∩ need_q).  Each dimension's need interval
// depends on one destination digit only (flatten: dims 1-3 on digit 1), so
// when the odometer advances digit d only dims d..3 get new overlap stats:
// ~1.1 dim_stats per q instead of 4.
__device__ inline int64_t xfer_maxvol_uniform(const EdgeDev &E, const int *cs, const int *cd, const int *ss,
                                              const int *spiece, const int *dpiece, int band) {
  const int td = cd[0] * cd[1] * cd[2] * cd[3];
  const int kind = E.kind;
  int par[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) par[k] = static_cast<int>(E.params[k]);
  int dig[4] = {0, 0, 0, 0};
  geo::DimStats<int> st[4];
  float rcp[4];
#pragma unroll
  for (int d = 0; d < 4; ++d) rcp[d] = 1.0f / static_cast<float>(spiece[d]);
  int64_t maxvol = 0;
  int changed = 0;
  for (int q = 0; q < td; ++q) {
    if (changed <= 3) {
      int olo[4], ohi[4], lo[4], hi[4];
#pragma unroll
      for (int d = 0; d < 4; ++d) olo[d] = dig[d] * dpiece[d], ohi[d] = olo[d] + dpiece[d];
      geo::required_box_owned<int, int>(kind, par, ss, band, olo, ohi, lo, hi);
#pragma unroll
      for (int d = 0; d < 4; ++d)
        if (d >= changed) st[d] = dim_stats_fast(lo[d], hi[d], spiece[d], rcp[d]);
    }
    // combine (geometry.hpp: max_offdiag_volume)
    const int64_t M = static_cast<int64_t>(st[0].best) * st[1].best * st[2].best * st[3].best;
    if (M > maxvol) {
      const bool unique = st[0].unique && st[1].unique && st[2].unique && st[3].unique;
      int64_t v = M;
      if (unique && ((st[0].arg * cs[1] + st[1].arg) * cs[2] + st[2].arg) * cs[3] + st[3].arg == q) {
        v = 0;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          int64_t x = st[d].second;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e != d) x *= st[e].best;
          v = x > v ? x : v;
        }
      }
      maxvol = v > maxvol ? v : maxvol;
    }
    // odometer over destination digits (W fastest), unrolled: constant indices
    changed = 3;
    if (++dig[3] == cd[3]) {
      dig[3] = 0, changed = 2;
      if (++dig[2] == cd[2]) {
        dig[2] = 0, changed = 1;
        if (++dig[1] == cd[1]) dig[1] = 0, changed = 0, ++dig[0];
      }
    }
  }
  return maxvol;
}

__device__ inline void xfer_cell(const BuildArgs &a, const EdgeDev &E, int64_t cell) {
  // cells are walked destination-config-major (consecutive threads share c_dst, so the
  // q loop has the same trip count across a warp); the table stays row-major [i][j]
  const int j = static_cast<int>(cell / E.nu), i = static_cast<int>(cell - static_cast<int64_t>(j) * E.nu);
  const int64_t out = E.out_off + static_cast<int64_t>(i) * E.nv + j;
  const int32_t *cs64 = a.cfg + 4 * (E.cat_u + i);
  const int32_t *cd64 = a.cfg + 4 * (E.cat_v + j);
  int cs[4], cd[4], ss[4], dpiece[4], spiece[4];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    cs[d] = static_cast<int>(cs64[d]);
    cd[d] = static_cast<int>(cd64[d]);
    ss[d] = static_cast<int>(E.sshape[d]);
    spiece[d] = ss[d] / cs[d];
    dpiece[d] = static_cast<int>(E.dshape[d]) / cd[d];
  }
  const int td = cd[0] * cd[1] * cd[2] * cd[3];
  const int band = static_cast<int>(E.band);
  double seconds = 0.0;
  if (a.bw_uniform > 0.0) {
    const int64_t maxvol = xfer_maxvol_uniform(E, cs, cd, ss, spiece, dpiece, band);
    if (maxvol > 0) seconds = 4.0 * static_cast<double>(maxvol) / a.bw_uniform;
    a.xfer[out] = seconds;
    return;
  }
  int dig[4] = {0, 0, 0, 0};
  int64_t maxvol = 0;
  for (int q = 0; q < td; ++q) {
    int olo[4], ohi[4], lo[4], hi[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) olo[d] = dig[d] * dpiece[d], ohi[d] = olo[d] + dpiece[d];
    geo::required_box_owned<int, int64_t>(E.kind, E.params, ss, band, olo, ohi, lo, hi);
    if (geo::box_volume<int>(lo, hi) != 0) {
      if (a.bw_uniform > 0.0) {
        maxvol = geo::imax<int64_t>(maxvol, geo::max_offdiag_volume<int>(spiece, cs, lo, hi, q));
      } else {
        int pd[4] = {0, 0, 0, 0};
        const int ts = cs[0] * cs[1] * cs[2] * cs[3];
        for (int p = 0; p < ts; ++p) {
          if (p != q) {
            int64_t vol = 1;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              const int plo = pd[d] * spiece[d];
              vol *= geo::imax<int>(0, geo::imin<int>(plo + spiece[d], hi[d]) - geo::imax<int>(plo, lo[d]));
            }
            if (vol > 0) seconds = fmax(seconds, 4.0 * static_cast<double>(vol) / a.bw[static_cast<int64_t>(p) * a.D + q]);
          }
          for (int d = 3; d >= 0; --d) { // odometer over source digits
            if (++pd[d] < cs[d]) break;
            pd[d] = 0;
          }
        }
      }
    }
    for (int d = 3; d >= 0; --d) { // odometer over destination digits
      if (++dig[d] < cd[d]) break;
      dig[d] = 0;
    }
  }
  if (a.bw_uniform > 0.0 && maxvol > 0) seconds = 4.0 * static_cast<double>(maxvol) / a.bw_uniform;
  a.xfer[out] = seconds;
}

} // namespace pp
