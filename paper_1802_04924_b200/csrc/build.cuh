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

// cat_off_s: the layers' catalog offsets staged in shared memory by the
// caller (or nullptr: read from the descriptors)
__device__ __forceinline__ void node_cost_cell(const BuildArgs &a, int64_t gi, const int64_t *cat_off_s = nullptr) {
  // layer with cat_off <= gi < cat_off + count (binary search)
  int lo = 0, hi = a.nl - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((cat_off_s ? cat_off_s[mid] : a.layers[mid].cat_off) <= gi)
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

// Geometry of one (c_src, c_dst) cell.  Coordinates are int32 (tensor
// extents < 2^22, checked on the host); volumes are int64.  Cells are walked
// destination-config-major (consecutive threads share c_dst); the table
// stays row-major [i][j].
struct XferCell {
  int cs[4], cd[4], ss[4], spiece[4], dpiece[4];
  float rcp[4];
  int par[7];
  int band, kind;
  int64_t out;
};

__device__ __forceinline__ void xfer_decode(const BuildArgs &a, const EdgeDev &E, int64_t cell, XferCell &c) {
  const int j = static_cast<int>(cell / E.nu), i = static_cast<int>(cell - static_cast<int64_t>(j) * E.nu);
  c.out = E.out_off + static_cast<int64_t>(i) * E.nv + j;
  const int32_t *cs32 = a.cfg + 4 * (E.cat_u + i);
  const int32_t *cd32 = a.cfg + 4 * (E.cat_v + j);
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    c.cs[d] = cs32[d];
    c.cd[d] = cd32[d];
    c.ss[d] = static_cast<int>(E.sshape[d]);
    c.spiece[d] = c.ss[d] / c.cs[d];
    c.dpiece[d] = static_cast<int>(E.dshape[d]) / c.cd[d];
    c.rcp[d] = 1.0f / static_cast<float>(c.spiece[d]);
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) c.par[k] = static_cast<int>(E.params[k]);
  c.band = static_cast<int>(E.band);
  c.kind = E.kind;
}

// Dimension d of required_box_owned (geometry.hpp) for an owned interval
// [olo, ohi) along d.  Every kind but Flatten maps each dimension of the
// need box from the same dimension of the owned box alone.
__device__ __forceinline__ void need_interval(const XferCell &c, int d, int olo, int ohi, int *lo, int *hi) {
  *lo = olo, *hi = ohi;
  switch (c.kind) {
  case geo::kConcat:
    if (d == c.par[0]) {
      int l = geo::imax<int>(olo, c.band), h = geo::imin<int>(ohi, c.band + c.ss[d]);
      if (h < l) h = l;
      *lo = l - c.band, *hi = h - c.band;
    }
    return;
  case geo::kSoftmax:
    return;
  case geo::kConv:
    if (d == 1) *lo = 0, *hi = c.ss[1];
    if (d == 2) geo::window<int>(olo, ohi, c.par[1], c.par[3], c.par[5], c.ss[2], lo, hi);
    if (d == 3) geo::window<int>(olo, ohi, c.par[2], c.par[4], c.par[6], c.ss[3], lo, hi);
    return;
  case geo::kPool:
    if (d == 2) geo::window<int>(olo, ohi, c.par[0], c.par[2], c.par[4], c.ss[2], lo, hi);
    if (d == 3) geo::window<int>(olo, ohi, c.par[1], c.par[3], c.par[5], c.ss[3], lo, hi);
    return;
  case geo::kFC:
    if (d > 0) *lo = 0, *hi = c.ss[d];
    return;
  default:
    if (d > 0) *lo = 0, *hi = 0;
    return;
  }
}

// Uniform bandwidth (the common case): seconds = RN(4 * maxvol / bw) with
// maxvol = max over destination partitions q of max_{p != q} vol(owned(p) ∩
// need_q) (cost.hpp:103-131).  With M(q) = prod_d best_d(q_d) the per-q
// maximum over all p, M is separable, so Mmax = prod_d max_x best_d(x) costs
// sum_d cd[d] dim_stats instead of prod_d cd[d].  Mmax is the answer unless
// every q attaining it has a unique maximiser p* equal to q itself; writing
// p* - q = sum_d delta_d(q_d) with delta_d(x) = arg_d(x) * S_d - x * D_d
// (S, D the flat strides of the two configs), some maximising q has p* != q
// iff a maximising digit has non-unique stats, or delta varies over the
// maximising digits of some dimension, or the constant deltas do not sum to
// 0.  Returns -1 when no such q exists (the diagonal cells) or the kind is
// Flatten; those cells take xfer_maxvol_walk.
__device__ __forceinline__ int64_t xfer_maxvol_separable(const XferCell &c) {
  if (c.kind == geo::kFlatten) return -1;
  int64_t mmax = 1;
  bool easy = false;
  int dsum = 0, S = 1, D = 1;
  int bm[4], sm2[4], b2[4]; // per dimension: max best, max second over the maximisers, best non-maximiser
#pragma unroll
  for (int d = 3; d >= 0; --d) {
    int bmax = -1, dfirst = 0, smax = 0, bnext = -1;
    bool nonunique = false, dvar = false;
    // Closed forms of the x loop below.  The need interval of an
    // x-invariant dimension (conv input channels, FC features) is the same
    // for every x: one dim_stats, all x tie, and delta(x) - delta(0) = -x*D.
    // An identity dimension (need = owned) whose piece sizes divide one
    // another has the same best overlap for every x: with cd = r*cs every
    // destination piece lies in source piece x/r (unique, second 0); with
    // cs = r*cd (r >= 2) each covers r whole source pieces (two maximisers).
    const bool invariant = (c.kind == geo::kConv && d == 1) || (c.kind == geo::kFC && d > 0);
    const bool identity = c.kind == geo::kConcat ? d != c.par[0]
                                                 : d == 0 || c.kind == geo::kSoftmax || (c.kind == geo::kPool && d == 1);
    const bool same_extent = c.spiece[d] * c.cs[d] == c.dpiece[d] * c.cd[d];
    if (invariant) {
      int lo, hi;
      need_interval(c, d, 0, c.dpiece[d], &lo, &hi);
      const geo::DimStats<int> st = dim_stats_fast(lo, hi, c.spiece[d], c.rcp[d]);
      bmax = st.best, nonunique = !st.unique, dvar = c.cd[d] > 1, dfirst = st.arg * S, smax = st.second;
    } else if (identity && same_extent && c.cd[d] % c.cs[d] == 0) {
      bmax = c.dpiece[d], dvar = c.cd[d] > 1 && (c.cd[d] != c.cs[d] || S != D);
    } else if (identity && same_extent && c.cs[d] % c.cd[d] == 0) {
      bmax = smax = c.spiece[d], nonunique = true, dvar = c.cd[d] > 1;
    } else
    for (int x = 0; x < c.cd[d]; ++x) {
      const int olo = x * c.dpiece[d];
      int lo, hi;
      need_interval(c, d, olo, olo + c.dpiece[d], &lo, &hi);
      const geo::DimStats<int> st = dim_stats_fast(lo, hi, c.spiece[d], c.rcp[d]);
      const int delta = st.arg * S - x * D;
      if (st.best > bmax) {
        bnext = bmax > bnext ? bmax : bnext;
        bmax = st.best, nonunique = !st.unique, dvar = false, dfirst = delta, smax = st.second;
      } else if (st.best == bmax) {
        nonunique |= !st.unique;
        dvar |= delta != dfirst;
        smax = st.second > smax ? st.second : smax;
      } else {
        bnext = st.best > bnext ? st.best : bnext;
      }
    }
    mmax *= bmax;
    easy |= nonunique | dvar;
    dsum += dfirst;
    bm[d] = bmax, sm2[d] = smax, b2[d] = bnext;
    S *= c.cs[d];
    D *= c.cd[d];
  }
  if (mmax == 0) return 0;
  if (easy || dsum != 0) return mmax;
  // Every maximising q is "diagonal" (its unique best source is q itself), so
  // over them the answer is the best other source: max_d S_d * prod_{e!=d}
  // bmax_e (S_d: largest second-best over the maximising digits).  Any other
  // q has M(q) <= U = max_d b2_d * prod_{e!=d} bmax_e; when U <= that value
  // (no non-maximising digit at all in the diagonal cells) it is exact.
  int64_t alt = 0, U = -1;
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    int64_t rest = 1;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e != d) rest *= bm[e];
    const int64_t a = rest * sm2[d];
    alt = a > alt ? a : alt;
    if (b2[d] >= 0) {
      const int64_t u = rest * b2[d];
      U = u > U ? u : U;
    }
  }
  if (U <= alt) return alt;
  return -1;
}

// The per-q walk (geometry.hpp: max_offdiag_volume) over destination
// partitions q = q0, q0 + dq, ... — one lane's share of a warp-cooperative walk.
__device__ __forceinline__ int64_t xfer_maxvol_walk(const XferCell &c, int q0, int dq) {
  const int td = c.cd[0] * c.cd[1] * c.cd[2] * c.cd[3];
  int64_t maxvol = 0;
  for (int q = q0; q < td; q += dq) {
    int dig[4], r = q;
#pragma unroll
    for (int d = 3; d >= 0; --d) dig[d] = r % c.cd[d], r /= c.cd[d];
    int olo[4], ohi[4], lo[4], hi[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) olo[d] = dig[d] * c.dpiece[d], ohi[d] = olo[d] + c.dpiece[d];
    geo::required_box_owned<int, int>(c.kind, c.par, c.ss, c.band, olo, ohi, lo, hi);
    geo::DimStats<int> st[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) st[d] = dim_stats_fast(lo[d], hi[d], c.spiece[d], c.rcp[d]);
    const int64_t M = static_cast<int64_t>(st[0].best) * st[1].best * st[2].best * st[3].best;
    if (M <= maxvol) continue;
    const bool unique = st[0].unique && st[1].unique && st[2].unique && st[3].unique;
    int64_t v = M;
    if (unique && ((st[0].arg * c.cs[1] + st[1].arg) * c.cs[2] + st[2].arg) * c.cs[3] + st[3].arg == q) {
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
  return maxvol;
}

__device__ __forceinline__ double xfer_seconds(const BuildArgs &a, int64_t maxvol) {
  return maxvol > 0 ? 4.0 * static_cast<double>(maxvol) / a.bw_uniform : 0.0;
}

// Per-pair bandwidth: every (q, p) pair in reference order (cost.hpp:113-129).
__device__ __forceinline__ double xfer_seconds_pairs(const BuildArgs &a, const XferCell &c) {
  const int td = c.cd[0] * c.cd[1] * c.cd[2] * c.cd[3];
  const int ts = c.cs[0] * c.cs[1] * c.cs[2] * c.cs[3];
  double seconds = 0.0;
  int dig[4] = {0, 0, 0, 0};
  for (int q = 0; q < td; ++q) {
    int olo[4], ohi[4], lo[4], hi[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) olo[d] = dig[d] * c.dpiece[d], ohi[d] = olo[d] + c.dpiece[d];
    geo::required_box_owned<int, int>(c.kind, c.par, c.ss, c.band, olo, ohi, lo, hi);
    if (geo::box_volume<int>(lo, hi) != 0) {
      int pd[4] = {0, 0, 0, 0};
      for (int p = 0; p < ts; ++p) {
        if (p != q) {
          int64_t vol = 1;
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const int plo = pd[d] * c.spiece[d];
            vol *= geo::imax<int>(0, geo::imin<int>(plo + c.spiece[d], hi[d]) - geo::imax<int>(plo, lo[d]));
          }
          if (vol > 0) seconds = fmax(seconds, 4.0 * static_cast<double>(vol) / a.bw[static_cast<int64_t>(p) * a.D + q]);
        }
        for (int d = 3; d >= 0; --d) { // odometer over source digits
          if (++pd[d] < c.cs[d]) break;
          pd[d] = 0;
        }
      }
    }
    for (int d = 3; d >= 0; --d) { // odometer over destination digits
      if (++dig[d] < c.cd[d]) break;
      dig[d] = 0;
    }
  }
  return seconds;
}

// One K1 cell per lane.  `edge` < 0 marks an inactive lane.  All 32 lanes of
// the warp must call this together: cells the separable bound cannot settle
// are then walked by the whole warp, one cell at a time, lanes striding q.
__device__ __forceinline__ void xfer_cells_warp(const BuildArgs &a, int edge, int64_t cell) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  bool hard = false;
  if (edge >= 0) {
    XferCell c;
    xfer_decode(a, a.edges[edge], cell, c);
    if (a.bw_uniform > 0.0) {
      const int64_t mv = xfer_maxvol_separable(c);
      if (mv >= 0)
        a.xfer[c.out] = xfer_seconds(a, mv);
      else
        hard = true;
    } else {
      a.xfer[c.out] = xfer_seconds_pairs(a, c);
    }
  }
  unsigned pending = __ballot_sync(kFull, hard);
  while (pending) {
    const int src = __ffs(pending) - 1;
    pending &= pending - 1;
    const int e = __shfl_sync(kFull, edge, src);
    const int64_t cl = __shfl_sync(kFull, cell, src);
    XferCell c;
    xfer_decode(a, a.edges[e], cl, c);
    int64_t mv = xfer_maxvol_walk(c, lane, 32);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t other = __shfl_xor_sync(kFull, mv, o);
      mv = other > mv ? other : mv;
    }
    if (lane == src) a.xfer[c.out] = xfer_seconds(a, mv);
  }
}

} // namespace pp
