/* parplan/geometry.hpp — the pure partition/cost formulas, shared verbatim by
 * the host API and the sm_100a kernels (PP_HD = __host__ __device__ under nvcc).
 *
 * Nothing here allocates or throws; every function works on plain integer
 * arrays in (sample, channel, height, width) order so the same definition runs
 * in the xfer-table kernel (K1, instantiated on int32 coordinates), the
 * node-cost kernel (K2) and the host-side single-call API (owned_region,
 * required_input_region, transfer_profile; int64).
 *
 * Citations: /root/reference/proj/include/parplan/partition.hpp and cost.hpp.
 */
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define PP_HD __host__ __device__ __forceinline__
#else
#define PP_HD inline
#endif

namespace parplan {
namespace geo {

using i64 = std::int64_t;

enum : int { kInput = 0, kConv = 1, kPool = 2, kFC = 3, kFlatten = 4, kConcat = 5, kSoftmax = 6 };

template <class I> PP_HD I imin(I a, I b) { return a < b ? a : b; }
template <class I> PP_HD I imax(I a, I b) { return a > b ? a : b; }

/* conv/pool output extent (graph.hpp:257-259) */
PP_HD i64 conv_out(i64 in, i64 k, i64 s, i64 p) { return (in + 2 * p - k) / s + 1; }

template <class I> PP_HD I config_total(const I *c) { return c[0] * c[1] * c[2] * c[3]; }

/* Row-major decode of a partition index, W fastest (partition.hpp:213-232). */
template <class I> PP_HD void decode_part(const I *cfg, I part, I *idx) {
  for (int d = 3; d >= 0; --d) {
    idx[d] = part % cfg[d];
    part /= cfg[d];
  }
}

/* owned_region: equal contiguous pieces of extent/deg per dimension */
template <class I> PP_HD void owned_box_digits(const I *shape, const I *cfg, const I *idx, I *lo, I *hi) {
  for (int d = 0; d < 4; ++d) {
    const I piece = shape[d] / cfg[d];
    lo[d] = idx[d] * piece;
    hi[d] = lo[d] + piece;
  }
}

template <class I> PP_HD void owned_box(const I *shape, const I *cfg, I part, I *lo, I *hi) {
  I idx[4];
  decode_part(cfg, part, idx);
  owned_box_digits(shape, cfg, idx, lo, hi);
}

/* map_spatial_window (partition.hpp:236-245) */
template <class I> PP_HD void window(I own_lo, I own_hi, I k, I s, I p, I ext, I *lo, I *hi) {
  const I a = own_lo * s - p;
  const I b = (own_hi - 1) * s - p + k;
  *lo = imax<I>(0, a);
  *hi = imin<I>(ext, b);
  if (*hi < *lo) *hi = *lo;
}

/* flat_range_box (partition.hpp:249-273): bounding box in (C, H, W) of the
 * flattened index range [flo, fhi), flat = (c*H + h)*W + w. */
template <class I> PP_HD void flat_box(I flo, I fhi, I H, I W, I *lo, I *hi) {
  const I plane = H * W;
  const I clo = flo / plane, chi = (fhi - 1) / plane;
  lo[1] = clo;
  hi[1] = chi + 1;
  if (clo != chi) {
    lo[2] = 0, hi[2] = H, lo[3] = 0, hi[3] = W;
    return;
  }
  const I rlo = (flo % plane) / W, rhi = ((fhi - 1) % plane) / W;
  lo[2] = rlo;
  hi[2] = rhi + 1;
  if (rlo != rhi) {
    lo[3] = 0, hi[3] = W;
    return;
  }
  lo[3] = flo % W;
  hi[3] = (fhi - 1) % W + 1;
}

/* required_input_region (partition.hpp:283-350) for the destination partition
 * owning [olo, ohi).  `p` = destination kind parameters, `ins` = the edge's
 * tensor shape (source output), `band_offset` = for Concat, the sum of the
 * preceding siblings' extents on the concat axis (partition.hpp:331-337,
 * precomputed by the caller).  Returns false for kinds that consume no inputs. */
template <class I, class P>
PP_HD bool required_box_owned(int kind, const P *p, const I *ins, I band_offset, const I *olo, const I *ohi, I *lo,
                              I *hi) {
  for (int d = 0; d < 4; ++d) lo[d] = 0, hi[d] = 0;
  lo[0] = olo[0];
  hi[0] = ohi[0];
  switch (kind) {
  case kConv:
    lo[1] = 0, hi[1] = ins[1];
    window<I>(olo[2], ohi[2], static_cast<I>(p[1]), static_cast<I>(p[3]), static_cast<I>(p[5]), ins[2], &lo[2], &hi[2]);
    window<I>(olo[3], ohi[3], static_cast<I>(p[2]), static_cast<I>(p[4]), static_cast<I>(p[6]), ins[3], &lo[3], &hi[3]);
    return true;
  case kPool:
    lo[1] = olo[1], hi[1] = ohi[1];
    window<I>(olo[2], ohi[2], static_cast<I>(p[0]), static_cast<I>(p[2]), static_cast<I>(p[4]), ins[2], &lo[2], &hi[2]);
    window<I>(olo[3], ohi[3], static_cast<I>(p[1]), static_cast<I>(p[3]), static_cast<I>(p[5]), ins[3], &lo[3], &hi[3]);
    return true;
  case kFC:
    lo[1] = 0, hi[1] = ins[1];
    lo[2] = 0, hi[2] = ins[2];
    lo[3] = 0, hi[3] = ins[3];
    return true;
  case kFlatten:
    flat_box<I>(olo[1], ohi[1], ins[2], ins[3], lo, hi);
    return true;
  case kConcat: {
    const int A = static_cast<int>(p[0]);
    for (int d = 0; d < 4; ++d) { // constant indices only: keeps the box in registers on the device
      if (d == A) {
        lo[d] = imax<I>(olo[d], band_offset);
        hi[d] = imin<I>(ohi[d], band_offset + ins[d]);
        if (hi[d] < lo[d]) hi[d] = lo[d];
        lo[d] -= band_offset;
        hi[d] -= band_offset;
      } else {
        lo[d] = olo[d], hi[d] = ohi[d];
      }
    }
    return true;
  }
  case kSoftmax:
    for (int d = 0; d < 4; ++d) lo[d] = olo[d], hi[d] = ohi[d];
    return true;
  default:
    return false;
  }
}

template <class I, class P>
PP_HD bool required_box(int kind, const P *p, const I *ins, const I *outs, I band_offset, const I *dcfg, I part, I *lo,
                        I *hi) {
  I olo[4], ohi[4];
  owned_box<I>(outs, dcfg, part, olo, ohi);
  return required_box_owned<I, P>(kind, p, ins, band_offset, olo, ohi, lo, hi);
}

template <class I> PP_HD i64 box_volume(const I *lo, const I *hi) {
  i64 v = 1;
  for (int d = 0; d < 4; ++d) v *= hi[d] > lo[d] ? static_cast<i64>(hi[d] - lo[d]) : 0;
  return v;
}

/* Per-dimension statistics of the overlaps o(x) = |[xP,(x+1)P) ∩ [a,b)| over
 * the source pieces x, in O(1): the best overlap, whether exactly one piece
 * attains it (and which), and the best over every other piece.  Used by K1 to
 * take max_{p != q} prod_d o_d(p_d) without enumerating p. */
template <class I> struct DimStats {
  I best, second, arg;
  bool unique;
};

template <class I> PP_HD DimStats<I> dim_stats(I a, I b, I P) {
  DimStats<I> s{0, 0, 0, false};
  if (b <= a) return s; /* every piece overlaps nothing */
  const I x0 = a / P, x1 = (b - 1) / P;
  if (x0 == x1) {
    s.best = b - a, s.arg = x0, s.unique = true, s.second = 0;
    return s;
  }
  const I o0 = (x0 + 1) * P - a, o1 = b - x1 * P;
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
  /* x1 >= x0 + 2: the middle pieces are fully covered (overlap P >= o0, o1) */
  const I full = (x1 - x0 - 1) + (o0 == P) + (o1 == P);
  s.best = P;
  if (full >= 2) {
    s.second = P, s.unique = false;
  } else {
    s.unique = true, s.arg = x0 + 1, s.second = imax<I>(o0, o1);
  }
  return s;
}

/* max over source partitions p != q of vol(owned_src(p) ∩ need), source config
 * `scfg` with piece sizes `piece` (cost.hpp:108-112: identity placement, so
 * p == q means the same device). */
template <class I> PP_HD i64 max_offdiag_volume(const I *piece, const I *scfg, const I *nlo, const I *nhi, I q) {
  DimStats<I> st[4];
  i64 M = 1;
  bool unique = true;
  for (int d = 0; d < 4; ++d) {
    st[d] = dim_stats<I>(nlo[d], nhi[d], piece[d]);
    M *= static_cast<i64>(st[d].best);
    unique = unique && st[d].unique;
  }
  if (M == 0) return 0;
  if (!unique) return M; /* two or more maximisers: one of them is != q */
  const I pstar = ((st[0].arg * scfg[1] + st[1].arg) * scfg[2] + st[2].arg) * scfg[3] + st[3].arg;
  if (pstar != q) return M;
  i64 best = 0;
  for (int d = 0; d < 4; ++d) {
    i64 v = st[d].second;
    for (int e = 0; e < 4; ++e)
      if (e != d) v *= static_cast<i64>(st[e].best);
    best = imax<i64>(best, v);
  }
  return best;
}

/* ---- cost formulas (cost.hpp:28-94) ---------------------------------------- */

PP_HD i64 layer_flops(int kind, const i64 *p, const i64 *o, const i64 *in) {
  switch (kind) {
  case kConv:
    return 2 * o[0] * o[1] * o[2] * o[3] * in[1] * p[1] * p[2];
  case kPool:
    return o[0] * o[1] * o[2] * o[3] * p[0] * p[1];
  case kFC:
    return 2 * o[0] * (in[0] * in[1] * in[2] * in[3]) / in[0] * o[1];
  case kSoftmax:
    return 5 * o[0] * o[1];
  default:
    return 0;
  }
}

PP_HD double parameter_bytes(int kind, const i64 *p, const i64 *o, const i64 *in) {
  if (kind == kConv)
    return 4.0 * static_cast<double>(o[1]) * static_cast<double>(in[1]) * static_cast<double>(p[1]) *
           static_cast<double>(p[2]);
  if (kind == kFC) return 4.0 * static_cast<double>((in[0] * in[1] * in[2] * in[3]) / in[0]) * static_cast<double>(o[1]);
  return 0.0;
}

/* compute_cost with the slowest assigned device's rate already reduced */
PP_HD double compute_seconds(i64 flops, i64 total, double slowest) {
  if (flops == 0) return 0.0;
  return static_cast<double>(flops) / static_cast<double>(total) * 3.0 / slowest;
}

} // namespace geo
} // namespace parplan
