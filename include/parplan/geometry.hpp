/* parplan/geometry.hpp — the pure partition/cost formulas, shared verbatim by
 * the host API and the sm_100a kernels (PP_HD = __host__ __device__ under nvcc).
 *
 * Nothing here allocates or throws; every function works on plain int64
 * arrays in (sample, channel, height, width) order so the same definition runs
 * in the xfer-table kernel (K1), the node-cost kernel (K2) and the host-side
 * single-call API (owned_region, required_input_region, transfer_profile).
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

PP_HD i64 imin(i64 a, i64 b) { return a < b ? a : b; }
PP_HD i64 imax(i64 a, i64 b) { return a > b ? a : b; }

/* conv/pool output extent (graph.hpp:257-259) */
PP_HD i64 conv_out(i64 in, i64 k, i64 s, i64 p) { return (in + 2 * p - k) / s + 1; }

PP_HD i64 config_total(const i64 *c) { return c[0] * c[1] * c[2] * c[3]; }

/* Row-major decode of a partition index, W fastest (partition.hpp:213-232). */
PP_HD void decode_part(const i64 *cfg, i64 part, i64 *idx) {
  for (int d = 3; d >= 0; --d) {
    idx[d] = part % cfg[d];
    part /= cfg[d];
  }
}

/* owned_region: equal contiguous pieces of extent/deg per dimension */
PP_HD void owned_box(const i64 *shape, const i64 *cfg, i64 part, i64 *lo, i64 *hi) {
  i64 idx[4];
  decode_part(cfg, part, idx);
  for (int d = 0; d < 4; ++d) {
    const i64 piece = shape[d] / cfg[d];
    lo[d] = idx[d] * piece;
    hi[d] = lo[d] + piece;
  }
}

/* map_spatial_window (partition.hpp:236-245) */
PP_HD void window(i64 own_lo, i64 own_hi, i64 k, i64 s, i64 p, i64 ext, i64 *lo, i64 *hi) {
  const i64 a = own_lo * s - p;
  const i64 b = (own_hi - 1) * s - p + k;
  *lo = imax(0, a);
  *hi = imin(ext, b);
  if (*hi < *lo) *hi = *lo;
}

/* flat_range_box (partition.hpp:249-273): bounding box in (C, H, W) of the
 * flattened index range [flo, fhi), flat = (c*H + h)*W + w. */
PP_HD void flat_box(i64 flo, i64 fhi, i64 H, i64 W, i64 *lo, i64 *hi) {
  const i64 plane = H * W;
  const i64 clo = flo / plane, chi = (fhi - 1) / plane;
  lo[1] = clo;
  hi[1] = chi + 1;
  if (clo != chi) {
    lo[2] = 0, hi[2] = H, lo[3] = 0, hi[3] = W;
    return;
  }
  const i64 rlo = (flo % plane) / W, rhi = ((fhi - 1) % plane) / W;
  lo[2] = rlo;
  hi[2] = rhi + 1;
  if (rlo != rhi) {
    lo[3] = 0, hi[3] = W;
    return;
  }
  lo[3] = flo % W;
  hi[3] = (fhi - 1) % W + 1;
}

/* required_input_region (partition.hpp:283-350) for destination partition
 * `part` under config `dcfg`.  `p` = destination kind parameters, `ins` = the
 * edge's tensor shape (source output), `outs` = destination output shape,
 * `band_offset` = for Concat, the sum of the preceding siblings' extents on the
 * concat axis (partition.hpp:331-337, precomputed by the caller).
 * Returns false for kinds that consume no inputs (Input). */
PP_HD bool required_box(int kind, const i64 *p, const i64 *ins, const i64 *outs, i64 band_offset, const i64 *dcfg,
                        i64 part, i64 *lo, i64 *hi) {
  i64 olo[4], ohi[4];
  owned_box(outs, dcfg, part, olo, ohi);
  for (int d = 0; d < 4; ++d) lo[d] = 0, hi[d] = 0;
  lo[0] = olo[0];
  hi[0] = ohi[0];
  switch (kind) {
  case kConv:
    lo[1] = 0, hi[1] = ins[1];
    window(olo[2], ohi[2], p[1], p[3], p[5], ins[2], &lo[2], &hi[2]);
    window(olo[3], ohi[3], p[2], p[4], p[6], ins[3], &lo[3], &hi[3]);
    return true;
  case kPool:
    lo[1] = olo[1], hi[1] = ohi[1];
    window(olo[2], ohi[2], p[0], p[2], p[4], ins[2], &lo[2], &hi[2]);
    window(olo[3], ohi[3], p[1], p[3], p[5], ins[3], &lo[3], &hi[3]);
    return true;
  case kFC:
    lo[1] = 0, hi[1] = ins[1];
    lo[2] = 0, hi[2] = ins[2];
    lo[3] = 0, hi[3] = ins[3];
    return true;
  case kFlatten:
    flat_box(olo[1], ohi[1], ins[2], ins[3], lo, hi);
    return true;
  case kConcat: {
    const int A = static_cast<int>(p[0]);
    for (int d = 0; d < 4; ++d) lo[d] = olo[d], hi[d] = ohi[d];
    lo[A] = imax(olo[A], band_offset);
    hi[A] = imin(ohi[A], band_offset + ins[A]);
    if (hi[A] < lo[A]) hi[A] = lo[A];
    lo[A] -= band_offset;
    hi[A] -= band_offset;
    return true;
  }
  case kSoftmax:
    for (int d = 0; d < 4; ++d) lo[d] = olo[d], hi[d] = ohi[d];
    return true;
  default:
    return false;
  }
}

PP_HD i64 box_volume(const i64 *lo, const i64 *hi) {
  i64 v = 1;
  for (int d = 0; d < 4; ++d) v *= hi[d] > lo[d] ? hi[d] - lo[d] : 0;
  return v;
}

/* Overlap of piece x (of size P) with [a, b). */
PP_HD i64 piece_overlap(i64 x, i64 P, i64 a, i64 b) { return imax(0, imin((x + 1) * P, b) - imax(x * P, a)); }

/* Per-dimension statistics of the overlaps o(x) = |[xP,(x+1)P) ∩ [a,b)| over
 * the deg source pieces x, in O(1): the best overlap, whether it is attained
 * by exactly one piece (and which), and the best over every other piece.
 * Used by K1 to take max_{p != q} prod_d o_d(p_d) without enumerating p. */
struct DimStats {
  i64 best, second, arg;
  bool unique;
};

PP_HD DimStats dim_stats(i64 a, i64 b, i64 P, i64 deg) {
  DimStats s{0, 0, 0, false};
  if (b <= a) return s; /* every piece overlaps nothing; best 0 attained by all */
  const i64 x0 = a / P, x1 = (b - 1) / P;
  if (x0 == x1) {
    s.best = b - a, s.arg = x0, s.unique = true, s.second = 0;
    return s;
  }
  const i64 o0 = (x0 + 1) * P - a, o1 = b - x1 * P;
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
  /* x1 >= x0 + 2: middle pieces are fully covered (overlap P >= o0, o1) */
  const i64 full = (x1 - x0 - 1) + (o0 == P) + (o1 == P);
  s.best = P;
  if (full >= 2) {
    s.second = P, s.unique = false;
  } else {
    s.unique = true, s.arg = x0 + 1, s.second = imax(o0, o1);
  }
  (void)deg;
  return s;
}

/* max over source partitions p != q of vol(owned_src(p) ∩ need), with the
 * source config `scfg` over source shape `sshape` (cost.hpp:108-112 semantics:
 * identity placement, so p == q means the same device). */
PP_HD i64 max_offdiag_volume(const i64 *sshape, const i64 *scfg, const i64 *nlo, const i64 *nhi, i64 q) {
  DimStats st[4];
  i64 M = 1;
  bool unique = true;
  for (int d = 0; d < 4; ++d) {
    st[d] = dim_stats(nlo[d], nhi[d], sshape[d] / scfg[d], scfg[d]);
    M *= st[d].best;
    unique = unique && st[d].unique;
  }
  if (M == 0) return 0;
  if (!unique) return M; /* two or more maximisers: one of them is != q */
  const i64 pstar = ((st[0].arg * scfg[1] + st[1].arg) * scfg[2] + st[2].arg) * scfg[3] + st[3].arg;
  if (pstar != q) return M;
  i64 best = 0;
  for (int d = 0; d < 4; ++d) {
    i64 v = st[d].second;
    for (int e = 0; e < 4; ++e)
      if (e != d) v *= st[e].best;
    best = imax(best, v);
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
