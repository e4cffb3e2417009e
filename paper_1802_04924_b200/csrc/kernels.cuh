// kernels.cuh — device kernels of the elimination DP.
//
//   K3 fold   Eq. 2 node elimination (planner.hpp:139-155):
//             out[i][k] = min_j ((w[j] + t1[i][j]) + t2[j][k]), argmin = lowest j
//   K4 merge  Eq. 3 edge elimination (planner.hpp:194-199): out = t1 + t2
//   K5 enum   enumerate_final (planner.hpp:256-304) / brute_force_plan
//             (oracle.hpp:52-93): odometer over the joint index space with the
//             reference summation order, lowest linear index on ties
//   finish    K5 block reduce + unwind (planner.hpp:309-319) + cost re-sum
//             (cost.hpp:235-246)
// T = double (analytic tables) or int32_t (certified fixed point).
#pragma once

#include <cstdint>
#include <climits>

namespace pp {

template <class T> struct FoldDesc {
  const T *t1; // [nu][nw]
  const T *t2; // [nw][nv]
  const T *w;  // [nw]
  T *out;      // [nu][nv]
  uint16_t *am;
  int32_t nu, nw, nv;
  int32_t tiles_k;    // tiles along nv
  int64_t tile_begin; // first global tile id of this fold
};

template <class T> struct MergeDesc {
  const T *a, *b;
  T *out;
  int64_t n;
  int64_t blk_begin;
};

constexpr int kTile = 32;
constexpr int kFoldThreads = 256;
constexpr int kMergeThreads = 256;
constexpr int kMergePerBlock = kMergeThreads * 8;

// One launch per wave: blocks [0, fold_tiles) fold 32x32 output tiles, the
// rest add merge chunks.
template <class T>
__global__ void __launch_bounds__(kFoldThreads) wave_kernel(const FoldDesc<T> *folds, int n_folds, int64_t fold_tiles,
                                                            const MergeDesc<T> *merges, int n_merges) {
  __shared__ T As[kTile][kTile + 1];
  __shared__ T Bs[kTile][kTile];
  const int64_t b = blockIdx.x;
  if (b < fold_tiles) {
    int lo = 0, hi = n_folds - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (folds[mid].tile_begin <= b)
        lo = mid;
      else
        hi = mid - 1;
    }
    const FoldDesc<T> f = folds[lo];
    const int64_t tile = b - f.tile_begin;
    const int i0 = static_cast<int>(tile / f.tiles_k) * kTile;
    const int k0 = static_cast<int>(tile % f.tiles_k) * kTile;
    const int ty = threadIdx.x >> 3, tx = (threadIdx.x & 7) * 4;
    T best[4];
    int bj[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) best[c] = T(0), bj[c] = 0;
    for (int j0 = 0; j0 < f.nw; j0 += kTile) {
      for (int idx = threadIdx.x; idx < kTile * kTile; idx += kFoldThreads) {
        const int r = idx >> 5, c = idx & 31;
        const int i = i0 + r, j = j0 + c;
        As[r][c] = (i < f.nu && j < f.nw) ? T(f.w[j] + f.t1[static_cast<int64_t>(i) * f.nw + j]) : T(0);
        const int jj = j0 + r, k = k0 + c;
        Bs[r][c] = (jj < f.nw && k < f.nv) ? f.t2[static_cast<int64_t>(jj) * f.nv + k] : T(0);
      }
      __syncthreads();
      const int jn = min(kTile, f.nw - j0);
      for (int jj = 0; jj < jn; ++jj) {
        const T a = As[ty][jj];
        const int j = j0 + jj;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const T cand = a + Bs[jj][tx + c];
          if (j == 0 || cand < best[c]) best[c] = cand, bj[c] = j; // strict <: lowest j wins
        }
      }
      __syncthreads();
    }
    const int i = i0 + ty;
    if (i < f.nu)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int k = k0 + tx + c;
        if (k < f.nv) {
          f.out[static_cast<int64_t>(i) * f.nv + k] = best[c];
          f.am[static_cast<int64_t>(i) * f.nv + k] = static_cast<uint16_t>(bj[c]);
        }
      }
    return;
  }
  const int64_t mb = b - fold_tiles;
  int lo = 0, hi = n_merges - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (merges[mid].blk_begin <= mb)
      lo = mid;
    else
      hi = mid - 1;
  }
  const MergeDesc<T> m = merges[lo];
  const int64_t base = (mb - m.blk_begin) * kMergePerBlock;
  for (int64_t k = base + threadIdx.x; k < m.n && k < base + kMergePerBlock; k += kMergeThreads)
    m.out[k] = m.a[k] + m.b[k];
}

// K5: odometer over prod(counts) candidates (last digit fastest); cost =
// 0 + sum nodes (list order) + sum edges (list order); per-block best.
struct EnumNode {
  const void *tab;
  int32_t count;
  int32_t pad;
};
struct EnumEdge {
  const void *tab;
  int32_t ps, pd; // positions of the endpoints in the node list
  int32_t cols;
  int32_t pad;
};

template <class T> struct Acc;
template <> struct Acc<double> {
  using type = double;
};
template <> struct Acc<int32_t> {
  using type = long long;
};

constexpr int kEnumThreads = 256;
constexpr int kMaxEnumNodes = 128;

template <class T>
__global__ void __launch_bounds__(kEnumThreads)
    enum_kernel(const EnumNode *nodes, int k, const EnumEdge *edges, int m, int64_t total, int64_t per_thread,
                typename Acc<T>::type *blk_val, int64_t *blk_idx) {
  using A = typename Acc<T>::type;
  const int64_t t = blockIdx.x * static_cast<int64_t>(kEnumThreads) + threadIdx.x;
  int64_t start = t * per_thread, end = min(total, start + per_thread);
  A best = A(0);
  int64_t bidx = INT64_MAX;
  if (start < end) {
    int digit[kMaxEnumNodes];
    int64_t r = start;
    for (int d = k - 1; d >= 0; --d) {
      digit[d] = static_cast<int>(r % nodes[d].count);
      r /= nodes[d].count;
    }
    for (int64_t lin = start; lin < end; ++lin) {
      A c = A(0);
      for (int d = 0; d < k; ++d) c += static_cast<A>(static_cast<const T *>(nodes[d].tab)[digit[d]]);
      for (int e = 0; e < m; ++e)
        c += static_cast<A>(static_cast<const T *>(
            edges[e].tab)[static_cast<int64_t>(digit[edges[e].ps]) * edges[e].cols + digit[edges[e].pd]]);
      if (bidx == INT64_MAX || c < best) best = c, bidx = lin;
      for (int d = k - 1; d >= 0; --d) { // odometer step
        if (++digit[d] < nodes[d].count) break;
        digit[d] = 0;
      }
    }
  }
  __shared__ A sv[kEnumThreads];
  __shared__ int64_t si[kEnumThreads];
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = kEnumThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const A ov = sv[threadIdx.x + s];
      const int64_t oi = si[threadIdx.x + s];
      if (oi != INT64_MAX &&
          (si[threadIdx.x] == INT64_MAX || ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])))
        sv[threadIdx.x] = ov, si[threadIdx.x] = oi;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) blk_val[blockIdx.x] = sv[0], blk_idx[blockIdx.x] = si[0];
}

struct UnwindRec {
  const uint16_t *am;
  int32_t removed, src, dst, cols;
};

struct FinishArgs {
  const void *blk_val;
  const int64_t *blk_idx;
  int nblk;
  const EnumNode *nodes;
  int k;
  const int32_t *node_layer;
  int32_t *digits;
  double *final_cost;
  int shift;
  // unwind + re-sum (n_rec < 0 skips both)
  const UnwindRec *recs;
  int n_rec;
  int32_t *indices;
  int nl;
  const void *onode, *oxfer;
  const int64_t *cat_off, *xoff;
  const int32_t *esrc, *edst, *counts;
  int ne;
  double *cost;
};

// Reduces the per-block bests, decodes the winner's digits and — when records
// are given — unwinds the log and re-sums the plan cost from the ORIGINAL
// tables in the pinned order.
template <class T> __global__ void finish_kernel(FinishArgs a) {
  using A = typename Acc<T>::type;
  if (threadIdx.x != 0) return;
  const A *bv = static_cast<const A *>(a.blk_val);
  A best = A(0);
  int64_t bi = INT64_MAX;
  for (int b = 0; b < a.nblk; ++b) {
    const int64_t oi = a.blk_idx[b];
    if (oi == INT64_MAX) continue;
    const A ov = bv[b];
    if (bi == INT64_MAX || ov < best || (ov == best && oi < bi)) best = ov, bi = oi;
  }
  int64_t r = bi;
  for (int d = a.k - 1; d >= 0; --d) {
    a.digits[d] = static_cast<int32_t>(r % a.nodes[d].count);
    r /= a.nodes[d].count;
  }
  *a.final_cost = ldexp(static_cast<double>(best), -a.shift);
  if (a.n_rec < 0) return;
  for (int l = 0; l < a.nl; ++l) a.indices[l] = -1;
  for (int d = 0; d < a.k; ++d) a.indices[a.node_layer[d]] = a.digits[d];
  for (int q = a.n_rec - 1; q >= 0; --q) { // planner.hpp:309-319
    const UnwindRec &u = a.recs[q];
    a.indices[u.removed] = u.am[static_cast<int64_t>(a.indices[u.src]) * u.cols + a.indices[u.dst]];
  }
  const T *onode = static_cast<const T *>(a.onode);
  const T *oxfer = static_cast<const T *>(a.oxfer);
  double t = 0.0; // cost.hpp:235-246
  for (int l = 0; l < a.nl; ++l) t += ldexp(static_cast<double>(onode[a.cat_off[l] + a.indices[l]]), -a.shift);
  for (int e = 0; e < a.ne; ++e)
    t += ldexp(static_cast<double>(oxfer[a.xoff[e] + static_cast<int64_t>(a.indices[a.esrc[e]]) * a.counts[a.edst[e]] +
                                         a.indices[a.edst[e]]]),
               -a.shift);
  *a.cost = t;
}

template <class T> __global__ void to_double_kernel(const T *in, double *out, int64_t n, int shift) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = ldexp(static_cast<double>(in[k]), -shift);
}

static __global__ void widen_u16_kernel(const uint16_t *in, int32_t *out, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = in[k];
}

} // namespace pp
