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
  int32_t small;      // 1: 16x16 output tiles (one cell per thread) for waves too small to fill the GPU
};

constexpr int kSmallTile = 16;

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

template <class T> struct WaveSmem {
  T As[kTile][kTile + 1];
  T Bs[kTile][kTile];
};

// Work item b of a wave: b < fold_tiles folds one 32x32 output tile of a fold
// (block-cooperative, uses `sm`); otherwise it adds one merge chunk.
template <class T>
__device__ __forceinline__ void wave_item(const FoldDesc<T> *folds, int n_folds, int64_t fold_tiles,
                                          const MergeDesc<T> *merges, int n_merges, int64_t b, WaveSmem<T> &sm) {
  auto &As = sm.As;
  auto &Bs = sm.Bs;
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
    if (f.small) { // 16x16 tile, one cell per thread, two interleaved scans
      const int i0 = static_cast<int>(tile / f.tiles_k) * kSmallTile;
      const int k0 = static_cast<int>(tile % f.tiles_k) * kSmallTile;
      const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
      T be = T(0), bo = T(0);
      int je = 0, jo = -1;
      T pa[2], pb[2];
      auto fetch = [&](int j0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int idx = threadIdx.x + q * kFoldThreads;
          const int r = idx >> 5, c = idx & 31; // A: 16 rows x 32 j
          const int i = i0 + r, j = j0 + c;
          pa[q] = (i < f.nu && j < f.nw) ? T(f.w[j] + f.t1[static_cast<int64_t>(i) * f.nw + j]) : T(0);
          const int jr = idx >> 4, kc = idx & 15; // B: 32 j x 16 cols
          const int jj = j0 + jr, k = k0 + kc;
          pb[q] = (jj < f.nw && k < f.nv) ? f.t2[static_cast<int64_t>(jj) * f.nv + k] : T(0);
        }
      };
      fetch(0);
      for (int j0 = 0; j0 < f.nw; j0 += kTile) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int idx = threadIdx.x + q * kFoldThreads;
          As[idx >> 5][idx & 31] = pa[q];
          Bs[idx >> 4][idx & 15] = pb[q];
        }
        __syncthreads();
        if (j0 + kTile < f.nw) fetch(j0 + kTile);
        const int jn = min(kTile, f.nw - j0);
        int jj = 0;
        for (; jj + 1 < jn; jj += 2) {
          const T c0 = As[ty][jj] + Bs[jj][tx];
          const T c1 = As[ty][jj + 1] + Bs[jj + 1][tx];
          const int j = j0 + jj;
          if (j == 0 || c0 < be) be = c0, je = j;
          if (jo < 0 || c1 < bo) bo = c1, jo = j + 1;
        }
        if (jj < jn) {
          const T c0 = As[ty][jj] + Bs[jj][tx];
          const int j = j0 + jj;
          if (j == 0 || c0 < be) be = c0, je = j;
        }
        __syncthreads();
      }
      const int i = i0 + ty, k = k0 + tx;
      if (i < f.nu && k < f.nv) {
        const bool odd = jo >= 0 && (bo < be || (bo == be && jo < je));
        f.out[static_cast<int64_t>(i) * f.nv + k] = odd ? bo : be;
        f.am[static_cast<int64_t>(i) * f.nv + k] = static_cast<uint16_t>(odd ? jo : je);
      }
      return;
    }
    const int i0 = static_cast<int>(tile / f.tiles_k) * kTile;
    const int k0 = static_cast<int>(tile % f.tiles_k) * kTile;
    const int ty = threadIdx.x >> 3, tx = (threadIdx.x & 7) * 4;
    // two interleaved scans per cell (even / odd j) halve the compare chain;
    // each keeps its lowest j under strict <, and the merge prefers the lower
    // j on equal values — the reference's lowest-index argmin
    T be[4], bo[4];
    int je[4], jo[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) be[c] = bo[c] = T(0), je[c] = 0, jo[c] = -1;
    // register prefetch of the next 32-j chunk overlaps its load with compute
    T pa[4], pb[4];
    auto fetch = [&](int j0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = threadIdx.x + q * kFoldThreads, r = idx >> 5, c = idx & 31;
        const int i = i0 + r, j = j0 + c;
        pa[q] = (i < f.nu && j < f.nw) ? T(f.w[j] + f.t1[static_cast<int64_t>(i) * f.nw + j]) : T(0);
        const int jj = j0 + r, k = k0 + c;
        pb[q] = (jj < f.nw && k < f.nv) ? f.t2[static_cast<int64_t>(jj) * f.nv + k] : T(0);
      }
    };
    fetch(0);
    for (int j0 = 0; j0 < f.nw; j0 += kTile) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = threadIdx.x + q * kFoldThreads;
        As[idx >> 5][idx & 31] = pa[q];
        Bs[idx >> 5][idx & 31] = pb[q];
      }
      __syncthreads();
      if (j0 + kTile < f.nw) fetch(j0 + kTile);
      const int jn = min(kTile, f.nw - j0);
      int jj = 0;
      for (; jj + 1 < jn; jj += 2) {
        const T a0 = As[ty][jj], a1 = As[ty][jj + 1];
        const int j = j0 + jj;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const T c0 = a0 + Bs[jj][tx + c];
          const T c1 = a1 + Bs[jj + 1][tx + c];
          if (j == 0 || c0 < be[c]) be[c] = c0, je[c] = j;
          if (jo[c] < 0 || c1 < bo[c]) bo[c] = c1, jo[c] = j + 1;
        }
      }
      if (jj < jn) { // odd chunk length (the last chunk only)
        const T a0 = As[ty][jj];
        const int j = j0 + jj;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const T c0 = a0 + Bs[jj][tx + c];
          if (j == 0 || c0 < be[c]) be[c] = c0, je[c] = j;
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
          const bool odd = jo[c] >= 0 && (bo[c] < be[c] || (bo[c] == be[c] && jo[c] < je[c]));
          f.out[static_cast<int64_t>(i) * f.nv + k] = odd ? bo[c] : be[c];
          f.am[static_cast<int64_t>(i) * f.nv + k] = static_cast<uint16_t>(odd ? jo[c] : je[c]);
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

// One launch per wave: blocks [0, fold_tiles) fold 32x32 output tiles, the
// rest add merge chunks.
template <class T>
__global__ void __launch_bounds__(kFoldThreads) wave_kernel(const FoldDesc<T> *folds, int n_folds, int64_t fold_tiles,
                                                            const MergeDesc<T> *merges, int n_merges) {
  __shared__ WaveSmem<T> sm;
  wave_item<T>(folds, n_folds, fold_tiles, merges, n_merges, blockIdx.x, sm);
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

// Virtual block vb of the enumeration: kEnumThreads threads x per_thread
// consecutive candidates each; writes the block's best to blk_val/blk_idx[vb].
template <class T>
__device__ __forceinline__ void enum_block(const EnumNode *nodes, int k, const EnumEdge *edges, int m, int64_t total,
                                           int64_t per_thread, typename Acc<T>::type *blk_val, int64_t *blk_idx,
                                           int64_t vb) {
  using A = typename Acc<T>::type;
  const int64_t t = vb * static_cast<int64_t>(kEnumThreads) + threadIdx.x;
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
  if (threadIdx.x == 0) blk_val[vb] = sv[0], blk_idx[vb] = si[0];
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(kEnumThreads)
    enum_kernel(const EnumNode *nodes, int k, const EnumEdge *edges, int m, int64_t total, int64_t per_thread,
                typename Acc<T>::type *blk_val, int64_t *blk_idx) {
  enum_block<T>(nodes, k, edges, m, total, per_thread, blk_val, blk_idx, blockIdx.x);
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
  // unwind + re-sum (n_rec < 0 skips both); recs sorted by wave, last wave
  // first; group g = recs[group_begin[g], group_begin[g+1])
  const UnwindRec *recs;
  int n_rec;
  const int32_t *group_begin;
  int n_groups;
  double *terms; // [nl + ne] scratch
  // optional zero-copy of the result block (indices, digits, final cost, cost)
  unsigned char *host_res;
  const unsigned char *dev_res;
  size_t res_bytes; // multiple of 4
  int32_t *indices;
  int nl;
  const void *onode, *oxfer;
  const int64_t *cat_off, *xoff;
  const int32_t *esrc, *edst, *counts;
  int ne;
  double *cost;
};

constexpr int kFinishThreads = 256;

// One CTA: reduces the per-block bests (value, then lowest linear index),
// decodes the winner's digits and — when records are given — unwinds the log
// and re-sums the plan cost from the ORIGINAL tables in the pinned order.
// The unwind walks dependency waves backwards: the endpoints of a record of
// wave w are eliminated (if ever) at waves > w, so every record of a wave is
// independent and the CTA processes a wave in parallel (planner.hpp:309-319).
// The cost terms are gathered in parallel, then summed by one thread in the
// reference's order (cost.hpp:235-246) — bit-identical.
template <class T> __device__ __forceinline__ void finish_block(const FinishArgs &a);

template <class T> __global__ void __launch_bounds__(kFinishThreads) finish_kernel(FinishArgs a) {
  finish_block<T>(a);
}

template <class T> __device__ __forceinline__ void finish_block(const FinishArgs &a) {
  using A = typename Acc<T>::type;
  __shared__ A sv[kFinishThreads];
  __shared__ int64_t si[kFinishThreads];
  const A *bv = static_cast<const A *>(a.blk_val);
  A best = A(0);
  int64_t bi = INT64_MAX;
  for (int b = threadIdx.x; b < a.nblk; b += kFinishThreads) {
    const int64_t oi = a.blk_idx[b];
    if (oi == INT64_MAX) continue;
    const A ov = bv[b];
    if (bi == INT64_MAX || ov < best || (ov == best && oi < bi)) best = ov, bi = oi;
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = kFinishThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const A ov = sv[threadIdx.x + s];
      const int64_t oi = si[threadIdx.x + s];
      if (oi != INT64_MAX &&
          (si[threadIdx.x] == INT64_MAX || ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])))
        sv[threadIdx.x] = ov, si[threadIdx.x] = oi;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int64_t r = si[0];
    for (int d = a.k - 1; d >= 0; --d) {
      a.digits[d] = static_cast<int32_t>(r % a.nodes[d].count);
      r /= a.nodes[d].count;
    }
    *a.final_cost = ldexp(static_cast<double>(sv[0]), -a.shift);
  }
  if (a.n_rec < 0) return;
  __syncthreads();
  for (int l = threadIdx.x; l < a.nl; l += kFinishThreads) a.indices[l] = -1;
  __syncthreads();
  for (int d = threadIdx.x; d < a.k; d += kFinishThreads) a.indices[a.node_layer[d]] = a.digits[d];
  __syncthreads();
  for (int gidx = 0; gidx < a.n_groups; ++gidx) { // waves, last first
    for (int q = a.group_begin[gidx] + threadIdx.x; q < a.group_begin[gidx + 1]; q += kFinishThreads) {
      const UnwindRec u = a.recs[q];
      a.indices[u.removed] = u.am[static_cast<int64_t>(a.indices[u.src]) * u.cols + a.indices[u.dst]];
    }
    __syncthreads();
  }
  const T *onode = static_cast<const T *>(a.onode);
  const T *oxfer = static_cast<const T *>(a.oxfer);
  for (int l = threadIdx.x; l < a.nl; l += kFinishThreads)
    a.terms[l] = ldexp(static_cast<double>(onode[a.cat_off[l] + a.indices[l]]), -a.shift);
  for (int e = threadIdx.x; e < a.ne; e += kFinishThreads)
    a.terms[a.nl + e] = ldexp(
        static_cast<double>(oxfer[a.xoff[e] + static_cast<int64_t>(a.indices[a.esrc[e]]) * a.counts[a.edst[e]] +
                                  a.indices[a.edst[e]]]),
        -a.shift);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int x = 0; x < a.nl + a.ne; ++x) t += a.terms[x];
    *a.cost = t;
  }
  if (a.host_res) { // zero-copy: results straight into pinned host memory
    __syncthreads();
    for (size_t b = threadIdx.x; b < a.res_bytes / 4; b += kFinishThreads)
      reinterpret_cast<volatile uint32_t *>(a.host_res)[b] = reinterpret_cast<const uint32_t *>(a.dev_res)[b];
    __threadfence_system();
  }
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
