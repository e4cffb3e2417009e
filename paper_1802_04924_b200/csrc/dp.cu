// dp.cu — the elimination dynamic program on the device.
//
//   K3 fold   Eq. 2 node elimination (planner.hpp:139-155):
//             out[i][k] = min_j ((w[j] + t1[i][j]) + t2[j][k]), argmin = lowest j
//   K4 merge  Eq. 3 edge elimination (planner.hpp:194-199): out = t1 + t2
//   K5 enum   enumerate_final (planner.hpp:256-304) / brute_force_plan
//             (oracle.hpp:52-93): odometer over the joint index space with
//             the reference summation order, lowest linear index on ties
//   unwind    planner.hpp:309-319 + total_cost_by_index (cost.hpp:235-246)
//
// The host scheduler (scheduler.cpp) fixes the whole log up front; every
// wave of independent folds/merges is ONE launch over a work list, and the
// plan is: upload descriptors (1 copy) -> waves -> enum -> unwind -> 1 copy back.
// Arithmetic is FP64 (analytic tables) or exact int32 fixed point (certified
// dyadic tables); both reproduce the reference's FP64 results bit for bit.
#include "dp.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>

namespace pp {

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

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
        c += static_cast<A>(
            static_cast<const T *>(edges[e].tab)[static_cast<int64_t>(digit[edges[e].ps]) * edges[e].cols + digit[edges[e].pd]]);
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
      if (oi != INT64_MAX && (si[threadIdx.x] == INT64_MAX || ov < sv[threadIdx.x] ||
                              (ov == sv[threadIdx.x] && oi < si[threadIdx.x])))
        sv[threadIdx.x] = ov, si[threadIdx.x] = oi;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) blk_val[blockIdx.x] = sv[0], blk_idx[blockIdx.x] = si[0];
}

// Reduces the per-block bests, decodes the winner's digits into `digits`, and
// — when records are given — unwinds the log and re-sums the plan cost from
// the ORIGINAL tables in the pinned order.
struct UnwindRec {
  const uint16_t *am;
  int32_t removed, src, dst, cols;
};

template <class T>
__global__ void finish_kernel(const typename Acc<T>::type *blk_val, const int64_t *blk_idx, int nblk,
                              const EnumNode *nodes, int k, const int32_t *node_layer, int32_t *digits,
                              double *final_cost, int shift,
                              // unwind (optional: n_rec < 0 skips)
                              const UnwindRec *recs, int n_rec, int32_t *indices, int nl,
                              // re-sum (optional)
                              const T *onode, const T *oxfer, const int64_t *cat_off, const int64_t *xoff,
                              const int32_t *esrc, const int32_t *edst, const int32_t *counts, int ne, double *cost) {
  using A = typename Acc<T>::type;
  if (threadIdx.x != 0) return;
  A best = A(0);
  int64_t bi = INT64_MAX;
  for (int b = 0; b < nblk; ++b) {
    const int64_t oi = blk_idx[b];
    if (oi == INT64_MAX) continue;
    const A ov = blk_val[b];
    if (bi == INT64_MAX || ov < best || (ov == best && oi < bi)) best = ov, bi = oi;
  }
  int64_t r = bi;
  for (int d = k - 1; d >= 0; --d) {
    digits[d] = static_cast<int32_t>(r % nodes[d].count);
    r /= nodes[d].count;
  }
  *final_cost = ldexp(static_cast<double>(best), -shift);
  if (n_rec < 0) return;
  for (int l = 0; l < nl; ++l) indices[l] = -1;
  for (int d = 0; d < k; ++d) indices[node_layer[d]] = digits[d];
  for (int q = n_rec - 1; q >= 0; --q) { // planner.hpp:309-319
    const UnwindRec &u = recs[q];
    indices[u.removed] = u.am[static_cast<int64_t>(indices[u.src]) * u.cols + indices[u.dst]];
  }
  double t = 0.0; // cost.hpp:235-246
  for (int l = 0; l < nl; ++l) t += ldexp(static_cast<double>(onode[cat_off[l] + indices[l]]), -shift);
  for (int e = 0; e < ne; ++e)
    t += ldexp(static_cast<double>(oxfer[xoff[e] + static_cast<int64_t>(indices[esrc[e]]) * counts[edst[e]] + indices[edst[e]]]),
               -shift);
  *cost = t;
}

template <class T> __global__ void to_double_kernel(const T *in, double *out, int64_t n, int shift) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = ldexp(static_cast<double>(in[k]), -shift);
}

__global__ void widen_u16_kernel(const uint16_t *in, int32_t *out, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = in[k];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

template <class T> const T *orig_node(const Tables &t) {
  if constexpr (std::is_same_v<T, double>)
    return t.node.p;
  else
    return t.node32.p;
}
template <class T> const T *orig_xfer(const Tables &t) {
  if constexpr (std::is_same_v<T, double>)
    return t.xfer64.p;
  else
    return t.xfer32.p;
}

// Device memory of one DP run: derived tables + argmins.
struct Arena {
  DBuf<unsigned char> buf;
  size_t top = 0;
};

// First-fit allocator with liveness: offsets of derived tables; blocks freed
// after the wave that consumes them (never reused inside that wave).
class OffsetPlanner {
public:
  size_t alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= bytes) {
        const size_t off = it->first, rest = it->second - bytes;
        free_.erase(it);
        if (rest) free_[off + bytes] = rest;
        return off;
      }
    const size_t off = end_;
    end_ += bytes;
    return off;
  }
  void release(size_t off, size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    auto it = free_.emplace(off, bytes).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) it->second += nx->second, free_.erase(nx);
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) pv->second += it->second, free_.erase(it);
    }
  }
  size_t end() const { return end_; }

private:
  std::map<size_t, size_t> free_;
  size_t end_ = 0;
};

template <class T>
static void launch_wave(pp_context *ctx, const FoldDesc<T> *dfolds, int n_folds, int64_t fold_tiles,
                        const MergeDesc<T> *dmerges, int n_merges, int64_t merge_blocks) {
  const int64_t grid = fold_tiles + merge_blocks;
  if (!grid) return;
  PP_REQUIRE(grid < (int64_t(1) << 31), "wave too large for one launch");
  wave_kernel<T><<<static_cast<unsigned>(grid), kFoldThreads, 0, ctx->stream>>>(dfolds, n_folds, fold_tiles, dmerges,
                                                                                n_merges);
  check_launch(ctx);
}

template <class T>
static void plan_impl(pp_context *ctx, Graph &g, Tables &t, int k_bound, int32_t *indices, pp_plan_result *res) {
  const Schedule &s = g.schedule();
  const int K = static_cast<int>(s.final_nodes.size());
  if (K > k_bound)
    throw parplan::LimitError("final graph has " + std::to_string(K) + " nodes, exceeding the enumeration bound of " +
                              std::to_string(k_bound) + " (graph is not reducible enough)");
  PP_REQUIRE(K <= kMaxEnumNodes, "final graph too large for the enumeration kernel");

  const int E_total = static_cast<int>(s.esrc.size());
  std::vector<int32_t> rows(static_cast<size_t>(E_total)), cols(static_cast<size_t>(E_total));
  for (int id = 0; id < E_total; ++id) {
    rows[static_cast<size_t>(id)] = t.counts[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])];
    cols[static_cast<size_t>(id)] = t.counts[static_cast<size_t>(s.edst[static_cast<size_t>(id)])];
  }
  for (const Op &op : s.ops)
    if (!op.type) PP_REQUIRE(t.counts[static_cast<size_t>(op.removed)] <= 65535, "argmin index exceeds 16 bits");

  // ---- memory plan: derived tables (liveness-reused) + argmins (kept) ----
  const bool keep_all = [&] {
    size_t total = 0;
    for (const Op &op : s.ops) total += static_cast<size_t>(rows[static_cast<size_t>(op.ne)]) * cols[static_cast<size_t>(op.ne)] * sizeof(T);
    return total <= (size_t(4) << 30);
  }();
  std::vector<int> consumer_wave(static_cast<size_t>(E_total), INT_MAX);
  for (const Op &op : s.ops) {
    consumer_wave[static_cast<size_t>(op.e1)] = op.wave;
    consumer_wave[static_cast<size_t>(op.e2)] = op.wave;
  }
  OffsetPlanner tab_plan;
  std::vector<size_t> tab_off(static_cast<size_t>(E_total), 0);
  std::vector<size_t> am_off(s.ops.size(), 0);
  size_t am_bytes = 0;
  for (int w = 1; w <= s.n_waves; ++w) {
    for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
      const Op &op = s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])];
      const size_t cells = static_cast<size_t>(rows[static_cast<size_t>(op.ne)]) * cols[static_cast<size_t>(op.ne)];
      tab_off[static_cast<size_t>(op.ne)] = tab_plan.alloc(cells * sizeof(T));
      if (!op.type) {
        am_off[static_cast<size_t>(s.exec[static_cast<size_t>(x)])] = am_bytes;
        am_bytes += (cells * 2 + 255) & ~size_t(255);
      }
    }
    if (!keep_all)
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const Op &op = s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])];
        for (int in : {op.e1, op.e2})
          if (in >= t.ne)
            tab_plan.release(tab_off[static_cast<size_t>(in)],
                             static_cast<size_t>(rows[static_cast<size_t>(in)]) * cols[static_cast<size_t>(in)] * sizeof(T));
      }
  }
  const size_t tab_bytes = tab_plan.end();
  ctx->scratch.ensure(tab_bytes + am_bytes + 256);
  unsigned char *tab_base = ctx->scratch.p;
  unsigned char *am_base = ctx->scratch.p + ((tab_bytes + 255) & ~size_t(255));

  const T *onode = orig_node<T>(t);
  const T *oxfer = orig_xfer<T>(t);
  auto table = [&](int id) -> const T * {
    if (id < t.ne) return oxfer + t.xoff[static_cast<size_t>(id)];
    return reinterpret_cast<const T *>(tab_base + tab_off[static_cast<size_t>(id)]);
  };

  // ---- descriptors ----
  std::vector<FoldDesc<T>> folds;
  std::vector<MergeDesc<T>> merges;
  struct WaveRange {
    int f0, nf, m0, nm;
    int64_t ftiles, mblocks;
  };
  std::vector<WaveRange> waves;
  for (int w = 1; w <= s.n_waves; ++w) {
    WaveRange wr{static_cast<int>(folds.size()), 0, static_cast<int>(merges.size()), 0, 0, 0};
    for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
      const int oi = s.exec[static_cast<size_t>(x)];
      const Op &op = s.ops[static_cast<size_t>(oi)];
      T *out = reinterpret_cast<T *>(tab_base + tab_off[static_cast<size_t>(op.ne)]);
      if (!op.type) {
        FoldDesc<T> f;
        f.t1 = table(op.e1);
        f.t2 = table(op.e2);
        f.w = onode + t.cat_off[static_cast<size_t>(op.removed)];
        f.out = out;
        f.am = reinterpret_cast<uint16_t *>(am_base + am_off[static_cast<size_t>(oi)]);
        f.nu = rows[static_cast<size_t>(op.e1)];
        f.nw = t.counts[static_cast<size_t>(op.removed)];
        f.nv = cols[static_cast<size_t>(op.e2)];
        f.tiles_k = (f.nv + kTile - 1) / kTile;
        f.tile_begin = wr.ftiles;
        wr.ftiles += static_cast<int64_t>((f.nu + kTile - 1) / kTile) * f.tiles_k;
        folds.push_back(f);
        ++wr.nf;
      } else {
        MergeDesc<T> m;
        m.a = table(op.e1);
        m.b = table(op.e2);
        m.out = out;
        m.n = static_cast<int64_t>(rows[static_cast<size_t>(op.ne)]) * cols[static_cast<size_t>(op.ne)];
        m.blk_begin = wr.mblocks;
        wr.mblocks += (m.n + kMergePerBlock - 1) / kMergePerBlock;
        merges.push_back(m);
        ++wr.nm;
      }
    }
    waves.push_back(wr);
  }
  // enumeration over the final graph (live nodes ascending, live edges by id)
  std::vector<EnumNode> en(static_cast<size_t>(K));
  std::vector<int32_t> node_layer(static_cast<size_t>(K));
  std::vector<int> pos(static_cast<size_t>(t.nl), -1);
  int64_t space = 1;
  for (int d = 0; d < K; ++d) {
    const int l = s.final_nodes[static_cast<size_t>(d)];
    en[static_cast<size_t>(d)] = EnumNode{onode + t.cat_off[static_cast<size_t>(l)], t.counts[static_cast<size_t>(l)], 0};
    node_layer[static_cast<size_t>(d)] = l;
    pos[static_cast<size_t>(l)] = d;
    PP_REQUIRE(space <= INT64_MAX / std::max(1, t.counts[static_cast<size_t>(l)]), "final enumeration space overflows");
    space *= t.counts[static_cast<size_t>(l)];
  }
  std::vector<EnumEdge> ee;
  for (int id : s.final_edges)
    ee.push_back(EnumEdge{table(id), pos[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])],
                          pos[static_cast<size_t>(s.edst[static_cast<size_t>(id)])], cols[static_cast<size_t>(id)], 0});
  std::vector<UnwindRec> recs;
  for (size_t oi = 0; oi < s.ops.size(); ++oi) {
    const Op &op = s.ops[oi];
    if (op.type) continue;
    recs.push_back(UnwindRec{reinterpret_cast<const uint16_t *>(am_base + am_off[oi]), op.removed, op.u, op.v,
                             cols[static_cast<size_t>(op.ne)]});
  }
  const int64_t per_thread = std::max<int64_t>(1, (space + int64_t(ctx->sms) * 8 * kEnumThreads - 1) /
                                                      (int64_t(ctx->sms) * 8 * kEnumThreads));
  const int64_t threads = (space + per_thread - 1) / per_thread;
  const int nblk = static_cast<int>((threads + kEnumThreads - 1) / kEnumThreads);

  using A = typename Acc<T>::type;
  std::vector<int32_t> es(t.esrc.begin(), t.esrc.end()), ed(t.edst.begin(), t.edst.end());
  Packer pk;
  const size_t oF = pk.put(folds), oM = pk.put(merges), oN = pk.put(en), oE = pk.put(ee), oR = pk.put(recs),
               oL = pk.put(node_layer), oCO = pk.put(t.cat_off), oXO = pk.put(t.xoff), oS = pk.put(es),
               oD = pk.put(ed), oC = pk.put(t.counts);
  const size_t oBV = pk.put(std::vector<A>(static_cast<size_t>(nblk))),
               oBI = pk.put(std::vector<int64_t>(static_cast<size_t>(nblk)));
  // results: digits[K], indices[nl], final_cost, cost (one contiguous copy back)
  const size_t oOut = pk.put(std::vector<unsigned char>(static_cast<size_t>(K) * 4 + static_cast<size_t>(t.nl) * 4 + 32));

  ctx->begin();
  const int64_t launches0 = ctx->launches;
  unsigned char *b = ctx->upload(pk);
  for (const WaveRange &wr : waves)
    launch_wave<T>(ctx, reinterpret_cast<const FoldDesc<T> *>(b + oF) + wr.f0, wr.nf, wr.ftiles,
                   reinterpret_cast<const MergeDesc<T> *>(b + oM) + wr.m0, wr.nm, wr.mblocks);
  enum_kernel<T><<<nblk, kEnumThreads, 0, ctx->stream>>>(
      reinterpret_cast<const EnumNode *>(b + oN), K, reinterpret_cast<const EnumEdge *>(b + oE),
      static_cast<int>(ee.size()), space, per_thread, reinterpret_cast<A *>(b + oBV), reinterpret_cast<int64_t *>(b + oBI));
  check_launch(ctx);
  unsigned char *outp = b + oOut;
  int32_t *d_digits = reinterpret_cast<int32_t *>(outp);
  int32_t *d_idx = d_digits + K;
  double *d_fc = reinterpret_cast<double *>(outp + ((static_cast<size_t>(K) * 4 + static_cast<size_t>(t.nl) * 4 + 7) & ~size_t(7)));
  finish_kernel<T><<<1, 32, 0, ctx->stream>>>(
      reinterpret_cast<const A *>(b + oBV), reinterpret_cast<const int64_t *>(b + oBI), nblk,
      reinterpret_cast<const EnumNode *>(b + oN), K, reinterpret_cast<const int32_t *>(b + oL), d_digits, d_fc,
      t.shift, reinterpret_cast<const UnwindRec *>(b + oR), static_cast<int>(recs.size()), d_idx, t.nl, onode, oxfer,
      reinterpret_cast<const int64_t *>(b + oCO), reinterpret_cast<const int64_t *>(b + oXO),
      reinterpret_cast<const int32_t *>(b + oS), reinterpret_cast<const int32_t *>(b + oD),
      reinterpret_cast<const int32_t *>(b + oC), t.ne, d_fc + 1);
  check_launch(ctx);
  const size_t out_bytes = (reinterpret_cast<unsigned char *>(d_fc + 2) - outp);
  unsigned char *h = static_cast<unsigned char *>(ctx->staging.p) + oOut; // staging holds the packed image
  PP_CUDA(cudaMemcpyAsync(h, outp, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  const double ms = ctx->end_ms();
  std::memcpy(indices, h + static_cast<size_t>(K) * 4, static_cast<size_t>(t.nl) * 4);
  double fc[2];
  std::memcpy(fc, h + (reinterpret_cast<unsigned char *>(d_fc) - outp), 16);
  if (res) {
    res->cost = fc[1];
    res->final_graph_nodes = K;
    res->node_eliminations = s.node_ops;
    res->edge_eliminations = s.edge_ops;
    res->precision = t.mode;
    res->waves = s.n_waves;
    res->launches = static_cast<int32_t>(ctx->launches - launches0);
    res->device_ms = ms;
  }
}

void run_plan(pp_context *ctx, Graph &g, Tables &t, int k_bound, int32_t *indices, pp_plan_result *res) {
  PP_REQUIRE(t.nl == g.nl && t.ne == g.ne, "tables do not match the graph");
  if (t.mode == kFP64)
    plan_impl<double>(ctx, g, t, k_bound, indices, res);
  else
    plan_impl<int32_t>(ctx, g, t, k_bound, indices, res);
}

// ---------------------------------------------------------------------------
// enumeration helper shared by ReducedGraph::enumerate_final and brute force
// ---------------------------------------------------------------------------

template <class T>
static void enumerate_impl(pp_context *ctx, const std::vector<EnumNode> &en, const std::vector<EnumEdge> &ee,
                           int shift, int32_t *digits, double *cost) {
  const int K = static_cast<int>(en.size());
  PP_REQUIRE(K <= kMaxEnumNodes, "too many nodes for the enumeration kernel");
  int64_t space = 1;
  for (const EnumNode &n : en) {
    PP_REQUIRE(space <= INT64_MAX / std::max(1, n.count), "enumeration space overflows");
    space *= n.count;
  }
  const int64_t per_thread = std::max<int64_t>(1, (space + int64_t(ctx->sms) * 8 * kEnumThreads - 1) /
                                                      (int64_t(ctx->sms) * 8 * kEnumThreads));
  const int64_t threads = (space + per_thread - 1) / per_thread;
  const int nblk = static_cast<int>((threads + kEnumThreads - 1) / kEnumThreads);
  using A = typename Acc<T>::type;
  Packer pk;
  const size_t oN = pk.put(en), oE = pk.put(ee), oBV = pk.put(std::vector<A>(static_cast<size_t>(nblk))),
               oBI = pk.put(std::vector<int64_t>(static_cast<size_t>(nblk))),
               oOut = pk.put(std::vector<unsigned char>(static_cast<size_t>(K) * 4 + 16));
  ctx->begin();
  unsigned char *b = ctx->upload(pk);
  enum_kernel<T><<<nblk, kEnumThreads, 0, ctx->stream>>>(reinterpret_cast<const EnumNode *>(b + oN), K,
                                                          reinterpret_cast<const EnumEdge *>(b + oE),
                                                          static_cast<int>(ee.size()), space, per_thread,
                                                          reinterpret_cast<A *>(b + oBV), reinterpret_cast<int64_t *>(b + oBI));
  check_launch(ctx);
  int32_t *d_digits = reinterpret_cast<int32_t *>(b + oOut);
  double *d_fc = reinterpret_cast<double *>(b + oOut + ((static_cast<size_t>(K) * 4 + 7) & ~size_t(7)));
  finish_kernel<T><<<1, 32, 0, ctx->stream>>>(reinterpret_cast<const A *>(b + oBV),
                                              reinterpret_cast<const int64_t *>(b + oBI), nblk,
                                              reinterpret_cast<const EnumNode *>(b + oN), K, nullptr, d_digits, d_fc,
                                              shift, nullptr, -1, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                                              nullptr, nullptr, nullptr, 0, nullptr);
  check_launch(ctx);
  unsigned char *h = static_cast<unsigned char *>(ctx->staging.p) + oOut;
  const size_t nbytes = (reinterpret_cast<unsigned char *>(d_fc + 1) - (b + oOut));
  PP_CUDA(cudaMemcpyAsync(h, b + oOut, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->end_ms();
  std::memcpy(digits, h, static_cast<size_t>(K) * 4);
  std::memcpy(cost, h + (reinterpret_cast<unsigned char *>(d_fc) - (b + oOut)), 8);
}

void run_enumerate(pp_context *ctx, int mode, int shift, const std::vector<const void *> &node_tabs,
                   const std::vector<int32_t> &counts, const std::vector<const void *> &edge_tabs,
                   const std::vector<int32_t> &eps, const std::vector<int32_t> &epd, const std::vector<int32_t> &ecols,
                   int32_t *digits, double *cost) {
  std::vector<EnumNode> en;
  for (size_t d = 0; d < node_tabs.size(); ++d) en.push_back(EnumNode{node_tabs[d], counts[d], 0});
  std::vector<EnumEdge> ee;
  for (size_t e = 0; e < edge_tabs.size(); ++e) ee.push_back(EnumEdge{edge_tabs[e], eps[e], epd[e], ecols[e], 0});
  if (mode == kFP64)
    enumerate_impl<double>(ctx, en, ee, 0, digits, cost);
  else
    enumerate_impl<int32_t>(ctx, en, ee, shift, digits, cost);
}

// ---------------------------------------------------------------------------
// single-op execution for the ReducedGraph step API
// ---------------------------------------------------------------------------

void run_single_op(pp_context *ctx, int mode, const Op &op, const void *t1, const void *t2, const void *w, void *out,
                   uint16_t *am, int nu, int nw, int nv) {
  Packer pk;
  int64_t tiles = 0, blocks = 0;
  size_t off;
  if (mode == kFP64) {
    if (!op.type) {
      FoldDesc<double> f{static_cast<const double *>(t1), static_cast<const double *>(t2), static_cast<const double *>(w),
                         static_cast<double *>(out), am, nu, nw, nv, (nv + kTile - 1) / kTile, 0};
      tiles = static_cast<int64_t>((nu + kTile - 1) / kTile) * f.tiles_k;
      off = pk.put(&f, 1);
    } else {
      MergeDesc<double> m{static_cast<const double *>(t1), static_cast<const double *>(t2), static_cast<double *>(out),
                          static_cast<int64_t>(nu) * nv, 0};
      blocks = (m.n + kMergePerBlock - 1) / kMergePerBlock;
      off = pk.put(&m, 1);
    }
  } else {
    if (!op.type) {
      FoldDesc<int32_t> f{static_cast<const int32_t *>(t1), static_cast<const int32_t *>(t2),
                          static_cast<const int32_t *>(w), static_cast<int32_t *>(out), am, nu, nw, nv,
                          (nv + kTile - 1) / kTile, 0};
      tiles = static_cast<int64_t>((nu + kTile - 1) / kTile) * f.tiles_k;
      off = pk.put(&f, 1);
    } else {
      MergeDesc<int32_t> m{static_cast<const int32_t *>(t1), static_cast<const int32_t *>(t2),
                           static_cast<int32_t *>(out), static_cast<int64_t>(nu) * nv, 0};
      blocks = (m.n + kMergePerBlock - 1) / kMergePerBlock;
      off = pk.put(&m, 1);
    }
  }
  ctx->begin();
  unsigned char *b = ctx->upload(pk);
  if (mode == kFP64)
    launch_wave<double>(ctx, reinterpret_cast<const FoldDesc<double> *>(b + off), op.type ? 0 : 1, tiles,
                        reinterpret_cast<const MergeDesc<double> *>(b + off), op.type ? 1 : 0, blocks);
  else
    launch_wave<int32_t>(ctx, reinterpret_cast<const FoldDesc<int32_t> *>(b + off), op.type ? 0 : 1, tiles,
                         reinterpret_cast<const MergeDesc<int32_t> *>(b + off), op.type ? 1 : 0, blocks);
  ctx->end_ms();
}

void download_table(pp_context *ctx, int mode, int shift, const void *src, int64_t n, double *out) {
  if (!n) return;
  ctx->begin();
  if (mode == kFP64) {
    PP_CUDA(cudaMemcpyAsync(out, src, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    DBuf<double> tmp(static_cast<size_t>(n));
    to_double_kernel<int32_t><<<ctx->sms * 4, 256, 0, ctx->stream>>>(static_cast<const int32_t *>(src), tmp.p, n, shift);
    check_launch(ctx);
    PP_CUDA(cudaMemcpyAsync(out, tmp.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    PP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->end_ms();
}

void download_argmin(pp_context *ctx, const uint16_t *src, int64_t n, int32_t *out) {
  if (!n) return;
  ctx->begin();
  DBuf<int32_t> tmp(static_cast<size_t>(n));
  widen_u16_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(src, tmp.p, n);
  check_launch(ctx);
  PP_CUDA(cudaMemcpyAsync(out, tmp.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->end_ms();
}

} // namespace pp
