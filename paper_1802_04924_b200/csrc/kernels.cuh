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
#include <type_traits>

namespace pp {

constexpr int kMaxEpi = 4;

template <class T> struct FoldDesc {
  const T *t1; // [nu][nw]
  const T *t2; // [nw][nv]
  const T *w;  // [nw]
  T *out;      // [nu][nv]
  uint16_t *am;
  int32_t nu, nw, nv;
  int32_t tiles_k;    // tiles along nv
  int64_t tile_begin; // first global tile id of this fold
  int32_t small;      // tile mode: 0 32x32 chunked, 1 16x16 chunked, kPanel16/8/4 panel tiles (nw <= kPanel)
  int32_t late;       // fused kernel: operands written by the previous wave (kPanelT1 | kPanelT2)
  // fused kernel: edge eliminations absorbed into this fold (Eq. 3 merges
  // whose other operand is ready before it runs): out = ((v + epi[0]) + epi[1]) ...,
  // one IEEE add per merge in the reference's merge order
  const T *epi[kMaxEpi];  // added table; with epi2: the merge (epi + epi2) is added
  const T *epi2[kMaxEpi];
  int32_t n_epi;
  int32_t pad;
};

// v with the fold's absorbed merges added, cell o of the [nu][nv] output
template <class T> __device__ __forceinline__ T fold_epilogue(const FoldDesc<T> &f, int64_t o, T v) {
  for (int e = 0; e < f.n_epi; ++e) {
    T x = __ldcg(&f.epi[e][o]);
    if (f.epi2[e]) x = x + __ldcg(&f.epi2[e][o]);
    v = v + x;
  }
  return v;
}

// Panel tiles: small-wave folds with nw <= kPanel stage the whole j range of
// an R x R output tile in shared memory with one batch of loads (one memory
// latency instead of one per 32-j chunk); 256 / R^2 thread groups split the j
// range (R = 16, 8, 4: 1, 4, 16 groups), shortening the per-thread scan when
// a wave has few tiles.  In the fused kernel the operands the previous wave
// did not write (w always, t1/t2 unless `late`) are staged before the barrier
// that ends that wave.
constexpr int kPanel = 128;
enum : int { kPanelW = 1, kPanelT1 = 2, kPanelT2 = 4, kPanelAll = 7 };
enum : int { kPanel16 = 2, kPanel8 = 3, kPanel4 = 4 };
__host__ __device__ constexpr int panel_side(int mode) { return mode == kPanel16 ? 16 : mode == kPanel8 ? 8 : 4; }

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

template <class T> struct TileSmem {
  T As[kTile][kTile + 1];
  T Bs[kTile][kTile];
};
template <class T> struct PanelSmem {
  T W[kPanel];
  T A[16 * (kPanel + 1)]; // w[j] + t1[i][j], R rows of stride kPanel + 1
  T B[kPanel * 17];       // t2[j][k], nw rows of R, stride R + 1 (conflict-free column reads)
};
// Chain segments (fused kernel): a run of waves whose folds form chains
// f1 -> f2 -> ... (f_{k+1}.t1 = f_k.out) with every t2 ready before the run.
// Row r of f_{k+1}.out depends on row r of f_k.out alone (Eq. 2 folds t1 row
// by row), so one block carries a few rows through the whole chain in shared
// memory: one grid barrier per segment instead of one per wave.
constexpr int kChainRows = 8;  // rows per item (max)
constexpr int kChainMax = 128; // max nw / nv of a chain fold
struct ChainDesc {
  int32_t first, n;  // folds [first, first + n) of the segment's fold list
  int32_t nu, rows;  // t1 rows, rows per item
  int64_t item_begin;
  // optional unwind path table [nu][nv of the last fold][n]: entry k = the
  // argmin of fold k along the chain's backtrack from (row, final column), so
  // the finish phase assigns the whole chain with one lookup
  uint16_t *path;
};

template <class T> union WaveSmem {
  TileSmem<T> t;
  PanelSmem<T> p;
};

// Shared memory of a chain item (dynamic, 16-byte-aligned sections):
// 2 mbarriers | fold descriptors[max_len] | A'[rows][kChainMax + 1] |
// cur[rows][kChainMax] | group minima (value, j)[kChainGroups][rows][kChainMax]
// | 2 staging buffers (a fold's t2 bytes + w bytes, each 16-byte-rounded).
constexpr int kChainGroups = kFoldThreads / 32; // j-groups = warps
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
template <class T> __host__ __device__ constexpr size_t chain_stage_bytes(int nw, int nv) {
  return align16(static_cast<size_t>(nw) * nv * sizeof(T) + 16) + align16(static_cast<size_t>(nw) * sizeof(T) + 16);
}
template <class T> __host__ __device__ constexpr size_t chain_smem_bytes(int rows, int max_len, size_t stage, bool path) {
  return 16 + align16(static_cast<size_t>(max_len) * sizeof(FoldDesc<T>)) +
         align16(static_cast<size_t>(rows) * (2 * kChainMax + 1) * sizeof(T)) +
         align16(static_cast<size_t>(kChainGroups) * rows * kChainMax * (sizeof(T) + 4)) + 2 * stage +
         (path ? align16(static_cast<size_t>(max_len) * rows * kChainMax * 2) : 0);
}

// A work item whose descriptor (and, for a panel tile, the operands the
// previous wave does not write) was staged before the barrier that starts its
// wave (fused kernel; lives in shared memory).
template <class T> struct StagedItem {
  FoldDesc<T> f;
  MergeDesc<T> m;
  int64_t b;    // work item, -1: none
  int32_t mask; // panel operands already in shared memory
  int32_t pad;
};

template <class T> __device__ __forceinline__ bool panel_fold(const FoldDesc<T> &f) {
  return f.small >= kPanel16;
}

// Stages operands `mask` of output tile `tile` of f (an R x R panel tile) into
// p.  Every global load is issued before the first shared-memory store, so
// the panel costs one memory latency; A holds w[j] + t1[i][j] (the
// reference's first addition), reading w from p.W when it was staged earlier.
template <class T, int R>
__device__ __forceinline__ void panel_load_r(const FoldDesc<T> &f, int64_t tile, int mask, PanelSmem<T> &p) {
  constexpr int kIt = R * kPanel / kFoldThreads;
  static_assert(kPanel <= kFoldThreads, "one w entry per thread");
  const int i0 = static_cast<int>(tile / f.tiles_k) * R;
  const int k0 = static_cast<int>(tile % f.tiles_k) * R;
  const bool lw = mask & kPanelW, l1 = mask & kPanelT1, l2 = mask & kPanelT2;
  const bool own_w = lw && static_cast<int>(threadIdx.x) < f.nw;
  const T vw = own_w ? f.w[threadIdx.x] : T(0);
  T v1[kIt], w1[kIt], v2[kIt];
#pragma unroll
  for (int q = 0; q < kIt; ++q) {
    const int idx = threadIdx.x + q * kFoldThreads;
    const int r = idx / kPanel, j = idx % kPanel;
    const bool in1 = l1 && j < f.nw && i0 + r < f.nu;
    v1[q] = in1 ? __ldcg(&f.t1[static_cast<int64_t>(i0 + r) * f.nw + j]) : T(0);
    w1[q] = in1 && lw ? f.w[j] : T(0);
    const int jj = idx / R, c = idx % R;
    v2[q] = (l2 && jj < f.nw && k0 + c < f.nv) ? __ldcg(&f.t2[static_cast<int64_t>(jj) * f.nv + k0 + c]) : T(0);
  }
  if (own_w) p.W[threadIdx.x] = vw;
#pragma unroll
  for (int q = 0; q < kIt; ++q) {
    const int idx = threadIdx.x + q * kFoldThreads;
    const int r = idx / kPanel, j = idx % kPanel;
    if (l1 && j < f.nw) p.A[r * (kPanel + 1) + j] = (lw ? w1[q] : p.W[j]) + v1[q];
    if (l2) p.B[(idx / R) * (R + 1) + idx % R] = v2[q];
  }
}

template <class T>
__device__ __forceinline__ void panel_load(const FoldDesc<T> &f, int64_t tile, int mask, PanelSmem<T> &p) {
  if (f.small == kPanel16)
    panel_load_r<T, 16>(f, tile, mask, p);
  else if (f.small == kPanel8)
    panel_load_r<T, 8>(f, tile, mask, p);
  else
    panel_load_r<T, 4>(f, tile, mask, p);
}

__device__ __forceinline__ uint64_t trace_ns() {
#ifdef PP_TRACE_CLOCK // microbenchmarks: SM cycles instead of ns
  return static_cast<uint64_t>(clock64());
#else
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
#endif
}

// Scan keys: candidates are compared as int64 keys, branch-free, starting
// from LLONG_MAX (above every key).  FP64 keys are order-preserving bit
// maps; -0.0 shares +0.0's key since the two compare equal.  Tables never
// hold NaN (rejected at upload; analytic costs are finite).
template <class T> __device__ __forceinline__ long long scan_key(T x);
template <> __device__ __forceinline__ long long scan_key<double>(double x) {
  long long b = __double_as_longlong(x);
  b = b == LLONG_MIN ? 0 : b;
  return b ^ ((b >> 63) & LLONG_MAX);
}
template <> __device__ __forceinline__ long long scan_key<int32_t>(int32_t x) { return x; }

// keep (k, j) if it precedes (bk, bj) in the reference's argmin order: lower
// value, then lower j
__device__ __forceinline__ void keep_min(long long k, int j, long long &bk, int &bj) {
  const bool t = k < bk || (k == bk && j < bj);
  bk = t ? k : bk;
  bj = t ? j : bj;
}

// One R x R panel tile: thread t owns cell t / G and scans j = g, g + G, ...
// (G = 256 / R^2 groups, g = t % G); every merge prefers the lower j on
// equal values, which reproduces the reference's ascending strict-< scan.
template <class T, int R>
__device__ __forceinline__ void panel_tile_r(const FoldDesc<T> &f, int64_t tile, int staged, PanelSmem<T> &p,
                                             uint64_t *tr) {
  constexpr int kCells = R * R, kG = kFoldThreads / kCells, kRS = R + 1;
  if (staged != kPanelAll) panel_load_r<T, R>(f, tile, kPanelAll & ~staged, p);
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[1] = trace_ns();
  // the kG groups of a cell are adjacent lanes: a shuffle tree merges them
  const int g = threadIdx.x % kG, cell = threadIdx.x / kG;
  const int ty = cell / R, tx = cell % R;
  const T *Ar = p.A + ty * (kPanel + 1);
  const T *Bc = p.B + tx;
  // two chains (alternate candidates), four candidates per step with every
  // shared-memory read issued before the compares; within a chain strict <
  // keeps the lowest j, as the reference's ascending scan does
  long long k0 = LLONG_MAX, k1 = LLONG_MAX;
  int j0 = INT_MAX, j1 = INT_MAX;
  const int nw = f.nw;
  int j = g;
  for (; j + 3 * kG < nw; j += 4 * kG) {
    T a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = Ar[j + u * kG], b[u] = Bc[(j + u * kG) * kRS];
    long long c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = scan_key<T>(a[u] + b[u]);
#pragma unroll
    for (int u = 0; u < 4; u += 2) {
      if (c[u] < k0) k0 = c[u], j0 = j + u * kG;
      if (c[u + 1] < k1) k1 = c[u + 1], j1 = j + (u + 1) * kG;
    }
  }
  for (; j < nw; j += kG) {
    const long long c = scan_key<T>(Ar[j] + Bc[j * kRS]);
    if (c < k0) k0 = c, j0 = j;
  }
  keep_min(k1, j1, k0, j0);
  if (tr && threadIdx.x == 0) tr[5] = trace_ns();
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) {
    const long long ok = __shfl_xor_sync(0xffffffffu, k0, o);
    const int oj = __shfl_xor_sync(0xffffffffu, j0, o);
    keep_min(ok, oj, k0, j0);
  }
  const int i = static_cast<int>(tile / f.tiles_k) * R + ty;
  const int k = static_cast<int>(tile % f.tiles_k) * R + tx;
  if (tr && threadIdx.x == 0) tr[6] = trace_ns();
  if (g == 0 && i < f.nu && k < f.nv) {
    const int64_t o = static_cast<int64_t>(i) * f.nv + k;
    f.out[o] = fold_epilogue(f, o, Ar[j0] + Bc[j0 * kRS]); // the winner's own sum (keeps -0.0)
    f.am[static_cast<int64_t>(i) * f.nv + k] = static_cast<uint16_t>(j0);
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = trace_ns();
}

template <class T>
__device__ __forceinline__ void panel_tile(const FoldDesc<T> &f, int64_t tile, int staged, PanelSmem<T> &p,
                                           uint64_t *tr = nullptr) {
  if (f.small == kPanel16)
    panel_tile_r<T, 16>(f, tile, staged, p, tr);
  else if (f.small == kPanel8)
    panel_tile_r<T, 8>(f, tile, staged, p, tr);
  else
    panel_tile_r<T, 4>(f, tile, staged, p, tr);
}

template <class T> __device__ __forceinline__ void cp_async(T *dst, const T *src) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte elements");
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- bulk async copies (TMA, non-tensor) into shared memory ---------------
__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// generic-proxy writes to GLOBAL memory (earlier phases of the same launch,
// ordered by the grid barrier) before async-proxy (bulk copy) reads of them
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Copies the 16-byte-rounded byte range of [p, p + n) to dst; returns the
// element offset of p inside dst.  (Device allocations are whole 256-byte
// granules, so the rounded range stays inside p's allocation.)
template <class T> __device__ __forceinline__ unsigned bulk_range(T *dst, const T *p, int64_t n, uint64_t *bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), lo = a & ~uintptr_t(15);
  const uintptr_t hi = (a + static_cast<uintptr_t>(n) * sizeof(T) + 15) & ~uintptr_t(15);
  bulk_g2s(dst, reinterpret_cast<const void *>(lo), static_cast<unsigned>(hi - lo), bar);
  return static_cast<unsigned>((a - lo) / sizeof(T));
}
template <class T> __device__ __forceinline__ unsigned bulk_bytes(const T *p, int64_t n) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), lo = a & ~uintptr_t(15);
  return static_cast<unsigned>(((a + static_cast<uintptr_t>(n) * sizeof(T) + 15) & ~uintptr_t(15)) - lo);
}

// Thread 0: stream fold f's t2 and w into staging buffer `buf` (t2 at the
// front, w after it at `w_at` bytes), completing on `bar`.
template <class T>
__device__ __forceinline__ void chain_stage(const FoldDesc<T> &f, unsigned char *buf, size_t w_at, uint64_t *bar,
                                            bool first) {
  const int64_t n2 = static_cast<int64_t>(f.nw) * f.nv;
  // earlier generic reads of buf happen before the async-proxy copies; the
  // first copies of an item also order the generic global stores that
  // produced t2 / w (table build, earlier phases: every chain fold's t2 is
  // written before its segment starts, w are node tables)
  if (first)
    fence_proxy_async_all();
  else
    fence_proxy_async();
  mbar_expect_tx(bar, bulk_bytes(f.t2, n2) + bulk_bytes(f.w, f.nw));
  bulk_range(reinterpret_cast<T *>(buf), f.t2, n2, bar);
  bulk_range(reinterpret_cast<T *>(buf + w_at), f.w, f.nw, bar);
}

// Keeps (v, j) if it precedes (bv, bj): lower value, then lower j.
template <class T> __device__ __forceinline__ void keep_min_v(T v, int j, T &bv, int &bj) {
  const bool t = v < bv || (v == bv && j < bj);
  bv = t ? v : bv;
  bj = t ? j : bj;
}

// One warp's share of a chain fold: cells lane + 32u (u < U) of one row, the
// j values g, g + G, ... two per step into separate chains; A'[j] = w[j] +
// row[j] (the reference's first addition) is formed on the fly.  Writes the
// per-cell (value, j) minima of this j-group.
template <class T, int U>
__device__ __forceinline__ void chain_scan(const T *ws, const T *cr, const T *t2s, int nw, int nv, int g, int G, int lane,
                                           T *ogv, int *ogj) {
  int vv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) vv[u] = min(lane + 32 * u, nv - 1); // clamped: dead cells re-read a live one
  T b0[U], b1[U];
  int j0[U], j1[U];
#pragma unroll
  for (int u = 0; u < U; ++u) b0[u] = b1[u] = T(0), j0[u] = j1[u] = INT_MAX;
  int j = g;
  for (; j + G < nw; j += 2 * G) {
    const T a0 = ws[j] + cr[j], a1 = ws[j + G] + cr[j + G];
    const T *t0 = t2s + j * nv, *t1 = t0 + G * nv;
    T x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x0[u] = t0[vv[u]], x1[u] = t1[vv[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T c0 = a0 + x0[u], c1 = a1 + x1[u];
      if (j0[u] == INT_MAX || c0 < b0[u]) b0[u] = c0, j0[u] = j;
      if (j1[u] == INT_MAX || c1 < b1[u]) b1[u] = c1, j1[u] = j + G;
    }
  }
  if (j < nw) {
    const T a0 = ws[j] + cr[j];
    const T *t0 = t2s + j * nv;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T c0 = a0 + t0[vv[u]];
      if (j0[u] == INT_MAX || c0 < b0[u]) b0[u] = c0, j0[u] = j;
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (j1[u] != INT_MAX) keep_min_v<T>(b1[u], j1[u], b0[u], j0[u]);
    const int v = lane + 32 * u;
    if (v < nv) ogv[v] = b0[u], ogj[v] = j0[u];
  }
}

// Item `it` of a chain segment: rows [r0, r0 + rows) of one chain, through
// all its folds; the rows live in shared memory between folds, and fold
// k + 1's t2 and w stream in (two bulk copies, mbarrier-completed) while
// fold k scans.  Per fold: A' = w + t1 rows (the reference's first
// addition); warp g of the rows' warps scans j = g, g + G, ... over the
// row's cells (lane l: cells l, l + 32, ...: conflict-free reads of the
// unpadded t2 rows), strict < in ascending j keeping the lowest j; the G
// group minima then merge per cell (lower value, then lower j), so the
// result is the reference's ascending strict-< scan.  Writes every fold's
// argmins and the last fold's table; the intermediate tables have no other
// reader.
template <class T>
__device__ __forceinline__ void chain_item(const ChainDesc *chains, int n_chains, const FoldDesc<T> *cf, int64_t it,
                                           unsigned char *smem, size_t stage, uint64_t *tr = nullptr,
                                           const uint16_t *chain_of = nullptr) {
  const bool stamp = tr && threadIdx.x == 0;
  // the item's chain: one load from the per-item index when the image has it
  int lo = chain_of ? chain_of[it] : 0, hi = chain_of ? lo : n_chains - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (chains[mid].item_begin <= it)
      lo = mid;
    else
      hi = mid - 1;
  }
  const ChainDesc c = chains[lo];
  const int r0 = static_cast<int>(it - c.item_begin) * c.rows;
  const int nr = min(c.rows, c.nu - r0);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  unsigned char *p = smem + 16;
  FoldDesc<T> *fd = reinterpret_cast<FoldDesc<T> *>(p);
  p += align16(static_cast<size_t>(c.n) * sizeof(FoldDesc<T>));
  T *A = reinterpret_cast<T *>(p);
  T *cur = A + c.rows * (kChainMax + 1);
  p += align16(static_cast<size_t>(c.rows) * (2 * kChainMax + 1) * sizeof(T));
  T *gv = reinterpret_cast<T *>(p);
  int *gj = reinterpret_cast<int *>(gv + kChainGroups * c.rows * kChainMax);
  p += align16(static_cast<size_t>(kChainGroups) * c.rows * kChainMax * (sizeof(T) + 4));
  unsigned char *buf[2] = {p, p + stage};
  uint16_t *amS = reinterpret_cast<uint16_t *>(p + 2 * stage); // [n][rows][kChainMax] when c.path
  __syncthreads(); // the block's previous item may still read smem
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_proxy_async();
  }
  for (int k = threadIdx.x; k < c.n; k += kFoldThreads) fd[k] = cf[c.first + k];
  __syncthreads();
  auto w_at = [&](int k) { return align16(static_cast<size_t>(fd[k].nw) * fd[k].nv * sizeof(T) + 16); };
  if (threadIdx.x == 0) { // folds 0 and 1 stream in now; fold k + 2 once fold k's scan frees its buffer
    chain_stage<T>(fd[0], buf[0], w_at(0), &bar[0], true);
    if (c.n > 1) chain_stage<T>(fd[1], buf[1], w_at(1), &bar[1], false);
  }
  {
    const FoldDesc<T> &f0 = fd[0];
    for (int x = threadIdx.x; x < nr * f0.nw; x += kFoldThreads) {
      const int r = x / f0.nw, j = x - r * f0.nw;
      cur[r * kChainMax + j] = __ldcg(&f0.t1[static_cast<int64_t>(r0 + r) * f0.nw + j]);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpr = kChainGroups / c.rows; // warps (j-groups) per row
  for (int k = 0; k < c.n; ++k) {
    const FoldDesc<T> &f = fd[k];
    const int nw = f.nw, nv = f.nv;
    if (stamp && k < 4) tr[4 * k] = trace_ns();
    mbar_wait(&bar[k & 1], static_cast<unsigned>(k >> 1) & 1u);
    const T *t2s = reinterpret_cast<const T *>(buf[k & 1]) + (reinterpret_cast<uintptr_t>(f.t2) & 15) / sizeof(T);
    const T *ws = reinterpret_cast<const T *>(buf[k & 1] + w_at(k)) + (reinterpret_cast<uintptr_t>(f.w) & 15) / sizeof(T);
    if (stamp && k < 4) tr[4 * k + 1] = tr[4 * k + 2] = trace_ns();
    { // scan: warp -> (row, j-group), lane -> cells lane, lane + 32, ...
      const int r = warp / wpr, g = warp - r * wpr;
      if (r < nr) {
        T *ogv = gv + (g * c.rows + r) * kChainMax;
        int *ogj = gj + (g * c.rows + r) * kChainMax;
        const T *cr = cur + r * kChainMax;
        switch ((nv + 31) >> 5) {
        case 1: chain_scan<T, 1>(ws, cr, t2s, nw, nv, g, wpr, lane, ogv, ogj); break;
        case 2: chain_scan<T, 2>(ws, cr, t2s, nw, nv, g, wpr, lane, ogv, ogj); break;
        case 3: chain_scan<T, 3>(ws, cr, t2s, nw, nv, g, wpr, lane, ogv, ogj); break;
        default: chain_scan<T, 4>(ws, cr, t2s, nw, nv, g, wpr, lane, ogv, ogj); break;
        }
      }
    }
    __syncthreads();
    if (stamp && k < 4) tr[4 * k + 3] = trace_ns();
    if (k + 2 < c.n && threadIdx.x == kFoldThreads - 1) { // buf[k & 1] is free again
      if (tr && k < 4) tr[16 + 2 * k] = trace_ns();
      chain_stage<T>(fd[k + 2], buf[k & 1], w_at(k + 2), &bar[k & 1], false);
      if (tr && k < 4) tr[17 + 2 * k] = trace_ns();
    }
    const bool last = k + 1 == c.n;
    const int ng = min(wpr, nw); // groups that scanned anything
    for (int x = threadIdx.x; x < nr * nv; x += kFoldThreads) {
      const int r = x / nv, v = x - r * nv;
      // (value, j) minimum over the groups as a tree (the order is
      // irrelevant: ties resolve on the distinct j); groups past ng repeat
      // group 0, which changes nothing
      T gvl[kChainGroups];
      int gjl[kChainGroups];
#pragma unroll
      for (int g = 0; g < kChainGroups; ++g) {
        const int gg = g < ng ? g : 0;
        gvl[g] = gv[(gg * c.rows + r) * kChainMax + v], gjl[g] = gj[(gg * c.rows + r) * kChainMax + v];
      }
#pragma unroll
      for (int h = kChainGroups / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int g = 0; g < h; ++g) keep_min_v<T>(gvl[g + h], gjl[g + h], gvl[g], gjl[g]);
      T b = gvl[0];
      int j = gjl[0];
      const int64_t o = static_cast<int64_t>(r0 + r) * nv + v;
      f.am[o] = static_cast<uint16_t>(j);
      if (c.path) amS[(k * c.rows + r) * kChainMax + v] = static_cast<uint16_t>(j);
      b = fold_epilogue(f, o, b);
      if (last)
        f.out[o] = b;
      else
        cur[r * kChainMax + v] = b;
    }
    __syncthreads();
  }
  if (c.path) { // backtrack every (row, final column) through the chain
    const int nvl = fd[c.n - 1].nv;
    for (int x = threadIdx.x; x < nr * nvl; x += kFoldThreads) {
      const int r = x / nvl, v = x - r * nvl;
      uint16_t *out = c.path + (static_cast<int64_t>(r0 + r) * nvl + v) * c.n;
      int col = v;
      for (int k = c.n - 1; k >= 0; --k) {
        const uint16_t j = amS[(k * c.rows + r) * kChainMax + col];
        out[k] = j;
        col = j;
      }
    }
  }
  if (threadIdx.x == 0) {
    mbar_inval(&bar[0]);
    mbar_inval(&bar[1]);
  }
}

// fold of work item b: the wave's per-tile fold index when the image has one
// (fused plans: one load instead of a chain of dependent ones), else a binary
// search over the folds' first tiles
template <class T>
__device__ __forceinline__ int find_fold(const FoldDesc<T> *folds, int n_folds, int64_t b, const uint16_t *fold_of = nullptr) {
  if (fold_of) return fold_of[b];
  int lo = 0, hi = n_folds - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (folds[mid].tile_begin <= b)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <class T> __device__ __forceinline__ int find_merge(const MergeDesc<T> *merges, int n_merges, int64_t mb) {
  int lo = 0, hi = n_merges - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (merges[mid].blk_begin <= mb)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Work item b of a wave: b < fold_tiles folds one 32x32 output tile of a fold
// (block-cooperative, uses `sm`); otherwise it adds one merge chunk.
template <class T>
__device__ __forceinline__ void wave_item(const FoldDesc<T> *folds, int n_folds, int64_t fold_tiles,
                                          const MergeDesc<T> *merges, int n_merges, int64_t b, WaveSmem<T> &sm,
                                          const StagedItem<T> *pre = nullptr, uint64_t *tr = nullptr,
                                          const uint16_t *fold_of = nullptr) {
  auto &As = sm.t.As;
  auto &Bs = sm.t.Bs;
  const bool staged = pre && pre->b == b;
  if (b < fold_tiles) {
    const FoldDesc<T> f = staged ? pre->f : folds[find_fold(folds, n_folds, b, fold_of)];
    const int64_t tile = b - f.tile_begin;
    if (panel_fold(f)) {
      panel_tile<T>(f, tile, staged ? pre->mask : 0, sm.p, tr);
      return;
    }
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
          pa[q] = (i < f.nu && j < f.nw) ? T(f.w[j] + __ldcg(&f.t1[static_cast<int64_t>(i) * f.nw + j])) : T(0);
          const int jr = idx >> 4, kc = idx & 15; // B: 32 j x 16 cols
          const int jj = j0 + jr, k = k0 + kc;
          pb[q] = (jj < f.nw && k < f.nv) ? __ldcg(&f.t2[static_cast<int64_t>(jj) * f.nv + k]) : T(0);
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
        f.out[static_cast<int64_t>(i) * f.nv + k] = fold_epilogue(f, static_cast<int64_t>(i) * f.nv + k, odd ? bo : be);
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
        pa[q] = (i < f.nu && j < f.nw) ? T(f.w[j] + __ldcg(&f.t1[static_cast<int64_t>(i) * f.nw + j])) : T(0);
        const int jj = j0 + r, k = k0 + c;
        pb[q] = (jj < f.nw && k < f.nv) ? __ldcg(&f.t2[static_cast<int64_t>(jj) * f.nv + k]) : T(0);
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
          f.out[static_cast<int64_t>(i) * f.nv + k] =
              fold_epilogue(f, static_cast<int64_t>(i) * f.nv + k, odd ? bo[c] : be[c]);
          f.am[static_cast<int64_t>(i) * f.nv + k] = static_cast<uint16_t>(odd ? jo[c] : je[c]);
        }
      }
    return;
  }
  const int64_t mb = b - fold_tiles;
  const MergeDesc<T> m = staged ? pre->m : merges[find_merge(merges, n_merges, mb)];
  const int64_t base = (mb - m.blk_begin) * kMergePerBlock;
  for (int64_t k = base + threadIdx.x; k < m.n && k < base + kMergePerBlock; k += kMergeThreads)
    m.out[k] = __ldcg(&m.a[k]) + __ldcg(&m.b[k]);
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

template <class A> __device__ __forceinline__ A shfl_xor_any(A v, int o) {
  if constexpr (sizeof(A) == 8) {
    long long x;
    memcpy(&x, &v, 8);
    x = __shfl_xor_sync(0xffffffffu, x, o);
    memcpy(&v, &x, 8);
    return v;
  } else {
    return __shfl_xor_sync(0xffffffffu, v, o);
  }
}

// (value, linear index) order of the enumeration: lower value, then lower
// index; INT64_MAX marks "no candidate".
template <class A> __device__ __forceinline__ void keep_best(A ov, int64_t oi, A &bv, int64_t &bi) {
  if (oi != INT64_MAX && (bi == INT64_MAX || ov < bv || (ov == bv && oi < bi))) bv = ov, bi = oi;
}

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
  // (value, index) minimum: shuffles within each warp, then warp 0 over the
  // warps' results (one barrier instead of one per tree level)
  __shared__ A sv[kEnumThreads / 32];
  __shared__ int64_t si[kEnumThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) keep_best<A>(shfl_xor_any<A>(best, o), __shfl_xor_sync(0xffffffffu, bidx, o), best, bidx);
  if (lane == 0) sv[warp] = best, si[warp] = bidx;
  __syncthreads();
  if (warp == 0) {
    best = lane < kEnumThreads / 32 ? sv[lane] : A(0);
    bidx = lane < kEnumThreads / 32 ? si[lane] : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) keep_best<A>(shfl_xor_any<A>(best, o), __shfl_xor_sync(0xffffffffu, bidx, o), best, bidx);
    if (lane == 0) blk_val[vb] = best, blk_idx[vb] = bidx;
  }
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(kEnumThreads)
    enum_kernel(const EnumNode *nodes, int k, const EnumEdge *edges, int m, int64_t total, int64_t per_thread,
                typename Acc<T>::type *blk_val, int64_t *blk_idx) {
  enum_block<T>(nodes, k, edges, m, total, per_thread, blk_val, blk_idx, blockIdx.x);
}

struct UnwindRec {
  const uint16_t *am; // argmins [rows][cols]; a chain record: path table [rows][cols][n]
  int32_t removed, src, dst, cols;
  int32_t n;          // 0: one fold; n > 0: a chain of n folds whose removed nodes are chain_nodes[removed, removed + n)
  int32_t blk;        // row-sharded plan: rows per rank; `am` is then the table's byte offset in every
                      // rank's plan memory and row r is read from rank r / blk (FinishArgs::peer)
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
  const int32_t *chain_nodes;
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
  uint64_t *trace; // optional: stamps after each finish step (profiling)
  const unsigned char *const *peer; // row-sharded: plan memory base of every rank (peer / IPC mapped)
  int32_t smem_ok;  // the caller's shared memory holds indices[nl] + terms[nl + ne]
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
template <class T>
__device__ __forceinline__ void finish_block(const FinishArgs &a, unsigned char *smem = nullptr, bool staged = false);

template <class T> __global__ void __launch_bounds__(kFinishThreads) finish_kernel(FinishArgs a) {
  finish_block<T>(a);
}


// Shared-memory layout of finish_block (when a.smem_ok): terms[nl + ne] |
// cat_off[nl] | xoff[ne] (8-byte) | indices[nl] | counts[nl] | esrc[ne] |
// edst[ne] | enumeration node counts[k] (4-byte).
__host__ __device__ constexpr size_t finish_smem_bytes(int nl, int ne, int k) {
  return static_cast<size_t>(nl + ne) * 8 + static_cast<size_t>(nl + ne) * 8 +
         (static_cast<size_t>(nl) * 2 + static_cast<size_t>(ne) * 2 + k) * 4 + 16;
}

// smem (optional): the fused kernel's dynamic region.  With it (a.smem_ok)
// the static lookup arrays are staged up front and the unwind and re-sum
// touch global memory only for the argmin and cost-table values.
// Stages finish_block's lookup arrays into smem (independent loads, all in
// flight at once).  The fused kernel runs it on block 0 before the barrier
// that precedes the finish, off the critical path.
__device__ __forceinline__ void finish_stage(const FinishArgs &a, unsigned char *smem) {
  double *terms = reinterpret_cast<double *>(smem);
  int64_t *co = reinterpret_cast<int64_t *>(terms + a.nl + a.ne), *xo = co + a.nl;
  int32_t *ix = reinterpret_cast<int32_t *>(xo + a.ne), *cn = ix + a.nl, *es = cn + a.nl, *ed = es + a.ne;
  int32_t *ncount = ed + a.ne;
  for (int l = threadIdx.x; l < a.nl; l += kFinishThreads) co[l] = a.cat_off[l], cn[l] = a.counts[l];
  for (int e = threadIdx.x; e < a.ne; e += kFinishThreads) xo[e] = a.xoff[e], es[e] = a.esrc[e], ed[e] = a.edst[e];
  for (int d = threadIdx.x; d < a.k; d += kFinishThreads) ncount[d] = a.nodes[d].count;
}

template <class T> __device__ __forceinline__ void finish_block(const FinishArgs &a, unsigned char *smem, bool staged) {
  using A = typename Acc<T>::type;
  const bool stamp = a.trace && threadIdx.x == 0;
  if (stamp) a.trace[0] = trace_ns();
  const bool sm = a.smem_ok && smem;
  double *terms = sm ? reinterpret_cast<double *>(smem) : a.terms;
  const int64_t *cat_off = a.cat_off, *xoff = a.xoff;
  int32_t *idx = a.indices;
  const int32_t *counts = a.counts, *esrc = a.esrc, *edst = a.edst;
  int32_t *ncount = nullptr;
  if (sm) {
    if (!staged) finish_stage(a, smem);
    int64_t *co = reinterpret_cast<int64_t *>(terms + a.nl + a.ne), *xo = co + a.nl;
    int32_t *ix = reinterpret_cast<int32_t *>(xo + a.ne), *cn = ix + a.nl, *es = cn + a.nl, *ed = es + a.ne;
    ncount = ed + a.ne;
    cat_off = co, xoff = xo, idx = ix, counts = cn, esrc = es, edst = ed;
  }
  __shared__ A sv[kFinishThreads / 32];
  __shared__ int64_t si[kFinishThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const A *bv = static_cast<const A *>(a.blk_val);
  A best = A(0);
  int64_t bi = INT64_MAX;
  if (stamp) a.trace[5] = trace_ns();
  for (int b = threadIdx.x; b < a.nblk; b += kFinishThreads) keep_best<A>(bv[b], a.blk_idx[b], best, bi);
  if (stamp) a.trace[6] = trace_ns();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) keep_best<A>(shfl_xor_any<A>(best, o), __shfl_xor_sync(0xffffffffu, bi, o), best, bi);
  if (lane == 0) sv[warp] = best, si[warp] = bi;
  __syncthreads();
  if (stamp) a.trace[7] = trace_ns();
  if (warp == 0) {
    best = lane < kFinishThreads / 32 ? sv[lane] : A(0);
    bi = lane < kFinishThreads / 32 ? si[lane] : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) keep_best<A>(shfl_xor_any<A>(best, o), __shfl_xor_sync(0xffffffffu, bi, o), best, bi);
    if (lane == 0) {
      int64_t r = bi;
      for (int d = a.k - 1; d >= 0; --d) {
        const int32_t cnt = ncount ? ncount[d] : a.nodes[d].count;
        a.digits[d] = static_cast<int32_t>(r % cnt);
        r /= cnt;
      }
      *a.final_cost = ldexp(static_cast<double>(best), -a.shift);
    }
  }
  if (stamp) a.trace[1] = trace_ns();
  if (a.n_rec < 0) return;
  for (int l = threadIdx.x; l < a.nl; l += kFinishThreads) idx[l] = -1;
  __syncthreads();
  for (int d = threadIdx.x; d < a.k; d += kFinishThreads) idx[a.node_layer[d]] = a.digits[d];
  // waves, last first; each thread's record of the next group is fetched
  // before the barrier that ends the current one
  UnwindRec u{};
  bool have = false;
  if (a.n_groups > 0) {
    const int q = a.group_begin[0] + threadIdx.x;
    have = q < a.group_begin[1];
    if (have) u = a.recs[q];
  }
  __syncthreads();
  for (int gidx = 0; gidx < a.n_groups; ++gidx) {
    for (int q = a.group_begin[gidx] + threadIdx.x; q < a.group_begin[gidx + 1]; q += kFinishThreads) {
      const UnwindRec r = q == a.group_begin[gidx] + static_cast<int>(threadIdx.x) && have ? u : a.recs[q];
      const int64_t at = static_cast<int64_t>(idx[r.src]) * r.cols + idx[r.dst];
      if (r.blk > 0) { // distributed unwind: the owner rank's argmin row, read over NVLink / peer memory
        const int row = idx[r.src], q = row / r.blk;
        const uint16_t *am = reinterpret_cast<const uint16_t *>(a.peer[q] + reinterpret_cast<uintptr_t>(r.am));
        idx[r.removed] = am[static_cast<int64_t>(row - q * r.blk) * r.cols + idx[r.dst]];
      } else if (r.n == 0) {
        idx[r.removed] = r.am[at];
      } else {
        // the path in batches: all loads of a batch in flight before its
        // stores (idx may alias global memory, so a plain loop serialises)
        const uint16_t *pth = r.am + at * r.n;
        for (int k0 = 0; k0 < r.n; k0 += 8) {
          int32_t node[8], val[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k0 + k < r.n) node[k] = a.chain_nodes[r.removed + k0 + k], val[k] = pth[k0 + k];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k0 + k < r.n) idx[node[k]] = val[k];
        }
      }
    }
    have = false;
    if (gidx + 1 < a.n_groups) {
      const int q = a.group_begin[gidx + 1] + threadIdx.x;
      have = q < a.group_begin[gidx + 2];
      if (have) u = a.recs[q];
    }
    __syncthreads();
  }
  if (stamp) a.trace[2] = trace_ns();
  const T *onode = static_cast<const T *>(a.onode);
  const T *oxfer = static_cast<const T *>(a.oxfer);
  for (int l = threadIdx.x; l < a.nl; l += kFinishThreads) {
    terms[l] = ldexp(static_cast<double>(onode[cat_off[l] + idx[l]]), -a.shift);
    if (idx != a.indices) a.indices[l] = idx[l];
  }
  for (int e = threadIdx.x; e < a.ne; e += kFinishThreads)
    terms[a.nl + e] = ldexp(
        static_cast<double>(oxfer[xoff[e] + static_cast<int64_t>(idx[esrc[e]]) * counts[edst[e]] + idx[edst[e]]]), -a.shift);
  __syncthreads();
  // zero-copy results (indices, digits, final cost) go to pinned host memory
  // from threads 1.. while thread 0 re-sums the cost serially and writes it
  const size_t cost_w = static_cast<size_t>(reinterpret_cast<const unsigned char *>(a.cost) - a.dev_res) / 4;
  if (threadIdx.x == 0) { // the reference's order: nodes by layer, then edges by id
    double t = 0.0;
    for (int x = 0; x < a.nl + a.ne; ++x) t += terms[x];
    *a.cost = t;
    if (a.host_res) *reinterpret_cast<volatile double *>(a.host_res + 4 * cost_w) = t;
  } else if (a.host_res) {
    for (size_t b = threadIdx.x - 1; b < a.res_bytes / 4; b += kFinishThreads - 1)
      if (b < cost_w || b >= cost_w + 2)
        reinterpret_cast<volatile uint32_t *>(a.host_res)[b] = reinterpret_cast<const uint32_t *>(a.dev_res)[b];
  }
  if (stamp) a.trace[3] = trace_ns();
  // no system fence: the host reads the block after synchronising with the
  // kernel's completion, which orders these writes
  if (stamp) a.trace[4] = trace_ns();
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
