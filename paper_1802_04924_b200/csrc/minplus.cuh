// minplus.cuh — the large-table Eq. 2 fold (K3-U16) for exact fixed-point tables.
//
// out[i][k] = min_j (a[i][j] + b[j][k]),  a = w[j] + t1[i][j],  b = t2[j][k],
// argmin = lowest j (planner.hpp:139-155), all in int32 units of 2^-s.
//
// Min-plus is shift-invariant per row of a and per column of b, so with
// ra[i] = min_j a[i][j] and cb[k] = min_j b[j][k] the normalised operands
// a' = a - ra, b' = b - cb lie in [0, rowspan(a)] x [0, colspan(b)].  The host
// propagates span bounds through the schedule and picks JB in {5, 4, 3} with
//   ((rowspan(a) + colspan(b)) << JB) + 2^JB - 1 <= 65534,
// so every candidate fits an unsigned 16-bit lane with its j carried along:
//   a'' = (a' << JB) | (j mod 2^JB),   b'' = b' << JB,
//   a'' + b'' = ((a' + b') << JB) | (j mod 2^JB).
// The low bits never carry into the value, so a lane-wise u16 min over the
// 2^JB candidates of one aligned j-group yields the minimum AND, among equal
// values, the lowest j of the group.  VIADDMNMX.U16x2 = min(a'' + b'', m) on a
// (cell, cell+1) pair is one instruction per two (add, min) cell updates — the
// FP32 CUDA-core roofline of one lane-op per cell.  Across groups the kernel
// keeps key = (value << (16 + JB) | group << JB | j-low) with an unsigned min:
// smallest value first, then the lowest j.  So the exact value AND the exact
// reference argmin come out of the fold itself:
//   out = ra + cb + (key >> (16 + JB)),   am = key & 0xFFFF.
// Padding: j >= nw has a'' = 0xFFFF, b'' = 0 (sum 0xFFFF above every real
// candidate, no wrap); padded rows / columns are never stored.
//
// Cap: operands are stored as min(x', cap).  If a cell's computed minimum m''
// is < cap, its minimising candidates have uncapped operands, so m'' is the
// true minimum (every true candidate >= its capped one >= m''), and a j
// attains m'' after capping iff it does before (a capped candidate is
// >= cap > m''): value and lowest-index argmin are exact.  With j0 the
// minimum of b's column k (b'[j0][k] = 0) the true minimum is <= a'[i][j0] <=
// rowspan(a), and likewise <= colspan(b), so cap = M + 1 with
// M = min(rowspan bound, colspan bound) is always safe (proven); only 2 cap,
// not spanA + spanB, must fit: (2 cap << JB) + 2^JB - 1 <= 65534.  Static
// bounds on derived tables are loose and minima of many candidates are small,
// so folds run optimistically at JB = 6 (64-j groups: half the key updates of
// JB = 5; the largest JB-6 cap, 511), or JB = 7 (cap 255) when nw >= 2048: the
// epilogue checks m'' < cap for every stored cell and raises `ovf` otherwise,
// and the host then re-runs the plan with the proven caps (JB <= 5).
//
// The group key must order (value, group, j mod 2^JB): per group and cell
// pair, one LOP3 moves the two j-low fields next to the group id
// (gj = (m & LOW2) | G2) and one clears them from the values (mv = m & ~LOW2);
// then per cell one PRMT builds (value << (16 + JB) | group << JB | j-low) and
// one UMNMX keeps the minimum — 3 instructions per cell and group.
//
//   mp_minima  (once per plan) cb of every fold whose t2 is an original table,
//              ra of every fold whose t1 is one
//   mp_merge   Eq. 3 (out = t1 + t2) for merges whose output is a large
//              fold's t2, with that fold's column minima (block min + atomicMin)
//   mp_prep    (per wave) the operand blocks: a'' -> A [tile_i][chunk][32 j]
//              [128 i] (u32, a'' in both halves), b'' -> B [tile_k][chunk]
//              [32 j][128 k] (u16), each (tile, chunk) block contiguous (one
//              bulk copy).  ra comes from the producing fold's epilogue when
//              t1 is a fold output, else from a row pass here; cb likewise.
//   mp_fold    persistent stream-K over (tile, 32-j chunk) units: 1 producer
//              warp (cp.async.bulk -> 4-stage mbarrier ring) + 8 consumer warps
//              (128x128 tile, 8x8 cells per thread).  A tile covered by one CTA
//              is stored directly; a tile split between CTAs is combined and
//              stored by the CTA holding its first chunk, from the other
//              CTAs' part slots (per-tile release counter).  The epilogue also feeds the
//              consuming large fold's row minima (out is its t1) or column
//              minima (out is its t2) with warp-reduced atomicMin.
#pragma once

#include "kernels.cuh"

#include <climits>
#include <cstdint>

namespace pp {

constexpr int kMpTile = 128;                    // output rows/cols per tile
constexpr int kMpChunk = 32;                    // j per pipeline stage
constexpr int kMpStages = 4;
constexpr int kMpConsumers = 256;               // 8 warps
constexpr int kMpThreads = kMpConsumers + 32;   // + 1 producer warp
constexpr int kMpTileCells = kMpTile * kMpTile;
constexpr unsigned kMpStageA = kMpChunk * kMpTile * 4; // 16 KiB
constexpr unsigned kMpStageB = kMpChunk * kMpTile * 2; // 8 KiB
constexpr unsigned kMpStageBytes = kMpStageA + kMpStageB;
constexpr size_t kMpSmem = kMpStages * kMpStageBytes + 2 * kMpStages * 8 + 16;
constexpr int kMpPrepRows = 32;  // rows per A-prep block
constexpr int kMpPrepCols = 32;  // columns per B-prep block

struct MpFold {
  // inputs (original or derived tables, int32 units)
  const int32_t *t1; // [nu][nw]
  const int32_t *t2; // [nw][nv]
  const int32_t *w;  // [nw]
  // outputs
  int32_t *out;  // [nu][nv]
  uint16_t *am;  // [nu][nv]
  // row / column minima, order-preserving unsigned (x ^ 2^31); 0xFFFFFFFF
  // before the producer's atomics (ready) or the prep pass
  uint32_t *ra; // [nu]
  uint32_t *cb; // [nv]
  uint32_t *A;  // [tiles_i][nchunks][32][128]
  uint16_t *B;  // [tiles_k][nchunks][32][128]
  uint32_t *part; // [gridDim][128 * 128] stream-K part keys (a CTA's first segment, when split)
  uint32_t *cnt;  // [tiles_i * tiles_k] arrivals, 0 at rest
  // the large fold consuming `out` as its t1 (w_next, ra_next) or t2 (cb_next)
  const int32_t *w_next;
  uint32_t *ra_next, *cb_next;
  int32_t nu, nw, nv, tiles_i, tiles_k, nchunks, jb;
  int32_t cap;   // operand cap: M + 1 (proven), or the JB's largest when optimistic
  uint32_t *ovf; // optimistic cap: set when a minimum reaches the cap (the host re-plans conservatively)
  int32_t ra_ready, cb_ready; // minima supplied before mp_prep (epilogue / mp_colmin)
  int32_t a_batches, b_batches; // mp_prep blocks per row group / column group (chunk batches; 0: none)
  int32_t b_cols;               // B row width: 0 = 128-column tiles (mp_fold); kMpChainCols (mp_chain)
  int64_t prep_begin;   // first mp_prep block (A blocks, then B blocks)
  int64_t colmin_begin; // first mp_minima column block (blocks only for an original t2)
  int64_t rowmin_begin; // first mp_minima row block, counted after all column blocks (original t1)
  int64_t unit_begin;   // first stream-K unit (tile-major, chunk fastest)
  int64_t tile_begin;   // first tile (data-parallel mode)
};

constexpr int kMpPrepBatch = 8; // chunks per mp_prep block when the minima are ready

__host__ __device__ inline int64_t mp_prep_blocks(const MpFold &f) {
  return static_cast<int64_t>((f.nu + kMpPrepRows - 1) / kMpPrepRows) * f.a_batches +
         static_cast<int64_t>((f.nv + kMpPrepCols - 1) / kMpPrepCols) * f.b_batches;
}

__device__ __forceinline__ uint32_t mm_enc(int32_t x) { return static_cast<uint32_t>(x) ^ 0x80000000u; }
__device__ __forceinline__ int32_t mm_dec(uint32_t x) { return static_cast<int32_t>(x ^ 0x80000000u); }

// JB for a fold whose minima are <= M (operands capped at M + 1; 0: too wide)
inline int mp_jbits(int64_t M) {
  for (int jb = 5; jb >= 3; --jb)
    if (((2 * M + 2) << jb) + (1 << jb) - 1 <= 65534) return jb;
  return 0;
}
constexpr int kMpOptJB = 6;       // optimistic plans: 64-j argmin groups, cap 511 (checked on the device)
constexpr int kMpOptJBWide = 7;   // folds with nw >= kMpWideNw: 128-j groups, cap 255 (minima of more candidates are smaller)
constexpr int kMpWideNw = 2048;
// the largest cap JB bits allow
inline int32_t mp_max_cap(int jb) { return static_cast<int32_t>((65534 - ((1 << jb) - 1)) >> (jb + 1)); }

// Eq. 3 for a merge feeding a large fold's t2: out = a + b (planner.hpp:194-199,
// one int32 add), plus that fold's column minima
struct MpMerge {
  const int32_t *a, *b;
  int32_t *out;
  uint32_t *cb; // consumer's column minima (encoded), 0xFF.. before
  int32_t nr, nc;
  int64_t blk_begin; // blocks: (32-column strip) x (64-row band)
};
constexpr int kMpMergeRows = 64;

template <class F> __device__ __forceinline__ int find_desc(const MpFold *d, int n, int64_t b, F key) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (key(d[mid]) <= b)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// ---- mp_minima (once per plan): cb of folds whose t2 is an original table,
// then ra of folds whose t1 is one (row blocks of 8 rows, one warp each) --------
__global__ void __launch_bounds__(256) mp_minima_kernel(const MpFold *folds, int n, int64_t col_blocks) {
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b >= col_blocks) {
    const int64_t rb = b - col_blocks;
    const MpFold &f = folds[find_desc(folds, n, rb, [](const MpFold &x) { return x.rowmin_begin; })];
    const int i = static_cast<int>(rb - f.rowmin_begin) * 8 + warp;
    if (i >= f.nu) return;
    const int32_t *row = f.t1 + static_cast<int64_t>(i) * f.nw;
    int m = INT_MAX;
    int j = lane;
    for (; j + 96 < f.nw; j += 128) { // four independent loads in flight
      const int a0 = f.w[j] + row[j], a1 = f.w[j + 32] + row[j + 32];
      const int a2 = f.w[j + 64] + row[j + 64], a3 = f.w[j + 96] + row[j + 96];
      m = min(m, min(min(a0, a1), min(a2, a3)));
    }
    for (; j < f.nw; j += 32) m = min(m, f.w[j] + row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) f.ra[i] = mm_enc(m);
    return;
  }
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.colmin_begin; })];
  const int k = static_cast<int>(b - f.colmin_begin) * 32 + lane;
  __shared__ int part[8][33];
  int m = INT_MAX;
  if (k < f.nv) {
    int j = warp;
    for (; j + 24 < f.nw; j += 32) { // four independent loads in flight
      const int a0 = f.t2[static_cast<int64_t>(j) * f.nv + k], a1 = f.t2[static_cast<int64_t>(j + 8) * f.nv + k];
      const int a2 = f.t2[static_cast<int64_t>(j + 16) * f.nv + k], a3 = f.t2[static_cast<int64_t>(j + 24) * f.nv + k];
      m = min(m, min(min(a0, a1), min(a2, a3)));
    }
    for (; j < f.nw; j += 8) m = min(m, f.t2[static_cast<int64_t>(j) * f.nv + k]);
  }
  part[warp][lane] = m;
  __syncthreads();
  if (tid < 32 && k < f.nv) {
    int r = part[0][tid];
#pragma unroll
    for (int q = 1; q < 8; ++q) r = min(r, part[q][tid]);
    f.cb[k] = mm_enc(r);
  }
}

__global__ void __launch_bounds__(256) mp_merge_kernel(const MpMerge *ms, int n) {
  const int64_t b = blockIdx.x;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ms[mid].blk_begin <= b)
      lo = mid;
    else
      hi = mid - 1;
  }
  const MpMerge &m = ms[lo];
  const int64_t lb = b - m.blk_begin;
  const int strips = (m.nc + 31) / 32;
  const int k = static_cast<int>(lb % strips) * 32 + (threadIdx.x & 31);
  const int r0 = static_cast<int>(lb / strips) * kMpMergeRows, rl = threadIdx.x >> 5;
  __shared__ int part[8][33];
  int cm = INT_MAX;
  if (k < m.nc) {
    int v[kMpMergeRows / 8];
#pragma unroll
    for (int q = 0; q < kMpMergeRows / 8; ++q) { // all loads first
      const int r = r0 + rl + 8 * q;
      const int64_t o = static_cast<int64_t>(r) * m.nc + k;
      v[q] = r < m.nr ? m.a[o] + m.b[o] : INT_MAX;
    }
#pragma unroll
    for (int q = 0; q < kMpMergeRows / 8; ++q) {
      const int r = r0 + rl + 8 * q;
      if (r < m.nr) m.out[static_cast<int64_t>(r) * m.nc + k] = v[q];
      cm = min(cm, v[q]);
    }
  }
  part[rl][threadIdx.x & 31] = cm;
  __syncthreads();
  if (threadIdx.x < 32 && k < m.nc) {
    int r = part[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < 8; ++q) r = min(r, part[q][threadIdx.x]);
    atomicMin(m.cb + k, mm_enc(r));
  }
}

// ---- mp_prep ------------------------------------------------------------------
// A block (row group of kMpPrepRows, chunk batch): the row pass (one warp per
// four rows) when ra is not ready, then per chunk a 32x32 tile of a'' through
// shared memory into the transposed, duplicated A layout: 16-byte loads (eight
// lanes per 128-byte row segment), kMpPrepBatch chunks' loads in flight, and
// 16-byte stores of four rows.  B block (column group of kMpPrepCols, chunk
// batch): the column pass when cb is not ready, then the shifted u16 values
// (no transpose).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__global__ void __launch_bounds__(256, 3) mp_prep_kernel(const MpFold *folds, int n) {
  pdl_launch_dependents(); // the fold may be scheduled now; it waits for this grid in griddepcontrol.wait
  const int64_t b = blockIdx.x;
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.prep_begin; })];
  int64_t pb = b - f.prep_begin;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jb = f.jb;
  const uint32_t jmask = (1u << jb) - 1;
  const int64_t a_blocks = static_cast<int64_t>((f.nu + kMpPrepRows - 1) / kMpPrepRows) * f.a_batches;
  pdl_wait(); // t1 / ra / cb come from the previous wave
  if (pb < a_blocks) {
    __shared__ int ras[kMpPrepRows];
    __shared__ uint32_t tr[kMpPrepBatch][kMpChunk][kMpPrepRows + 1];
    const int i0 = static_cast<int>(pb / f.a_batches) * kMpPrepRows;
    const int batch = static_cast<int>(pb % f.a_batches);
    const int c0 = f.a_batches > 1 ? batch * kMpPrepBatch : 0, c1 = f.a_batches > 1 ? min(f.nchunks, c0 + kMpPrepBatch) : f.nchunks;
    if (!f.ra_ready) { // a_batches == 1: the whole row here
#pragma unroll 1
      for (int rr = 0; rr < kMpPrepRows / 8; ++rr) {
        const int r = warp * (kMpPrepRows / 8) + rr, i = i0 + r;
        int m = INT_MAX;
        if (i < f.nu) {
          const int32_t *row = f.t1 + static_cast<int64_t>(i) * f.nw;
          int j = lane;
          for (; j + 96 < f.nw; j += 128) { // four independent loads in flight
            const int a0 = f.w[j] + row[j], a1 = f.w[j + 32] + row[j + 32];
            const int a2 = f.w[j + 64] + row[j + 64], a3 = f.w[j + 96] + row[j + 96];
            m = min(m, min(min(a0, a1), min(a2, a3)));
          }
          for (; j < f.nw; j += 32) m = min(m, f.w[j] + row[j]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
          ras[r] = m;
          if (i < f.nu) f.ra[i] = mm_enc(m);
        }
      }
    } else if (tid < kMpPrepRows) {
      ras[tid] = i0 + tid < f.nu ? mm_dec(f.ra[i0 + tid]) : 0;
    }
    __syncthreads();
    const int ti = i0 / kMpTile, ii0 = i0 % kMpTile;
    const int lr = tid >> 3, lj = (tid & 7) * 4; // load: row lr, columns lj..lj+3 of each chunk
    const int sj = tid >> 3, sr = (tid & 7) * 4; // store: j sj, rows sr..sr+3
    const int i = i0 + lr;
    const int32_t *row = f.t1 + static_cast<int64_t>(i) * f.nw;
    const bool vec = ((f.nw & 3) | (reinterpret_cast<uintptr_t>(f.t1) & 15) | (reinterpret_cast<uintptr_t>(f.w) & 15)) == 0;
    const int rai = ras[lr];
    for (int cb0 = c0; cb0 < c1; cb0 += kMpPrepBatch) {
      const int nb = min(kMpPrepBatch, c1 - cb0);
      int4 v[kMpPrepBatch], wv[kMpPrepBatch];
      if (vec && i0 + kMpPrepRows <= f.nu && (cb0 + kMpPrepBatch) * kMpChunk <= f.nw) { // interior: all loads first
#pragma unroll
        for (int q = 0; q < kMpPrepBatch; ++q) {
          const int j = (cb0 + q) * kMpChunk + lj;
          v[q] = __ldg(reinterpret_cast<const int4 *>(row + j));
          wv[q] = __ldg(reinterpret_cast<const int4 *>(f.w + j));
        }
      } else {
#pragma unroll
      for (int q = 0; q < kMpPrepBatch; ++q) {
        const int j = (cb0 + q) * kMpChunk + lj;
        v[q] = wv[q] = make_int4(0, 0, 0, 0);
        if (q < nb && i < f.nu) {
          if (vec && j + 3 < f.nw) {
            v[q] = *reinterpret_cast<const int4 *>(row + j);
            wv[q] = *reinterpret_cast<const int4 *>(f.w + j);
          } else {
            int *pv = &v[q].x, *pw = &wv[q].x;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (j + e < f.nw) pv[e] = row[j + e], pw[e] = f.w[j + e];
          }
        }
      }
      }
#pragma unroll
      for (int q = 0; q < kMpPrepBatch; ++q) {
        const int *pv = &v[q].x, *pw = &wv[q].x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = (cb0 + q) * kMpChunk + lj + e;
          tr[q][lj + e][lr] = i >= f.nu ? 0u
                              : j < f.nw ? (static_cast<uint32_t>(min(pw[e] + pv[e] - rai, f.cap)) << jb) |
                                               (static_cast<uint32_t>(j) & jmask)
                                         : 0xFFFFu;
        }
      }
      __syncthreads();
      for (int q = 0; q < nb; ++q) {
        uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = tr[q][sj][sr + e] * 0x10001u; // a'' in both halves
        *reinterpret_cast<uint4 *>(f.A + (static_cast<int64_t>(ti) * f.nchunks + cb0 + q) * (kMpChunk * kMpTile) +
                                   sj * kMpTile + ii0 + sr) = make_uint4(x[0], x[1], x[2], x[3]);
      }
      __syncthreads();
    }
    return;
  }
  pb -= a_blocks;
  __shared__ int part[8][kMpPrepCols + 1];
  __shared__ int cbs[kMpPrepCols];
  const int k0 = static_cast<int>(pb / f.b_batches) * kMpPrepCols;
  const int batch = static_cast<int>(pb % f.b_batches);
  const int c0 = f.b_batches > 1 ? batch * kMpPrepBatch : 0, c1 = f.b_batches > 1 ? min(f.nchunks, c0 + kMpPrepBatch) : f.nchunks;
  if (!f.cb_ready) {
    const int k = k0 + lane;
    int m = INT_MAX;
    if (k < f.nv) {
      int j = warp;
      for (; j + 24 < f.nw; j += 32) {
        const int a0 = f.t2[static_cast<int64_t>(j) * f.nv + k], a1 = f.t2[static_cast<int64_t>(j + 8) * f.nv + k];
        const int a2 = f.t2[static_cast<int64_t>(j + 16) * f.nv + k], a3 = f.t2[static_cast<int64_t>(j + 24) * f.nv + k];
        m = min(m, min(min(a0, a1), min(a2, a3)));
      }
      for (; j < f.nw; j += 8) m = min(m, f.t2[static_cast<int64_t>(j) * f.nv + k]);
    }
    part[warp][lane] = m;
    __syncthreads();
    if (tid < kMpPrepCols) {
      int r = part[0][tid];
#pragma unroll
      for (int q = 1; q < 8; ++q) r = min(r, part[q][tid]);
      cbs[tid] = r;
      if (k0 + tid < f.nv) f.cb[k0 + tid] = mm_enc(r);
    }
  } else if (tid < kMpPrepCols) {
    cbs[tid] = k0 + tid < f.nv ? mm_dec(f.cb[k0 + tid]) : 0;
  }
  __syncthreads();
  const int bw = f.b_cols ? f.b_cols : kMpTile; // B rows: one 128-column tile, or a chain fold's whole row
  const int tk = k0 / bw, kk0 = k0 % bw;
  const int sj = tid >> 3, kq = (tid & 7) * 4; // j sj, columns kq..kq+3
  int cbq[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) cbq[e] = cbs[kq + e];
  const bool bvec = ((f.nv & 3) | (reinterpret_cast<uintptr_t>(f.t2) & 15)) == 0;
  for (int cb0 = c0; cb0 < c1; cb0 += kMpPrepBatch) {
    const int nb = min(kMpPrepBatch, c1 - cb0);
    uint32_t v[kMpPrepBatch][4];
    if (bvec && k0 + kMpPrepCols <= f.nv && (cb0 + kMpPrepBatch) * kMpChunk <= f.nw) { // interior: 16-byte loads first
      int4 x[kMpPrepBatch];
#pragma unroll
      for (int q = 0; q < kMpPrepBatch; ++q)
        x[q] = __ldg(reinterpret_cast<const int4 *>(f.t2 + static_cast<int64_t>((cb0 + q) * kMpChunk + sj) * f.nv + k0 + kq));
#pragma unroll
      for (int q = 0; q < kMpPrepBatch; ++q) {
        const int *px = &x[q].x;
#pragma unroll
        for (int e = 0; e < 4; ++e) v[q][e] = static_cast<uint32_t>(min(px[e] - cbq[e], f.cap)) << jb;
      }
    } else {
#pragma unroll
    for (int q = 0; q < kMpPrepBatch; ++q) {
      const int j = (cb0 + q) * kMpChunk + sj;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = k0 + kq + e;
        v[q][e] = q < nb && j < f.nw && k < f.nv
                      ? static_cast<uint32_t>(min(f.t2[static_cast<int64_t>(j) * f.nv + k] - cbq[e], f.cap)) << jb : 0u;
      }
    }
    }
#pragma unroll
    for (int q = 0; q < kMpPrepBatch; ++q)
      if (q < nb)
        *reinterpret_cast<uint2 *>(f.B + ((static_cast<int64_t>(tk) * f.nchunks + cb0 + q) * kMpChunk + sj) * bw + kk0 +
                                   kq) = make_uint2(v[q][0] | (v[q][1] << 16), v[q][2] | (v[q][3] << 16));
  }
}

// ---- mp_fold ------------------------------------------------------------------

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMpConsumers) : "memory"); }

// stream-K ranges: CTA b owns units [b * units / G, (b + 1) * units / G)
__device__ __forceinline__ int64_t mp_first(int64_t b, int64_t units, int64_t G) { return b * units / G; }
// the CTA owning unit u: the largest b with b * units / G <= u
__device__ __forceinline__ int64_t mp_owner(int64_t u, int64_t units, int64_t G) { return ((u + 1) * G - 1) / units; }

// dp_tiles > 0: data-parallel mode for wide launches — CTA b takes whole tiles
// b, b + G, ... (tile_begin order), so co-running CTAs share operand blocks in
// L2 and no tile is split; 0: stream-K over the contiguous unit ranges.
template <int JB>
__global__ void __launch_bounds__(kMpThreads, 1) mp_fold_kernel(const MpFold *folds, int n, int64_t units, int64_t dp_tiles) {
  extern __shared__ __align__(128) unsigned char mp_smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(mp_smem + kMpStages * kMpStageBytes);
  uint64_t *empty = full + kMpStages;
  const int64_t G = gridDim.x;
  const int64_t u_begin = mp_first(blockIdx.x, units, G), u_end = mp_first(blockIdx.x + 1, units, G);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_launch_dependents(); // the next wave's kernels may be scheduled; they wait in griddepcontrol.wait
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kMpStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMpConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait(); // operand blocks / minima from mp_prep, counters from the previous fold
  __syncthreads();

  if (warp == kMpConsumers / 32) { // producer: one thread streams the CTA's units in order
    if (lane == 0) {
      int64_t nn = 0;
      auto stage = [&](const MpFold *f, int tile, int c) {
        const int ti = tile / f->tiles_k, tk = tile % f->tiles_k;
        const int s = static_cast<int>(nn % kMpStages);
        const unsigned ph = static_cast<unsigned>(nn / kMpStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        unsigned char *st = mp_smem + s * kMpStageBytes;
        mbar_expect_tx(&full[s], kMpStageBytes);
        bulk_g2s(st, f->A + (static_cast<int64_t>(ti) * f->nchunks + c) * (kMpChunk * kMpTile), kMpStageA, &full[s]);
        bulk_g2s(st + kMpStageA, f->B + (static_cast<int64_t>(tk) * f->nchunks + c) * (kMpChunk * kMpTile), kMpStageB,
                 &full[s]);
        ++nn;
      };
      if (dp_tiles > 0) {
        for (int64_t tg = blockIdx.x; tg < dp_tiles; tg += G) {
          const MpFold *f = &folds[find_desc(folds, n, tg, [](const MpFold &x) { return x.tile_begin; })];
          for (int c = 0; c < f->nchunks; ++c) stage(f, static_cast<int>(tg - f->tile_begin), c);
        }
      } else {
        int64_t seg_hi = -1;
        const MpFold *f = nullptr;
        for (int64_t u = u_begin; u < u_end; ++u) {
          if (u >= seg_hi) {
            const int fi = find_desc(folds, n, u, [](const MpFold &x) { return x.unit_begin; });
            f = &folds[fi];
            seg_hi = fi + 1 < n ? folds[fi + 1].unit_begin : units;
          }
          const int64_t local = u - f->unit_begin;
          stage(f, static_cast<int>(local / f->nchunks), static_cast<int>(local % f->nchunks));
        }
      }
    }
    return;
  }

  // consumers: thread (ty, tx) owns rows ty*8..+7, columns tx*8..+7 of the tile
  const int ty = (warp >> 1) * 4 + (lane >> 3), tx = (warp & 1) * 8 + (lane & 7);
  // argmin groups of 2^JB j: GPS per stage (JB <= 5) or one per CPG stages (JB = 6)
  constexpr int GL = (1 << JB) < kMpChunk ? (1 << JB) : kMpChunk; // j of a group inside one stage
  constexpr int GPS = kMpChunk / GL, CPG = (1 << JB) / GL;
  constexpr uint32_t LOW2 = ((1u << JB) - 1) * 0x10001u;
  int64_t u = u_begin, nn = 0, tg = blockIdx.x;
  while (dp_tiles > 0 ? tg < dp_tiles : u < u_end) {
    int fi, tile, c_first;
    int64_t tile_lo, tile_hi, seg_lo, seg_end;
    if (dp_tiles > 0) { // a whole tile
      fi = find_desc(folds, n, tg, [](const MpFold &x) { return x.tile_begin; });
      tile = static_cast<int>(tg - folds[fi].tile_begin);
      c_first = 0;
      tile_lo = seg_lo = folds[fi].unit_begin + static_cast<int64_t>(tile) * folds[fi].nchunks;
      tile_hi = seg_end = tile_lo + folds[fi].nchunks;
      tg += G;
      u = seg_lo;
    } else {
      fi = find_desc(folds, n, u, [](const MpFold &x) { return x.unit_begin; });
      const int64_t local = u - folds[fi].unit_begin;
      tile = static_cast<int>(local / folds[fi].nchunks);
      c_first = static_cast<int>(local % folds[fi].nchunks);
      tile_lo = folds[fi].unit_begin + static_cast<int64_t>(tile) * folds[fi].nchunks;
      tile_hi = tile_lo + folds[fi].nchunks;
      seg_lo = u;
      seg_end = min(u_end, tile_hi);
    }
    const MpFold &f = folds[fi];

    // key = value << (16 + JB) | j (group << JB | j-low): lowest value, then lowest j.
    // A group cut by a segment boundary contributes its part; parts combine by min.
    uint32_t key[8][8], m[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int q = 0; q < 8; ++q) key[r][q] = 0xFFFFFFFFu;
#pragma unroll
      for (int q = 0; q < 4; ++q) m[r][q] = 0xFFFFFFFFu; // defined on every path (reset at each group start)
    }

    for (int c = c_first; u < seg_end; ++u, ++nn, ++c) {
      const int s = static_cast<int>(nn % kMpStages);
      mbar_wait(&full[s], static_cast<unsigned>(nn / kMpStages) & 1u);
      const uint32_t *As = reinterpret_cast<const uint32_t *>(mp_smem + s * kMpStageBytes) + ty * 8;
      const uint32_t *Bs = reinterpret_cast<const uint32_t *>(mp_smem + s * kMpStageBytes + kMpStageA) + tx * 4;
      const bool g_start = CPG == 1 || c % CPG == 0 || c == c_first;
      const bool g_end = CPG == 1 || c % CPG == CPG - 1 || u + 1 == seg_end;
#pragma unroll
      for (int g = 0; g < GPS; ++g) {
        if (g_start) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) m[r][q] = 0xFFFFFFFFu; // min(a'' + b'', 0xFFFF) = a'' + b''
        }
#pragma unroll
        for (int jj = g * GL; jj < (g + 1) * GL; ++jj) {
          uint32_t a[8], bb[4];
          *reinterpret_cast<uint4 *>(&a[0]) = *reinterpret_cast<const uint4 *>(As + jj * kMpTile);
          *reinterpret_cast<uint4 *>(&a[4]) = *reinterpret_cast<const uint4 *>(As + jj * kMpTile + 4);
          *reinterpret_cast<uint4 *>(&bb[0]) = *reinterpret_cast<const uint4 *>(Bs + jj * (kMpTile / 2));
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) m[r][q] = __viaddmin_u16x2(a[r], bb[q], m[r][q]);
        }
        if (g_end) {
          const uint32_t G2 = static_cast<uint32_t>((c * kMpChunk + g * GL) >> JB) * ((1u << JB) * 0x10001u); // group << JB, both halves
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t gj = (m[r][q] & LOW2) | G2, mv = m[r][q] & ~LOW2;
              key[r][2 * q] = min(key[r][2 * q], __byte_perm(mv, gj, 0x1054));
              key[r][2 * q + 1] = min(key[r][2 * q + 1], __byte_perm(mv, gj, 0x3276));
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- epilogue -----------------------------------------------------------
    const int ti = tile / f.tiles_k, tk = tile % f.tiles_k;
    const int i0 = ti * kMpTile + ty * 8, k0 = tk * kMpTile + tx * 8;
    bool store = c_first == 0 && seg_end == tile_hi;
    if (!store) {
      // split tile.  Its owner is the CTA holding its first chunk: the tile is
      // the owner's LAST segment, and every other part is a later CTA's FIRST
      // segment, deposited early in that CTA's run; so the owner rarely waits.
      // Parts: keys to the CTA's slot, then one release increment (no round
      // trip on the consumers' path).  Owner: acquire the count, combine, store.
      const int64_t b0 = mp_owner(tile_lo, units, G), b1 = mp_owner(tile_hi - 1, units, G);
      if (seg_lo != tile_lo) {
        uint32_t *mine = f.part + static_cast<int64_t>(blockIdx.x) * kMpTileCells + (ty * 8) * kMpTile + tx * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          *reinterpret_cast<uint4 *>(mine + r * kMpTile) = make_uint4(key[r][0], key[r][1], key[r][2], key[r][3]);
          *reinterpret_cast<uint4 *>(mine + r * kMpTile + 4) = make_uint4(key[r][4], key[r][5], key[r][6], key[r][7]);
        }
        consumer_sync(); // the CTA's part stores precede thread 0's release
        if (tid == 0) {
          __threadfence();
          atomicAdd(f.cnt + tile, 1u);
        }
        continue;
      }
      if (tid == 0) {
        const unsigned want = static_cast<unsigned>(b1 - b0);
        unsigned got;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(f.cnt + tile) : "memory");
          if (got >= want) break;
          __nanosleep(64);
        }
        f.cnt[tile] = 0; // every part has arrived: restore for the next use
      }
      consumer_sync();
      for (int64_t ob = b0 + 1; ob <= b1; ++ob) {
        const uint32_t *other = f.part + ob * kMpTileCells + (ty * 8) * kMpTile + tx * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint4 lo = __ldcg(reinterpret_cast<const uint4 *>(other + r * kMpTile));
          const uint4 hi = __ldcg(reinterpret_cast<const uint4 *>(other + r * kMpTile + 4));
          key[r][0] = min(key[r][0], lo.x), key[r][1] = min(key[r][1], lo.y);
          key[r][2] = min(key[r][2], lo.z), key[r][3] = min(key[r][3], lo.w);
          key[r][4] = min(key[r][4], hi.x), key[r][5] = min(key[r][5], hi.y);
          key[r][6] = min(key[r][6], hi.z), key[r][7] = min(key[r][7], hi.w);
        }
      }
      store = true;
    }
    if (store) {
      int cbk[8], wn[8], cm[8]; // cm: the consumer's column minima over this thread's rows
      bool capped = false;      // a minimum reached the (optimistic) cap
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        cbk[q] = k0 + q < f.nv ? mm_dec(f.cb[k0 + q]) : 0;
        wn[q] = f.ra_next && k0 + q < f.nv ? f.w_next[k0 + q] : 0;
        cm[q] = INT_MAX;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r;
        const bool row_ok = i < f.nu;
        const int rai = row_ok ? mm_dec(f.ra[i]) : 0;
        int32_t ov[8];
        uint16_t av[8];
        int nm = INT_MAX; // the consumer's row minimum over these columns
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int32_t best = static_cast<int32_t>(key[r][q] >> (16 + JB));
          if (row_ok && k0 + q < f.nv && best >= f.cap) capped = true;
          ov[q] = rai + cbk[q] + best;
          av[q] = static_cast<uint16_t>(key[r][q] & 0xFFFFu);
          if (k0 + q < f.nv) nm = min(nm, ov[q] + wn[q]);
          if (row_ok) cm[q] = min(cm[q], ov[q]);
        }
        if (f.ra_next) { // 8 lanes share the row: reduce, one atomic per warp and row
          nm = min(nm, __shfl_xor_sync(0xffffffffu, nm, 1));
          nm = min(nm, __shfl_xor_sync(0xffffffffu, nm, 2));
          nm = min(nm, __shfl_xor_sync(0xffffffffu, nm, 4));
          if ((lane & 7) == 0 && row_ok && nm != INT_MAX) atomicMin(f.ra_next + i, mm_enc(nm));
        }
        if (!row_ok) continue;
        int32_t *orow = f.out + static_cast<int64_t>(i) * f.nv + k0;
        uint16_t *arow = f.am + static_cast<int64_t>(i) * f.nv + k0;
        if (k0 + 8 <= f.nv && (f.nv & 7) == 0) {
          *reinterpret_cast<int4 *>(orow) = *reinterpret_cast<const int4 *>(&ov[0]);
          *reinterpret_cast<int4 *>(orow + 4) = *reinterpret_cast<const int4 *>(&ov[4]);
          *reinterpret_cast<uint4 *>(arow) = *reinterpret_cast<const uint4 *>(&av[0]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (k0 + q < f.nv) orow[q] = ov[q], arow[q] = av[q];
        }
      }
      if (capped && f.ovf) atomicOr(f.ovf, 1u);
      if (f.cb_next) { // 4 lanes of a warp share each column: reduce, one atomic per warp and column
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cm[q] = min(cm[q], __shfl_xor_sync(0xffffffffu, cm[q], 8));
          cm[q] = min(cm[q], __shfl_xor_sync(0xffffffffu, cm[q], 16));
          if (lane < 8 && k0 + q < f.nv && cm[q] != INT_MAX) atomicMin(f.cb_next + k0 + q, mm_enc(cm[q]));
        }
      }
    }
  }
}

// ---- mp_chain: a run of one-fold waves, row-parallel ---------------------------
// A run of waves whose folds F_1 -> F_2 -> ... chain through t1 (F_{k+1}.t1 =
// F_k.out) and whose t2 are all written before the run (config 5: 314 of its
// 329 waves).  Eq. 2 works row by row, so each CTA carries R rows of the
// source node through EVERY fold of the run with no grid-wide dependency:
// per fold it normalises its rows of t1 (row minima over the full row, in the
// CTA) into shared memory, streams the fold's whole B'' (packed once before the
// run, [j][kMpChainCols] u16) through a bulk-copy ring fed by a producer warp
// that runs ahead across fold boundaries, and writes out / argmins.  Each
// consumer thread owns 4 columns (2 U16x2 pairs) of all R <= 8 rows.  Same
// arithmetic, caps and keys as mp_fold.
constexpr int kMpChainCols = 1024;                     // columns per B'' row (nv <= 1024)
constexpr int kMpChainRows = 8;                        // rows per CTA at most
constexpr int kMpChainJ = 32;                          // j per stage
constexpr int kMpChainStages = 3;
constexpr unsigned kMpChainStageBytes = kMpChainJ * kMpChainCols * 2; // 32 KiB
constexpr int kMpChainNw = 1024;                       // padded nw at most (A in shared memory)
constexpr size_t kMpChainSmem = kMpChainStages * kMpChainStageBytes + static_cast<size_t>(kMpChainNw) * kMpChainRows * 4 +
                                2 * kMpChainStages * 8 + 64;

template <int JB, int RR> // RR: rows per CTA computed (>= R; the unrolled register tile)
__global__ void __launch_bounds__(kMpThreads, 1) mp_chain_kernel(const MpFold *folds, int K, int R) {
  extern __shared__ __align__(128) unsigned char ch_smem[];
  uint32_t *As = reinterpret_cast<uint32_t *>(ch_smem + kMpChainStages * kMpChainStageBytes); // [j][8] a'' (dup)
  uint64_t *full = reinterpret_cast<uint64_t *>(As + kMpChainNw * kMpChainRows);
  uint64_t *empty = full + kMpChainStages;
  int *ras = reinterpret_cast<int *>(empty + kMpChainStages); // [8]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kMpChainStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMpConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kMpConsumers / 32) { // producer: every fold's B'' stages, in order
    if (lane == 0) {
      int s = 0; // ring slot and its phase, advanced incrementally (5 stages: no division per stage)
      unsigned ph = 0;
      for (int k = 0; k < K; ++k) {
        const MpFold &f = folds[k];
        const int stages = f.nchunks * (kMpChunk / kMpChainJ);
        for (int st = 0; st < stages; ++st, s = s + 1 == kMpChainStages ? (ph ^= 1u, 0) : s + 1) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], kMpChainStageBytes);
          bulk_g2s(ch_smem + s * kMpChainStageBytes, f.B + static_cast<int64_t>(st) * kMpChainJ * kMpChainCols,
                   kMpChainStageBytes, &full[s]);
        }
      }
    }
    return;
  }
  constexpr uint32_t LOW2 = ((1u << JB) - 1) * 0x10001u;
  constexpr int SPG = (1 << JB) >= kMpChainJ ? (1 << JB) / kMpChainJ : 1; // stages per argmin group
  static_assert((1 << JB) >= kMpChainJ, "argmin groups span whole stages");
  const int c4 = tid * 4; // this thread's columns c4..c4+3
  int s = 0; // ring slot and phase (as the producer's)
  unsigned ph = 0;
  for (int k = 0; k < K; ++k) {
    const MpFold &f = folds[k];
    const int r0 = static_cast<int>(blockIdx.x) * R, nr = min(R, f.nu - r0);
    const int nwp = f.nchunks * kMpChunk;
    // ---- A: one warp per row loads the row once (all loads in flight), takes
    // its minimum and writes a'' into shared memory (rows >= nr are never stored)
    if (warp < nr) {
      constexpr int kPer = kMpChainNw / 32;
      const int32_t *row = f.t1 + static_cast<int64_t>(r0 + warp) * f.nw;
      int v[kPer];
      int m = INT_MAX;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int j = i * 32 + lane;
        v[i] = j < f.nw ? f.w[j] + row[j] : INT_MAX;
        m = min(m, v[i]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) ras[warp] = m;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int j = i * 32 + lane;
        if (j < nwp)
          As[j * kMpChainRows + warp] =
              (j < f.nw ? (static_cast<uint32_t>(min(v[i] - m, f.cap)) << JB) | (static_cast<uint32_t>(j) & ((1u << JB) - 1))
                        : 0xFFFFu) * 0x10001u;
      }
    }
    consumer_sync();
    // ---- the fold: RR rows x 2 column pairs per thread over all j
    uint32_t key[RR][4], m[RR][2];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q) key[r][q] = 0xFFFFFFFFu;
      m[r][0] = m[r][1] = 0xFFFFFFFFu;
    }
    const int stages = nwp / kMpChainJ;
    for (int st = 0; st < stages; ++st, s = s + 1 == kMpChainStages ? (ph ^= 1u, 0) : s + 1) {
      mbar_wait(&full[s], ph);
      const uint32_t *Bs = reinterpret_cast<const uint32_t *>(ch_smem + s * kMpChainStageBytes) + tid * 2;
      if (st % SPG == 0) {
#pragma unroll
        for (int r = 0; r < RR; ++r) m[r][0] = m[r][1] = 0xFFFFFFFFu;
      }
#pragma unroll
      for (int jj = 0; jj < kMpChainJ; ++jj) {
        const int j = st * kMpChainJ + jj;
        uint32_t a[8];
        *reinterpret_cast<uint4 *>(&a[0]) = *reinterpret_cast<const uint4 *>(As + j * kMpChainRows);
        if constexpr (RR > 4) *reinterpret_cast<uint4 *>(&a[4]) = *reinterpret_cast<const uint4 *>(As + j * kMpChainRows + 4);
        const uint2 b = *reinterpret_cast<const uint2 *>(Bs + jj * (kMpChainCols / 2));
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          m[r][0] = __viaddmin_u16x2(a[r], b.x, m[r][0]);
          m[r][1] = __viaddmin_u16x2(a[r], b.y, m[r][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (st % SPG == SPG - 1 || st == stages - 1) {
        const uint32_t G2 = static_cast<uint32_t>((st * kMpChainJ) >> JB) * ((1u << JB) * 0x10001u);
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t gj = (m[r][q] & LOW2) | G2, mv = m[r][q] & ~LOW2;
            key[r][2 * q] = min(key[r][2 * q], __byte_perm(mv, gj, 0x1054));
            key[r][2 * q + 1] = min(key[r][2 * q + 1], __byte_perm(mv, gj, 0x3276));
          }
      }
    }
    // ---- epilogue: out = ra + cb + best, am = j
    bool capped = false;
    if (c4 < f.nv) {
      int cbk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) cbk[q] = c4 + q < f.nv ? mm_dec(f.cb[c4 + q]) : 0;
      const bool vec = c4 + 4 <= f.nv && (f.nv & 3) == 0;
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        if (r >= nr) break;
        int32_t ov[4];
        uint16_t av[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int32_t best = static_cast<int32_t>(key[r][q] >> (16 + JB));
          if (c4 + q < f.nv && best >= f.cap) capped = true;
          ov[q] = ras[r] + cbk[q] + best;
          av[q] = static_cast<uint16_t>(key[r][q] & 0xFFFFu);
        }
        int32_t *orow = f.out + static_cast<int64_t>(r0 + r) * f.nv + c4;
        uint16_t *arow = f.am + static_cast<int64_t>(r0 + r) * f.nv + c4;
        if (vec) {
          *reinterpret_cast<int4 *>(orow) = *reinterpret_cast<const int4 *>(&ov[0]);
          *reinterpret_cast<uint2 *>(arow) = *reinterpret_cast<const uint2 *>(&av[0]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c4 + q < f.nv) orow[q] = ov[q], arow[q] = av[q];
        }
      }
    }
    if (capped && f.ovf) atomicOr(f.ovf, 1u);
    // the next fold reads this CTA's rows of out (its t1) from global memory
    __threadfence_block();
    consumer_sync();
  }
}

} // namespace pp
