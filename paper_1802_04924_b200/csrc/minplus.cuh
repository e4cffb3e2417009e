// minplus.cuh — the large-table Eq. 2 fold (K3) for exact fixed-point tables.
//
// out[i][k] = min_j (a[i][j] + b[j][k]),  a = w[j] + t1[i][j],  b = t2[j][k],
// argmin = lowest j (planner.hpp:139-155), all in int32 units of 2^-s.
//
// Min-plus is shift-invariant per row of a and per column of b, so with
// ra[i] = min_j a[i][j] and cb[k] = min_j b[j][k] the normalised operands
// a' = a - ra, b' = b - cb lie in [0, rowspan(a)] x [0, colspan(b)].  When the
// host's span bounds (propagated through the schedule) prove rowspan(a) <=
// 16383 and colspan(b) <= 16382, every candidate a' + b' fits a signed 16-bit
// lane with no overflow, and the fold runs two cells per instruction:
// VIADDMNMX.S16x2 = min(a' + b', m) on a (cell, cell+1) pair — one
// instruction per two (add, min) cell updates, i.e. the FP32 CUDA-core
// roofline of one lane-op per cell (measured: tools/microbench).
//
// Argmin: per 32-j chunk the kernel keeps the chunk minimum and, with a strict
// lane-wise "<" against the running best, the first chunk that attains the
// final minimum (earlier chunks win ties).  A rescan of that chunk's 32
// candidates — identical integer arithmetic — returns the first j with the
// minimum value: exactly the reference's lowest-index tie-break.
//
//   mp_reduce  ra[i], cb[k]
//   mp_pack    a' -> A2T [j][i] (u32, a' in both halves) and A16 [i][j];
//              b' -> B16 [j][k] and B16T [k][j]  (s16), padded with 16383
//   mp_fold    128x128 tile per CTA, 8x8 cells per thread, cp.async 4-stage
//              pipeline over 32-j chunks; split-j across CTAs combine with
//              atomicMin on (best << 16 | chunk)
//   mp_rescan  first j of the winning chunk; out = ra + cb + best, am = j
#pragma once

#include "kernels.cuh"

#include <climits>
#include <cstdint>

namespace pp {

constexpr int kMpTile = 128;   // output rows/cols per CTA
constexpr int kMpChunk = 32;   // j per pipeline stage (and argmin chunk)
constexpr int kMpStages = 4;
constexpr int kMpThreads = 256;
constexpr int kMpPad = 16383;  // padding value of a' and b'
constexpr size_t kMpStageBytes = kMpChunk * kMpTile * 4 + kMpChunk * kMpTile * 2; // 24 KiB
constexpr size_t kMpSmem = kMpStages * kMpStageBytes;                            // 96 KiB

struct MpFold {
  // inputs (original or derived tables, int32 units)
  const int32_t *t1; // [nu][nw]
  const int32_t *t2; // [nw][nv]
  const int32_t *w;  // [nw]
  // outputs
  int32_t *out;  // [nu][nv]
  uint16_t *am;  // [nu][nv]
  // scratch
  int32_t *ra, *cb;   // [nu], [nv]
  int32_t *cbp;       // [col_segs][nv] partial column minima (mp_reduce), folded into cb by mp_pack
  int32_t col_segs;   // j segments of kMpRedColJ per column block
  uint32_t *A2T;      // [nwp][nup]
  uint16_t *A16;      // [nu][nwp]
  uint16_t *B16;      // [nwp][nvp]
  uint16_t *B16T;     // [nv][nwp]
  int32_t *P;         // [nup][nvp] packed (best << 16 | chunk)
  int32_t nu, nw, nv, nup, nwp, nvp;
  int32_t tiles_i, tiles_k, splits, chunks_per_split;
  int64_t fold_begin;   // first mp_fold block of this fold
  int64_t red_begin;    // first mp_reduce block
  int64_t pack_begin;   // first mp_pack block
  int64_t rescan_begin; // first mp_rescan block
};

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

// ---- mp_reduce: ra (one warp per row) and partial cb (32 columns x one
// j segment per block: 8 warps x kMpRedColJ / 8 rows each, loads unrolled) --
constexpr int kMpRedRowsPerBlock = 8; // 8 warps
constexpr int kMpRedColJ = 128;       // j rows per column block
__global__ void __launch_bounds__(256) mp_reduce_kernel(const MpFold *folds, int n) {
  const int64_t b = blockIdx.x;
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.red_begin; })];
  const int64_t rb = b - f.red_begin;
  const int64_t row_blocks = (f.nu + kMpRedRowsPerBlock - 1) / kMpRedRowsPerBlock;
  if (rb < row_blocks) {
    const int i = static_cast<int>(rb) * kMpRedRowsPerBlock + (threadIdx.x >> 5);
    if (i >= f.nu) return;
    const int lane = threadIdx.x & 31;
    int m = INT_MAX;
    const int32_t *row = f.t1 + static_cast<int64_t>(i) * f.nw;
    int j = lane;
    for (; j + 96 < f.nw; j += 128) { // four independent loads in flight
      const int a0 = f.w[j] + row[j], a1 = f.w[j + 32] + row[j + 32];
      const int a2 = f.w[j + 64] + row[j + 64], a3 = f.w[j + 96] + row[j + 96];
      m = min(m, min(min(a0, a1), min(a2, a3)));
    }
    for (; j < f.nw; j += 32) m = min(m, f.w[j] + row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) f.ra[i] = m;
    return;
  }
  // columns: block (column block, j segment); 8 j-lanes x kMpRedColJ / 8 rows
  __shared__ int part[8][33];
  const int64_t cbk = rb - row_blocks;
  const int seg = static_cast<int>(cbk % f.col_segs);
  const int kc = static_cast<int>(cbk / f.col_segs) * 32 + (threadIdx.x & 31), lane_j = threadIdx.x >> 5;
  const int jend = min(f.nw, (seg + 1) * kMpRedColJ);
  int m = INT_MAX;
  if (kc < f.nv) {
    int j = seg * kMpRedColJ + lane_j;
    for (; j + 24 < jend; j += 32) { // four independent loads in flight
      const int a0 = f.t2[static_cast<int64_t>(j) * f.nv + kc], a1 = f.t2[static_cast<int64_t>(j + 8) * f.nv + kc];
      const int a2 = f.t2[static_cast<int64_t>(j + 16) * f.nv + kc], a3 = f.t2[static_cast<int64_t>(j + 24) * f.nv + kc];
      m = min(m, min(min(a0, a1), min(a2, a3)));
    }
    for (; j < jend; j += 8) m = min(m, f.t2[static_cast<int64_t>(j) * f.nv + kc]);
  }
  part[lane_j][threadIdx.x & 31] = m;
  __syncthreads();
  if (threadIdx.x < 32 && kc < f.nv) {
    int r = part[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < 8; ++q) r = min(r, part[q][threadIdx.x]);
    f.cbp[static_cast<int64_t>(seg) * f.nv + kc] = r;
  }
}

// cb[k] = min over the column's segment minima
__device__ __forceinline__ int mp_colmin(const MpFold &f, int k) {
  int m = f.cbp[k];
  for (int s = 1; s < f.col_segs; ++s) m = min(m, f.cbp[static_cast<int64_t>(s) * f.nv + k]);
  return m;
}

// ---- mp_pack: 32x32 tiles; A part over (i, j) then B part over (j, k) -------
__global__ void __launch_bounds__(256) mp_pack_kernel(const MpFold *folds, int n) {
  __shared__ int32_t tile[32][33];
  const int64_t b = blockIdx.x;
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.pack_begin; })];
  int64_t pb = b - f.pack_begin;
  const int ti_a = f.nup / 32, tj = f.nwp / 32, tk = f.nvp / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5; // 32 x 8
  if (pb < static_cast<int64_t>(ti_a) * tj) {
    const int i0 = static_cast<int>(pb / tj) * 32, j0 = static_cast<int>(pb % tj) * 32;
    // all four rows' loads first (the stores below could alias them as far
    // as the compiler knows, which would serialise load -> store per row)
    int v[4];
    const int j = j0 + tx;
#pragma unroll
    for (int q = 0; q < 4; ++q) { // row i = i0 + ty + 8q, col j
      const int i = i0 + ty + 8 * q;
      v[q] = i < f.nu && j < f.nw ? f.w[j] + f.t1[static_cast<int64_t>(i) * f.nw + j] - f.ra[i] : kMpPad;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q, i = i0 + r;
      tile[r][tx] = v[q];
      if (i < f.nu) f.A16[static_cast<int64_t>(i) * f.nwp + j] = static_cast<uint16_t>(v[q]);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) { // A2T[j0 + r][i0 + tx]
      const uint32_t v = static_cast<uint32_t>(tile[tx][r]) & 0xffffu;
      f.A2T[static_cast<int64_t>(j0 + r) * f.nup + i0 + tx] = v | (v << 16);
    }
    return;
  }
  pb -= static_cast<int64_t>(ti_a) * tj;
  const int j0 = static_cast<int>(pb / tk) * 32, k0 = static_cast<int>(pb % tk) * 32;
  const int cbk = k0 + tx < f.nv ? mp_colmin(f, k0 + tx) : 0;
  if (j0 == 0 && ty == 0 && k0 + tx < f.nv) f.cb[k0 + tx] = cbk; // for mp_rescan
  {
    int v[4];
    const int k = k0 + tx;
#pragma unroll
    for (int q = 0; q < 4; ++q) { // row j = j0 + ty + 8q, col k
      const int j = j0 + ty + 8 * q;
      v[q] = j < f.nw && k < f.nv ? f.t2[static_cast<int64_t>(j) * f.nv + k] - cbk : kMpPad;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q;
      tile[r][tx] = v[q];
      f.B16[static_cast<int64_t>(j0 + r) * f.nvp + k] = static_cast<uint16_t>(v[q]);
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) { // B16T[k0 + r][j0 + tx]
    const int k = k0 + r;
    if (k < f.nv) f.B16T[static_cast<int64_t>(k) * f.nwp + j0 + tx] = static_cast<uint16_t>(tile[tx][r]);
  }
}

// ---- mp_fold ----------------------------------------------------------------

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// cp_async_commit / cp_async_wait: kernels.cuh

__global__ void __launch_bounds__(kMpThreads, 1) mp_fold_kernel(const MpFold *folds, int n) {
  extern __shared__ __align__(16) unsigned char mp_smem[];
  const int64_t b = blockIdx.x;
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.fold_begin; })];
  int64_t lb = b - f.fold_begin;
  const int tiles = f.tiles_i * f.tiles_k;
  const int split = static_cast<int>(lb / tiles);
  lb -= static_cast<int64_t>(split) * tiles;
  const int i0 = static_cast<int>(lb / f.tiles_k) * kMpTile, k0 = static_cast<int>(lb % f.tiles_k) * kMpTile;
  const int nchunks = f.nwp / kMpChunk;
  const int c_begin = split * f.chunks_per_split;
  const int c_end = min(nchunks, c_begin + f.chunks_per_split);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ty = (warp >> 1) * 4 + (lane >> 3), tx = (warp & 1) * 8 + (lane & 7);

  auto stageA = [&](int s) { return reinterpret_cast<uint32_t *>(mp_smem + s * kMpStageBytes); };
  auto stageB = [&](int s) {
    return reinterpret_cast<uint32_t *>(mp_smem + s * kMpStageBytes + kMpChunk * kMpTile * 4);
  };
  auto load = [&](int c, int s) {
    const int j0 = c * kMpChunk;
    uint32_t *As = stageA(s);
    uint32_t *Bs = stageB(s);
#pragma unroll
    for (int q = 0; q < 4; ++q) { // A: 32 rows x 512 B = 1024 x 16 B
      const int e = tid + q * kMpThreads, r = e >> 5, c16 = e & 31;
      cp_async16(As + r * kMpTile + c16 * 4, f.A2T + static_cast<int64_t>(j0 + r) * f.nup + i0 + c16 * 4);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) { // B: 32 rows x 256 B = 512 x 16 B
      const int e = tid + q * kMpThreads, r = e >> 4, c16 = e & 15;
      cp_async16(Bs + r * (kMpTile / 2) + c16 * 4, f.B16 + static_cast<int64_t>(j0 + r) * f.nvp + k0 + c16 * 8);
    }
  };

  // per cell: packed (chunk minimum << 16 | chunk); an integer min keeps the
  // smallest value and, among equal values, the earliest chunk
  int32_t key[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) key[r][c] = INT_MAX;

  // prologue: stages 0..S-2
#pragma unroll
  for (int s = 0; s < kMpStages - 1; ++s) {
    if (c_begin + s < c_end) load(c_begin + s, s);
    cp_async_commit();
  }
  for (int c = c_begin; c < c_end; ++c) {
    const int s = (c - c_begin) % kMpStages;
    cp_async_wait<kMpStages - 2>();
    __syncthreads();
    { // prefetch chunk c + S - 1 into the stage freed last iteration
      const int cn = c + kMpStages - 1;
      if (cn < c_end) load(cn, (cn - c_begin) % kMpStages);
      cp_async_commit();
    }
    const uint32_t *As = stageA(s) + ty * 8;
    const uint32_t *Bs = stageB(s) + tx * 4;
    uint32_t m[8][4];
#pragma unroll
    for (int jj = 0; jj < kMpChunk; ++jj) {
      uint32_t a[8], bb[4];
      *reinterpret_cast<uint4 *>(&a[0]) = *reinterpret_cast<const uint4 *>(As + jj * kMpTile);
      *reinterpret_cast<uint4 *>(&a[4]) = *reinterpret_cast<const uint4 *>(As + jj * kMpTile + 4);
      *reinterpret_cast<uint4 *>(&bb[0]) = *reinterpret_cast<const uint4 *>(Bs + jj * (kMpTile / 2));
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          m[r][q] = jj == 0 ? __vadd2(a[r], bb[q]) : __viaddmin_s16x2(a[r], bb[q], m[r][q]);
    }
    const uint32_t cid = static_cast<uint32_t>(c);
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) { // PRMT builds (half << 16 | chunk) for each half
        key[r][2 * q] = min(key[r][2 * q], static_cast<int32_t>(__byte_perm(m[r][q], cid, 0x1054)));
        key[r][2 * q + 1] = min(key[r][2 * q + 1], static_cast<int32_t>(__byte_perm(m[r][q], cid, 0x3254)));
      }
  }
  cp_async_wait<0>();

  // epilogue: packed (best << 16 | chunk), lexicographic min across splits
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + ty * 8 + r;
    int32_t *prow = f.P + static_cast<int64_t>(i) * f.nvp + k0 + tx * 8;
    const int32_t *v = key[r];
    if (f.splits == 1) {
      *reinterpret_cast<int4 *>(prow) = *reinterpret_cast<const int4 *>(&v[0]);
      *reinterpret_cast<int4 *>(prow + 4) = *reinterpret_cast<const int4 *>(&v[4]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) atomicMin(prow + q, v[q]);
    }
  }
}

// ---- mp_rescan: one thread per output cell ------------------------------------
__global__ void __launch_bounds__(256) mp_rescan_kernel(const MpFold *folds, int n) {
  const int64_t b = blockIdx.x;
  const MpFold &f = folds[find_desc(folds, n, b, [](const MpFold &x) { return x.rescan_begin; })];
  const int64_t cell = (b - f.rescan_begin) * 256 + threadIdx.x;
  if (cell >= static_cast<int64_t>(f.nu) * f.nv) return;
  const int i = static_cast<int>(cell / f.nv), k = static_cast<int>(cell % f.nv);
  const int32_t p = f.P[static_cast<int64_t>(i) * f.nvp + k];
  const int bestv = p >> 16, chunk = p & 0xffff;
  const int j0 = chunk * kMpChunk;
  const uint4 *ar = reinterpret_cast<const uint4 *>(f.A16 + static_cast<int64_t>(i) * f.nwp + j0);
  const uint4 *br = reinterpret_cast<const uint4 *>(f.B16T + static_cast<int64_t>(k) * f.nwp + j0);
  int jbest = j0 + kMpChunk; // sentinel
#pragma unroll
  for (int q = 3; q >= 0; --q) { // scan backwards so the first match wins without a branch
    const uint4 av = ar[q], bv = br[q];
    const uint32_t aw[4] = {av.x, av.y, av.z, av.w}, bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
    for (int e = 3; e >= 0; --e) {
      const int hi = static_cast<int>(aw[e] >> 16) + static_cast<int>(bw[e] >> 16);
      const int lo = static_cast<int>(aw[e] & 0xffffu) + static_cast<int>(bw[e] & 0xffffu);
      const int j = j0 + q * 8 + e * 2;
      if (hi == bestv) jbest = j + 1;
      if (lo == bestv) jbest = j;
    }
  }
  f.out[cell] = f.ra[i] + f.cb[k] + bestv;
  f.am[cell] = static_cast<uint16_t>(jbest);
}

} // namespace pp
