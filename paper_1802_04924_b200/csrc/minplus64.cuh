// minplus64.cuh — the large-table Eq. 2 fold for FP64 tables (analytic or
// measured costs that the fixed-point certificate rejects).
//
// cand = (w[j] + t1[i][j]) + t2[j][k] in the reference's summation order
// (planner.hpp:139-155): the first add is done once per (i, j) in the prep
// (the same IEEE rounding), the second per cell; strict '<' over ascending j
// keeps the lowest index among equal candidates.  64x64 output tile per CTA,
// 4x4 cells per thread: per j, 16 DADD + 16 DSETP on the FP64 pipe, per cell
// two predicated IMADs (the value halves, FMA pipe) and one select (j, ALU);
// operands staged by bulk copies
// (thread 0, mbarrier ring) from per-(tile, 32-j chunk) contiguous blocks.
//
//   mp64_prep  a = w + t1 -> A [tile_i][chunk][32 j][64 i]  (+inf for padded j)
//              t2         -> B [tile_k][chunk][32 j][64 k]  (0 for padded j)
//   mp64_fold  one CTA per (fold, tile), all chunks; out, argmin
#pragma once

#include "kernels.cuh"

#include <cstdint>

namespace pp {

constexpr int kMp64Tile = 64;
constexpr int kMp64Chunk = 32;
constexpr int kMp64Stages = 3;
constexpr int kMp64Threads = 256;
constexpr int kMp64MinSide = 512; // folds with nu, nv >= this take mp64 (per-wave executor)
constexpr unsigned kMp64StageA = kMp64Chunk * kMp64Tile * 8; // 16 KiB
constexpr unsigned kMp64StageBytes = 2 * kMp64StageA;
constexpr size_t kMp64Smem = kMp64Stages * kMp64StageBytes + 2 * kMp64Stages * 8;

struct Mp64Fold {
  const double *t1, *t2, *w;
  double *out;
  uint16_t *am;
  double *A, *B;
  int32_t nu, nw, nv, tiles_i, tiles_k, nchunks;
  int32_t one; // 1 (a value the compiler cannot fold: the fold's predicated IMAD selects)
  int64_t prep_begin; // A prep blocks (row groups of 32 x chunk groups), then B prep blocks (chunk x tile groups)
  int64_t prep_a;
  int64_t tile_begin; // first mp64_fold block
};

__device__ __forceinline__ int find64(const Mp64Fold *d, int n, int64_t b, bool tiles) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((tiles ? d[mid].tile_begin : d[mid].prep_begin) <= b)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// A blocks: 32 rows x kMp64PrepChunks chunks (32x32 tiles transposed through
// shared memory); B blocks: one 32-j chunk of t2 x kMp64PrepTiles column tiles.
// Enough blocks per fold to keep every SM streaming (HBM-bound copy).
constexpr int kMp64PrepChunks = 4;
constexpr int kMp64PrepTiles = 4;
__host__ __device__ inline int64_t mp64_prep_a_blocks(int nu, int nchunks) {
  return static_cast<int64_t>((nu + 31) / 32) * ((nchunks + kMp64PrepChunks - 1) / kMp64PrepChunks);
}
__host__ __device__ inline int64_t mp64_prep_b_blocks(int nchunks, int tiles_k) {
  return static_cast<int64_t>(nchunks) * ((tiles_k + kMp64PrepTiles - 1) / kMp64PrepTiles);
}

__global__ void __launch_bounds__(256) mp64_prep_kernel(const Mp64Fold *folds, int n) {
  const int64_t b = blockIdx.x;
  const Mp64Fold &f = folds[find64(folds, n, b, false)];
  const int64_t pb = b - f.prep_begin;
  const int tid = threadIdx.x;
  if (pb < f.prep_a) {
    __shared__ double tr[32][33];
    const int ncg = (f.nchunks + kMp64PrepChunks - 1) / kMp64PrepChunks;
    const int i0 = static_cast<int>(pb / ncg) * 32, ti = i0 / kMp64Tile, ii0 = i0 % kMp64Tile;
    const int c0 = static_cast<int>(pb % ncg) * kMp64PrepChunks, c1 = min(f.nchunks, c0 + kMp64PrepChunks);
    const int lr = tid >> 3, lj = (tid & 7) * 4; // load: row lr, j lj..lj+3
    const int sj = tid >> 3, sr = (tid & 7) * 4; // store: j sj, rows sr..sr+3
    const int i = i0 + lr;
    for (int c = c0; c < c1; ++c) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = c * kMp64Chunk + lj + e;
        tr[lj + e][lr] = i < f.nu && j < f.nw ? f.w[j] + f.t1[static_cast<int64_t>(i) * f.nw + j] // reference: w + t1 first
                                              : __longlong_as_double(0x7ff0000000000000LL);        // +inf: never a minimum
      }
      __syncthreads();
      double *dst = f.A + (static_cast<int64_t>(ti) * f.nchunks + c) * (kMp64Chunk * kMp64Tile) + sj * kMp64Tile + ii0 + sr;
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = tr[sj][sr + e];
      __syncthreads();
    }
    return;
  }
  // B: chunk c, column tiles [t0, t0 + kMp64PrepTiles): each thread one column, all 32 j
  const int64_t bb = pb - f.prep_a;
  const int ntg = (f.tiles_k + kMp64PrepTiles - 1) / kMp64PrepTiles;
  const int c = static_cast<int>(bb / ntg), t0 = static_cast<int>(bb % ntg) * kMp64PrepTiles;
  const int k = t0 * kMp64Tile + tid, tk = k / kMp64Tile;
  if (tk >= f.tiles_k) return;
  double *dst = f.B + (static_cast<int64_t>(tk) * f.nchunks + c) * (kMp64Chunk * kMp64Tile) + (k - tk * kMp64Tile);
#pragma unroll 4
  for (int jj = 0; jj < kMp64Chunk; ++jj) {
    const int j = c * kMp64Chunk + jj;
    dst[jj * kMp64Tile] = j < f.nw && k < f.nv ? f.t2[static_cast<int64_t>(j) * f.nv + k] : 0.0;
  }
}

__global__ void __launch_bounds__(kMp64Threads, 2) mp64_fold_kernel(const Mp64Fold *folds, int n) {
  extern __shared__ __align__(128) unsigned char m64_smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(m64_smem + kMp64Stages * kMp64StageBytes);
  const int64_t b = blockIdx.x;
  const Mp64Fold &f = folds[find64(folds, n, b, true)];
  const int tile = static_cast<int>(b - f.tile_begin);
  const int ti = tile / f.tiles_k, tk = tile % f.tiles_k;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kMp64Stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double *Ab = f.A + static_cast<int64_t>(ti) * f.nchunks * (kMp64Chunk * kMp64Tile);
  const double *Bb = f.B + static_cast<int64_t>(tk) * f.nchunks * (kMp64Chunk * kMp64Tile);
  auto issue = [&](int c) {
    const int s = c % kMp64Stages;
    unsigned char *st = m64_smem + s * kMp64StageBytes;
    mbar_expect_tx(&full[s], kMp64StageBytes);
    bulk_g2s(st, Ab + static_cast<int64_t>(c) * (kMp64Chunk * kMp64Tile), kMp64StageA, &full[s]);
    bulk_g2s(st + kMp64StageA, Bb + static_cast<int64_t>(c) * (kMp64Chunk * kMp64Tile), kMp64StageA, &full[s]);
  };
  if (tid == 0)
    for (int c = 0; c < kMp64Stages - 1 && c < f.nchunks; ++c) issue(c);
  // best value (as its two 32-bit halves) and argmin per cell.  The value
  // selects are predicated IMADs by a runtime 1 (f.one): they issue on the FMA
  // pipe, which is otherwise idle, instead of two ALU selects per cell (ptxas
  // keeps the j update a select; measured best among the variants tried)
  uint32_t blo[4][4], bhi[4][4], bj[4][4];
  const uint32_t one = static_cast<uint32_t>(f.one);
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) blo[r][q] = 0u, bhi[r][q] = 0x7ff00000u, bj[r][q] = 0u;
  for (int c = 0; c < f.nchunks; ++c) {
    const int s = c % kMp64Stages;
    // the stage refilled below was last read in iteration c - 1: every thread is past it
    __syncthreads();
    if (tid == 0 && c + kMp64Stages - 1 < f.nchunks) {
      fence_proxy_async(); // generic reads of that stage before the async writes
      issue(c + kMp64Stages - 1);
    }
    mbar_wait(&full[s], static_cast<unsigned>(c / kMp64Stages) & 1u);
    const double *As = reinterpret_cast<const double *>(m64_smem + s * kMp64StageBytes) + ty * 4;
    const double *Bs = reinterpret_cast<const double *>(m64_smem + s * kMp64StageBytes + kMp64StageA) + tx * 4;
#pragma unroll 8
    for (int jj = 0; jj < kMp64Chunk; ++jj) {
      double a[4], bv[4];
      *reinterpret_cast<double2 *>(&a[0]) = *reinterpret_cast<const double2 *>(As + jj * kMp64Tile);
      *reinterpret_cast<double2 *>(&a[2]) = *reinterpret_cast<const double2 *>(As + jj * kMp64Tile + 2);
      *reinterpret_cast<double2 *>(&bv[0]) = *reinterpret_cast<const double2 *>(Bs + jj * kMp64Tile);
      *reinterpret_cast<double2 *>(&bv[2]) = *reinterpret_cast<const double2 *>(Bs + jj * kMp64Tile + 2);
      const int j = c * kMp64Chunk + jj;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double cand = __dadd_rn(a[r], bv[q]);
          // strict: the lowest j wins ties
          asm("{\n\t.reg .pred p;\n\t.reg .f64 b;\n\t.reg .b32 cl, ch;\n\t"
              "mov.b64 b, {%0, %1};\n\t"
              "mov.b64 {cl, ch}, %3;\n\t"
              "setp.lt.f64 p, %3, b;\n\t"
              "@p mad.lo.u32 %0, cl, %5, 0;\n\t"
              "@p mad.lo.u32 %1, ch, %5, 0;\n\t"
              "@p mad.lo.u32 %2, %4, %5, 0;\n\t}"
              : "+r"(blo[r][q]), "+r"(bhi[r][q]), "+r"(bj[r][q])
              : "d"(cand), "r"(static_cast<uint32_t>(j)), "r"(one));
        }
    }
  }
  const int i0 = ti * kMp64Tile + ty * 4, k0 = tk * kMp64Tile + tx * 4;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + r;
    if (i >= f.nu) break;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (k0 + q < f.nv) {
        f.out[static_cast<int64_t>(i) * f.nv + k0 + q] =
            __hiloint2double(static_cast<int>(bhi[r][q]), static_cast<int>(blo[r][q]));
        f.am[static_cast<int64_t>(i) * f.nv + k0 + q] = static_cast<uint16_t>(bj[r][q]);
      }
  }
}

} // namespace pp
