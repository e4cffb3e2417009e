// fused.cuh — the whole plan in ONE cooperative kernel, for plans whose folds
// all take the generic tiled kernel (the real-model regime: <= a few hundred
// configs per layer, where launch latency, not arithmetic, bounds a search).
//
//   phase 0   K2 node costs + K1 xfer cells (plan() only), grid-stride
//   waves     every fold tile / merge chunk of dependency wave w, grid-stride;
//             grid.sync() between waves (the scheduler's DAG levels)
//   enum      K5 virtual blocks, grid-stride
//   finish    block 0: reduce, unwind by reverse waves, cost re-sum
//
// The grid is sized to the co-resident capacity (occupancy x SMs) and launched
// with the cooperative attribute, so grid.sync() is a legal device-wide
// barrier; one launch replaces 1 + waves + 2 launches and their gaps.
#pragma once

#include "build.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>

namespace pp {

template <class T> struct FusedWave {
  const FoldDesc<T> *folds;
  const MergeDesc<T> *merges;
  int32_t nf, nm;
  int64_t ftiles, items;
};

template <class T> struct FusedArgs {
  int32_t has_build;
  BuildArgs build;
  int64_t xcells;
  const FusedWave<T> *waves;
  int32_t n_waves;
  const EnumNode *en;
  const EnumEdge *ee;
  int32_t k, m;
  int64_t space, per_thread;
  void *blk_val;
  int64_t *blk_idx;
  int32_t nblk;
  FinishArgs fin;
  uint64_t *stamps; // optional: %globaltimer after each phase (profiling)
};

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kFusedThreads = 256;

template <class T> __global__ void __launch_bounds__(kFusedThreads) dp_fused_kernel(FusedArgs<T> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ WaveSmem<T> sm;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kFusedThreads;
  const bool stamp = a.stamps && blockIdx.x == 0 && threadIdx.x == 0;
  int ph = 0;
  if (stamp) a.stamps[ph++] = global_ns();
  if (a.has_build) {
    const BuildArgs &B = a.build;
    const int64_t n = B.ncells + a.xcells;
    // block-uniform trip count: xfer_cells_warp needs whole warps
    for (int64_t g0 = static_cast<int64_t>(blockIdx.x) * kFusedThreads; g0 < n; g0 += stride) {
      const int64_t g = g0 + threadIdx.x;
      if (g < B.ncells) {
        node_cost_cell(B, g);
      }
      int edge = -1;
      int64_t x = g - B.ncells;
      if (g >= B.ncells && g < n) {
        int lo = 0, hi = B.ne - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (B.edges[mid].out_off <= x)
            lo = mid;
          else
            hi = mid - 1;
        }
        edge = lo;
        x -= B.edges[lo].out_off;
      }
      xfer_cells_warp(B, edge, x);
    }
    grid.sync();
  }
  if (stamp) a.stamps[ph++] = global_ns();
  for (int w = 0; w < a.n_waves; ++w) {
    const FusedWave<T> W = a.waves[w];
    for (int64_t it = blockIdx.x; it < W.items; it += gridDim.x)
      wave_item<T>(W.folds, W.nf, W.ftiles, W.merges, W.nm, it, sm);
    grid.sync();
    if (stamp) a.stamps[ph++] = global_ns();
  }
  using A = typename Acc<T>::type;
  for (int64_t vb = blockIdx.x; vb < a.nblk; vb += gridDim.x)
    enum_block<T>(a.en, a.k, a.ee, a.m, a.space, a.per_thread, static_cast<A *>(a.blk_val), a.blk_idx, vb);
  grid.sync();
  if (stamp) a.stamps[ph++] = global_ns();
  if (blockIdx.x == 0) finish_block<T>(a.fin);
  if (stamp) a.stamps[ph++] = global_ns();
}

} // namespace pp
