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
  int64_t rot; // items before this wave: block (b + rot) mod grid runs item b, so
               // a small wave's blocks are idle in the previous wave and stage early
  int32_t narrow; // run by the first cluster alone (cluster barrier to a narrow successor)
  int32_t n_chains; // > 0: a chain segment (several waves), items = its row groups
  const ChainDesc *chains;
  int64_t stage;    // chain segment: bytes per staging buffer
  const FoldDesc<T> *cfolds;
  const uint16_t *fold_of;  // per fold tile: its fold in `folds` (null: binary search)
  const uint16_t *chain_of; // chain segment, per item: its chain in `chains` (null: binary search)
};

__device__ __forceinline__ int64_t first_item(int64_t rot) {
  // (blockIdx + g - rot mod g) mod g, in 32-bit arithmetic when rot fits
  // (a 64-bit remainder is ~70 instructions right after a barrier)
  const unsigned g = gridDim.x;
  const unsigned r = rot < (int64_t(1) << 32) ? static_cast<unsigned>(rot) % g : static_cast<unsigned>(rot % g);
  const unsigned b = blockIdx.x >= r ? blockIdx.x - r : blockIdx.x + g - r;
  return static_cast<int64_t>(b);
}

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
  int32_t stage;    // stage each wave's first item before the preceding barrier
  uint64_t *trace;  // optional: 8 stamps per wave from the block running item 0
  int32_t nc;       // cluster size (narrow waves run on blocks [0, nc))
  unsigned int *gbar; // hand-rolled grid barrier word (scratch), nullptr: cooperative_groups grid.sync
  unsigned long long *build_ctr; // build chunks claimed past the static first round (0 between launches)
};

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kFusedThreads = 256;

// Grid barrier for the cooperative launch.  Same arrive / flip protocol as
// cooperative_groups (one atomic per CTA; the first CTA's increment flips the
// counter's top bit once all have arrived), but the waiting thread polls with
// relaxed loads and backs off, and the acquire is one fence after the flip:
// the co-resident CTA of a still-working SM does not have its L1 invalidated
// on every poll.  `bar` must start with its low 31 bits zero (they return
// there after every barrier).
#ifndef PP_BARRIER_SLEEP_NS
#define PP_BARRIER_SLEEP_NS 20
#endif
__device__ __forceinline__ void grid_barrier(unsigned int *bar, uint64_t *ts = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence(); // release this CTA's writes
    if (ts) ts[0] = global_ns();
    const unsigned int old = atomicAdd(bar, nb);
    if (ts) ts[2048] = global_ns();
    unsigned int cur;
    for (;;) {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      if ((old ^ cur) & 0x80000000u) break;
      __nanosleep(PP_BARRIER_SLEEP_NS);
    }
    if (ts) ts[4096] = global_ns();
    __threadfence(); // acquire: later reads see every CTA's writes
  }
  __syncthreads();
}

// Stages this block's first item of wave W: its descriptor and, for a panel
// tile, the operands not in f.late (all of them when `ready` == kPanelAll).
template <class T>
__device__ __forceinline__ void stage_item(const FusedWave<T> &W, int ready, PanelSmem<T> &p, StagedItem<T> &st) {
  __syncthreads(); // the block's last item of the finishing wave may still read p / st
  const int64_t b = first_item(W.rot);
  if (b >= W.items || W.n_chains) {
    if (threadIdx.x == 0) st.b = -1;
    return;
  }
  if (b < W.ftiles) {
    const FoldDesc<T> f = W.folds[find_fold(W.folds, W.nf, b, W.fold_of)];
    int mask = 0;
    if (panel_fold(f)) {
      mask = (kPanelAll & ~f.late) | ready;
      panel_load<T>(f, b - f.tile_begin, mask, p);
    }
    if (threadIdx.x == 0) st.f = f, st.mask = mask, st.b = b;
  } else {
    const MergeDesc<T> m = W.merges[find_merge(W.merges, W.nm, b - W.ftiles)];
    if (threadIdx.x == 0) st.m = m, st.b = b;
  }
}

// kBuild: the image holds the K1/K2 phase.  Plans whose tables are built by a
// separate launch (one-shot plans build them while the host prepares the DP
// image) run the variant without it: a ~25 % smaller instruction image.
template <class T, bool kBuild> __global__ void __launch_bounds__(kFusedThreads, 2) dp_fused_kernel(FusedArgs<T> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // dynamic: max(WaveSmem, the largest chain item) bytes
  extern __shared__ __align__(16) unsigned char fused_smem[];
  WaveSmem<T> &sm = *reinterpret_cast<WaveSmem<T> *>(fused_smem);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kFusedThreads;
  const bool stamp = a.stamps && blockIdx.x == 0 && threadIdx.x == 0;
  auto gsync = [&] {
    if (a.gbar)
      grid_barrier(a.gbar);
    else
      grid.sync();
  };
  int ph = 0;
  if (stamp) a.stamps[ph++] = global_ns();
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 2048) a.trace[16 * a.n_waves + 16 + 2048 + blockIdx.x] = global_ns();
  if (kBuild && a.has_build) {
    const BuildArgs &B = a.build;
    const int64_t n = B.ncells + a.xcells;
    // the binary searches over layers and edges read their offsets from
    // shared memory (a dependent chain of descriptor loads otherwise)
    int64_t *cat_off_s = reinterpret_cast<int64_t *>(fused_smem), *out_off_s = cat_off_s + B.nl;
    const bool offs_in_smem = static_cast<size_t>(B.nl + B.ne) * 8 <= sizeof(WaveSmem<T>);
    if (offs_in_smem) {
      for (int l = threadIdx.x; l < B.nl; l += kFusedThreads) cat_off_s[l] = B.layers[l].cat_off;
      for (int e = threadIdx.x; e < B.ne; e += kFusedThreads) out_off_s[e] = B.edges[e].out_off;
      __syncthreads();
    }
    // 32-cell chunks, one per warp at a time (xfer_cells_warp needs whole
    // warps): the first chunk of each warp is static, later ones come from a
    // counter, so warps that drew cheap cells take more (a static grid-stride
    // split leaves a third round on a few blocks).  The next chunk is claimed
    // before the current one is computed: the atomic's latency overlaps it.
    const int64_t nchunks = (n + 31) >> 5;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kFusedThreads / 32);
    const int lane = threadIdx.x & 31;
    int64_t chunk = static_cast<int64_t>(blockIdx.x) * (kFusedThreads / 32) + (threadIdx.x >> 5);
    while (chunk < nchunks) {
      unsigned long long claim = 0;
      if (a.build_ctr && lane == 0) claim = atomicAdd(a.build_ctr, 1ull);
      const int64_t g = (chunk << 5) + lane;
      if (g < B.ncells) {
        node_cost_cell(B, g, offs_in_smem ? cat_off_s : nullptr);
      }
      int edge = -1;
      int64_t x = g - B.ncells;
      if (g >= B.ncells && g < n) {
        int lo = 0, hi = B.ne - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if ((offs_in_smem ? out_off_s[mid] : B.edges[mid].out_off) <= x)
            lo = mid;
          else
            hi = mid - 1;
        }
        edge = lo;
        x -= B.edges[lo].out_off;
      }
      xfer_cells_warp(B, edge, x);
      chunk = a.build_ctr ? nwarps + static_cast<int64_t>(__shfl_sync(0xffffffffu, claim, 0)) : chunk + nwarps;
    }
    if (a.trace) { // per-block end of the build loop (profiling)
      __syncthreads();
      if (threadIdx.x == 0 && blockIdx.x < 2048) a.trace[16 * a.n_waves + 16 + blockIdx.x] = global_ns();
    }
    if (a.gbar)
      grid_barrier(a.gbar, a.trace && blockIdx.x < 2048 ? a.trace + 16 * a.n_waves + 16 + 6144 + blockIdx.x : nullptr);
    else
      grid.sync();
    if (a.trace && threadIdx.x == 0 && blockIdx.x < 2048) a.trace[16 * a.n_waves + 16 + 4096 + blockIdx.x] = global_ns();
    // every claim of this launch precedes the barrier: rearm the counter
    if (a.build_ctr && blockIdx.x == 0 && threadIdx.x == 0) *a.build_ctr = 0;
  }
  if (stamp) a.stamps[ph++] = global_ns();
  // this block's first item of each wave is staged one wave early: its
  // descriptor, and everything but the operands the finishing wave writes,
  // load before the barrier, off the critical path after it
  __shared__ StagedItem<T> st;
  FusedWave<T> W;
  if (a.n_waves > 0) {
    W = a.waves[0];
    stage_item<T>(W, kPanelAll, sm.p, st);
    __syncthreads();
  }
  for (int w = 0; w < a.n_waves; ++w) {
    const bool narrow = W.narrow;
    const int64_t b0 = narrow ? static_cast<int64_t>(blockIdx.x) : first_item(W.rot);
    const int64_t step = narrow ? a.nc : gridDim.x;
    uint64_t *tr = a.trace && b0 == 0 ? a.trace + 16 * w : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = global_ns();
    if (W.n_chains)
      for (int64_t it = blockIdx.x; it < W.items; it += gridDim.x) chain_item<T>(W.chains, W.n_chains, W.cfolds, it, fused_smem, static_cast<size_t>(W.stage), nullptr,
                                  W.chain_of);
    else if (!narrow || static_cast<int>(blockIdx.x) < a.nc)
      for (int64_t it = b0; it < W.items; it += step)
        wave_item<T>(W.folds, W.nf, W.ftiles, W.merges, W.nm, it, sm, narrow ? nullptr : &st, it == 0 ? tr : nullptr,
                     W.fold_of);
    bool next_narrow = false;
    if (w + 1 < a.n_waves) {
      W = a.waves[w + 1];
      next_narrow = W.narrow;
      if (a.stage && !next_narrow)
        stage_item<T>(W, 0, sm.p, st);
      else {
        __syncthreads();
        if (threadIdx.x == 0) st.b = -1;
      }
    }
    if (tr && threadIdx.x == 0) tr[3] = global_ns();
    if (narrow && next_narrow) {
      // both waves live in the first cluster: a cluster barrier (release /
      // acquire at cluster scope) orders its writes; other clusters skip ahead
      if (static_cast<int>(blockIdx.x) < a.nc) cg::this_cluster().sync();
    } else {
      gsync();
    }
    if (tr && threadIdx.x == 0) tr[4] = global_ns();
    if (stamp) a.stamps[ph++] = global_ns();
  }
  using A = typename Acc<T>::type;
  for (int64_t vb = blockIdx.x; vb < a.nblk; vb += gridDim.x)
    enum_block<T>(a.en, a.k, a.ee, a.m, a.space, a.per_thread, static_cast<A *>(a.blk_val), a.blk_idx, vb);
  // block 0's own DP items are done: it stages the finish lookups now
  const bool staged = blockIdx.x == 0 && a.fin.smem_ok;
  if (staged) finish_stage(a.fin, fused_smem);
  gsync();
  if (stamp) a.stamps[ph++] = global_ns();
  if (blockIdx.x == 0) finish_block<T>(a.fin, fused_smem, staged);
  if (stamp) a.stamps[ph++] = global_ns();
}

} // namespace pp
