// plan_builder.cuh — prepare stages of a plan (plan.cu's prepare()):
//
//   1. final-graph check, and for one-shot plan() calls the early table build
//      (K1/K2 launched before the host builds anything else)
//   2. MemoryPlan        table shapes, row shards, derived-table liveness
//   3. MinplusPlan       which folds take the U16x2 / FP64 large-fold kernels
//                        (span certificate, caps, JB, chain runs, scratch)
//   4. EffectiveSchedule merge absorption for the fused kernel
//   5. sections          plan memory: tables | derived | argmins | min-plus
//                        scratch | gather targets | descriptor image
//   6. image             ONE descriptor image holding every launch's work list
//                        (folds, merges, large folds, chain segments, unwind
//                        records, fused phases) plus the result slots; built
//                        against the final device base
//   7. steps             the launch list (plan_steps.cuh)
//
// Every stage is host work over the symbolic schedule (scheduler.hpp); the
// device only ever sees the image.
#pragma once

#include "fused.cuh"
#include "kernels.cuh"
#include "minplus.cuh"
#include "minplus64.cuh"
#include "mp_plan.hpp"
#include "plan_memory.hpp"
#include "plan_state.hpp"
#include "shard.hpp"

#include <algorithm>
#include <climits>
#include <cstring>
#include <functional>
#include <string>
#include <type_traits>
#include <vector>

namespace pp {

using MpChainFn = void (*)(const MpFold *, int, int);
// the chain kernel for a run: optimistic runs (JB 6) get the exact row count
// per CTA, proven-cap runs (JB <= 5) the 8-row tile
inline MpChainFn mp_chain_launch(int jb, int R) {
  if (jb < kMpOptJB) return mp_chain_kernel<5, 8>; // runs need JB >= 5 (argmin groups cover whole stages)
  switch (R) {
  case 1: return mp_chain_kernel<kMpOptJB, 1>;
  case 2: return mp_chain_kernel<kMpOptJB, 2>;
  case 3: return mp_chain_kernel<kMpOptJB, 3>;
  case 4: return mp_chain_kernel<kMpOptJB, 4>;
  case 5: return mp_chain_kernel<kMpOptJB, 5>;
  case 6: return mp_chain_kernel<kMpOptJB, 6>;
  case 7: return mp_chain_kernel<kMpOptJB, 7>;
  default: return mp_chain_kernel<kMpOptJB, 8>;
  }
}

template <class T> class PlanBuilder {
public:
  PlanBuilder(pp_prepared *P, const BuildPlan *bp) : P(P), bp(bp), ctx(P->ctx), t(*P->t), s(P->g->schedule()) {}
  void build(int k_bound);

private:
  using A = typename Acc<T>::type;
  using MpLayout = MinplusPlan::Layout;
  using MpRun = MinplusPlan::Run;

  // per-wave work lists inside the image
  struct WaveRange {
    size_t f0 = 0, m0 = 0; // generic folds [f0, f0 + nf), merges [m0, m0 + nm)
    int nf = 0, nm = 0;
    int64_t ftiles = 0, mblocks = 0;
    double cells = 0.0;
    struct MpGroup {
      size_t p0 = 0; // large folds [p0, p0 + np) in mpf, one prep + fold launch pair
      int np = 0;
      int64_t units = 0, prep_blocks = 0, tiles = 0; // stream-K units, mp_prep blocks, tiles
      int jb = 5;
      double cells = 0.0;
    };
    std::vector<MpGroup> mg;
    struct Mp64Group {
      size_t p0 = 0; // FP64 large folds [p0, p0 + np) in m64
      int np = 0;
      int64_t prep_blocks = 0, tiles = 0;
      double cells = 0.0;
    };
    std::vector<Mp64Group> mg64;
    size_t mm0 = 0; // min-plus merges: [mm0, mm0 + nmm) in mmv
    int nmm = 0;
    int64_t mm_blocks = 0;
    double mm_cells = 0.0;
    CopyList gathers; // sharded: derived t2 -> full, before the wave
  };
  struct Image {
    Packer pk;
    std::vector<WaveRange> waves;
    CopyList final_gathers; // sharded: derived final edges
    size_t oF, oM, oN, oE, oR, oL, oCO, oXO, oS, oD, oC, oBV, oBI, oRes, oIdx, oFC, oLay, oEdg, oCfg, oRat, oBw, oMP;
    size_t oG, oT, oFW, oST, oTR, oCN; // oT, oST, oTR (+1), oBV, oBI: scratch offsets
    size_t oOvf = 0;                   // min-plus optimistic-cap overflow flag (result slot)
    size_t oPeer = 0;                  // row-sharded: NR plan memory bases
    size_t scratch = 0;                // bytes of the scratch section
    int n_phases = 0;                  // fused kernel: waves / chain segments
    size_t dyn_smem = 0;               // fused kernel dynamic shared memory
    std::vector<char> phase_chain;     // phase is a chain segment
    std::vector<double> phase_work;    // cells per fused phase
    int nG = 0;
    size_t res_bytes = 0;
    size_t oMM = 0;   // min-plus merges (all waves)
    size_t oM64 = 0;  // FP64 large folds (all waves)
    int n_mp = 0;     // large folds (all waves)
    int64_t colmin_blocks = 0, rowmin_blocks = 0; // mp_minima blocks
  };
  // chain runs in the image: folds [p0, p0 + n) of mpf, B prep blocks, JB, cells, rows per CTA, first wave
  struct RunImg {
    size_t p0;
    int n;
    int64_t prep_blocks;
    double cells;
    int R, w0;
    int jb = 6;
    int nu = 0;
  };
  // chain segments (fused kernel, chain_item): maximal runs of >= 2 waves of
  // folds only, each fold's t2 written before the run and its t1 before the
  // run or by a fold of the run (whose chain it extends)
  struct Segment {
    int ws, we; // waves [ws, we]
    std::vector<ChainDesc> chains;
    std::vector<FoldDesc<T>> cf;
    int64_t items = 0;
    size_t smem = 0;  // dynamic shared memory of its items
    size_t stage = 0; // bytes per staging buffer
  };
  // chains with unwind path tables: one finish record each
  struct ChainRec {
    int node_off, n;
    const uint16_t *path;
  };
  struct FoldOps {
    int e1, e2, ne, wave, oi;
  };
  // the work lists while one image is built
  struct Work {
    std::vector<FoldDesc<T>> folds;
    std::vector<FoldOps> fold_ops;
    std::vector<MergeDesc<T>> merges;
    std::vector<MpFold> mpf;
    std::vector<Mp64Fold> m64;
    std::vector<MpMerge> mmv;
    int64_t colmin_blocks = 0, rowmin_blocks = 0; // mp_minima blocks over all large folds (one launch per plan)
    std::vector<Segment> segs;
    std::vector<int> seg_of;   // effective wave -> segment (-1: none)
    std::vector<char> narrow;  // effective wave runs on the first cluster alone
    std::vector<ChainRec> chain_recs;
    std::vector<int> chain_last_op;
    std::vector<int32_t> chain_nodes;
    std::vector<int> chain_of_op;
  };

  pp_prepared *P;
  const BuildPlan *bp;
  pp_context *ctx;
  Tables &t;
  const Schedule &s;
  const Knobs kn;
  StageClock clk;
  int K = 0;
  bool early = false; // K1/K2 launched before the descriptor image is built

  MemoryPlan mem;
  MinplusPlan mp;
  EffectiveSchedule es;
  bool use_fused = false;
  size_t off_tables = 0, off_derived = 0, off_am = 0, off_mp = 0, off_mpp = 0, off_gat = 0, off_image = 0;
  // final enumeration (K5) geometry
  std::vector<int> pos;
  std::vector<int32_t> node_layer;
  int64_t space = 1, per_thread = 1;
  int nblk = 0;
  std::vector<RunImg> run_img;
  // bases the image is being built against (sizing pass: null)
  unsigned char *db = nullptr, *sb = nullptr;
  size_t oOvf_ = 0;

  void check_final(int k_bound);
  void early_table_build();
  void plan_minplus();
  void plan_sections();
  void plan_enumeration();
  Image make_image(unsigned char *dbase, unsigned char *sbase);
  void image_waves(Image &im, Work &wk);
  void image_segments(Image &im, Work &wk);
  void image_staging(Image &im, Work &wk);
  void image_unwind(Image &im, Work &wk, std::vector<UnwindRec> &recs, std::vector<int32_t> &groups);
  void image_phases(Image &im, Work &wk);
  Image place_image();
  // plan_steps.cuh: the launch list
  int launches = 0; // kernel launches per run
  void step(int kind, double work, std::function<void(cudaStream_t)> fn, int n_launches);
  void emit_steps(const Image &im);
  BuildArgs build_args(const Image &im) const;
  void emit_table_build(const BuildArgs &ba, bool split_build);
  void emit_minima(const Image &im);
  void emit_gathers(const CopyList &list);
  void emit_waves(const Image &im);
  FinishArgs finish_args(const Image &im) const;
  void emit_fused(const Image &im, const BuildArgs &ba, bool split_build, const FinishArgs &fa);

  // ---- device pointers of the image being built -----------------------------
  int cnt(int layer) const { return t.counts[static_cast<size_t>(layer)]; }
  size_t scr(Image &im, size_t bytes) const {
    const size_t off = im.scratch;
    im.scratch = off + align256(bytes);
    return off;
  }
  uint32_t *ovf_ptr() const { return reinterpret_cast<uint32_t *>(db + off_image + oOvf_); }
  const T *onode() const {
    return bp ? reinterpret_cast<const T *>(db + off_tables)
              : (t.mode == kFP64 ? reinterpret_cast<const T *>(t.node.p) : reinterpret_cast<const T *>(t.node32.p));
  }
  const T *tabp(int id) const {
    if (id < t.ne) {
      const T *ox = bp ? reinterpret_cast<const T *>(db + off_tables + 3 * align256(static_cast<size_t>(t.ncells) * 8))
                       : (t.mode == kFP64 ? reinterpret_cast<const T *>(t.xfer64.p)
                                          : reinterpret_cast<const T *>(t.xfer32.p));
      return ox + t.xoff[static_cast<size_t>(id)];
    }
    return reinterpret_cast<const T *>(db + off_derived + mem.tab_off[static_cast<size_t>(id)]);
  }
  // this rank's first row of a table (original tables are replicated in full)
  const T *rowp(int id) const {
    return id < t.ne && mem.shard ? tabp(id) + static_cast<int64_t>(mem.lr0(id)) * mem.ncols(id) : tabp(id);
  }
  T *gatp(int id) const { return reinterpret_cast<T *>(db + off_gat + mem.gat_off[static_cast<size_t>(id)]); }
  const T *t2p(int id) const { return mem.shard && id >= t.ne ? gatp(id) : tabp(id); }
  uint16_t *amp(int oi) const { return reinterpret_cast<uint16_t *>(db + off_am + mem.am_off[static_cast<size_t>(oi)]); }
  // min-plus persistent section: part | cnt | ra | cb | chain B''
  unsigned char *mpp() const { return db + off_mpp; }
  uint32_t *rap(int oi) const {
    return reinterpret_cast<uint32_t *>(mpp() + mp.part + mp.cnt + mp.mpl[static_cast<size_t>(oi)].ra);
  }
  uint32_t *cbp(int oi) const {
    return reinterpret_cast<uint32_t *>(mpp() + mp.part + mp.cnt + mp.ra + mp.mpl[static_cast<size_t>(oi)].cb);
  }
};

// ---- stage 1 -------------------------------------------------------------------
template <class T> void PlanBuilder<T>::check_final(int k_bound) {
  K = static_cast<int>(s.final_nodes.size());
  if (K > k_bound)
    throw parplan::LimitError("final graph has " + std::to_string(K) + " nodes, exceeding the enumeration bound of " +
                              std::to_string(k_bound) + " (graph is not reducible enough)");
  PP_REQUIRE(K <= kMaxEnumNodes, "final graph too large for the enumeration kernel");
  P->K = K;
  P->n_waves = s.n_waves;
  P->node_ops = s.node_ops;
  P->edge_ops = s.edge_ops;
  for (const Op &op : s.ops)
    if (!op.type) PP_REQUIRE(cnt(op.removed) <= 65535, "argmin index exceeds 16 bits");
}

// One-shot plans overlap the host's descriptor build with the device's table
// build: K1/K2 launch first (their descriptors go up in a small separate
// upload), the image is built while they run, and the fused kernel follows
// without its build phase.  The pool must already hold the final layout; if
// the image outgrows the estimate, place_image falls back.
template <class T> void PlanBuilder<T>::early_table_build() {
  if (!(P->transient && bp && !ctx->no_fused && ctx->nranks <= 1 && bp->grid > 0 && kn.early_build &&
        ctx->last_pool_bytes > 0))
    return;
  // at least the table region (a larger final layout falls back below)
  ctx->plan_pool.ensure(std::max(ctx->last_pool_bytes, align256(static_cast<size_t>(t.ncells) * 8) * 3 +
                                                           align256(static_cast<size_t>(t.xcells) * 8)));
  unsigned char *pb = ctx->plan_pool.p;
  // descriptor arrays straight into pinned staging, one H2D copy
  size_t o = 0;
  auto slot = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 15) & ~size_t(15);
    return at;
  };
  const size_t oL = slot(bp->L.size() * sizeof(LayerDev)), oE = slot(bp->E.size() * sizeof(EdgeDev)),
               oC = slot(bp->cfg32->size() * 4), oR = slot(bp->rates.size() * 8), oB = slot(bp->bw.size() * 8);
  unsigned char *h = static_cast<unsigned char *>(ctx->staging.ensure(o + 16));
  std::memcpy(h + oL, bp->L.data(), bp->L.size() * sizeof(LayerDev));
  std::memcpy(h + oE, bp->E.data(), bp->E.size() * sizeof(EdgeDev));
  std::memcpy(h + oC, bp->cfg32->data(), bp->cfg32->size() * 4);
  std::memcpy(h + oR, bp->rates.data(), bp->rates.size() * 8);
  std::memcpy(h + oB, bp->bw.data(), bp->bw.size() * 8);
  ctx->desc.ensure(o + 16);
  ctx->begin(); // the plan's device time starts with the table build
  unsigned char *base = ctx->desc.p;
  PP_CUDA(cudaMemcpyAsync(base, h, o, cudaMemcpyHostToDevice, ctx->stream));
  BuildArgs a{};
  a.layers = reinterpret_cast<const LayerDev *>(base + oL);
  a.edges = reinterpret_cast<const EdgeDev *>(base + oE);
  a.cfg = reinterpret_cast<const int32_t *>(base + oC);
  a.rates = reinterpret_cast<const double *>(base + oR);
  a.bw = reinterpret_cast<const double *>(base + oB);
  const size_t nb = align256(static_cast<size_t>(t.ncells) * 8); // the table region opens the pool
  a.node = reinterpret_cast<double *>(pb);
  a.compute = reinterpret_cast<double *>(pb + nb);
  a.sync = reinterpret_cast<double *>(pb + 2 * nb);
  a.xfer = reinterpret_cast<double *>(pb + 3 * nb);
  a.ncells = t.ncells;
  a.nl = t.nl, a.ne = t.ne, a.D = bp->D;
  a.node_blocks = static_cast<int32_t>(bp->node_blocks);
  a.bw_uniform = bp->bw_uniform;
  clk.mark("early-upload");
  launch_build(ctx, ctx->stream, a, bp->grid);
  clk.mark("early-launch");
  early = true;
  P->early_built = true;
}

// ---- stage 3: large folds (U16 fixed point / FP64) -------------------------------
template <class T> void PlanBuilder<T>::plan_minplus() {
  mp.build<T>(MinplusPlan::In{s, t, mem.rows, mem.cols, [this](int id) { return mem.nu_eff(id); }, mem.shard,
                              P->mp_conservative || ctx->mp_conservative, ctx->no_minplus, ctx->sms,
                              kn.mp_chain != 0, kn.mp_chain_min, mem.prod_wave});
  // dynamic shared memory allowances: per device, so set on every prepare (cheap)
  for (const MpRun &run : mp.runs)
    for (int jb : {5, kMpOptJB})
      PP_CUDA(cudaFuncSetAttribute(mp_chain_launch(jb, run.R), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kMpChainSmem)));
  if (mp.part)
    for (auto fn : {mp_fold_kernel<7>, mp_fold_kernel<6>, mp_fold_kernel<5>, mp_fold_kernel<4>, mp_fold_kernel<3>})
      PP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMpSmem)));
  if (mp.bytes && std::is_same_v<T, double>)
    PP_CUDA(cudaFuncSetAttribute(mp64_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMp64Smem)));
  // one cooperative kernel for the whole plan when no fold needs a large-fold kernel
  use_fused = mp.bytes == 0 && mp.pbytes() == 0 && !ctx->no_fused && !mem.shard;
}

// ---- stage 5: plan memory sections ------------------------------------------------
template <class T> void PlanBuilder<T>::plan_sections() {
  const size_t tables_bytes =
      bp ? align256(static_cast<size_t>(t.ncells) * 8) * 3 + align256(static_cast<size_t>(t.xcells) * 8) : 0;
  off_tables = 0;
  off_derived = tables_bytes;
  off_am = off_derived + align256(mem.tab_end);
  off_mp = off_am + align256(mem.am_bytes);
  off_mpp = off_mp + align256(mp.bytes);
  off_gat = off_mpp + align256(mp.pbytes());
  off_image = off_gat + align256(mem.gat_bytes);
}

// final enumeration (K5): mixed-radix space over the final nodes' configs
template <class T> void PlanBuilder<T>::plan_enumeration() {
  pos.assign(static_cast<size_t>(t.nl), -1);
  node_layer.assign(static_cast<size_t>(K), 0);
  space = 1;
  for (int d = 0; d < K; ++d) {
    const int l = s.final_nodes[static_cast<size_t>(d)];
    node_layer[static_cast<size_t>(d)] = l;
    pos[static_cast<size_t>(l)] = d;
    PP_REQUIRE(space <= INT64_MAX / std::max(1, cnt(l)), "final enumeration space overflows");
    space *= cnt(l);
  }
  const int64_t lanes = int64_t(ctx->sms) * 8 * kEnumThreads;
  per_thread = std::max<int64_t>(1, (space + lanes - 1) / lanes);
  nblk = static_cast<int>(((space + per_thread - 1) / per_thread + kEnumThreads - 1) / kEnumThreads);
}

// ---- stage 6: the descriptor image ------------------------------------------------
// Work lists per effective wave: generic folds (32x32 / 16x16 / panel tiles),
// merges, large U16 folds (per launch group, or as mp_chain run members),
// FP64 large folds, min-plus merges.
template <class T> void PlanBuilder<T>::image_waves(Image &im, Work &wk) {
  const T *on = onode();
  for (int w = 1; w <= es.n_waves; ++w) {
    WaveRange wr;
    wr.f0 = wk.folds.size(), wr.m0 = wk.merges.size(), wr.mm0 = wk.mmv.size();
    // a wave whose generic folds cover fewer than 2 x SMs 32x32 tiles uses
    // 16x16 tiles: 4x the blocks, a quarter of the per-tile latency
    int64_t big_tiles = 0;
    for (int x = es.begin[static_cast<size_t>(w)]; x < es.begin[static_cast<size_t>(w) + 1]; ++x) {
      const int oi = es.exec[static_cast<size_t>(x)];
      const Op &op = s.ops[static_cast<size_t>(oi)];
      if (op.type || mp.large[static_cast<size_t>(oi)]) continue;
      big_tiles += static_cast<int64_t>((mem.nu_eff(op.e1) + kTile - 1) / kTile) * ((mem.ncols(op.e2) + kTile - 1) / kTile);
    }
    const bool small_wave = big_tiles < 2 * int64_t(ctx->sms);
    // panel tiles: the smallest side whose tile count still fits one round
    // of co-resident blocks (more j-split groups, shorter scans)
    int panel_mode = kPanel16;
    if (small_wave && kn.panel) {
      const int forced = kn.panel_side;
      for (int mode : {kPanel4, kPanel8}) {
        const int R = panel_side(mode);
        int64_t n = 0;
        for (int x = es.begin[static_cast<size_t>(w)]; x < es.begin[static_cast<size_t>(w) + 1]; ++x) {
          const int oi = es.exec[static_cast<size_t>(x)];
          const Op &op = s.ops[static_cast<size_t>(oi)];
          if (op.type || mp.large[static_cast<size_t>(oi)]) continue;
          n += static_cast<int64_t>((mem.nu_eff(op.e1) + R - 1) / R) * ((mem.ncols(op.e2) + R - 1) / R);
        }
        if (forced ? R == forced : n <= 2 * int64_t(ctx->sms)) {
          panel_mode = mode;
          break;
        }
      }
    }
    for (int x = es.begin[static_cast<size_t>(w)]; x < es.begin[static_cast<size_t>(w) + 1]; ++x) {
      const int oi = es.exec[static_cast<size_t>(x)];
      const Op &op = s.ops[static_cast<size_t>(oi)];
      T *out = const_cast<T *>(tabp(es.out_table[static_cast<size_t>(oi)]));
      if (mem.shard && !op.type && op.e2 >= t.ne)
        wr.gathers.emplace_back(tabp(op.e2), gatp(op.e2), static_cast<size_t>(mem.blk(op.e2)) * mem.ncols(op.e2) * sizeof(T));
      if (mem.nu_eff(op.e1) == 0) continue; // no rows of this op on this rank
      if constexpr (std::is_same_v<T, int32_t>) {
        if (mp.large[static_cast<size_t>(oi)] && mp.run_of[static_cast<size_t>(oi)] >= 0) { // chain run member
          const MpRun &run = mp.runs[static_cast<size_t>(mp.run_of[static_cast<size_t>(oi)])];
          const MpLayout &L = mp.mpl[static_cast<size_t>(oi)];
          if (oi == run.ops.front()) run_img.push_back(RunImg{wk.mpf.size(), 0, 0, 0.0, run.R, w, 6, mem.nu_eff(op.e1)});
          RunImg &rn = run_img.back();
          MpFold f{};
          f.t1 = rowp(op.e1);
          f.t2 = t2p(op.e2);
          f.w = on + t.cat_off[static_cast<size_t>(op.removed)];
          f.out = out;
          f.am = amp(oi);
          f.cb = cbp(oi);
          f.ra = rap(oi);
          f.B = reinterpret_cast<uint16_t *>(mpp() + mp.part + mp.cnt + mp.ra + mp.cb + L.B);
          f.b_cols = kMpChainCols;
          f.nu = mem.nu_eff(op.e1);
          f.nw = cnt(op.removed);
          f.nv = mem.ncols(op.e2);
          f.tiles_i = f.tiles_k = 1;
          f.nchunks = L.nchunks;
          f.jb = mp.fold_jb[static_cast<size_t>(oi)];
          for (int o2 : run.ops) f.jb = std::min(f.jb, mp.fold_jb[static_cast<size_t>(o2)]); // one JB per run
          f.jb = std::max(f.jb, 5);
          if (mp.fold_opt[static_cast<size_t>(oi)]) {
            f.cap = mp_max_cap(f.jb);
            f.ovf = ovf_ptr();
          } else {
            f.cap = static_cast<int32_t>(mp.fold_m[static_cast<size_t>(oi)] + 1);
          }
          PP_REQUIRE(((2 * int64_t(f.cap)) << f.jb) + (1 << f.jb) - 1 <= 65534, "min-plus operand cap exceeds 16 bits");
          f.cb_ready = op.e2 < t.ne || mp.mp_producer[static_cast<size_t>(op.e2)] >= 0 || mp.mp_merge_out[static_cast<size_t>(op.e2)];
          f.a_batches = 0; // the chain kernel normalises its own rows
          f.b_batches = f.cb_ready ? (f.nchunks + kMpPrepBatch - 1) / kMpPrepBatch : 1;
          f.prep_begin = rn.prep_blocks;
          rn.prep_blocks += mp_prep_blocks(f);
          f.colmin_begin = wk.colmin_blocks;
          if (op.e2 < t.ne) wk.colmin_blocks += (f.nv + 31) / 32;
          f.rowmin_begin = wk.rowmin_blocks;
          rn.jb = f.jb;
          rn.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          ++rn.n;
          wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          wk.mpf.push_back(f);
          continue;
        }
        if (mp.large[static_cast<size_t>(oi)]) {
          const MpLayout &L = mp.mpl[static_cast<size_t>(oi)];
          unsigned char *scratch = db + off_mp;
          MpFold f{};
          f.t1 = rowp(op.e1);
          f.t2 = t2p(op.e2);
          f.w = on + t.cat_off[static_cast<size_t>(op.removed)];
          f.out = out;
          f.am = amp(oi);
          f.ra = rap(oi);
          f.cb = cbp(oi);
          f.A = reinterpret_cast<uint32_t *>(scratch + L.A);
          f.B = reinterpret_cast<uint16_t *>(scratch + L.B);
          f.part = reinterpret_cast<uint32_t *>(mpp());
          f.cnt = reinterpret_cast<uint32_t *>(mpp() + mp.part + L.cnt);
          const int nxt = mp.mp_consumer[static_cast<size_t>(op.ne)];
          if (nxt >= 0) {
            f.w_next = on + t.cat_off[static_cast<size_t>(s.ops[static_cast<size_t>(nxt)].removed)];
            f.ra_next = rap(nxt);
          }
          const int nxt2 = mp.mp_consumer2[static_cast<size_t>(op.ne)];
          if (nxt2 >= 0 && !mem.shard) f.cb_next = cbp(nxt2); // row-sharded: a rank sees only its rows
          f.ra_ready = op.e1 < t.ne || mp.mp_producer[static_cast<size_t>(op.e1)] >= 0; // mp_minima / producer
          // original t2: mp_colmin (once per plan); a large fold's or an mp_merge's output: their epilogues
          f.cb_ready = op.e2 < t.ne || (!mem.shard && (mp.mp_producer[static_cast<size_t>(op.e2)] >= 0 ||
                                                       mp.mp_merge_out[static_cast<size_t>(op.e2)]));
          f.nu = mem.nu_eff(op.e1);
          f.nw = cnt(op.removed);
          f.nv = mem.ncols(op.e2);
          f.tiles_i = L.tiles_i;
          f.tiles_k = L.tiles_k;
          f.nchunks = L.nchunks;
          const int gi = mp.mp_group[static_cast<size_t>(oi)];
          if (static_cast<int>(wr.mg.size()) <= gi) wr.mg.resize(static_cast<size_t>(gi) + 1);
          auto &G = wr.mg[static_cast<size_t>(gi)];
          if (G.np == 0) G.p0 = wk.mpf.size();
          G.jb = mp.wave_group_jb[static_cast<size_t>(op.wave)][static_cast<size_t>(gi)];
          f.jb = G.jb;
          // operand cap (minplus.cuh): optimistic = the largest the launch's JB allows, checked on
          // the device; proven = M + 1, which fits the fold's (and so the group's smaller) JB
          if (mp.fold_opt[static_cast<size_t>(oi)]) {
            f.cap = mp_max_cap(f.jb);
            f.ovf = ovf_ptr();
          } else {
            f.cap = static_cast<int32_t>(mp.fold_m[static_cast<size_t>(oi)] + 1);
          }
          PP_REQUIRE(((2 * int64_t(f.cap)) << f.jb) + (1 << f.jb) - 1 <= 65534, "min-plus operand cap exceeds 16 bits");
          const int batches = (f.nchunks + kMpPrepBatch - 1) / kMpPrepBatch;
          f.a_batches = f.ra_ready ? batches : 1;
          f.b_batches = f.cb_ready ? batches : 1;
          f.prep_begin = G.prep_blocks;
          G.prep_blocks += mp_prep_blocks(f);
          f.colmin_begin = wk.colmin_blocks;
          if (op.e2 < t.ne) wk.colmin_blocks += (f.nv + 31) / 32; // original t2 only (derived: producers)
          f.rowmin_begin = wk.rowmin_blocks;
          if (op.e1 < t.ne) wk.rowmin_blocks += (f.nu + 7) / 8;
          f.unit_begin = G.units;
          G.units += static_cast<int64_t>(f.tiles_i) * f.tiles_k * f.nchunks;
          f.tile_begin = G.tiles;
          G.tiles += static_cast<int64_t>(f.tiles_i) * f.tiles_k;
          G.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          wk.mpf.push_back(f);
          ++G.np;
          continue;
        }
      }
      if constexpr (std::is_same_v<T, double>) {
        if (mp.large64[static_cast<size_t>(oi)]) {
          const int gi = mp.mp64_group[static_cast<size_t>(oi)];
          if (static_cast<int>(wr.mg64.size()) <= gi) wr.mg64.resize(static_cast<size_t>(gi) + 1);
          auto &G = wr.mg64[static_cast<size_t>(gi)];
          if (G.np == 0) G.p0 = wk.m64.size();
          Mp64Fold f{};
          f.t1 = rowp(op.e1);
          f.t2 = t2p(op.e2);
          f.w = on + t.cat_off[static_cast<size_t>(op.removed)];
          f.out = out;
          f.am = amp(oi);
          f.A = reinterpret_cast<double *>(db + off_mp + mp.mp64_off[static_cast<size_t>(oi)][0]);
          f.B = reinterpret_cast<double *>(db + off_mp + mp.mp64_off[static_cast<size_t>(oi)][1]);
          f.nu = mem.nu_eff(op.e1);
          f.nw = cnt(op.removed);
          f.nv = mem.ncols(op.e2);
          f.tiles_i = (f.nu + kMp64Tile - 1) / kMp64Tile;
          f.tiles_k = (f.nv + kMp64Tile - 1) / kMp64Tile;
          f.nchunks = (f.nw + kMp64Chunk - 1) / kMp64Chunk;
          f.one = 1;
          f.prep_a = mp64_prep_a_blocks(f.nu, f.nchunks);
          f.prep_begin = G.prep_blocks;
          G.prep_blocks += f.prep_a + mp64_prep_b_blocks(f.nchunks, f.tiles_k);
          f.tile_begin = G.tiles;
          G.tiles += static_cast<int64_t>(f.tiles_i) * f.tiles_k;
          G.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          wk.m64.push_back(f);
          ++G.np;
          continue;
        }
      }
      if (!op.type) {
        FoldDesc<T> f{};
        f.t1 = rowp(op.e1);
        f.t2 = t2p(op.e2);
        f.w = on + t.cat_off[static_cast<size_t>(op.removed)];
        f.out = out;
        f.am = amp(oi);
        f.nu = mem.nu_eff(op.e1);
        f.nw = cnt(op.removed);
        f.nv = mem.ncols(op.e2);
        f.small = small_wave ? (f.nw <= kPanel && kn.panel ? panel_mode : 1) : 0;
        const int ts = f.small >= kPanel16 ? panel_side(f.small) : f.small ? kSmallTile : kTile;
        f.late = 0; // set by image_staging, once the narrow waves are known
        wk.fold_ops.push_back({op.e1, op.e2, es.out_table[static_cast<size_t>(oi)], w, oi});
        const auto &ep = es.epi[static_cast<size_t>(oi)];
        f.n_epi = static_cast<int32_t>(ep.size());
        for (int e = 0; e < f.n_epi; ++e) {
          f.epi[e] = tabp(ep[static_cast<size_t>(e)].first);
          f.epi2[e] = ep[static_cast<size_t>(e)].second >= 0 ? tabp(ep[static_cast<size_t>(e)].second) : nullptr;
        }
        f.tiles_k = (f.nv + ts - 1) / ts;
        f.tile_begin = wr.ftiles;
        wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
        wr.ftiles += static_cast<int64_t>((f.nu + ts - 1) / ts) * f.tiles_k;
        wk.folds.push_back(f);
        ++wr.nf;
        continue;
      }
      if constexpr (std::is_same_v<T, int32_t>) {
        if (mp.mp_merge_out[static_cast<size_t>(op.ne)]) { // feeds a large fold's t2: with its column minima
          MpMerge mm{};
          mm.a = rowp(op.e1);
          mm.b = rowp(op.e2);
          mm.out = out;
          mm.cb = cbp(mp.mp_consumer2[static_cast<size_t>(op.ne)]);
          mm.nr = mem.nu_eff(op.e1);
          mm.nc = mem.ncols(op.ne);
          mm.blk_begin = wr.mm_blocks;
          wr.mm_blocks += static_cast<int64_t>((mm.nc + 31) / 32) * ((mm.nr + kMpMergeRows - 1) / kMpMergeRows);
          wr.cells += static_cast<double>(mm.nr) * mm.nc;
          wr.mm_cells += static_cast<double>(mm.nr) * mm.nc;
          wk.mmv.push_back(mm);
          ++wr.nmm;
          continue;
        }
      }
      MergeDesc<T> m;
      m.a = rowp(op.e1);
      m.b = rowp(op.e2);
      m.out = out;
      m.n = static_cast<int64_t>(mem.nu_eff(op.e1)) * mem.ncols(op.ne);
      m.blk_begin = wr.mblocks;
      wr.cells += static_cast<double>(m.n);
      wr.mblocks += (m.n + kMergePerBlock - 1) / kMergePerBlock;
      wk.merges.push_back(m);
      ++wr.nm;
    }
    im.waves.push_back(std::move(wr));
  }
}

// Chain segments of the fused kernel.  A segment has no grid barrier between
// its waves, so a later wave's output must never reuse a table an earlier
// chain item still reads: segments need every derived table kept.
template <class T> void PlanBuilder<T>::image_segments(Image &im, Work &wk) {
  const int nwv = es.n_waves;
  wk.seg_of.assign(static_cast<size_t>(nwv) + 2, -1);
  wk.chain_of_op.assign(s.ops.size(), -1);
  if (!(use_fused && kn.chains && mem.keep_all)) return;
  const size_t chain_smem_max = static_cast<size_t>(kn.chain_smem_kb) * 1024;
  auto fits = [&](int w, int ws, size_t limit) {
    const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
    if (wr.nm || wr.nf == 0) return false;
    for (size_t q = wr.f0; q < wr.f0 + static_cast<size_t>(wr.nf); ++q) {
      const FoldOps &o = wk.fold_ops[q];
      if (wk.folds[q].nw > kChainMax || wk.folds[q].nv > kChainMax) return false;
      if (chain_smem_bytes<T>(1, 64, chain_stage_bytes<T>(wk.folds[q].nw, wk.folds[q].nv), false) > limit) return false;
      if (es.tab_wave[static_cast<size_t>(o.e2)] >= ws) return false;
      for (const auto &ab : es.epi[static_cast<size_t>(o.oi)]) // absorbed-merge operands: written before the run too
        if (es.tab_wave[static_cast<size_t>(ab.first)] >= ws || (ab.second >= 0 && es.tab_wave[static_cast<size_t>(ab.second)] >= ws))
          return false;
      const int p1 = es.tab_wave[static_cast<size_t>(o.e1)];
      if (p1 >= ws && p1 >= w) return false;
    }
    return true;
  };
  auto ranges = [&](size_t limit) {
    std::vector<std::pair<int, int>> r;
    for (int w = 1; w <= nwv;) {
      int we = w;
      if (fits(w, w, limit))
        while (we + 1 <= nwv && fits(we + 1, w, limit)) ++we;
      if (we - w + 1 >= kn.chain_min_waves) r.emplace_back(w, we);
      w = we + 1;
    }
    return r;
  };
  auto barriers_saved = [](const std::vector<std::pair<int, int>> &r) {
    int n = 0;
    for (const auto &x : r) n += x.second - x.first;
    return n;
  };
  // segments whose staging needs more than chain_smem_max run the kernel at one
  // CTA per SM (slower table build, fewer wave CTAs): only worth it when they
  // remove many more barriers (VGG-16: the whole network is one chain)
  std::vector<std::pair<int, int>> R = ranges(chain_smem_max);
  size_t limit = chain_smem_max;
  {
    const size_t big = static_cast<size_t>(kn.chain_smem_big_kb) * 1024;
    const auto R2 = ranges(big);
    if (barriers_saved(R2) - barriers_saved(R) >= kn.chain_big_gain) R = R2, limit = big;
  }
  for (const auto &[w, we] : R) {
    Segment sg{w, we, {}, {}, 0, 0, 0};
    std::vector<int> chain_of_table(static_cast<size_t>(mem.E_total), -1);
    std::vector<std::vector<size_t>> members;
    for (int x = w; x <= we; ++x) {
      const WaveRange &wr = im.waves[static_cast<size_t>(x) - 1];
      for (size_t q = wr.f0; q < wr.f0 + static_cast<size_t>(wr.nf); ++q) {
        const FoldOps &o = wk.fold_ops[q];
        int c = es.tab_wave[static_cast<size_t>(o.e1)] >= w ? chain_of_table[static_cast<size_t>(o.e1)] : -1;
        if (c < 0) {
          c = static_cast<int>(members.size());
          members.emplace_back();
        }
        members[static_cast<size_t>(c)].push_back(q);
        chain_of_table[static_cast<size_t>(o.ne)] = c;
      }
    }
    int max_len = 0, max_nw = 1;
    size_t stage = 0;
    for (const auto &m : members) {
      max_len = std::max(max_len, static_cast<int>(m.size()));
      for (size_t q : m) {
        stage = std::max(stage, chain_stage_bytes<T>(wk.folds[q].nw, wk.folds[q].nv));
        max_nw = std::max(max_nw, wk.folds[q].nw);
      }
    }
    // rows per item: the fewest rounds of items over the resident blocks (2
    // per SM; 1 with the large shared-memory layout) times the per-fold scan
    // length, kChainGroups / rows warps sharing a row's j range, plus a fixed
    // per-fold cost of ~14 j steps (measured: I16's first segment runs 6-row
    // items in one round faster than 4-row items in two)
    const int64_t blocks = (limit > chain_smem_max ? 1 : 2) * int64_t(ctx->sms);
    const bool want_path = max_len >= 3 && kn.chain_path; // unwind path tables for chains of >= 3 folds
    int rows = 1;
    bool path = false;
    int64_t best = INT64_MAX;
    for (int R = 1; R <= std::clamp(kn.chain_rows, 1, kChainRows); ++R) {
      const bool pr = want_path && chain_smem_bytes<T>(R, max_len, stage, true) <= limit;
      if (chain_smem_bytes<T>(R, max_len, stage, pr) > limit) break;
      int64_t items = 0;
      for (const auto &m : members) items += (wk.folds[m.front()].nu + R - 1) / R;
      const int wpr = std::max(1, kChainGroups / R);
      const int64_t cost = (items + blocks - 1) / blocks * (14 + (max_nw + wpr - 1) / wpr);
      if (cost < best || (cost == best && pr && !path)) best = cost, rows = R, path = pr;
    }
    sg.smem = chain_smem_bytes<T>(rows, max_len, stage, path);
    sg.stage = stage;
    for (const auto &m : members) {
      ChainDesc cd{static_cast<int32_t>(sg.cf.size()), static_cast<int32_t>(m.size()), wk.folds[m.front()].nu, rows,
                   sg.items, nullptr};
      for (size_t q : m) sg.cf.push_back(wk.folds[q]);
      sg.items += (cd.nu + rows - 1) / rows;
      if (path && m.size() >= 3) { // path table in the scratch section (rewritten by every run)
        const FoldDesc<T> &fl = wk.folds[m.back()];
        const size_t off = scr(im, static_cast<size_t>(cd.nu) * fl.nv * m.size() * sizeof(uint16_t));
        cd.path = reinterpret_cast<uint16_t *>(sb + off);
        ChainRec cr{static_cast<int>(wk.chain_nodes.size()), static_cast<int>(m.size()), cd.path};
        for (size_t q : m) wk.chain_nodes.push_back(s.ops[static_cast<size_t>(wk.fold_ops[q].oi)].removed);
        for (size_t q : m) wk.chain_of_op[static_cast<size_t>(wk.fold_ops[q].oi)] = static_cast<int>(wk.chain_recs.size());
        wk.chain_last_op.push_back(wk.fold_ops[m.back()].oi);
        wk.chain_recs.push_back(cr);
      }
      sg.chains.push_back(cd);
    }
    for (int x = w; x <= we; ++x) wk.seg_of[static_cast<size_t>(x)] = static_cast<int>(wk.segs.size());
    wk.segs.push_back(std::move(sg));
  }
}

// Which waves run on the first cluster alone, and which operands of a wave's
// first item may be staged during the previous wave: those every block has
// seen through a grid barrier that ended a wave x <= w - 2 (a
// narrow-to-narrow step ends in a cluster barrier only).  Chain segment folds
// were copied before this (they stage nothing across waves).
template <class T> void PlanBuilder<T>::image_staging(Image &im, Work &wk) {
  const int nwv = es.n_waves;
  const int64_t narrow_items = use_fused ? kn.narrow_items : 0;
  wk.narrow.assign(static_cast<size_t>(nwv) + 2, 0);
  std::vector<char> gbar(static_cast<size_t>(nwv) + 2, 1);
  for (int w = 1; w <= nwv; ++w) {
    const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
    wk.narrow[static_cast<size_t>(w)] = wk.seg_of[static_cast<size_t>(w)] < 0 && wr.ftiles + wr.mblocks <= narrow_items;
  }
  for (int w = 1; w < nwv; ++w) // inside a segment no barrier separates the waves
    if (wk.seg_of[static_cast<size_t>(w)] >= 0 && wk.seg_of[static_cast<size_t>(w)] == wk.seg_of[static_cast<size_t>(w) + 1])
      gbar[static_cast<size_t>(w)] = 0;
  for (int w = 1; w < nwv; ++w)
    if (wk.narrow[static_cast<size_t>(w)] && wk.narrow[static_cast<size_t>(w) + 1]) gbar[static_cast<size_t>(w)] = 0;
  std::vector<int> seen(static_cast<size_t>(nwv) + 2, 0); // data of waves <= seen[w] is visible while wave w - 1 runs
  for (int w = 3; w <= nwv; ++w)
    seen[static_cast<size_t>(w)] = gbar[static_cast<size_t>(w) - 2] ? w - 2 : seen[static_cast<size_t>(w) - 1];
  for (size_t q = 0; q < wk.folds.size(); ++q) {
    const FoldOps &o = wk.fold_ops[q];
    const int vis = seen[static_cast<size_t>(o.wave)];
    wk.folds[q].late = (es.tab_wave[static_cast<size_t>(o.e1)] > vis ? kPanelT1 : 0) |
                       (es.tab_wave[static_cast<size_t>(o.e2)] > vis || (mem.shard && o.e2 >= t.ne) ? kPanelT2 : 0);
  }
}

// Unwind records (kernels.cuh finish_block), visited last wave first and
// grouped by dependency level: a record's endpoints are final nodes (level 0)
// or removed by records of lower levels, so one group per level (the unwind's
// critical path) instead of one per wave.  Row-sharded: argmin tables stay on
// their ranks; a record holds the table's byte offset in every rank's plan
// memory and the finish phase reads the owner's row through the peer bases.
template <class T>
void PlanBuilder<T>::image_unwind(Image &im, Work &wk, std::vector<UnwindRec> &recs, std::vector<int32_t> &groups) {
  (void)im;
  std::vector<int> rlevel;
  std::vector<int> lvl(static_cast<size_t>(t.nl), -1);
  for (int d = 0; d < K; ++d) lvl[static_cast<size_t>(node_layer[static_cast<size_t>(d)])] = 0;
  for (int w = es.n_waves; w >= 1; --w) {
    for (int x = es.begin[static_cast<size_t>(w)]; x < es.begin[static_cast<size_t>(w) + 1]; ++x) {
      const int oi = es.exec[static_cast<size_t>(x)];
      const Op &op = s.ops[static_cast<size_t>(oi)];
      if (op.type) continue;
      const int ch = wk.chain_of_op[static_cast<size_t>(oi)];
      if (ch >= 0 && wk.chain_last_op[static_cast<size_t>(ch)] != oi) continue; // a chain: at its last fold
      const int lu = lvl[static_cast<size_t>(op.u)], lv = lvl[static_cast<size_t>(op.v)];
      PP_REQUIRE(lu >= 0 && lv >= 0, "unwind: record endpoint not yet assigned");
      const int level = std::max(lu, lv) + 1;
      if (ch < 0) {
        if (mem.shard) // byte offset of the table in every rank's plan memory (identical layouts)
          recs.push_back(UnwindRec{reinterpret_cast<const uint16_t *>(off_am + mem.am_off[static_cast<size_t>(oi)]),
                                   op.removed, op.u, op.v, mem.ncols(op.ne), 0, mem.blk(op.ne)});
        else
          recs.push_back(UnwindRec{amp(oi), op.removed, op.u, op.v, mem.ncols(op.ne), 0, 0});
        lvl[static_cast<size_t>(op.removed)] = level;
      } else {
        const ChainRec &cr = wk.chain_recs[static_cast<size_t>(ch)];
        recs.push_back(UnwindRec{cr.path, cr.node_off, op.u, op.v, mem.ncols(op.ne), cr.n, 0});
        for (int k = 0; k < cr.n; ++k) lvl[static_cast<size_t>(wk.chain_nodes[static_cast<size_t>(cr.node_off + k)])] = level;
      }
      rlevel.push_back(level);
    }
  }
  groups.assign(1, 0);
  std::vector<size_t> order(recs.size());
  for (size_t q = 0; q < order.size(); ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return rlevel[x] < rlevel[y]; });
  std::vector<UnwindRec> sorted;
  sorted.reserve(recs.size());
  for (size_t q = 0; q < order.size(); ++q) {
    if (q > 0 && rlevel[order[q]] != rlevel[order[q - 1]]) groups.push_back(static_cast<int32_t>(sorted.size()));
    sorted.push_back(recs[order[q]]);
  }
  if (!sorted.empty()) groups.push_back(static_cast<int32_t>(sorted.size()));
  recs.swap(sorted);
}

// Per-phase work lists of the fused kernel (pointers into the fold / merge
// sections already packed): one entry per wave, or per chain segment.
template <class T> void PlanBuilder<T>::image_phases(Image &im, Work &wk) {
  Packer &pk = im.pk;
  std::vector<FusedWave<T>> fw;
  im.phase_work.clear();
  int64_t rot = 0;
  for (int w = 1; w <= es.n_waves;) {
    const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
    const int sg = wk.seg_of[static_cast<size_t>(w)];
    if (sg >= 0) {
      const Segment &S = wk.segs[static_cast<size_t>(sg)];
      const size_t oc = pk.put(S.chains), of = pk.put(S.cf);
      FusedWave<T> e{};
      e.items = S.items;
      e.n_chains = static_cast<int32_t>(S.chains.size());
      e.stage = static_cast<int64_t>(S.stage);
      e.chains = reinterpret_cast<const ChainDesc *>(db + off_image + oc);
      e.cfolds = reinterpret_cast<const FoldDesc<T> *>(db + off_image + of);
      if (S.chains.size() > 1) { // per-item chain index (replaces a binary search per item)
        PP_REQUIRE(S.chains.size() <= 65535, "too many chains in one segment");
        std::vector<uint16_t> chain_of(static_cast<size_t>(S.items));
        for (size_t q = 0; q < S.chains.size(); ++q) {
          const int64_t i1 = q + 1 < S.chains.size() ? S.chains[q + 1].item_begin : S.items;
          for (int64_t x = S.chains[q].item_begin; x < i1; ++x) chain_of[static_cast<size_t>(x)] = static_cast<uint16_t>(q);
        }
        e.chain_of = reinterpret_cast<const uint16_t *>(db + off_image + pk.put(chain_of));
      }
      fw.push_back(e);
      double cells = 0.0;
      for (int x = S.ws; x <= S.we; ++x) cells += im.waves[static_cast<size_t>(x) - 1].cells;
      im.phase_work.push_back(cells);
      w = S.we + 1;
      continue;
    }
    const int64_t items = wr.ftiles + wr.mblocks;
    FusedWave<T> e{};
    if (wr.nf > 1) { // per-tile fold index (replaces a binary search per work item)
      std::vector<uint16_t> fold_of(static_cast<size_t>(wr.ftiles));
      PP_REQUIRE(wr.nf <= 65535, "too many folds in one wave");
      for (int q = 0; q < wr.nf; ++q) {
        const int64_t t0 = wk.folds[wr.f0 + static_cast<size_t>(q)].tile_begin;
        const int64_t t1 = q + 1 < wr.nf ? wk.folds[wr.f0 + static_cast<size_t>(q) + 1].tile_begin : wr.ftiles;
        for (int64_t x = t0; x < t1; ++x) fold_of[static_cast<size_t>(x)] = static_cast<uint16_t>(q);
      }
      e.fold_of = reinterpret_cast<const uint16_t *>(db + off_image + pk.put(fold_of));
    }
    e.folds = reinterpret_cast<const FoldDesc<T> *>(db + off_image + im.oF) + wr.f0;
    e.merges = reinterpret_cast<const MergeDesc<T> *>(db + off_image + im.oM) + wr.m0;
    e.nf = wr.nf, e.nm = wr.nm, e.ftiles = wr.ftiles, e.items = items, e.rot = rot;
    e.narrow = wk.narrow[static_cast<size_t>(w)];
    fw.push_back(e);
    im.phase_work.push_back(wr.cells);
    if (kn.rotate) rot += items;
    ++w;
  }
  im.oFW = pk.put(fw);
  im.n_phases = static_cast<int>(fw.size());
  im.dyn_smem = sizeof(WaveSmem<T>);
  for (const Segment &S : wk.segs) im.dyn_smem = std::max(im.dyn_smem, S.smem);
  im.phase_chain.clear();
  for (const auto &e : fw) im.phase_chain.push_back(e.n_chains > 0);
  im.oST = scr(im, (fw.size() + 4) * sizeof(uint64_t));
  im.oTR = kn.wave_trace ? scr(im, (16 * fw.size() + 16 + 12288) * sizeof(uint64_t)) + 1 : 0; // +1: nonzero flag
}

// The whole image against device bases dbase (plan memory) and sbase
// (device-only scratch: enumeration block results, cost terms, stamps, chain
// path tables; not uploaded).  Null bases: a sizing pass.
template <class T> typename PlanBuilder<T>::Image PlanBuilder<T>::make_image(unsigned char *dbase, unsigned char *sbase) {
  db = dbase, sb = sbase;
  Image im;
  Work wk;
  im.pk.bytes.reserve(ctx->last_image_bytes + 4096);
  // result slots first, contiguous: indices[nl] | digits[K] | final_cost |
  // cost | min-plus cap overflow flag
  im.oRes = im.pk.put(std::vector<int32_t>(static_cast<size_t>(t.nl) + static_cast<size_t>(K) + 2));
  im.oIdx = im.oRes;
  im.oFC = im.pk.put(std::vector<double>(2));
  im.oOvf = im.pk.put(std::vector<int32_t>(4));
  oOvf_ = im.oOvf;
  // row-sharded: every rank's plan memory base (filled before upload: IPC-mapped peers, or the virtual ranks')
  im.oPeer = mem.shard ? im.pk.put(std::vector<uint64_t>(static_cast<size_t>(mem.NR))) : 0;
  im.res_bytes = im.oOvf + 16 - im.oRes;
  run_img.clear();
  image_waves(im, wk);
  image_segments(im, wk);
  image_staging(im, wk);
  const T *on = onode();
  std::vector<EnumNode> en(static_cast<size_t>(K));
  for (int d = 0; d < K; ++d) {
    const int l = node_layer[static_cast<size_t>(d)];
    en[static_cast<size_t>(d)] = EnumNode{on + t.cat_off[static_cast<size_t>(l)], cnt(l), 0};
  }
  std::vector<EnumEdge> ee;
  for (int id : s.final_edges) {
    if (mem.shard && id >= t.ne)
      im.final_gathers.emplace_back(tabp(id), gatp(id), static_cast<size_t>(mem.blk(id)) * mem.ncols(id) * sizeof(T));
    ee.push_back(EnumEdge{t2p(id), pos[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])],
                          pos[static_cast<size_t>(s.edst[static_cast<size_t>(id)])], mem.ncols(id), 0});
  }
  if (mem.shard) { // the gathers issued above follow shard.hpp's schedule (pp_shard_layout, host-tested)
    size_t n = im.final_gathers.size();
    for (const auto &w : im.waves) n += w.gathers.size();
    PP_REQUIRE(n == shard_gathers(s, t.ne).size(), "row-sharded plan: all-gather schedule mismatch");
  }
  std::vector<UnwindRec> recs;
  std::vector<int32_t> groups;
  image_unwind(im, wk, recs, groups);
  Packer &pk = im.pk;
  im.oG = pk.put(groups);
  im.nG = static_cast<int>(groups.size()) - 1;
  im.oT = scr(im, static_cast<size_t>(t.nl + t.ne) * sizeof(double));
  im.oMP = pk.put(wk.mpf);
  im.oMM = pk.put(wk.mmv);
  im.oM64 = pk.put(wk.m64);
  im.n_mp = static_cast<int>(wk.mpf.size());
  im.colmin_blocks = wk.colmin_blocks;
  im.rowmin_blocks = wk.rowmin_blocks;
  im.oF = pk.put(wk.folds);
  im.oM = pk.put(wk.merges);
  image_phases(im, wk);
  im.oN = pk.put(en);
  im.oE = pk.put(ee);
  im.oR = pk.put(recs);
  im.oCN = pk.put(wk.chain_nodes.empty() ? std::vector<int32_t>{0} : wk.chain_nodes);
  im.oL = pk.put(node_layer);
  im.oCO = pk.put(t.cat_off);
  im.oXO = pk.put(t.xoff);
  im.oS = pk.put(std::vector<int32_t>(t.esrc.begin(), t.esrc.end()));
  im.oD = pk.put(std::vector<int32_t>(t.edst.begin(), t.edst.end()));
  im.oC = pk.put(t.counts);
  if (bp && !early) {
    im.oLay = pk.put(bp->L);
    im.oEdg = pk.put(bp->E);
    im.oCfg = pk.put(*bp->cfg32);
    im.oRat = pk.put(bp->rates);
    im.oBw = pk.put(bp->bw);
  }
  im.oBV = scr(im, static_cast<size_t>(nblk) * sizeof(A));
  im.oBI = scr(im, static_cast<size_t>(nblk) * sizeof(int64_t));
  return im;
}

// The image holds absolute device pointers, so it is built against the final
// base.  One-shot plans reuse the context pool: build against the current pool
// and rebuild only when the pool has to grow (first calls).  Prepared plans own
// their memory: a sizing pass, the allocation, the real image.
template <class T> typename PlanBuilder<T>::Image PlanBuilder<T>::place_image() {
  Image im;
  if (P->transient) {
    im = make_image(ctx->plan_pool.p, ctx->plan_scratch.p);
    const size_t total = off_image + align256(im.pk.size());
    if (total > ctx->plan_pool.n || !ctx->plan_pool.p || im.scratch > ctx->plan_scratch.n || !ctx->plan_scratch.p) {
      if (early) { // the pool moves: rebuild the tables in the fused kernel instead
        PP_CUDA(cudaStreamSynchronize(ctx->stream));
        early = false;
        P->early_built = false;
      }
      ctx->plan_pool.ensure(total + total / 4);
      ctx->plan_scratch.ensure(std::max<size_t>(im.scratch + im.scratch / 4, 256));
      im = make_image(ctx->plan_pool.p, ctx->plan_scratch.p);
    }
    ctx->last_pool_bytes = std::max(ctx->last_pool_bytes, off_image + align256(im.pk.size()) + 65536);
    P->dbase = ctx->plan_pool.p;
    P->sbase = ctx->plan_scratch.p;
    P->hbase = static_cast<unsigned char *>(ctx->plan_pinned.ensure(align256(im.pk.size())));
    clk.mark("image");
  } else {
    const Image sizing = make_image(nullptr, nullptr);
    const size_t total = off_image + align256(sizing.pk.size());
    P->dmem.alloc(total);
    P->dscratch.alloc(std::max<size_t>(sizing.scratch, 256));
    P->dbase = P->dmem.p;
    P->sbase = P->dscratch.p;
    // poison: a slot the device work fails to write shows up as garbage
    PP_CUDA(cudaMemsetAsync(P->dbase, 0xFF, total, ctx->stream));
    im = make_image(P->dbase, P->sbase);
    P->hbase = static_cast<unsigned char *>(P->hmem.ensure(align256(im.pk.size())));
  }
  ctx->last_image_bytes = std::max(ctx->last_image_bytes, im.pk.size());
  std::memcpy(P->hbase, im.pk.bytes.data(), im.pk.size());
  P->image_off = off_image;
  P->image_bytes = im.pk.size();
  P->res_off = im.oRes;
  P->res_bytes = im.res_bytes;
  P->off_idx = im.oIdx;
  P->off_cost = im.oFC;
  P->off_ovf = im.oOvf;
  P->off_peer = mem.shard ? im.oPeer : SIZE_MAX;
  P->nranks = mem.NR;
  if (bp) { // tables live in the plan's memory
    unsigned char *d = P->dbase + off_tables;
    const size_t nb = align256(static_cast<size_t>(t.ncells) * 8);
    t.node.view(d, static_cast<size_t>(t.ncells));
    t.compute.view(d + nb, static_cast<size_t>(t.ncells));
    t.sync.view(d + 2 * nb, static_cast<size_t>(t.ncells));
    t.xfer64.view(d + 3 * nb, static_cast<size_t>(t.xcells));
  }
  return im;
}

template <class T> void PlanBuilder<T>::build(int k_bound) {
  check_final(k_bound);
  early_table_build();
  mem.build(s, t.counts, t.ne, sizeof(T), ctx->nranks, ctx->rank);
  plan_minplus();
  es.build(s, mem.prod_wave, use_fused && mem.keep_all && kn.merge_fuse, kMaxEpi);
  plan_sections();
  plan_enumeration();
  clk.mark("memplan");
  const Image im = place_image();
  db = P->dbase, sb = P->sbase;
  emit_steps(im);
}

} // namespace pp
