// plan.cu — the batched plan executor: plan() / plan_with_tables() on the device.
//
// prepare (host, once):  catalogs + K1/K2 descriptors (plan()), the cached
//                        symbolic schedule, a liveness memory plan for derived
//                        tables, and ONE descriptor image holding every launch's
//                        work list plus the result slots
// launch  (device only): [H2D image] -> K1/K2 -> one wave kernel per dependency
//                        wave -> K5 enumerate -> finish (unwind + cost re-sum)
//                        -> D2H of indices + cost; captured as a CUDA graph
//                        for prepared plans
// fetch:                 stream sync, parse results
#include "dp.hpp"
#include "fused.cuh"
#include "kernels.cuh"
#include "minplus.cuh"
#include "minplus64.cuh"
#include "mp_plan.hpp"
#include "shard.hpp"

#include <array>
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstring>
#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

namespace pp {
// tuning knobs read once per prepare (A/B experiments in one process)
static int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}
struct Knobs {
  int cluster, narrow_items, chain_smem_kb, chain_smem_big_kb, chain_big_gain, mp_chain, mp_chain_min, merge_fuse,
      chain_min_waves, early_build, grid_barrier, build_dynamic, panel,
      panel_side, chains,
      chain_path, rotate,
      wave_trace, stage, blocks_per_sm, split_build;
  Knobs()
      : cluster(env_int("PARPLAN_CLUSTER", 1)), narrow_items(env_int("PARPLAN_NARROW_ITEMS", 0)),
        chain_smem_kb(env_int("PARPLAN_CHAIN_SMEM_KB", 110)), chain_smem_big_kb(env_int("PARPLAN_CHAIN_SMEM_BIG_KB", 216)),
        chain_big_gain(env_int("PARPLAN_CHAIN_BIG_GAIN", 6)), mp_chain(env_int("PARPLAN_MP_CHAIN", 1)),
        mp_chain_min(std::max(1, env_int("PARPLAN_MP_CHAIN_MIN", 4))),
        merge_fuse(env_int("PARPLAN_MERGE_FUSE", 1)), chain_min_waves(std::max(2, env_int("PARPLAN_CHAIN_MIN_WAVES", 2))),
        early_build(env_int("PARPLAN_EARLY_BUILD", 1)), grid_barrier(env_int("PARPLAN_GRID_BARRIER", 1)),
        build_dynamic(env_int("PARPLAN_BUILD_DYNAMIC", 1)),
        panel(env_int("PARPLAN_PANEL", 1)),
        panel_side(env_int("PARPLAN_PANEL_SIDE", 0)), chains(env_int("PARPLAN_CHAINS", 1)),
        chain_path(env_int("PARPLAN_CHAIN_PATH", 1)), rotate(env_int("PARPLAN_ROTATE", 1)),
        wave_trace(env_int("PARPLAN_WAVE_TRACE", 0)), stage(env_int("PARPLAN_STAGE", 1)),
        blocks_per_sm(env_int("PARPLAN_FUSED_BLOCKS_PER_SM", 0)), split_build(env_int("PARPLAN_SPLIT_BUILD", 1)) {}
};
}

namespace pp {

namespace {

// First-fit offset allocator with coalescing; derived tables are released
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

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

} // namespace
} // namespace pp

using namespace pp;

struct pp_prepared {
  pp_context *ctx = nullptr;
  Graph *g = nullptr;
  Tables *t = nullptr;
  std::unique_ptr<Tables> own_t;
  bool transient = true;
  DBuf<unsigned char> dmem, dscratch;
  PinnedBuf hmem;
  unsigned char *dbase = nullptr, *hbase = nullptr;
  unsigned char *sbase = nullptr; // device-only scratch (kernel-written buffers)
  size_t image_off = 0, image_bytes = 0, res_off = 0, res_bytes = 0, off_idx = 0, off_cost = 0, off_ovf = 0;
  bool mp_conservative = false; // min-plus folds with proven caps only (after an optimistic overflow)
  int k_bound = 8;
  // row-sharded plans: image offset of the peer bases, rank count, the block
  // lists of the collective steps (kind 15 all-gathers, kind 19 edge-range
  // broadcasts; in order), IPC-opened peer bases
  size_t off_peer = SIZE_MAX;
  int nranks = 1;
  std::vector<std::vector<std::tuple<const void *, void *, size_t>>> gather_lists;
  std::vector<void *> ipc_opened;
  std::vector<std::function<void(cudaStream_t)>> steps;
  int launches_per_run = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int K = 0, n_waves = 0, node_ops = 0, edge_ops = 0;
  std::vector<int32_t> step_kind; // 0 K1/K2, 1 wave, 2 K5, 3 finish, 4 D2H
  std::vector<double> step_work;  // cells: K1/K2 table cells, wave min-plus cells (nu*nw*nv) + merge cells
  bool launched = false, uploaded = false;
  bool early_built = false; // transient plan: the table build was launched during prepare (ev0 already recorded)
  size_t stamp_off = 0; // fused kernel phase stamps (image offset), n_stamps entries
  int n_stamps = 0;
  size_t trace_off = 0; // PARPLAN_WAVE_TRACE: 8 stamps per wave (printed by pp_plan_profile)
  std::vector<char> phase_chain; // fused phases that are chain segments (profile kind 16)
  int nblk_dbg = 0, ngroups_dbg = 0;
  std::vector<double> fused_wave_work;

  ~pp_prepared() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (void *p : ipc_opened) cudaIpcCloseMemHandle(p);
  }
};

namespace pp {

// PARPLAN_TRACE=2: host-side timing of build_steps' stages
struct StageClock {
  bool on = false;
  std::vector<std::pair<const char *, std::chrono::steady_clock::time_point>> marks;
  StageClock() {
    const char *e = std::getenv("PARPLAN_TRACE");
    on = e && std::atoi(e) >= 2;
    if (on) marks.emplace_back("start", std::chrono::steady_clock::now());
  }
  void mark(const char *name) {
    if (on) marks.emplace_back(name, std::chrono::steady_clock::now());
  }
  ~StageClock() {
    if (!on) return;
    std::fprintf(stderr, "[parplan] build_steps:");
    for (size_t k = 1; k < marks.size(); ++k)
      std::fprintf(stderr, " %s %.1f", marks[k].first,
                   std::chrono::duration<double, std::micro>(marks[k].second - marks[k - 1].second).count());
    std::fprintf(stderr, " us\n");
  }
};

using MpChainFn = void (*)(const MpFold *, int, int);
// the chain kernel for a run: optimistic runs (JB 6) get the exact row count
// per CTA, proven-cap runs (JB <= 5) the 8-row tile
static MpChainFn mp_chain_launch(int jb, int R) {
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

template <class T>
static void build_steps(pp_prepared *P, const BuildPlan *bp, int k_bound) {
  StageClock clk;
  const Knobs kn;
  pp_context *ctx = P->ctx;
  Graph &g = *P->g;
  Tables &t = *P->t;
  const Schedule &s = g.schedule();
  const int K = static_cast<int>(s.final_nodes.size());
  if (K > k_bound)
    throw parplan::LimitError("final graph has " + std::to_string(K) + " nodes, exceeding the enumeration bound of " +
                              std::to_string(k_bound) + " (graph is not reducible enough)");
  PP_REQUIRE(K <= kMaxEnumNodes, "final graph too large for the enumeration kernel");
  P->K = K;
  P->n_waves = s.n_waves;
  P->node_ops = s.node_ops;
  P->edge_ops = s.edge_ops;
  bool early = false; // transient plans: K1/K2 launched before the descriptor image is built
  {
    // One-shot plans overlap the host's descriptor build with the device's
    // table build: K1/K2 launch first (their descriptors go up in a small
    // separate upload), the image is built while they run, and the fused
    // kernel follows without its build phase.  The pool must already hold
    // the final layout; if the image outgrows the estimate, fall back.
    if (P->transient && bp && !ctx->no_fused && ctx->nranks <= 1 && bp->grid > 0 && kn.early_build && ctx->last_pool_bytes > 0) {
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
  }

  const int E_total = static_cast<int>(s.esrc.size());
  std::vector<int32_t> rows(static_cast<size_t>(E_total)), cols(static_cast<size_t>(E_total));
  for (int id = 0; id < E_total; ++id) {
    rows[static_cast<size_t>(id)] = t.counts[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])];
    cols[static_cast<size_t>(id)] = t.counts[static_cast<size_t>(s.edst[static_cast<size_t>(id)])];
  }
  for (const Op &op : s.ops)
    if (!op.type) PP_REQUIRE(t.counts[static_cast<size_t>(op.removed)] <= 65535, "argmin index exceeds 16 bits");

  // ---- row sharding across ranks (pp_context_attach_comm) --------------------
  // Every derived table is split by rows (= configs of its source node) into
  // NR blocks of blk rows; rank RK computes and stores rows [RK*blk, ...).
  // Original tables are replicated.  A fold needs its t2 in full: a derived t2
  // is all-gathered first (the re-association points); at the end the final
  // edges and every argmin table are all-gathered so every rank enumerates and
  // unwinds identically.
  const int NR = ctx->nranks > 1 ? ctx->nranks : 1, RK = NR > 1 ? ctx->rank : 0;
  const bool shard = NR > 1;
  auto blk = [&](int id) { return shard_blk(rows[static_cast<size_t>(id)], NR); };
  auto lr0 = [&](int id) { return shard_first(rows[static_cast<size_t>(id)], NR, RK); };
  auto lrows = [&](int id) { return shard_rows(rows[static_cast<size_t>(id)], NR, RK); };

  // ---- memory plan ----------------------------------------------------------
  auto cells = [&](int id) { return static_cast<size_t>(rows[static_cast<size_t>(id)]) * cols[static_cast<size_t>(id)]; };
  auto store_cells = [&](int id) { // storage of a derived table on this rank
    return shard ? static_cast<size_t>(blk(id)) * cols[static_cast<size_t>(id)] : cells(id);
  };
  auto full_cells = [&](int id) { // all-gather target (NR padded blocks)
    return static_cast<size_t>(NR) * blk(id) * cols[static_cast<size_t>(id)];
  };
  size_t derived_total = 0;
  for (const Op &op : s.ops) derived_total += align256(store_cells(op.ne) * sizeof(T));
  const bool keep_all = derived_total <= (size_t(4) << 30);
  OffsetPlanner tab_plan;
  std::vector<size_t> tab_off(static_cast<size_t>(E_total), 0), am_off(s.ops.size(), 0);
  std::vector<size_t> gat_off(static_cast<size_t>(E_total), SIZE_MAX);
  size_t am_bytes = 0, gat_bytes = 0;
  std::vector<int> prod_wave(static_cast<size_t>(E_total), 0); // wave writing each table (0: original)
  for (int w = 1; w <= s.n_waves; ++w) {
    const int x0 = s.wave_begin[static_cast<size_t>(w)], x1 = s.wave_begin[static_cast<size_t>(w) + 1];
    for (int x = x0; x < x1; ++x) {
      const int oi = s.exec[static_cast<size_t>(x)];
      const Op &op = s.ops[static_cast<size_t>(oi)];
      tab_off[static_cast<size_t>(op.ne)] = tab_plan.alloc(store_cells(op.ne) * sizeof(T));
      prod_wave[static_cast<size_t>(op.ne)] = w;
      if (!op.type) {
        am_off[static_cast<size_t>(oi)] = am_bytes;
        am_bytes += align256(store_cells(op.ne) * 2);
        if (shard) {
          if (op.e2 >= t.ne) { // derived t2: gathered in full before the fold
            gat_off[static_cast<size_t>(op.e2)] = gat_bytes;
            gat_bytes += align256(full_cells(op.e2) * sizeof(T));
          }
        }
      }
    }
    if (!keep_all)
      for (int x = x0; x < x1; ++x) {
        const Op &op = s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])];
        for (int in : {op.e1, op.e2})
          if (in >= t.ne) tab_plan.release(tab_off[static_cast<size_t>(in)], store_cells(in) * sizeof(T));
      }
  }
  if (shard)
    for (int id : s.final_edges)
      if (id >= t.ne && gat_off[static_cast<size_t>(id)] == SIZE_MAX) {
        gat_off[static_cast<size_t>(id)] = gat_bytes;
        gat_bytes += align256(full_cells(id) * sizeof(T));
      }
  // rows of a fold's t1 / a merge's operands this rank works on
  auto nu_eff = [&](int id) { return shard ? lrows(id) : rows[static_cast<size_t>(id)]; };
  // ---- large folds (U16 fixed point / FP64): certificate, chain runs, scratch layout
  MinplusPlan mp;
  mp.build<T>(MinplusPlan::In{s, t, rows, cols, nu_eff, shard, P->mp_conservative || ctx->mp_conservative || shard,
                              ctx->no_minplus, ctx->sms, kn.mp_chain != 0, kn.mp_chain_min, prod_wave});
  using MpLayout = MinplusPlan::Layout;
  using MpRun = MinplusPlan::Run;
  auto &large = mp.large;
  auto &fold_jb = mp.fold_jb;
  auto &fold_m = mp.fold_m;
  auto &fold_opt = mp.fold_opt;
  auto &mpl = mp.mpl;
  auto &wave_group_jb = mp.wave_group_jb;
  auto &mp_group = mp.mp_group;
  auto &mp_consumer = mp.mp_consumer;
  auto &mp_consumer2 = mp.mp_consumer2;
  auto &mp_producer = mp.mp_producer;
  auto &mp_merge_out = mp.mp_merge_out;
  auto &mp_runs = mp.runs;
  auto &mp_run_of = mp.run_of;
  auto &large64 = mp.large64;
  auto &mp64_group = mp.mp64_group;
  auto &mp64_off = mp.mp64_off;
  const size_t mp_bytes = mp.bytes, mp_part = mp.part, mp_cnt = mp.cnt, mp_ra = mp.ra, mp_cb = mp.cb,
               mp_chainb = mp.chainb;
  const size_t mp_pbytes = mp.pbytes();
  (void)mp_consumer;
  (void)mp_group;
  // dynamic shared memory allowances: per device, so set on every prepare (cheap)
  for (const MpRun &run : mp_runs)
    for (int jb : {5, kMpOptJB})
      PP_CUDA(cudaFuncSetAttribute(mp_chain_launch(jb, run.R), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kMpChainSmem)));
  if (mp_part)
    for (auto fn : {mp_fold_kernel<7>, mp_fold_kernel<6>, mp_fold_kernel<5>, mp_fold_kernel<4>, mp_fold_kernel<3>})
      PP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMpSmem)));
  if (mp_bytes && std::is_same_v<T, double>)
    PP_CUDA(cudaFuncSetAttribute(mp64_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMp64Smem)));

  const size_t tables_bytes =
      bp ? align256(static_cast<size_t>(t.ncells) * 8) * 3 + align256(static_cast<size_t>(t.xcells) * 8) : 0;
  const size_t off_tables = 0, off_derived = tables_bytes, off_am = off_derived + align256(tab_plan.end()),
               off_mp = off_am + align256(am_bytes), off_mpp = off_mp + align256(mp_bytes),
               off_gat = off_mpp + align256(mp_pbytes), off_image = off_gat + align256(gat_bytes);

  // ---- enumeration / unwind descriptors (pointer-free parts) ----------------
  std::vector<int> pos(static_cast<size_t>(t.nl), -1);
  int64_t space = 1;
  std::vector<int32_t> node_layer(static_cast<size_t>(K));
  for (int d = 0; d < K; ++d) {
    const int l = s.final_nodes[static_cast<size_t>(d)];
    node_layer[static_cast<size_t>(d)] = l;
    pos[static_cast<size_t>(l)] = d;
    PP_REQUIRE(space <= INT64_MAX / std::max(1, t.counts[static_cast<size_t>(l)]), "final enumeration space overflows");
    space *= t.counts[static_cast<size_t>(l)];
  }
  const int64_t lanes = int64_t(ctx->sms) * 8 * kEnumThreads;
  const int64_t per_thread = std::max<int64_t>(1, (space + lanes - 1) / lanes);
  const int nblk = static_cast<int>(((space + per_thread - 1) / per_thread + kEnumThreads - 1) / kEnumThreads);
  std::vector<int32_t> es(t.esrc.begin(), t.esrc.end()), ed(t.edst.begin(), t.edst.end());
  using A = typename Acc<T>::type;

  // ---- descriptor image, as a function of the device base --------------------
  struct WaveRange {
    size_t f0, m0;
    int nf, nm;
    int64_t ftiles, mblocks;
    double cells;
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
    std::vector<std::tuple<const void *, void *, size_t>> gathers; // sharded: derived t2 -> full, before the wave
  };
  struct Image {
    Packer pk;
    std::vector<WaveRange> waves;
    std::vector<std::tuple<const void *, void *, size_t>> final_gathers; // sharded: final edges + argmins
    size_t oF, oM, oN, oE, oR, oL, oCO, oXO, oS, oD, oC, oBV, oBI, oRes, oIdx, oFC, oLay, oEdg, oCfg, oRat, oBw, oMP;
    size_t oG, oT, oFW, oST, oTR, oCN; // oT, oST, oTR (+1), oBV, oBI: scratch offsets
    size_t oOvf = 0;                   // min-plus optimistic-cap overflow flag (result slot)
    size_t oPeer = 0;                  // row-sharded: NR plan memory bases
    size_t scratch = 0;                // bytes of the scratch section
    int n_phases = 0;                // fused kernel: waves / chain segments
    size_t dyn_smem = 0;             // fused kernel dynamic shared memory
    std::vector<char> phase_chain;   // phase is a chain segment
    std::vector<double> phase_work;  // cells per fused phase
    int nG;
    size_t res_bytes;
    size_t oMM = 0;            // min-plus merges (all waves)
    size_t oM64 = 0;           // FP64 large folds (all waves)
    int n_mp = 0;              // large folds (all waves)
    int64_t colmin_blocks = 0, rowmin_blocks = 0; // mp_minima blocks
  };
  const bool use_fused = mp_bytes == 0 && mp_pbytes == 0 && !ctx->no_fused && !shard; // no large (U16 or FP64) folds
  // ---- effective schedule of the fused kernel: merge absorption ------------
  // An edge elimination (Eq. 3, out = a + b) whose operand a comes from a fold
  // F (or from merges already absorbed into F) while b is ready before F runs
  // is folded into F's epilogue: F writes ((v + b1) + b2)..., one IEEE add per
  // merge in the reference's order (a single add is commutative, so which
  // operand F produced does not matter).  Merge-only waves disappear and later
  // folds move up.  Needs every derived table kept (keep_all: no memory reuse
  // across the reordered waves).
  const int n_ops = static_cast<int>(s.ops.size());
  std::vector<int> out_table(static_cast<size_t>(n_ops)), op_wave(static_cast<size_t>(n_ops));
  std::vector<std::vector<std::pair<int, int>>> epi(static_cast<size_t>(n_ops)); // (table, table or -1) per absorbed merge
  std::vector<char> absorbed(static_cast<size_t>(n_ops), 0);
  std::vector<int> tab_wave(static_cast<size_t>(E_total), 0); // effective wave writing each table
  int EWn = s.n_waves;
  std::vector<int> EWbegin(s.wave_begin.begin(), s.wave_begin.end()), EWexec(s.exec.begin(), s.exec.end());
  for (int oi = 0; oi < n_ops; ++oi) out_table[static_cast<size_t>(oi)] = s.ops[static_cast<size_t>(oi)].ne;
  for (int oi = 0; oi < n_ops; ++oi) op_wave[static_cast<size_t>(oi)] = s.ops[static_cast<size_t>(oi)].wave;
  for (int id = 0; id < E_total; ++id) tab_wave[static_cast<size_t>(id)] = prod_wave[static_cast<size_t>(id)];
  if (use_fused && keep_all && kn.merge_fuse) {
    // runs of fold-only waves that may become chain segments (original waves,
    // ignoring shared-memory limits): a host fold inside one only absorbs
    // operands written before the run, so absorption never breaks a segment
    std::vector<int> run_start(static_cast<size_t>(s.n_waves) + 2, 0);
    for (int w = 1; w <= s.n_waves; ++w) {
      bool folds_only = true;
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x)
        folds_only = folds_only && !s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])].type;
      int ws = w;
      if (folds_only && w > 1 && run_start[static_cast<size_t>(w) - 1] > 0) {
        const int cand = run_start[static_cast<size_t>(w) - 1];
        bool ok = true;
        for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x)
          ok = ok && prod_wave[static_cast<size_t>(s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])].e2)] < cand;
        if (ok) ws = cand;
      }
      run_start[static_cast<size_t>(w)] = folds_only ? ws : 0;
    }
    std::vector<int> owner(static_cast<size_t>(E_total), -1);    // fold writing a table (after absorption)
    std::vector<int> merge_of(static_cast<size_t>(E_total), -1); // real merge writing a table
    for (int id = 0; id < E_total; ++id) tab_wave[static_cast<size_t>(id)] = 0;
    for (int w = 1; w <= s.n_waves; ++w)
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        const int wa = tab_wave[static_cast<size_t>(op.e1)], wb = tab_wave[static_cast<size_t>(op.e2)];
        if (!op.type) {
          const int ew = 1 + std::max(wa, wb);
          op_wave[static_cast<size_t>(oi)] = ew;
          tab_wave[static_cast<size_t>(op.ne)] = ew;
          owner[static_cast<size_t>(op.ne)] = oi;
          continue;
        }
        // operands must be ready before the host runs (before its fold run,
        // when it sits in one); a not-yet-absorbed merge of two such tables
        // rides along as a pair
        int host = -1;
        std::pair<int, int> add{-1, -1};
        for (int side = 0; side < 2 && host < 0; ++side) {
          const int mine = side ? op.e2 : op.e1, oth = side ? op.e1 : op.e2;
          const int F = owner[static_cast<size_t>(mine)];
          if (F < 0 || out_table[static_cast<size_t>(F)] != mine || epi[static_cast<size_t>(F)].size() >= kMaxEpi) continue;
          const int rs = run_start[static_cast<size_t>(s.ops[static_cast<size_t>(F)].wave)];
          const int lim = rs > 0 ? std::min(op_wave[static_cast<size_t>(F)], rs) : op_wave[static_cast<size_t>(F)];
          auto old_enough = [&](int id) { return tab_wave[static_cast<size_t>(id)] == 0 || tab_wave[static_cast<size_t>(id)] < lim; };
          if (old_enough(oth)) {
            host = F, add = {oth, -1};
          } else if (merge_of[static_cast<size_t>(oth)] >= 0) {
            const int M2 = merge_of[static_cast<size_t>(oth)];
            const Op &o2 = s.ops[static_cast<size_t>(M2)];
            if (!absorbed[static_cast<size_t>(M2)] && old_enough(o2.e1) && old_enough(o2.e2)) {
              host = F, add = {o2.e1, o2.e2};
              absorbed[static_cast<size_t>(M2)] = 1;
            }
          }
        }
        if (host >= 0) {
          epi[static_cast<size_t>(host)].push_back(add);
          out_table[static_cast<size_t>(host)] = op.ne;
          owner[static_cast<size_t>(op.ne)] = host;
          tab_wave[static_cast<size_t>(op.ne)] = op_wave[static_cast<size_t>(host)];
          absorbed[static_cast<size_t>(oi)] = 1;
        } else {
          const int ew = 1 + std::max(wa, wb);
          op_wave[static_cast<size_t>(oi)] = ew;
          tab_wave[static_cast<size_t>(op.ne)] = ew;
          merge_of[static_cast<size_t>(op.ne)] = oi;
        }
      }
    // regroup the surviving ops by effective wave (stable: schedule order within a wave)
    EWn = 0;
    for (int oi = 0; oi < n_ops; ++oi)
      if (!absorbed[static_cast<size_t>(oi)]) EWn = std::max(EWn, op_wave[static_cast<size_t>(oi)]);
    std::vector<std::vector<int>> by(static_cast<size_t>(EWn) + 1);
    for (int w = 1; w <= s.n_waves; ++w)
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        if (!absorbed[static_cast<size_t>(oi)]) by[static_cast<size_t>(op_wave[static_cast<size_t>(oi)])].push_back(oi);
      }
    EWbegin.assign(static_cast<size_t>(EWn) + 2, 0);
    EWexec.clear();
    for (int w = 1; w <= EWn; ++w) {
      EWbegin[static_cast<size_t>(w)] = static_cast<int>(EWexec.size());
      EWexec.insert(EWexec.end(), by[static_cast<size_t>(w)].begin(), by[static_cast<size_t>(w)].end());
    }
    EWbegin[static_cast<size_t>(EWn) + 1] = static_cast<int>(EWexec.size());
  }
  // fused kernel: waves with at most kNarrowItems work items run on the first
  // thread-block cluster alone, with cluster barriers between consecutive
  // narrow waves instead of grid-wide ones
  const int fused_nc = use_fused ? std::max(1, kn.cluster) : 1;
  const int64_t narrow_items = use_fused ? kn.narrow_items : 0;
  const size_t kChainSmemMax = static_cast<size_t>(kn.chain_smem_kb) * 1024;
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
  std::vector<RunImg> run_img;
  // sb: base of the device-only scratch section (buffers the kernels write:
  // enumeration block results, cost terms, stamps, chain path tables), not uploaded
  auto make_image = [&](unsigned char *db, unsigned char *sb) {
    Image im;
    im.pk.bytes.reserve(ctx->last_image_bytes + 4096);
    // result slots first, contiguous: indices[nl] | digits[K] | final_cost |
    // cost | min-plus cap overflow flag
    im.oRes = im.pk.put(std::vector<int32_t>(static_cast<size_t>(t.nl) + static_cast<size_t>(K) + 2));
    im.oIdx = im.oRes;
    im.oFC = im.pk.put(std::vector<double>(2));
    im.oOvf = im.pk.put(std::vector<int32_t>(4));
    // row-sharded: every rank's plan memory base (filled before upload: IPC-mapped peers, or the virtual ranks')
    im.oPeer = shard ? im.pk.put(std::vector<uint64_t>(static_cast<size_t>(NR))) : 0;
    im.res_bytes = im.oOvf + 16 - im.oRes;
    auto ovf_ptr = [&] { return reinterpret_cast<uint32_t *>(db + off_image + im.oOvf); };
    auto scr = [&](size_t bytes) {
      const size_t off = im.scratch;
      im.scratch = off + align256(bytes);
      return off;
    };
    auto tabp = [&](int id) -> const T * {
      if (id < t.ne) {
        const T *ox = bp ? reinterpret_cast<const T *>(db + off_tables + 3 * align256(static_cast<size_t>(t.ncells) * 8))
                         : (t.mode == kFP64 ? reinterpret_cast<const T *>(t.xfer64.p)
                                            : reinterpret_cast<const T *>(t.xfer32.p));
        return ox + t.xoff[static_cast<size_t>(id)];
      }
      return reinterpret_cast<const T *>(db + off_derived + tab_off[static_cast<size_t>(id)]);
    };
    const T *onode = bp ? reinterpret_cast<const T *>(db + off_tables)
                        : (t.mode == kFP64 ? reinterpret_cast<const T *>(t.node.p)
                                           : reinterpret_cast<const T *>(t.node32.p));
    // this rank's first row of a table (original tables are replicated in full)
    auto rowp = [&](int id) -> const T * {
      return id < t.ne && shard ? tabp(id) + static_cast<int64_t>(lr0(id)) * cols[static_cast<size_t>(id)] : tabp(id);
    };
    auto gatp = [&](int id) -> T * { return reinterpret_cast<T *>(db + off_gat + gat_off[static_cast<size_t>(id)]); };
    auto t2p = [&](int id) -> const T * { return shard && id >= t.ne ? gatp(id) : tabp(id); };
    auto amp = [&](int oi) { return reinterpret_cast<uint16_t *>(db + off_am + am_off[static_cast<size_t>(oi)]); };
    std::vector<FoldDesc<T>> folds;
    struct FoldOps {
      int e1, e2, ne, wave, oi;
    };
    std::vector<FoldOps> fold_ops;
    std::vector<MergeDesc<T>> merges;
    std::vector<MpFold> mpf;
    std::vector<Mp64Fold> m64;
    std::vector<MpMerge> mmv;
    run_img.clear();
    int64_t colmin_blocks = 0, rowmin_blocks = 0; // mp_minima blocks over all large folds (one launch per plan)
    for (int w = 1; w <= EWn; ++w) {
      WaveRange wr{folds.size(), merges.size(), 0, 0, 0, 0, 0.0, {}, {}, mmv.size(), 0, 0, {}};
      // a wave whose generic folds cover fewer than 2 x SMs 32x32 tiles uses
      // 16x16 tiles: 4x the blocks, a quarter of the per-tile latency
      int64_t big_tiles = 0;
      for (int x = EWbegin[static_cast<size_t>(w)]; x < EWbegin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = EWexec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        if (op.type || large[static_cast<size_t>(oi)]) continue;
        big_tiles += static_cast<int64_t>((nu_eff(op.e1) + kTile - 1) / kTile) *
                     ((cols[static_cast<size_t>(op.e2)] + kTile - 1) / kTile);
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
          for (int x = EWbegin[static_cast<size_t>(w)]; x < EWbegin[static_cast<size_t>(w) + 1]; ++x) {
            const Op &op = s.ops[static_cast<size_t>(EWexec[static_cast<size_t>(x)])];
            if (op.type || large[static_cast<size_t>(EWexec[static_cast<size_t>(x)])]) continue;
            n += static_cast<int64_t>((nu_eff(op.e1) + R - 1) / R) * ((cols[static_cast<size_t>(op.e2)] + R - 1) / R);
          }
          if (forced ? R == forced : n <= 2 * int64_t(ctx->sms)) {
            panel_mode = mode;
            break;
          }
        }
      }
      for (int x = EWbegin[static_cast<size_t>(w)]; x < EWbegin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = EWexec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        T *out = const_cast<T *>(tabp(out_table[static_cast<size_t>(oi)]));
        if (shard && !op.type && op.e2 >= t.ne)
          wr.gathers.emplace_back(tabp(op.e2), gatp(op.e2),
                                  static_cast<size_t>(blk(op.e2)) * cols[static_cast<size_t>(op.e2)] * sizeof(T));
        if (nu_eff(op.e1) == 0) continue; // no rows of this op on this rank
        if constexpr (std::is_same_v<T, int32_t>) {
          if (large[static_cast<size_t>(oi)] && mp_run_of[static_cast<size_t>(oi)] >= 0) { // chain run member
            const int ri = mp_run_of[static_cast<size_t>(oi)];
            const MpRun &run = mp_runs[static_cast<size_t>(ri)];
            const MpLayout &L = mpl[static_cast<size_t>(oi)];
            unsigned char *pb = db + off_mpp;
            if (oi == run.ops.front()) run_img.push_back(RunImg{mpf.size(), 0, 0, 0.0, run.R, w, 6, nu_eff(op.e1)});
            RunImg &ri_ = run_img.back();
            MpFold f{};
            f.t1 = rowp(op.e1);
            f.t2 = t2p(op.e2);
            f.w = onode + t.cat_off[static_cast<size_t>(op.removed)];
            f.out = out;
            f.am = reinterpret_cast<uint16_t *>(db + off_am + am_off[static_cast<size_t>(oi)]);
            f.cb = reinterpret_cast<uint32_t *>(pb + mp_part + mp_cnt + mp_ra + L.cb);
            f.ra = reinterpret_cast<uint32_t *>(pb + mp_part + mp_cnt + L.ra);
            f.B = reinterpret_cast<uint16_t *>(pb + mp_part + mp_cnt + mp_ra + mp_cb + L.B);
            f.b_cols = kMpChainCols;
            f.nu = nu_eff(op.e1);
            f.nw = t.counts[static_cast<size_t>(op.removed)];
            f.nv = cols[static_cast<size_t>(op.e2)];
            f.tiles_i = f.tiles_k = 1;
            f.nchunks = L.nchunks;
            f.jb = fold_jb[static_cast<size_t>(oi)];
            for (int o2 : run.ops) f.jb = std::min(f.jb, fold_jb[static_cast<size_t>(o2)]); // one JB per run
            f.jb = std::max(f.jb, 5);
            if (fold_opt[static_cast<size_t>(oi)]) {
              f.cap = mp_max_cap(f.jb);
              f.ovf = ovf_ptr();
            } else {
              f.cap = static_cast<int32_t>(fold_m[static_cast<size_t>(oi)] + 1);
            }
            PP_REQUIRE(((2 * int64_t(f.cap)) << f.jb) + (1 << f.jb) - 1 <= 65534, "min-plus operand cap exceeds 16 bits");
            f.cb_ready = op.e2 < t.ne || mp_producer[static_cast<size_t>(op.e2)] >= 0 || mp_merge_out[static_cast<size_t>(op.e2)];
            f.a_batches = 0; // the chain kernel normalises its own rows
            f.b_batches = f.cb_ready ? (f.nchunks + kMpPrepBatch - 1) / kMpPrepBatch : 1;
            f.prep_begin = ri_.prep_blocks;
            ri_.prep_blocks += mp_prep_blocks(f);
            f.colmin_begin = colmin_blocks;
            if (op.e2 < t.ne) colmin_blocks += (f.nv + 31) / 32;
            f.rowmin_begin = rowmin_blocks;
            ri_.jb = f.jb;
            ri_.cells += static_cast<double>(f.nu) * f.nw * f.nv;
            ++ri_.n;
            wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
            mpf.push_back(f);
            continue;
          }
          if (large[static_cast<size_t>(oi)]) {
            const MpLayout &L = mpl[static_cast<size_t>(oi)];
            unsigned char *sb = db + off_mp, *pb = db + off_mpp;
            auto rap = [&](int o) { return reinterpret_cast<uint32_t *>(pb + mp_part + mp_cnt + mpl[static_cast<size_t>(o)].ra); };
            auto cbp = [&](int o) {
              return reinterpret_cast<uint32_t *>(pb + mp_part + mp_cnt + mp_ra + mpl[static_cast<size_t>(o)].cb);
            };
            MpFold f{};
            f.t1 = rowp(op.e1);
            f.t2 = t2p(op.e2);
            f.w = onode + t.cat_off[static_cast<size_t>(op.removed)];
            f.out = out;
            f.am = reinterpret_cast<uint16_t *>(db + off_am + am_off[static_cast<size_t>(oi)]);
            f.ra = rap(oi);
            f.cb = cbp(oi);
            f.A = reinterpret_cast<uint32_t *>(sb + L.A);
            f.B = reinterpret_cast<uint16_t *>(sb + L.B);
            f.part = reinterpret_cast<uint32_t *>(pb);
            f.cnt = reinterpret_cast<uint32_t *>(pb + mp_part + L.cnt);
            const int nxt = mp_consumer[static_cast<size_t>(op.ne)];
            if (nxt >= 0) {
              f.w_next = onode + t.cat_off[static_cast<size_t>(s.ops[static_cast<size_t>(nxt)].removed)];
              f.ra_next = rap(nxt);
            }
            const int nxt2 = mp_consumer2[static_cast<size_t>(op.ne)];
            if (nxt2 >= 0 && !shard) f.cb_next = cbp(nxt2); // row-sharded: a rank sees only its rows
            f.ra_ready = op.e1 < t.ne || mp_producer[static_cast<size_t>(op.e1)] >= 0; // mp_minima / producer
            // original t2: mp_colmin (once per plan); a large fold's or an mp_merge's output: their epilogues
            f.cb_ready = op.e2 < t.ne || (!shard && (mp_producer[static_cast<size_t>(op.e2)] >= 0 ||
                                                     mp_merge_out[static_cast<size_t>(op.e2)]));
            f.nu = nu_eff(op.e1);
            f.nw = t.counts[static_cast<size_t>(op.removed)];
            f.nv = cols[static_cast<size_t>(op.e2)];
            f.tiles_i = L.tiles_i;
            f.tiles_k = L.tiles_k;
            f.nchunks = L.nchunks;
            const int gi = mp_group[static_cast<size_t>(oi)];
            if (static_cast<int>(wr.mg.size()) <= gi) wr.mg.resize(static_cast<size_t>(gi) + 1);
            auto &G = wr.mg[static_cast<size_t>(gi)];
            if (G.np == 0) G.p0 = mpf.size();
            G.jb = wave_group_jb[static_cast<size_t>(s.ops[static_cast<size_t>(oi)].wave)][static_cast<size_t>(gi)];
            f.jb = G.jb;
            // operand cap (minplus.cuh): optimistic = the largest the launch's JB allows, checked on
            // the device; proven = M + 1, which fits the fold's (and so the group's smaller) JB
            if (fold_opt[static_cast<size_t>(oi)]) {
              f.cap = mp_max_cap(f.jb);
              f.ovf = ovf_ptr();
            } else {
              f.cap = static_cast<int32_t>(fold_m[static_cast<size_t>(oi)] + 1);
            }
            PP_REQUIRE(((2 * int64_t(f.cap)) << f.jb) + (1 << f.jb) - 1 <= 65534, "min-plus operand cap exceeds 16 bits");
            const int batches = (f.nchunks + kMpPrepBatch - 1) / kMpPrepBatch;
            f.a_batches = f.ra_ready ? batches : 1;
            f.b_batches = f.cb_ready ? batches : 1;
            f.prep_begin = G.prep_blocks;
            G.prep_blocks += mp_prep_blocks(f);
            f.colmin_begin = colmin_blocks;
            if (op.e2 < t.ne) colmin_blocks += (f.nv + 31) / 32; // original t2 only (derived: producers)
            f.rowmin_begin = rowmin_blocks;
            if (op.e1 < t.ne) rowmin_blocks += (f.nu + 7) / 8;
            f.unit_begin = G.units;
            G.units += static_cast<int64_t>(f.tiles_i) * f.tiles_k * f.nchunks;
            f.tile_begin = G.tiles;
            G.tiles += static_cast<int64_t>(f.tiles_i) * f.tiles_k;
            G.cells += static_cast<double>(f.nu) * f.nw * f.nv;
            mpf.push_back(f);
            ++G.np;
            continue;
          }
        }
        if constexpr (std::is_same_v<T, double>) {
          if (large64[static_cast<size_t>(oi)]) {
            const int gi = mp64_group[static_cast<size_t>(oi)];
            if (static_cast<int>(wr.mg64.size()) <= gi) wr.mg64.resize(static_cast<size_t>(gi) + 1);
            auto &G = wr.mg64[static_cast<size_t>(gi)];
            if (G.np == 0) G.p0 = m64.size();
            Mp64Fold f{};
            f.t1 = rowp(op.e1);
            f.t2 = t2p(op.e2);
            f.w = onode + t.cat_off[static_cast<size_t>(op.removed)];
            f.out = out;
            f.am = amp(oi);
            f.A = reinterpret_cast<double *>(db + off_mp + mp64_off[static_cast<size_t>(oi)][0]);
            f.B = reinterpret_cast<double *>(db + off_mp + mp64_off[static_cast<size_t>(oi)][1]);
            f.nu = nu_eff(op.e1);
            f.nw = t.counts[static_cast<size_t>(op.removed)];
            f.nv = cols[static_cast<size_t>(op.e2)];
            f.tiles_i = (f.nu + kMp64Tile - 1) / kMp64Tile;
            f.tiles_k = (f.nv + kMp64Tile - 1) / kMp64Tile;
            f.nchunks = (f.nw + kMp64Chunk - 1) / kMp64Chunk;
            f.prep_a = (f.nu + 31) / 32;
            f.prep_begin = G.prep_blocks;
            G.prep_blocks += f.prep_a + f.nchunks;
            f.tile_begin = G.tiles;
            G.tiles += static_cast<int64_t>(f.tiles_i) * f.tiles_k;
            G.cells += static_cast<double>(f.nu) * f.nw * f.nv;
            wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
            m64.push_back(f);
            ++G.np;
            continue;
          }
        }
        if (!op.type) {
          FoldDesc<T> f{};
          f.t1 = rowp(op.e1);
          f.t2 = t2p(op.e2);
          f.w = onode + t.cat_off[static_cast<size_t>(op.removed)];
          f.out = out;
          f.am = amp(oi);
          f.nu = nu_eff(op.e1);
          f.nw = t.counts[static_cast<size_t>(op.removed)];
          f.nv = cols[static_cast<size_t>(op.e2)];
          f.small = small_wave ? (f.nw <= kPanel && kn.panel ? panel_mode : 1) : 0;
          const int ts = f.small >= kPanel16 ? panel_side(f.small) : f.small ? kSmallTile : kTile;
          f.late = 0; // set below, once the narrow waves are known
          fold_ops.push_back({op.e1, op.e2, out_table[static_cast<size_t>(oi)], w, oi});
          f.n_epi = static_cast<int32_t>(epi[static_cast<size_t>(oi)].size());
          for (int e = 0; e < f.n_epi; ++e) {
            const auto &ab = epi[static_cast<size_t>(oi)][static_cast<size_t>(e)];
            f.epi[e] = tabp(ab.first);
            f.epi2[e] = ab.second >= 0 ? tabp(ab.second) : nullptr;
          }
          f.tiles_k = (f.nv + ts - 1) / ts;
          f.tile_begin = wr.ftiles;
          wr.cells += static_cast<double>(f.nu) * f.nw * f.nv;
          wr.ftiles += static_cast<int64_t>((f.nu + ts - 1) / ts) * f.tiles_k;
          folds.push_back(f);
          ++wr.nf;
        } else {
          if constexpr (std::is_same_v<T, int32_t>) {
            if (mp_merge_out[static_cast<size_t>(op.ne)]) { // feeds a large fold's t2: with its column minima
              const int nxt2 = mp_consumer2[static_cast<size_t>(op.ne)];
              MpMerge mm{};
              mm.a = rowp(op.e1);
              mm.b = rowp(op.e2);
              mm.out = out;
              mm.cb = reinterpret_cast<uint32_t *>(db + off_mpp + mp_part + mp_cnt + mp_ra +
                                                   mpl[static_cast<size_t>(nxt2)].cb);
              mm.nr = nu_eff(op.e1);
              mm.nc = cols[static_cast<size_t>(op.ne)];
              mm.blk_begin = wr.mm_blocks;
              wr.mm_blocks += static_cast<int64_t>((mm.nc + 31) / 32) * ((mm.nr + kMpMergeRows - 1) / kMpMergeRows);
              wr.cells += static_cast<double>(mm.nr) * mm.nc;
              wr.mm_cells += static_cast<double>(mm.nr) * mm.nc;
              mmv.push_back(mm);
              ++wr.nmm;
              continue;
            }
          }
          MergeDesc<T> m;
          m.a = rowp(op.e1);
          m.b = rowp(op.e2);
          m.out = out;
          m.n = static_cast<int64_t>(nu_eff(op.e1)) * cols[static_cast<size_t>(op.ne)];
          m.blk_begin = wr.mblocks;
          wr.cells += static_cast<double>(m.n);
          wr.mblocks += (m.n + kMergePerBlock - 1) / kMergePerBlock;
          merges.push_back(m);
          ++wr.nm;
        }
      }
      im.waves.push_back(wr);
    }
    // fused kernel: which waves run on the first cluster alone, and which
    // operands of a wave's first item may be staged during the previous wave:
    // those every block has seen through a grid barrier that ended a wave
    // x <= w - 2 (a narrow-to-narrow step ends in a cluster barrier only)
    const int nwv = EWn;
    // chain segments (fused kernel, chain_item): maximal runs of >= 2 waves of
    // folds only, each fold's t2 written before the run and its t1 before the
    // run or by a fold of the run (whose chain it extends)
    struct Segment {
      int ws, we; // waves [ws, we]
      std::vector<ChainDesc> chains;
      std::vector<FoldDesc<T>> cf;
      int64_t items;
      size_t smem = 0;  // dynamic shared memory of its items
      size_t stage = 0; // bytes per staging buffer
    };
    std::vector<Segment> segs;
    std::vector<int> seg_of(static_cast<size_t>(nwv) + 2, -1);
    // chains with unwind path tables: one finish record each
    struct ChainRec {
      int node_off, n;
      const uint16_t *path;
    };
    std::vector<ChainRec> chain_recs;
    std::vector<int> chain_last_op;
    std::vector<int32_t> chain_nodes;
    std::vector<int> chain_of_op(s.ops.size(), -1);
    // a segment has no grid barrier between its waves, so a later wave's
    // output must never reuse a table an earlier chain item still reads:
    // segments need every derived table kept (no liveness reuse)
    if (use_fused && kn.chains && keep_all) {
      auto fits = [&](int w, int ws, size_t limit) {
        const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
        if (wr.nm || wr.nf == 0) return false;
        for (size_t q = wr.f0; q < wr.f0 + static_cast<size_t>(wr.nf); ++q) {
          const FoldOps &o = fold_ops[q];
          if (folds[q].nw > kChainMax || folds[q].nv > kChainMax) return false;
          if (chain_smem_bytes<T>(1, 64, chain_stage_bytes<T>(folds[q].nw, folds[q].nv), false) > limit) return false;
          if (tab_wave[static_cast<size_t>(o.e2)] >= ws) return false;
          for (const auto &ab : epi[static_cast<size_t>(o.oi)]) // absorbed-merge operands: written before the run too
            if (tab_wave[static_cast<size_t>(ab.first)] >= ws || (ab.second >= 0 && tab_wave[static_cast<size_t>(ab.second)] >= ws))
              return false;
          const int p1 = tab_wave[static_cast<size_t>(o.e1)];
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
      // segments whose staging needs more than kChainSmemMax run the kernel at one
      // CTA per SM (slower table build, fewer wave CTAs): only worth it when they
      // remove many more barriers (VGG-16: the whole network is one chain)
      std::vector<std::pair<int, int>> R = ranges(kChainSmemMax);
      size_t limit = kChainSmemMax;
      {
        const size_t big = static_cast<size_t>(kn.chain_smem_big_kb) * 1024;
        const auto R2 = ranges(big);
        if (barriers_saved(R2) - barriers_saved(R) >= kn.chain_big_gain) R = R2, limit = big;
      }
      for (const auto &[w, we] : R) {
        {
          Segment sg{w, we, {}, {}, 0, 0, 0};
          std::vector<int> chain_of_table(static_cast<size_t>(E_total), -1);
          std::vector<std::vector<size_t>> members;
          for (int x = w; x <= we; ++x) {
            const WaveRange &wr = im.waves[static_cast<size_t>(x) - 1];
            for (size_t q = wr.f0; q < wr.f0 + static_cast<size_t>(wr.nf); ++q) {
              const FoldOps &o = fold_ops[q];
              int c = tab_wave[static_cast<size_t>(o.e1)] >= w ? chain_of_table[static_cast<size_t>(o.e1)] : -1;
              if (c < 0) {
                c = static_cast<int>(members.size());
                members.emplace_back();
              }
              members[static_cast<size_t>(c)].push_back(q);
              chain_of_table[static_cast<size_t>(o.ne)] = c;
            }
          }
          int64_t rows_total = 0;
          int max_len = 0;
          size_t stage = 0;
          for (const auto &m : members) {
            rows_total += folds[m.front()].nu;
            max_len = std::max(max_len, static_cast<int>(m.size()));
            for (size_t q : m) stage = std::max(stage, chain_stage_bytes<T>(folds[q].nw, folds[q].nv));
          }
          const int64_t cap = 2 * int64_t(ctx->sms);
          int rows = static_cast<int>(std::clamp<int64_t>((rows_total + cap - 1) / cap, 1, kChainRows));
          // unwind path tables for chains of >= 3 folds, when the argmins fit in shared memory
          bool path = max_len >= 3 && kn.chain_path;
          while (rows > 1 && chain_smem_bytes<T>(rows, max_len, stage, path) > limit) --rows;
          if (path && chain_smem_bytes<T>(rows, max_len, stage, path) > limit) path = false;
          sg.smem = chain_smem_bytes<T>(rows, max_len, stage, path);
          sg.stage = stage;
          for (const auto &m : members) {
            ChainDesc cd{static_cast<int32_t>(sg.cf.size()), static_cast<int32_t>(m.size()), folds[m.front()].nu, rows,
                         sg.items, nullptr};
            for (size_t q : m) sg.cf.push_back(folds[q]);
            sg.items += (cd.nu + rows - 1) / rows;
            if (path && m.size() >= 3) { // path table inside the image (rewritten by every run)
              const FoldDesc<T> &fl = folds[m.back()];
              const size_t off = scr(static_cast<size_t>(cd.nu) * fl.nv * m.size() * sizeof(uint16_t));
              cd.path = reinterpret_cast<uint16_t *>(sb + off);
              ChainRec cr{static_cast<int>(chain_nodes.size()), static_cast<int>(m.size()), cd.path};
              for (size_t q : m) chain_nodes.push_back(s.ops[static_cast<size_t>(fold_ops[q].oi)].removed);
              for (size_t q : m) chain_of_op[static_cast<size_t>(fold_ops[q].oi)] = static_cast<int>(chain_recs.size());
              chain_last_op.push_back(fold_ops[m.back()].oi);
              chain_recs.push_back(cr);
            }
            sg.chains.push_back(cd);
          }
          for (int x = w; x <= we; ++x) seg_of[static_cast<size_t>(x)] = static_cast<int>(segs.size());
          segs.push_back(std::move(sg));
        }
      }
    }
    std::vector<char> narrow(static_cast<size_t>(nwv) + 2, 0), gbar(static_cast<size_t>(nwv) + 2, 1);
    for (int w = 1; w <= nwv; ++w) {
      const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
      narrow[static_cast<size_t>(w)] = seg_of[static_cast<size_t>(w)] < 0 && wr.ftiles + wr.mblocks <= narrow_items;
    }
    for (int w = 1; w < nwv; ++w) // inside a segment no barrier separates the waves
      if (seg_of[static_cast<size_t>(w)] >= 0 && seg_of[static_cast<size_t>(w)] == seg_of[static_cast<size_t>(w) + 1])
        gbar[static_cast<size_t>(w)] = 0;
    for (int w = 1; w < nwv; ++w)
      if (narrow[static_cast<size_t>(w)] && narrow[static_cast<size_t>(w) + 1]) gbar[static_cast<size_t>(w)] = 0;
    std::vector<int> seen(static_cast<size_t>(nwv) + 2, 0); // data of waves <= seen[w] is visible while wave w - 1 runs
    for (int w = 3; w <= nwv; ++w)
      seen[static_cast<size_t>(w)] = gbar[static_cast<size_t>(w) - 2] ? w - 2 : seen[static_cast<size_t>(w) - 1];
    for (size_t q = 0; q < folds.size(); ++q) {
      const FoldOps &o = fold_ops[q];
      const int vis = seen[static_cast<size_t>(o.wave)];
      folds[q].late = (tab_wave[static_cast<size_t>(o.e1)] > vis ? kPanelT1 : 0) |
                      (tab_wave[static_cast<size_t>(o.e2)] > vis || (shard && o.e2 >= t.ne) ? kPanelT2 : 0);
    }
    std::vector<EnumNode> en(static_cast<size_t>(K));
    for (int d = 0; d < K; ++d) {
      const int l = node_layer[static_cast<size_t>(d)];
      en[static_cast<size_t>(d)] = EnumNode{onode + t.cat_off[static_cast<size_t>(l)], t.counts[static_cast<size_t>(l)], 0};
    }
    std::vector<EnumEdge> ee;
    for (int id : s.final_edges) {
      if (shard && id >= t.ne)
        im.final_gathers.emplace_back(tabp(id), gatp(id),
                                      static_cast<size_t>(blk(id)) * cols[static_cast<size_t>(id)] * sizeof(T));
      ee.push_back(EnumEdge{t2p(id), pos[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])],
                            pos[static_cast<size_t>(s.edst[static_cast<size_t>(id)])], cols[static_cast<size_t>(id)], 0});
    }
    if (shard) { // the gathers issued above follow shard.hpp's schedule (pp_shard_layout, host-tested)
      size_t n = im.final_gathers.size();
      for (const auto &w : im.waves) n += w.gathers.size();
      PP_REQUIRE(n == shard_gathers(s, t.ne).size(), "row-sharded plan: all-gather schedule mismatch");
    }
    // row-sharded: argmin tables stay on their ranks; the unwind reads the
    // owner's row through the peer bases (no gather of the argmin tables)
    // unwind records (kernels.cuh finish_block), visited last wave first and
    // grouped by dependency level: a record's endpoints are final nodes
    // (level 0) or removed by records of lower levels, so one group per
    // level (the unwind's critical path) instead of one per wave
    std::vector<UnwindRec> recs;
    std::vector<int> rlevel;
    {
      std::vector<int> lvl(static_cast<size_t>(t.nl), -1);
      for (int d = 0; d < K; ++d) lvl[static_cast<size_t>(node_layer[static_cast<size_t>(d)])] = 0;
      for (int w = EWn; w >= 1; --w) {
        for (int x = EWbegin[static_cast<size_t>(w)]; x < EWbegin[static_cast<size_t>(w) + 1]; ++x) {
          const int oi = EWexec[static_cast<size_t>(x)];
          const Op &op = s.ops[static_cast<size_t>(oi)];
          if (op.type) continue;
          const int ch = chain_of_op[static_cast<size_t>(oi)];
          if (ch >= 0 && chain_last_op[static_cast<size_t>(ch)] != oi) continue; // a chain: at its last fold
          const int lu = lvl[static_cast<size_t>(op.u)], lv = lvl[static_cast<size_t>(op.v)];
          PP_REQUIRE(lu >= 0 && lv >= 0, "unwind: record endpoint not yet assigned");
          const int level = std::max(lu, lv) + 1;
          if (ch < 0) {
            if (shard) // byte offset of the table in every rank's plan memory (identical layouts)
              recs.push_back(UnwindRec{reinterpret_cast<const uint16_t *>(off_am + am_off[static_cast<size_t>(oi)]),
                                       op.removed, op.u, op.v, cols[static_cast<size_t>(op.ne)], 0, blk(op.ne)});
            else
              recs.push_back(UnwindRec{amp(oi), op.removed, op.u, op.v, cols[static_cast<size_t>(op.ne)], 0, 0});
            lvl[static_cast<size_t>(op.removed)] = level;
          } else {
            const ChainRec &cr = chain_recs[static_cast<size_t>(ch)];
            recs.push_back(UnwindRec{cr.path, cr.node_off, op.u, op.v, cols[static_cast<size_t>(op.ne)], cr.n, 0});
            for (int k = 0; k < cr.n; ++k) lvl[static_cast<size_t>(chain_nodes[static_cast<size_t>(cr.node_off + k)])] = level;
          }
          rlevel.push_back(level);
        }
      }
    }
    std::vector<int32_t> groups{0};
    {
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
    Packer &pk = im.pk;
    im.oG = pk.put(groups);
    im.nG = static_cast<int>(groups.size()) - 1;
    im.oT = scr(static_cast<size_t>(t.nl + t.ne) * sizeof(double));
    im.oMP = pk.put(mpf);
    im.oMM = pk.put(mmv);
    im.oM64 = pk.put(m64);
    im.n_mp = static_cast<int>(mpf.size());
    im.colmin_blocks = colmin_blocks;
    im.rowmin_blocks = rowmin_blocks;
    im.oF = pk.put(folds);
    im.oM = pk.put(merges);
    { // per-phase work lists of the fused kernel (pointers into the sections above):
      // one entry per wave, or per chain segment
      std::vector<FusedWave<T>> fw;
      im.phase_work.clear();
      int64_t rot = 0;
      for (int w = 1; w <= nwv;) {
        const WaveRange &wr = im.waves[static_cast<size_t>(w) - 1];
        const int sg = seg_of[static_cast<size_t>(w)];
        if (sg >= 0) {
          const Segment &S = segs[static_cast<size_t>(sg)];
          const size_t oc = pk.put(S.chains), of = pk.put(S.cf);
          FusedWave<T> e{};
          e.items = S.items;
          e.n_chains = static_cast<int32_t>(S.chains.size());
          e.stage = static_cast<int64_t>(S.stage);
          e.chains = reinterpret_cast<const ChainDesc *>(db + off_image + oc);
          e.cfolds = reinterpret_cast<const FoldDesc<T> *>(db + off_image + of);
          fw.push_back(e);
          double cells = 0.0;
          for (int x = S.ws; x <= S.we; ++x) cells += im.waves[static_cast<size_t>(x) - 1].cells;
          im.phase_work.push_back(cells);
          w = S.we + 1;
          continue;
        }
        const int64_t items = wr.ftiles + wr.mblocks;
        FusedWave<T> e{};
        e.folds = reinterpret_cast<const FoldDesc<T> *>(db + off_image + im.oF) + wr.f0;
        e.merges = reinterpret_cast<const MergeDesc<T> *>(db + off_image + im.oM) + wr.m0;
        e.nf = wr.nf, e.nm = wr.nm, e.ftiles = wr.ftiles, e.items = items, e.rot = rot;
        e.narrow = narrow[static_cast<size_t>(w)];
        fw.push_back(e);
        im.phase_work.push_back(wr.cells);
        if (kn.rotate) rot += items;
        ++w;
      }
      im.oFW = pk.put(fw);
      im.n_phases = static_cast<int>(fw.size());
      im.dyn_smem = sizeof(WaveSmem<T>);
      for (const Segment &S : segs) im.dyn_smem = std::max(im.dyn_smem, S.smem);
      im.phase_chain.clear();
      for (const auto &e : fw) im.phase_chain.push_back(e.n_chains > 0);
      im.oST = scr((fw.size() + 4) * sizeof(uint64_t));
      im.oTR = kn.wave_trace ? scr((16 * fw.size() + 16 + 12288) * sizeof(uint64_t)) + 1 : 0; // +1: nonzero flag
    }
    im.oN = pk.put(en);
    im.oE = pk.put(ee);
    im.oR = pk.put(recs);
    im.oCN = pk.put(chain_nodes.empty() ? std::vector<int32_t>{0} : chain_nodes);
    im.oL = pk.put(node_layer);
    im.oCO = pk.put(t.cat_off);
    im.oXO = pk.put(t.xoff);
    im.oS = pk.put(es);
    im.oD = pk.put(ed);
    im.oC = pk.put(t.counts);
    if (bp && !early) {
      im.oLay = pk.put(bp->L);
      im.oEdg = pk.put(bp->E);
      im.oCfg = pk.put(*bp->cfg32);
      im.oRat = pk.put(bp->rates);
      im.oBw = pk.put(bp->bw);
    }
    im.oBV = scr(static_cast<size_t>(nblk) * sizeof(A));
    im.oBI = scr(static_cast<size_t>(nblk) * sizeof(int64_t));
    return im;
  };

  clk.mark("memplan");
  // sizes (pointer values do not change the layout)
  // The image holds absolute device pointers, so it is built against the final
  // base.  One-shot plans reuse the context pool: build against the current
  // pool and rebuild only when the pool has to grow (first calls).
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
  unsigned char *db = P->dbase;
  unsigned char *dimg = db + off_image;
  std::memcpy(P->hbase, im.pk.bytes.data(), im.pk.size());
  P->image_off = off_image;
  P->image_bytes = im.pk.size();
  P->res_off = im.oRes;
  P->res_bytes = im.res_bytes;
  P->off_idx = im.oIdx;
  P->off_cost = im.oFC;
  P->off_ovf = im.oOvf;
  P->off_peer = shard ? im.oPeer : SIZE_MAX;
  P->nranks = NR;

  if (bp) { // tables live in the plan's memory
    t.node.view(db + off_tables, static_cast<size_t>(t.ncells));
    t.compute.view(db + off_tables + align256(static_cast<size_t>(t.ncells) * 8), static_cast<size_t>(t.ncells));
    t.sync.view(db + off_tables + 2 * align256(static_cast<size_t>(t.ncells) * 8), static_cast<size_t>(t.ncells));
    t.xfer64.view(db + off_tables + 3 * align256(static_cast<size_t>(t.ncells) * 8), static_cast<size_t>(t.xcells));
  }

  // ---- launch steps -------------------------------------------------------------
  P->steps.clear();
  P->step_kind.clear();
  P->step_work.clear();
  P->gather_lists.clear();
  int launches = 0;
  // one cooperative kernel for the whole plan when no fold needs the S16x2 path
  // (use_fused / fused_nc are decided before the image is built)
  auto push_gathers = [&](const std::vector<std::tuple<const void *, void *, size_t>> &list) {
    for (size_t g0 = 0; g0 < list.size(); g0 += 256) { // NCCL groups of <= 256 all-gathers
      std::vector<std::tuple<const void *, void *, size_t>> part(list.begin() + static_cast<long>(g0),
                                                                 list.begin() + static_cast<long>(std::min(list.size(), g0 + 256)));
      double bytes = 0.0;
      for (const auto &x : part) bytes += static_cast<double>(std::get<2>(x)) * NR;
      P->steps.push_back([ctx, part](cudaStream_t st) {
        PP_REQUIRE(ctx->comm, "row-sharded plan without a communicator (virtual ranks run through pp_vgroup)");
        group_start();
        for (const auto &x : part) all_gather(ctx, std::get<0>(x), std::get<1>(x), std::get<2>(x), st);
        group_end();
      });
      P->gather_lists.push_back(part); // the k-th collective step (virtual ranks copy these blocks themselves)
      P->step_kind.push_back(15);
      P->step_work.push_back(bytes);
    }
  };
  BuildArgs ba{};
  if (bp && !early) {
    ba.layers = reinterpret_cast<const LayerDev *>(dimg + im.oLay);
    ba.edges = reinterpret_cast<const EdgeDev *>(dimg + im.oEdg);
    ba.cfg = reinterpret_cast<const int32_t *>(dimg + im.oCfg);
    ba.rates = reinterpret_cast<const double *>(dimg + im.oRat);
    ba.bw = reinterpret_cast<const double *>(dimg + im.oBw);
    ba.node = t.node.p, ba.compute = t.compute.p, ba.sync = t.sync.p, ba.xfer = t.xfer64.p;
    ba.ncells = t.ncells;
    ba.nl = t.nl, ba.ne = t.ne, ba.D = bp->D;
    ba.node_blocks = static_cast<int32_t>(bp->node_blocks);
    ba.bw_uniform = bp->bw_uniform;
  }
  // fused plans may build their tables in a separate launch before the DP
  // kernel (PARPLAN_SPLIT_BUILD): the DP kernel then runs without the K1/K2 code
  const bool split_build = use_fused && bp && bp->grid > 0 && !early && kn.split_build;
  if (bp && bp->grid > 0 && (!use_fused || split_build) && !shard) {
    const BuildArgs a = ba;
    const int64_t grid = bp->grid;
    P->steps.push_back([ctx, a, grid](cudaStream_t st) { launch_build(ctx, st, a, grid); });
    P->step_kind.push_back(0);
    P->step_work.push_back(static_cast<double>(t.ncells + t.xcells));
    ++launches;
  } else if (bp && bp->grid > 0 && !use_fused) {
    // row-sharded plan: K1 sharded by edge — rank q builds the xfer tables of
    // the edges whose blocks fall in its 1/NR of the edge blocks (whole edges),
    // K2 (node costs, tiny) on every rank; then every rank's edge range is
    // broadcast over NVLink (in place: the tables sit at offset 0 of every
    // rank's plan memory)
    const int64_t eblocks = bp->grid - bp->node_blocks;
    std::vector<int64_t> eb0(static_cast<size_t>(t.ne));
    for (int e = 0; e < t.ne; ++e) eb0[static_cast<size_t>(e)] = bp->E[static_cast<size_t>(e)].blk_begin;
    const std::vector<int> first = shard_edges(eb0, eblocks, NR);
    auto eblk = [&](int e) { return e < t.ne ? bp->E[static_cast<size_t>(e)].blk_begin : eblocks; };
    BuildArgs a = ba;
    a.edge_block0 = eblk(first[static_cast<size_t>(RK)]);
    const int64_t grid = bp->node_blocks + eblk(first[static_cast<size_t>(RK) + 1]) - a.edge_block0;
    P->steps.push_back([ctx, a, grid](cudaStream_t st) { launch_build(ctx, st, a, grid); });
    P->step_kind.push_back(0);
    P->step_work.push_back(static_cast<double>(t.ncells + t.xcells) / NR);
    ++launches;
    std::vector<std::tuple<const void *, void *, size_t>> ranges;
    double bytes = 0.0;
    for (int q = 0; q < NR; ++q) {
      const int64_t c0 = t.xoff[static_cast<size_t>(first[static_cast<size_t>(q)])];
      const int64_t c1 = t.xoff[static_cast<size_t>(first[static_cast<size_t>(q) + 1])];
      double *p = t.xfer64.p + c0;
      ranges.emplace_back(p, p, static_cast<size_t>(c1 - c0) * 8);
      bytes += static_cast<double>(c1 - c0) * 8;
    }
    P->steps.push_back([ctx, ranges](cudaStream_t st) {
      PP_REQUIRE(ctx->comm, "row-sharded plan without a communicator (virtual ranks run through pp_vgroup)");
      group_start();
      for (int q = 0; q < static_cast<int>(ranges.size()); ++q)
        if (std::get<2>(ranges[static_cast<size_t>(q)]))
          broadcast(ctx, std::get<1>(ranges[static_cast<size_t>(q)]), std::get<2>(ranges[static_cast<size_t>(q)]), q, st);
      group_end();
    });
    P->gather_lists.push_back(ranges); // kind 19: entry q = rank q's range (virtual ranks copy it)
    P->step_kind.push_back(19);
    P->step_work.push_back(bytes);
  }
  if (mp_pbytes) { // large folds: tile counters 0 at rest, row minima 0xFF.. before their producers
    unsigned char *pz = db + off_mpp + mp_part, *ovf = dimg + im.oOvf;
    const size_t nc_ = mp_cnt, nr_ = mp_ra + mp_cb;
    P->steps.push_back([pz, nc_, nr_, ovf](cudaStream_t st) {
      PP_CUDA(cudaMemsetAsync(pz, 0, nc_, st));
      PP_CUDA(cudaMemsetAsync(pz + nc_, 0xFF, nr_, st));
      PP_CUDA(cudaMemsetAsync(ovf, 0, 4, st));
    });
    P->step_kind.push_back(5);
    P->step_work.push_back(static_cast<double>(nc_ + nr_));
    if (im.colmin_blocks + im.rowmin_blocks > 0) {
      const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP);
      const int nmp = im.n_mp;
      const int64_t cbk = im.colmin_blocks, all = im.colmin_blocks + im.rowmin_blocks;
      PP_REQUIRE(all < (int64_t(1) << 31), "too many minima blocks");
      P->steps.push_back([ctx, mf, nmp, cbk, all](cudaStream_t st) {
        mp_minima_kernel<<<static_cast<unsigned>(all), 256, 0, st>>>(mf, nmp, cbk);
        check_launch(ctx);
      });
      P->step_kind.push_back(7);
      P->step_work.push_back(0.0);
      ++launches;
    }
  }
  size_t next_run = 0;
  for (size_t wi = 0; wi < im.waves.size(); ++wi) {
    const auto &wr = im.waves[wi];
    if (use_fused) break;
    if constexpr (std::is_same_v<T, int32_t>) {
      if (next_run < run_img.size() && run_img[next_run].w0 == static_cast<int>(wi) + 1) { // a chain run starts here
        const RunImg rn = run_img[next_run++];
        const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP) + rn.p0;
        const int64_t pb = rn.prep_blocks;
        const int n = rn.n, R = rn.R, jb = rn.jb;
        const int nu = rn.nu;
        const unsigned grid = static_cast<unsigned>((nu + R - 1) / R);
        P->steps.push_back([ctx, mf, n, pb](cudaStream_t st) { // every fold's B'' (and missing column minima)
          mp_prep_kernel<<<static_cast<unsigned>(pb), 256, 0, st>>>(mf, n);
          check_launch(ctx);
        });
        P->step_kind.push_back(6);
        P->step_work.push_back(0.0);
        P->steps.push_back([ctx, mf, n, R, grid, jb](cudaStream_t st) {
          mp_chain_launch(jb, R)<<<grid, kMpThreads, kMpChainSmem, st>>>(mf, n, R);
          check_launch(ctx);
        });
        P->step_kind.push_back(17);
        P->step_work.push_back(rn.cells);
        launches += 2;
      }
    }
    push_gathers(wr.gathers);
    if (wr.nmm > 0) { // merges feeding large folds' t2 (independent of this wave's folds)
      const MpMerge *mm = reinterpret_cast<const MpMerge *>(dimg + im.oMM) + wr.mm0;
      const int nmm = wr.nmm;
      const int64_t mb = wr.mm_blocks;
      PP_REQUIRE(mb < (int64_t(1) << 31), "wave too large");
      P->steps.push_back([ctx, mm, nmm, mb](cudaStream_t st) {
        mp_merge_kernel<<<static_cast<unsigned>(mb), 256, 0, st>>>(mm, nmm);
        check_launch(ctx);
      });
      P->step_kind.push_back(9);
      P->step_work.push_back(wr.mm_cells);
      ++launches;
    }
    for (const auto &grp : wr.mg64) { // large FP64 folds of this wave, per launch group: prep -> tile fold
      const Mp64Fold *mf = reinterpret_cast<const Mp64Fold *>(dimg + im.oM64) + grp.p0;
      const int np = grp.np;
      const int64_t pb = grp.prep_blocks, tiles = grp.tiles;
      PP_REQUIRE(pb < (int64_t(1) << 31) && tiles < (int64_t(1) << 31), "wave too large");
      P->steps.push_back([ctx, mf, np, pb](cudaStream_t st) {
        mp64_prep_kernel<<<static_cast<unsigned>(pb), 256, 0, st>>>(mf, np);
        check_launch(ctx);
      });
      P->step_kind.push_back(6);
      P->step_work.push_back(0.0);
      P->steps.push_back([ctx, mf, np, tiles](cudaStream_t st) {
        mp64_fold_kernel<<<static_cast<unsigned>(tiles), kMp64Threads, kMp64Smem, st>>>(mf, np);
        check_launch(ctx);
      });
      P->step_kind.push_back(18);
      P->step_work.push_back(grp.cells);
      launches += 2;
    }
    for (const auto &grp : wr.mg) { // large fixed-point folds of this wave, per launch group: prep -> stream-K fold
      const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP) + grp.p0;
      const int np = grp.np;
      const int64_t pb = grp.prep_blocks, units = grp.units;
      // wide launches: whole tiles round-robin (no split tiles, operand blocks shared in L2)
      const int64_t dp = grp.tiles >= 4 * int64_t(ctx->sms) ? grp.tiles : 0;
      PP_REQUIRE(pb < (int64_t(1) << 31), "wave too large");
      const unsigned G = static_cast<unsigned>(std::min<int64_t>(units, int64_t(ctx->sms)));
      const int jb = grp.jb;
      // programmatic dependent launches: each kernel of the prep -> fold ->
      // prep ... chain is scheduled while its predecessor drains and waits in
      // griddepcontrol.wait (minplus.cuh) for its results
      P->steps.push_back([ctx, mf, np, pb](cudaStream_t st) {
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(pb));
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PP_CUDA(cudaLaunchKernelEx(&cfg, mp_prep_kernel, mf, np));
        check_launch(ctx);
      });
      P->step_kind.push_back(6);
      P->step_work.push_back(0.0);
      P->steps.push_back([ctx, mf, np, units, G, jb, dp](cudaStream_t st) {
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kMpThreads);
        cfg.dynamicSmemBytes = kMpSmem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PP_CUDA(cudaLaunchKernelEx(&cfg,
                                   jb == 7   ? mp_fold_kernel<7>
                                   : jb == 6 ? mp_fold_kernel<6>
                                   : jb == 5 ? mp_fold_kernel<5>
                                   : jb == 4 ? mp_fold_kernel<4>
                                             : mp_fold_kernel<3>,
                                   mf, np, units, dp));
        check_launch(ctx);
      });
      P->step_kind.push_back(8);
      P->step_work.push_back(grp.cells);
      launches += 2;
    }
    const int64_t grid = wr.ftiles + wr.mblocks;
    if (!grid) continue;
    PP_REQUIRE(grid < (int64_t(1) << 31), "wave too large for one launch");
    const FoldDesc<T> *f = reinterpret_cast<const FoldDesc<T> *>(dimg + im.oF) + wr.f0;
    const MergeDesc<T> *m = reinterpret_cast<const MergeDesc<T> *>(dimg + im.oM) + wr.m0;
    const int nf = wr.nf, nm = wr.nm;
    const int64_t ft = wr.ftiles;
    P->steps.push_back([ctx, f, nf, ft, m, nm, grid](cudaStream_t st) {
      wave_kernel<T><<<static_cast<unsigned>(grid), kFoldThreads, 0, st>>>(f, nf, ft, m, nm);
      check_launch(ctx);
    });
    P->step_kind.push_back(1);
    P->step_work.push_back(wr.cells);
    ++launches;
  }
  push_gathers(im.final_gathers);
  {
    const EnumNode *en = reinterpret_cast<const EnumNode *>(dimg + im.oN);
    const EnumEdge *ee = reinterpret_cast<const EnumEdge *>(dimg + im.oE);
    const int m = static_cast<int>(s.final_edges.size());
    A *bv = reinterpret_cast<A *>(P->sbase + im.oBV);
    int64_t *bi = reinterpret_cast<int64_t *>(P->sbase + im.oBI);
    if (!use_fused) {
      P->steps.push_back([ctx, en, K, ee, m, space, per_thread, bv, bi, nblk](cudaStream_t st) {
        enum_kernel<T><<<nblk, kEnumThreads, 0, st>>>(en, K, ee, m, space, per_thread, bv, bi);
        check_launch(ctx);
      });
      P->step_kind.push_back(2);
      P->step_work.push_back(static_cast<double>(space));
    }
    FinishArgs fa{};
    fa.blk_val = bv;
    fa.blk_idx = bi;
    fa.nblk = nblk;
    P->nblk_dbg = nblk;
    P->ngroups_dbg = im.nG;
    fa.nodes = en;
    fa.k = K;
    fa.node_layer = reinterpret_cast<const int32_t *>(dimg + im.oL);
    fa.indices = reinterpret_cast<int32_t *>(dimg + im.oIdx);
    fa.digits = fa.indices + t.nl;
    fa.final_cost = reinterpret_cast<double *>(dimg + im.oFC);
    fa.cost = fa.final_cost + 1;
    fa.peer = shard ? reinterpret_cast<const unsigned char *const *>(dimg + im.oPeer) : nullptr;
    fa.shift = t.shift;
    fa.recs = reinterpret_cast<const UnwindRec *>(dimg + im.oR);
    fa.chain_nodes = reinterpret_cast<const int32_t *>(dimg + im.oCN);
    fa.n_rec = static_cast<int>(s.node_ops);
    fa.group_begin = reinterpret_cast<const int32_t *>(dimg + im.oG);
    fa.n_groups = im.nG;
    fa.terms = reinterpret_cast<double *>(P->sbase + im.oT);
    fa.nl = t.nl;
    fa.onode = bp ? static_cast<const void *>(t.node.p)
                  : (t.mode == kFP64 ? static_cast<const void *>(t.node.p) : static_cast<const void *>(t.node32.p));
    fa.oxfer = bp ? static_cast<const void *>(t.xfer64.p)
                  : (t.mode == kFP64 ? static_cast<const void *>(t.xfer64.p) : static_cast<const void *>(t.xfer32.p));
    fa.cat_off = reinterpret_cast<const int64_t *>(dimg + im.oCO);
    fa.xoff = reinterpret_cast<const int64_t *>(dimg + im.oXO);
    fa.esrc = reinterpret_cast<const int32_t *>(dimg + im.oS);
    fa.edst = reinterpret_cast<const int32_t *>(dimg + im.oD);
    fa.counts = reinterpret_cast<const int32_t *>(dimg + im.oC);
    fa.ne = t.ne;
    fa.host_res = P->hbase + P->res_off;
    fa.dev_res = dimg + P->res_off;
    fa.res_bytes = (P->res_bytes + 3) & ~size_t(3);
    if (!use_fused) {
      P->steps.push_back([ctx, fa](cudaStream_t st) {
        finish_kernel<T><<<1, kFinishThreads, 0, st>>>(fa);
        check_launch(ctx);
      });
      P->step_kind.push_back(3);
      P->step_work.push_back(0.0);
      launches += 2;
    } else {
      FusedArgs<T> fz{};
      fz.has_build = bp != nullptr && !early && !split_build;
      fz.build = ba;
      fz.xcells = fz.has_build ? t.xcells : 0;
      fz.waves = reinterpret_cast<const FusedWave<T> *>(dimg + im.oFW);
      fz.n_waves = static_cast<int32_t>(im.n_phases);
      fz.en = en, fz.ee = ee, fz.k = K, fz.m = m;
      fz.space = space, fz.per_thread = per_thread;
      fz.blk_val = bv, fz.blk_idx = bi, fz.nblk = nblk;
      fz.fin = fa;
      fz.stamps = reinterpret_cast<uint64_t *>(P->sbase + im.oST);
      fz.stage = kn.stage;
      if (!ctx->gbar.p) { // per context: its launches are ordered on ctx->stream
        ctx->gbar.alloc(64);
        PP_CUDA(cudaMemsetAsync(ctx->gbar.p, 0, ctx->gbar.bytes(), ctx->stream));
      }
      fz.gbar = kn.grid_barrier ? ctx->gbar.p : nullptr;
      fz.build_ctr = kn.build_dynamic ? reinterpret_cast<unsigned long long *>(ctx->gbar.p + 32) : nullptr;
      fz.trace = im.oTR ? reinterpret_cast<uint64_t *>(P->sbase + im.oTR - 1) : nullptr;
      if (fz.trace) fz.fin.trace = fz.trace + 16 * im.n_phases;
      fz.fin.smem_ok = finish_smem_bytes(t.nl, t.ne, K) <= im.dyn_smem;
      P->trace_off = im.oTR;
      P->stamp_off = im.oST;
      P->n_stamps = im.n_phases + 4; // start, tables, waves / segments..., enum, finish
      P->fused_wave_work = im.phase_work;
      P->phase_chain = im.phase_chain;
      clk.mark("steps");
      const size_t dyn = im.dyn_smem;
      void (*const fused_fn)(FusedArgs<T>) = fz.has_build ? dp_fused_kernel<T, true> : dp_fused_kernel<T, false>;
      {
        // grow the dynamic allowance monotonically; keep the shared-memory
        // carveout at what two co-resident blocks need (the rest stays L1,
        // which the table build and the wave folds lean on)
        // function attributes are per device: the allowance only ever grows,
        // tracked per device under a lock (several contexts / threads)
        static std::mutex mu;
        static std::map<int, std::array<size_t, 4>> dev_set; // per (T, with build phase)
        std::lock_guard<std::mutex> lock(mu);
        size_t *dyn_set = dev_set[ctx->device].data();
        const int fi = (sizeof(T) == 8 ? 2 : 0) + (fz.has_build ? 1 : 0);
        if (dyn_set[fi] < dyn) {
          PP_CUDA(cudaFuncSetAttribute(fused_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
          cudaFuncAttributes fa_{};
          PP_CUDA(cudaFuncGetAttributes(&fa_, fused_fn));
          const double need = 2.0 * static_cast<double>(dyn + fa_.sharedSizeBytes + 1024);
          const int pct = std::min(100, static_cast<int>(std::ceil(100.0 * need / (228.0 * 1024))));
          PP_CUDA(cudaFuncSetAttribute(fused_fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
          dyn_set[fi] = dyn;
        }
      }
      int occ = 0;
      PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_fn, kFusedThreads, dyn));
      PP_REQUIRE(occ > 0, "fused plan kernel does not fit on an SM");
      int64_t items = std::max<int64_t>(nblk, 1);
      if (fz.has_build) items = std::max<int64_t>(items, (t.ncells + t.xcells + kFusedThreads - 1) / kFusedThreads);
      for (const auto &wr : im.waves) items = std::max<int64_t>(items, wr.ftiles + wr.mblocks);
      const int per_sm_env = kn.blocks_per_sm;
      const int per_sm = per_sm_env > 0 ? std::min(per_sm_env, occ) : occ;
      // cooperative + cluster launch: the grid is whole clusters, all co-resident
      const int nc = fused_nc;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = static_cast<unsigned>(nc), attr[1].val.clusterDim.y = 1, attr[1].val.clusterDim.z = 1;
      int64_t cap = int64_t(ctx->sms) * per_sm;
      if (nc > 1) {
        PP_CUDA(cudaFuncSetAttribute(fused_fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(static_cast<unsigned>(nc));
        q.blockDim = dim3(kFusedThreads);
        q.attrs = attr;
        q.numAttrs = 2;
        q.dynamicSmemBytes = dyn;
        int clusters = 0;
        PP_CUDA(cudaOccupancyMaxActiveClusters(&clusters, fused_fn, &q));
        PP_REQUIRE(clusters > 0, "fused plan kernel: no co-resident cluster of " + std::to_string(nc));
        cap = std::min<int64_t>(cap, int64_t(clusters) * nc) / nc * nc;
      }
      clk.mark("occupancy");
      const int64_t want = (items + nc - 1) / nc * nc;
      const unsigned grid = static_cast<unsigned>(std::max<int64_t>(nc, std::min<int64_t>(want, cap)));
      fz.nc = nc;
      P->steps.push_back([ctx, fz, grid, attr, dyn, nc, fused_fn](cudaStream_t st) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kFusedThreads);
        cfg.dynamicSmemBytes = dyn;
        cfg.stream = st;
        cfg.attrs = const_cast<cudaLaunchAttribute *>(attr);
        cfg.numAttrs = nc > 1 ? 2 : 1;
        PP_CUDA(cudaLaunchKernelEx(&cfg, fused_fn, fz));
        check_launch(ctx);
      });
      P->step_kind.push_back(10);
      P->step_work.push_back(static_cast<double>(bp ? t.ncells + t.xcells : 0));
      launches += 1;
    }
  }
  // results reach the host by zero-copy stores at the end of the finish phase
  // (FinishArgs::host_res), so no D2H copy node follows
  P->launches_per_run = launches + (early ? 1 : 0);
}

// Row-sharded plans over NCCL: every rank's plan memory base, mapped into this
// process with CUDA IPC (peer memory over NVLink), so the finish phase reads
// each unwind record's argmin row from the rank that owns it instead of
// all-gathering every argmin table (planner.hpp:309-319 needs one entry per
// record).  Plan memory layouts are identical on all ranks up to the argmin
// tables (row blocks are padded to blk rows), so one offset serves every rank.
static void exchange_peers(pp_prepared *P) {
  pp_context *ctx = P->ctx;
  const int NR = P->nranks;
  PP_REQUIRE(!P->transient && P->dmem.p, "row-sharded plans own their memory");
  cudaIpcMemHandle_t mine;
  PP_CUDA(cudaIpcGetMemHandle(&mine, P->dmem.p));
  DBuf<unsigned char> buf(sizeof(mine) * static_cast<size_t>(NR));
  unsigned char *slot = buf.p + sizeof(mine) * static_cast<size_t>(ctx->rank);
  PP_CUDA(cudaMemcpyAsync(slot, &mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
  all_gather(ctx, slot, buf.p, sizeof(mine), ctx->stream); // in place
  std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(NR));
  PP_CUDA(cudaMemcpyAsync(all.data(), buf.p, buf.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<uint64_t> bases(static_cast<size_t>(NR));
  for (int q = 0; q < NR; ++q) {
    if (q == ctx->rank) {
      bases[static_cast<size_t>(q)] = reinterpret_cast<uint64_t>(P->dmem.p);
      continue;
    }
    void *p = nullptr;
    PP_CUDA(cudaIpcOpenMemHandle(&p, all[static_cast<size_t>(q)], cudaIpcMemLazyEnablePeerAccess));
    P->ipc_opened.push_back(p);
    bases[static_cast<size_t>(q)] = reinterpret_cast<uint64_t>(p);
  }
  std::memcpy(P->hbase + P->off_peer, bases.data(), bases.size() * 8);
  P->uploaded = false;
}

static void prepare(pp_prepared *P, const pp_device_desc *dev, int k_bound) {
  P->k_bound = k_bound;
  BuildPlan bp;
  if (dev) {
    P->own_t = std::make_unique<Tables>();
    P->t = P->own_t.get();
    P->t->ctx = P->ctx;
    bp = plan_build(*P->t, *P->g, dev, /*host_configs=*/false);
    bp.rates.assign(dev->compute_rates, dev->compute_rates + dev->count);
    bp.bw.assign(dev->bandwidth, dev->bandwidth + static_cast<size_t>(dev->count) * dev->count);
  }
  PP_REQUIRE(P->t->nl == P->g->nl && P->t->ne == P->g->ne, "tables do not match the graph");
  if (std::getenv("PARPLAN_TRACE") && std::atoi(std::getenv("PARPLAN_TRACE")) >= 2)
    std::fprintf(stderr, "[parplan] plan_build done\n");
  if (P->t->mode == kFP64)
    build_steps<double>(P, dev ? &bp : nullptr, k_bound);
  else
    build_steps<int32_t>(P, dev ? &bp : nullptr, k_bound);
  if (P->nranks > 1 && P->ctx->comm) exchange_peers(P);
}

// captures the plan's device work as one CUDA graph, on a private stream
// (the context stream may be the legacy default stream, which cannot
// capture); the graph is launched on the context stream
static void capture(pp_prepared *P) {
  pp_context *ctx = P->ctx;
  if (P->exec) cudaGraphExecDestroy(P->exec), P->exec = nullptr;
  if (P->graph) cudaGraphDestroy(P->graph), P->graph = nullptr;
  cudaStream_t cap = nullptr;
  PP_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  const int64_t l0 = ctx->launches;
  cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    try {
      for (auto &st : P->steps) st(cap);
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(cap, &dummy);
      cudaStreamDestroy(cap);
      throw;
    }
    e = cudaStreamEndCapture(cap, &P->graph);
  }
  ctx->launches = l0;
  cudaStreamDestroy(cap);
  PP_CUDA(e);
  PP_CUDA(cudaGraphInstantiate(&P->exec, P->graph, 0));
}

static void launch(pp_prepared *P, bool upload);

// An optimistic min-plus operand cap was reached (minplus.cuh): the plan is
// rebuilt with proven caps and run again, so results stay exact.  Only
// fixed-point tables reach the min-plus kernels, and those are given
// (plan_with_tables), so no table build is repeated.
static void rerun_conservative(pp_prepared *P) {
  PP_CUDA(cudaEventSynchronize(P->ctx->ev1));
  if (std::getenv("PARPLAN_TRACE")) std::fprintf(stderr, "[parplan] optimistic operand cap reached: re-planning with proven caps\n");
  P->mp_conservative = true;
  build_steps<int32_t>(P, nullptr, P->k_bound);
  P->uploaded = false;
  if (!P->transient) capture(P);
  launch(P, true);
}

static void launch(pp_prepared *P, bool upload) {
  pp_context *ctx = P->ctx;
  if (P->early_built)
    PP_CUDA(cudaSetDevice(ctx->device)); // ev0 was recorded before the early table build
  else
    ctx->begin();
  if (upload || !P->uploaded) {
    PP_CUDA(cudaMemcpyAsync(P->dbase + P->image_off, P->hbase, P->image_bytes, cudaMemcpyHostToDevice, ctx->stream));
    P->uploaded = true;
  }
  if (P->exec) {
    PP_CUDA(cudaGraphLaunch(P->exec, ctx->stream));
    ctx->launches += P->launches_per_run;
  } else {
    for (auto &st : P->steps) st(ctx->stream);
  }
  PP_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  P->launched = true;
}

static void fetch(pp_prepared *P, int32_t *indices, pp_plan_result *res) {
  PP_REQUIRE(P->launched, "plan was not launched");
  pp_context *ctx = P->ctx;
  PP_CUDA(cudaEventSynchronize(ctx->ev1));
  uint32_t ovf = 0;
  std::memcpy(&ovf, P->hbase + P->off_ovf, 4);
  if (ovf && !P->mp_conservative && P->t->mode != kFP64) {
    rerun_conservative(P);
    PP_CUDA(cudaEventSynchronize(ctx->ev1));
  }
  float ms = 0.f;
  PP_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  const unsigned char *h = P->hbase + P->res_off;
  if (indices) std::memcpy(indices, h, static_cast<size_t>(P->t->nl) * 4);
  double fc[2];
  std::memcpy(fc, P->hbase + P->off_cost, 16);
  if (res) {
    res->cost = fc[1];
    res->final_graph_nodes = P->K;
    res->node_eliminations = P->node_ops;
    res->edge_eliminations = P->edge_ops;
    res->precision = P->t->mode;
    res->waves = P->n_waves;
    res->launches = P->launches_per_run;
    res->device_ms = ms;
    res->h2d_bytes = static_cast<int64_t>(P->image_bytes);
    res->d2h_bytes = static_cast<int64_t>(P->res_bytes);
  }
}

void run_plan(pp_context *ctx, Graph &g, Tables *t, const pp_device_desc *dev, int k_bound, int32_t *indices,
              pp_plan_result *res) {
  static const bool trace = std::getenv("PARPLAN_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  pp_prepared P;
  P.ctx = ctx;
  P.g = &g;
  P.t = t;
  P.transient = ctx->nranks <= 1; // row-sharded plans own their memory (peer-mapped for the unwind)
  PP_CUDA(cudaSetDevice(ctx->device));
  prepare(&P, dev, k_bound);
  const auto t1 = std::chrono::steady_clock::now();
  launch(&P, true);
  const auto t2 = std::chrono::steady_clock::now();
  fetch(&P, indices, res);
  const auto t3 = std::chrono::steady_clock::now();
  if (trace) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "[parplan] plan: prepare %.1f us, launch %.1f us, fetch %.1f us, image %zu B\n", us(t0, t1),
                 us(t1, t2), us(t2, t3), P.image_bytes);
  }
}

} // namespace pp

extern "C" {

pp_status pp_plan_with_tables(pp_context *ctx, const pp_graph *g, pp_tables *t, int32_t k_bound, int32_t *indices,
                              pp_plan_result *res) {
  return guard([&] {
    PP_REQUIRE(ctx && g && t && indices, "pp_plan_with_tables: null argument");
    run_plan(ctx, const_cast<pp_graph *>(g)->impl, &t->impl, nullptr, k_bound, indices, res);
  });
}

pp_status pp_plan(pp_context *ctx, const pp_graph *g, const pp_device_desc *dev, int32_t k_bound, int32_t *indices,
                  pp_plan_result *res) {
  return guard([&] {
    PP_REQUIRE(ctx && g && dev && indices, "pp_plan: null argument");
    run_plan(ctx, const_cast<pp_graph *>(g)->impl, nullptr, dev, k_bound, indices, res);
  });
}

pp_status pp_plan_prepare(pp_context *ctx, const pp_graph *g, const pp_device_desc *dev, pp_tables *t, int32_t k_bound,
                          pp_prepared **out) {
  return guard([&] {
    PP_REQUIRE(ctx && g && out && (dev != nullptr) != (t != nullptr), "pp_plan_prepare: give exactly one of dev, t");
    auto P = std::make_unique<pp_prepared>();
    P->ctx = ctx;
    P->g = &const_cast<pp_graph *>(g)->impl;
    P->t = t ? &t->impl : nullptr;
    P->transient = false;
    PP_CUDA(cudaSetDevice(ctx->device));
    prepare(P.get(), dev, k_bound);
    capture(P.get());
    *out = P.release();
  });
}

pp_status pp_plan_launch(pp_prepared *P, int32_t upload_inputs) {
  return guard([&] {
    PP_REQUIRE(P, "null plan");
    launch(P, upload_inputs != 0);
  });
}

pp_status pp_plan_fetch(pp_prepared *P, int32_t *indices, pp_plan_result *res) {
  return guard([&] {
    PP_REQUIRE(P, "null plan");
    fetch(P, indices, res);
  });
}

pp_status pp_plan_profile(pp_prepared *P, int32_t cap, double *step_ms, int32_t *step_kind, double *step_work,
                          int32_t *n_steps) {
  return guard([&] {
    PP_REQUIRE(P && n_steps, "null argument");
    pp_context *ctx = P->ctx;
    const int n = static_cast<int>(P->steps.size());
    std::vector<cudaEvent_t> ev(static_cast<size_t>(n) + 1);
    for (auto &e : ev) PP_CUDA(cudaEventCreate(&e));
    PP_CUDA(cudaSetDevice(ctx->device));
    if (!P->uploaded) {
      PP_CUDA(cudaMemcpyAsync(P->dbase + P->image_off, P->hbase, P->image_bytes, cudaMemcpyHostToDevice, ctx->stream));
      P->uploaded = true;
    }
    PP_CUDA(cudaEventRecord(ev[0], ctx->stream));
    for (int k = 0; k < n; ++k) {
      P->steps[static_cast<size_t>(k)](ctx->stream);
      PP_CUDA(cudaEventRecord(ev[static_cast<size_t>(k) + 1], ctx->stream));
    }
    PP_CUDA(cudaEventSynchronize(ev.back()));
    std::vector<double> ms_v, work_v;
    std::vector<int32_t> kind_v;
    for (int k = 0; k < n; ++k) {
      float ms = 0.f;
      PP_CUDA(cudaEventElapsedTime(&ms, ev[static_cast<size_t>(k)], ev[static_cast<size_t>(k) + 1]));
      const int kind = P->step_kind[static_cast<size_t>(k)];
      if (kind == 10 && P->n_stamps > 1) { // fused kernel: expand its phases (globaltimer stamps)
        std::vector<uint64_t> st(static_cast<size_t>(P->n_stamps));
        PP_CUDA(cudaMemcpy(st.data(), P->sbase + P->stamp_off, st.size() * 8, cudaMemcpyDeviceToHost));
        const int waves = P->n_stamps - 4;
        if (P->trace_off) {
          std::vector<uint64_t> tr(static_cast<size_t>(16 * waves + 16 + 12288));
          PP_CUDA(cudaMemcpy(tr.data(), P->sbase + P->trace_off - 1, tr.size() * 8, cudaMemcpyDeviceToHost));
          for (int w = 0; w < waves; ++w) {
            const uint64_t *r = &tr[static_cast<size_t>(16 * w)];
            const uint64_t b0 = st[static_cast<size_t>(w) + 1]; // block 0 left the previous barrier
            auto rel = [&](uint64_t x) { return x ? static_cast<double>(static_cast<int64_t>(x - b0)) : -1.0; };
            std::fprintf(stderr,
                         "wave %2d worker start %6.0f tile %6.0f loaded %6.0f scanned %6.0f merged %6.0f stored %6.0f "
                         "arrive %6.0f leave %6.0f ns\n",
                         w, rel(r[0]), rel(r[7]), rel(r[1]), rel(r[5]), rel(r[6]), rel(r[2]), rel(r[3]), rel(r[4]));
          }
          {
            std::vector<double> be, bs, bx;
            for (int b = 0; b < 2048; ++b) {
              const uint64_t x = tr[static_cast<size_t>(16 * waves + 16 + b)];
              const uint64_t y = tr[static_cast<size_t>(16 * waves + 16 + 2048 + b)];
              const uint64_t z = tr[static_cast<size_t>(16 * waves + 16 + 4096 + b)];
              if (x && y && z) be.push_back(static_cast<double>(static_cast<int64_t>(x - st[0]))),
                  bs.push_back(static_cast<double>(static_cast<int64_t>(y - st[0]))),
                  bx.push_back(static_cast<double>(static_cast<int64_t>(z - st[0])));
            }
            if (!be.empty()) {
              std::sort(be.begin(), be.end());
              std::sort(bs.begin(), bs.end());
              std::sort(bx.begin(), bx.end());
              if (std::getenv("PARPLAN_TRACE_BLOCKS")) {
                std::fprintf(stderr, "build arrive by block:");
                for (int b = 0; b < 2048; ++b) {
                  const uint64_t x = tr[static_cast<size_t>(16 * waves + 16 + b)];
                  if (x) std::fprintf(stderr, " %d:%.0f", b, static_cast<double>(static_cast<int64_t>(x - st[0])));
                }
                std::fprintf(stderr, "\n");
              }
              { // hand-rolled barrier internals (PARPLAN_GRID_BARRIER=1).  "arrived" is warp 0 past the
                // block barrier, which defers blocking: the block's last warp may still be working
                std::vector<std::array<double, 5>> q;
                for (int b = 0; b < 2048; ++b) {
                  const uint64_t f = tr[static_cast<size_t>(16 * waves + 16 + 6144 + b)];
                  const uint64_t a = tr[static_cast<size_t>(16 * waves + 16 + 8192 + b)];
                  const uint64_t e = tr[static_cast<size_t>(16 * waves + 16 + 10240 + b)];
                  const uint64_t x = tr[static_cast<size_t>(16 * waves + 16 + b)];
                  if (f && a && e && x)
                    q.push_back({static_cast<double>(static_cast<int64_t>(x - st[0])),
                                 static_cast<double>(static_cast<int64_t>(f - st[0])),
                                 static_cast<double>(static_cast<int64_t>(a - st[0])),
                                 static_cast<double>(static_cast<int64_t>(e - st[0])), static_cast<double>(b)});
                }
                if (!q.empty()) {
                  std::sort(q.begin(), q.end(), [](const auto &x, const auto &y) { return x[2] < y[2]; });
                  std::fprintf(stderr, "barrier by atomic time (block: arrived/fenced/atomic returned/released):");
                  for (size_t i = 0; i < q.size(); ++i)
                    if (i < 4 || i + 12 >= q.size())
                      std::fprintf(stderr, " %.0f:%.0f/%.0f/%.0f/%.0f", q[i][4], q[i][0], q[i][1], q[i][2], q[i][3]);
                  std::fprintf(stderr, "\n");
                }
              }
              std::fprintf(stderr,
                           "build: %zu blocks start min %.0f max %.0f; arrive min %.0f median %.0f p90 %.0f max %.0f; "
                           "leave min %.0f max %.0f ns (phase %.0f)\n",
                           be.size(), bs.front(), bs.back(), be.front(), be[be.size() / 2], be[be.size() * 9 / 10], be.back(),
                           bx.front(), bx.back(), static_cast<double>(st[1] - st[0]));
            }
          }
          const uint64_t *fr = &tr[static_cast<size_t>(16 * waves)];
          std::fprintf(stderr, "finish: reduce %.0f unwind %.0f resum %.0f results %.0f ns (stage %.0f blk %.0f sync %.0f; nblk %d, unwind groups %d)\n",
                       static_cast<double>(fr[1] - fr[0]), static_cast<double>(fr[2] - fr[1]),
                       static_cast<double>(fr[3] - fr[2]), static_cast<double>(fr[4] - fr[3]),
                       static_cast<double>(fr[5] - fr[0]), static_cast<double>(fr[6] - fr[5]),
                       static_cast<double>(fr[7] - fr[6]), P->nblk_dbg, P->ngroups_dbg);
        }
        for (int ph = 0; ph + 1 < P->n_stamps; ++ph) {
          const int pk = ph == 0       ? 11
                         : ph <= waves ? (P->phase_chain[static_cast<size_t>(ph) - 1] ? 16 : 12)
                         : ph == waves + 1 ? 13
                                           : 14;
          kind_v.push_back(pk);
          ms_v.push_back(static_cast<double>(st[static_cast<size_t>(ph) + 1] - st[static_cast<size_t>(ph)]) * 1e-6);
          work_v.push_back(pk == 11 ? P->step_work[static_cast<size_t>(k)]
                                    : pk == 12 || pk == 16 ? P->fused_wave_work[static_cast<size_t>(ph - 1)] : 0.0);
        }
        kind_v.push_back(10); // launch + residual (kernel time not covered by phases)
        double covered = 0.0;
        for (size_t q = ms_v.size() - static_cast<size_t>(P->n_stamps - 1); q < ms_v.size(); ++q) covered += ms_v[q];
        ms_v.push_back(std::max(0.0, ms - covered));
        work_v.push_back(0.0);
        continue;
      }
      kind_v.push_back(kind);
      ms_v.push_back(ms);
      work_v.push_back(P->step_work[static_cast<size_t>(k)]);
    }
    *n_steps = static_cast<int32_t>(kind_v.size());
    for (size_t k = 0; k < kind_v.size() && static_cast<int>(k) < cap && step_ms; ++k) {
      step_ms[k] = ms_v[k];
      if (step_kind) step_kind[k] = kind_v[k];
      if (step_work) step_work[k] = work_v[k];
    }
    for (auto &e : ev) cudaEventDestroy(e);
  });
}

// ---- virtual ranks: the row-sharded plan on one device ----------------------
// n contexts on one GPU play the n ranks of a row-sharded plan (the multi-GPU
// code path: row blocks, all-gathers of derived t2 at re-association points and
// of the final edges, the distributed unwind through peer bases).  One host
// thread drives the ranks' step lists in lock-step; an all-gather is one
// device-to-device copy per (rank, block) after every rank's preceding steps.
struct pp_vgroup {
  int device = 0, n = 0;
  std::vector<pp_context *> ctx;
  ~pp_vgroup() {
    for (pp_context *c : ctx) pp_context_destroy(c);
  }
};

namespace pp {
static void run_group(std::vector<pp_prepared *> &Ps) {
  const int n = static_cast<int>(Ps.size());
  std::vector<uint64_t> bases(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) bases[static_cast<size_t>(r)] = reinterpret_cast<uint64_t>(Ps[static_cast<size_t>(r)]->dmem.p);
  std::vector<cudaEvent_t> ev(static_cast<size_t>(n));
  for (auto &e : ev) PP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int r = 0; r < n; ++r) {
    pp_prepared &P = *Ps[static_cast<size_t>(r)];
    std::memcpy(P.hbase + P.off_peer, bases.data(), bases.size() * 8);
    P.ctx->begin();
    PP_CUDA(cudaMemcpyAsync(P.dbase + P.image_off, P.hbase, P.image_bytes, cudaMemcpyHostToDevice, P.ctx->stream));
    P.uploaded = true;
  }
  std::vector<size_t> pos(static_cast<size_t>(n), 0);
  for (size_t k = 0;; ++k) {
    int at_gather = 0;
    for (int r = 0; r < n; ++r) {
      pp_prepared &P = *Ps[static_cast<size_t>(r)];
      size_t &i = pos[static_cast<size_t>(r)];
      while (i < P.steps.size() && P.step_kind[i] != 15 && P.step_kind[i] != 19) P.steps[i++](P.ctx->stream);
      PP_CUDA(cudaEventRecord(ev[static_cast<size_t>(r)], P.ctx->stream));
      at_gather += i < P.steps.size();
    }
    if (at_gather == 0) break;
    PP_REQUIRE(at_gather == n, "virtual ranks disagree on the all-gather schedule");
    for (int r = 0; r < n; ++r) {
      pp_prepared &P = *Ps[static_cast<size_t>(r)];
      for (int q = 0; q < n; ++q)
        if (q != r) PP_CUDA(cudaStreamWaitEvent(P.ctx->stream, ev[static_cast<size_t>(q)], 0));
      const auto &mine = P.gather_lists[k];
      if (P.step_kind[pos[static_cast<size_t>(r)]] == 19) { // edge-range broadcast: rank q's range from rank q
        for (int q = 0; q < n; ++q) {
          if (q == r || !std::get<2>(mine[static_cast<size_t>(q)])) continue;
          const auto &theirs = Ps[static_cast<size_t>(q)]->gather_lists[k][static_cast<size_t>(q)];
          PP_CUDA(cudaMemcpyAsync(std::get<1>(mine[static_cast<size_t>(q)]), std::get<0>(theirs), std::get<2>(theirs),
                                  cudaMemcpyDeviceToDevice, P.ctx->stream));
        }
        ++pos[static_cast<size_t>(r)];
        continue;
      }
      for (size_t j = 0; j < mine.size(); ++j) {
        const size_t bytes = std::get<2>(mine[j]);
        unsigned char *recv = static_cast<unsigned char *>(std::get<1>(mine[j]));
        for (int q = 0; q < n; ++q) {
          const auto &theirs = Ps[static_cast<size_t>(q)]->gather_lists[k];
          PP_REQUIRE(theirs.size() == mine.size() && std::get<2>(theirs[j]) == bytes, "all-gather blocks differ");
          PP_CUDA(cudaMemcpyAsync(recv + static_cast<size_t>(q) * bytes, std::get<0>(theirs[j]), bytes,
                                  cudaMemcpyDeviceToDevice, P.ctx->stream));
        }
      }
      ++pos[static_cast<size_t>(r)];
    }
    // the sends of this gather are read by every rank's copies: a rank may not
    // overwrite them (later waves) before those copies ran
    for (int r = 0; r < n; ++r) PP_CUDA(cudaEventRecord(ev[static_cast<size_t>(r)], Ps[static_cast<size_t>(r)]->ctx->stream));
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q)
        if (q != r) PP_CUDA(cudaStreamWaitEvent(Ps[static_cast<size_t>(r)]->ctx->stream, ev[static_cast<size_t>(q)], 0));
  }
  // the finish phase of each rank reads the other ranks' argmin tables
  for (int r = 0; r < n; ++r) {
    pp_prepared &P = *Ps[static_cast<size_t>(r)];
    PP_CUDA(cudaEventRecord(P.ctx->ev1, P.ctx->stream));
    P.launched = true;
  }
  for (auto &e : ev) cudaEventDestroy(e);
}
} // namespace pp

pp_status pp_vgroup_create(int32_t device, int32_t nranks, pp_vgroup **out) {
  return guard([&] {
    PP_REQUIRE(out && nranks >= 1 && nranks <= 64, "pp_vgroup_create: 1..64 ranks");
    auto g = std::make_unique<pp_vgroup>();
    g->device = device;
    g->n = nranks;
    for (int r = 0; r < nranks; ++r) {
      pp_context *c = nullptr;
      const pp_status st = pp_context_create(device, &c);
      if (st != PP_OK) fail(st, pp_last_error());
      c->nranks = nranks;
      c->rank = r;
      g->ctx.push_back(c);
    }
    *out = g.release();
  });
}

pp_status pp_vgroup_destroy(pp_vgroup *g) {
  delete g;
  return PP_OK;
}

pp_status pp_vgroup_plan(pp_vgroup *grp, const pp_graph *g, const pp_device_desc *dev, pp_tables *t, int32_t k_bound,
                         int32_t *indices, pp_plan_result *res) {
  return guard([&] {
    PP_REQUIRE(grp && g && indices && (dev != nullptr) != (t != nullptr), "pp_vgroup_plan: give exactly one of dev, t");
    std::vector<std::unique_ptr<pp_prepared>> own;
    std::vector<pp_prepared *> Ps;
    for (pp_context *c : grp->ctx) {
      auto P = std::make_unique<pp_prepared>();
      P->ctx = c;
      P->g = &const_cast<pp_graph *>(g)->impl;
      P->t = t ? &t->impl : nullptr;
      P->transient = false;
      PP_CUDA(cudaSetDevice(c->device));
      prepare(P.get(), dev, k_bound);
      Ps.push_back(P.get());
      own.push_back(std::move(P));
    }
    run_group(Ps);
    fetch(Ps[0], indices, res);
    for (size_t r = 1; r < Ps.size(); ++r) { // every rank unwinds the same plan
      std::vector<int32_t> mine(static_cast<size_t>(g->impl.nl));
      fetch(Ps[r], mine.data(), nullptr);
      PP_REQUIRE(std::equal(mine.begin(), mine.end(), indices), "virtual ranks returned different plans");
    }
  });
}

pp_status pp_plan_destroy(pp_prepared *P) {
  if (P && P->ctx) {
    cudaSetDevice(P->ctx->device);
    cudaStreamSynchronize(P->ctx->stream);
  }
  delete P;
  return PP_OK;
}

} // extern "C"
