// plan_state.hpp — a prepared plan (pp_prepared: its device memory, descriptor
// image, launch steps and CUDA graph) and the tuning knobs read once per
// prepare.  Built by PlanBuilder (plan_builder.cuh, plan_steps.cuh), run by
// plan.cu.
#pragma once

#include "tables.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <tuple>
#include <utility>
#include <vector>

namespace pp {

inline int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Tuning knobs, read once per prepare (A/B experiments in one process).  The
// defaults are the measured best; the settings read from the environment stay
// selectable because the parity tests run every plan shape through them.  The
// plain constants are fixed tuning values (they used to be switches).
struct Knobs {
  // fused kernel
  int cluster = env_int("PARPLAN_CLUSTER", 1);            // thread-block cluster size of the cooperative launch
  int narrow_items = env_int("PARPLAN_NARROW_ITEMS", 0);  // waves <= this many items run on the first cluster alone
  int grid_barrier = env_int("PARPLAN_GRID_BARRIER", 1);  // hand-rolled barrier (0: cooperative-groups grid sync)
  int build_dynamic = env_int("PARPLAN_BUILD_DYNAMIC", 1); // table build blocks claimed from a counter
  int split_build = env_int("PARPLAN_SPLIT_BUILD", 1);    // prepared plans: table build as its own launch
  int early_build = env_int("PARPLAN_EARLY_BUILD", 1);    // one-shot plans: table build launched before the image
  int stage = env_int("PARPLAN_STAGE", 1);                // stage the next wave's operands before the barrier
  int rotate = 1;                                         // rotate item -> block assignment across waves
  int blocks_per_sm = env_int("PARPLAN_FUSED_BLOCKS_PER_SM", 0); // 0: occupancy limit
  int wave_trace = env_int("PARPLAN_WAVE_TRACE", 0);      // per-wave globaltimer stamps (pp_plan_profile prints)
  // generic folds
  int panel = env_int("PARPLAN_PANEL", 1);           // small waves: 4/8-row panel tiles
  int panel_side = 0;                                // forced panel side (0: the smallest that fills the GPU)
  int merge_fuse = env_int("PARPLAN_MERGE_FUSE", 1); // merge absorption into fold epilogues
  // chain segments (fused kernel)
  int chains = env_int("PARPLAN_CHAINS", 1);
  int chain_path = 1;                                // unwind path tables for chains of >= 3 folds
  int chain_min_waves = 2;                           // shortest segment (waves)
  int chain_rows = env_int("PARPLAN_CHAIN_ROWS", 8); // rows per chain item at most (the cost model picks)
  int chain_smem_kb = 110;                           // segment shared memory at two CTAs per SM
  int chain_smem_big_kb = 216;                       // ... at one CTA per SM
  int chain_big_gain = 6;                            // barriers a one-CTA-per-SM segment layout must save
  // large min-plus folds
  int mp_chain = env_int("PARPLAN_MP_CHAIN", 1);                           // mp_chain runs
  int mp_chain_min = 4;                                                    // shortest run worth a chain launch
};

// PARPLAN_TRACE=2: host-side timing of the build stages
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
    std::fprintf(stderr, "[parplan] prepare stages:");
    for (size_t k = 1; k < marks.size(); ++k)
      std::fprintf(stderr, " %s %.1f", marks[k].first,
                   std::chrono::duration<double, std::micro>(marks[k].second - marks[k - 1].second).count());
    std::fprintf(stderr, " us\n");
  }
};

// device-to-device block copies of one collective step: (send, receive, bytes)
using CopyList = std::vector<std::tuple<const void *, void *, size_t>>;

} // namespace pp

struct pp_prepared {
  pp_context *ctx = nullptr;
  pp::Graph *g = nullptr;
  pp::Tables *t = nullptr;
  std::unique_ptr<pp::Tables> own_t;
  bool transient = true;
  pp::DBuf<unsigned char> dmem, dscratch;
  pp::PinnedBuf hmem;
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
  std::vector<pp::CopyList> gather_lists;
  std::vector<void *> ipc_opened;
  // the plan's device work: one entry per launch (or collective), with its
  // profile kind (pp_plan_profile) and work (cells, bytes)
  std::vector<std::function<void(cudaStream_t)>> steps;
  std::vector<int32_t> step_kind;
  std::vector<double> step_work;
  int launches_per_run = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int K = 0, n_waves = 0, node_ops = 0, edge_ops = 0;
  bool launched = false, uploaded = false;
  bool early_built = false; // transient plan: the table build was launched during prepare (ev0 already recorded)
  size_t stamp_off = 0; // fused kernel phase stamps (scratch offset), n_stamps entries
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
