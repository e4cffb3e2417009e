// plan_steps.cuh — stage 7 of PlanBuilder (plan_builder.cuh): the plan's
// launch list.  Every entry of pp_prepared::steps enqueues one launch (or one
// collective) on a stream; prepared plans capture the list once as a CUDA
// graph (plan.cu capture()).
//
//   fused plans     [K1/K2 build] -> dp_fused_kernel (waves / chain segments,
//                   K5 enumerate, unwind + cost re-sum; zero-copy results)
//   per-wave plans  K1/K2 build (row-sharded: by edge + broadcast) ->
//                   [min-plus counters, mp_minima] -> per wave: [all-gathers]
//                   [mp_prep + mp_chain run] [mp_merge] [mp64 prep + fold]
//                   [mp_prep + mp_fold per launch group] [wave_kernel] ->
//                   [final all-gathers] -> enum_kernel -> finish_kernel
#pragma once

#include "comm.hpp"
#include "plan_builder.cuh"

#include <array>
#include <cmath>
#include <map>
#include <mutex>

namespace pp {

template <class T>
void PlanBuilder<T>::step(int kind, double work, std::function<void(cudaStream_t)> fn, int n_launches) {
  P->steps.push_back(std::move(fn));
  P->step_kind.push_back(kind);
  P->step_work.push_back(work);
  launches += n_launches;
}

// K1/K2 arguments with the descriptors inside the image (not for early builds,
// whose descriptors went up separately)
template <class T> BuildArgs PlanBuilder<T>::build_args(const Image &im) const {
  BuildArgs ba{};
  if (!bp || early) return ba;
  const unsigned char *dimg = db + off_image;
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
  return ba;
}

// The table build as its own launch: per-wave plans, and fused plans with
// split_build (the DP kernel then runs without the K1/K2 code).  Row-sharded
// plans shard K1 by edge: rank q builds the xfer tables of the edges whose
// blocks fall in its 1/NR of the edge blocks (whole edges), K2 (node costs,
// tiny) on every rank; then every rank's edge range is broadcast over NVLink
// (in place: the tables sit at offset 0 of every rank's plan memory).
template <class T> void PlanBuilder<T>::emit_table_build(const BuildArgs &ba, bool split_build) {
  if (!bp || bp->grid <= 0) return;
  pp_context *c = ctx;
  if ((!use_fused || split_build) && !mem.shard) {
    const int64_t grid = bp->grid;
    step(0, static_cast<double>(t.ncells + t.xcells), [c, ba, grid](cudaStream_t st) { launch_build(c, st, ba, grid); }, 1);
    return;
  }
  if (use_fused) return; // built in the fused kernel's first phase
  const int NR = mem.NR, RK = mem.RK;
  const int64_t eblocks = bp->grid - bp->node_blocks;
  std::vector<int64_t> eb0(static_cast<size_t>(t.ne));
  for (int e = 0; e < t.ne; ++e) eb0[static_cast<size_t>(e)] = bp->E[static_cast<size_t>(e)].blk_begin;
  const std::vector<int> first = shard_edges(eb0, eblocks, NR);
  auto eblk = [&](int e) { return e < t.ne ? bp->E[static_cast<size_t>(e)].blk_begin : eblocks; };
  BuildArgs a = ba;
  a.edge_block0 = eblk(first[static_cast<size_t>(RK)]);
  const int64_t grid = bp->node_blocks + eblk(first[static_cast<size_t>(RK) + 1]) - a.edge_block0;
  step(0, static_cast<double>(t.ncells + t.xcells) / NR, [c, a, grid](cudaStream_t st) { launch_build(c, st, a, grid); }, 1);
  CopyList ranges;
  double bytes = 0.0;
  for (int q = 0; q < NR; ++q) {
    const int64_t c0 = t.xoff[static_cast<size_t>(first[static_cast<size_t>(q)])];
    const int64_t c1 = t.xoff[static_cast<size_t>(first[static_cast<size_t>(q) + 1])];
    double *p = t.xfer64.p + c0;
    ranges.emplace_back(p, p, static_cast<size_t>(c1 - c0) * 8);
    bytes += static_cast<double>(c1 - c0) * 8;
  }
  step(19, bytes, [c, ranges](cudaStream_t st) {
    PP_REQUIRE(c->comm, "row-sharded plan without a communicator (virtual ranks run through pp_vgroup)");
    group_start();
    for (int q = 0; q < static_cast<int>(ranges.size()); ++q)
      if (std::get<2>(ranges[static_cast<size_t>(q)]))
        broadcast(c, std::get<1>(ranges[static_cast<size_t>(q)]), std::get<2>(ranges[static_cast<size_t>(q)]), q, st);
    group_end();
  }, 0);
  P->gather_lists.push_back(ranges); // kind 19: entry q = rank q's range (virtual ranks copy it)
}

// large folds: tile counters 0 at rest, row / column minima 0xFF.. before
// their producers; then the minima of the original operands, one launch per plan
template <class T> void PlanBuilder<T>::emit_minima(const Image &im) {
  if (!mp.pbytes()) return;
  pp_context *c = ctx;
  unsigned char *dimg = db + off_image;
  unsigned char *pz = db + off_mpp + mp.part, *ovf = dimg + im.oOvf;
  const size_t nc_ = mp.cnt, nr_ = mp.ra + mp.cb;
  step(5, static_cast<double>(nc_ + nr_), [pz, nc_, nr_, ovf](cudaStream_t st) {
    PP_CUDA(cudaMemsetAsync(pz, 0, nc_, st));
    PP_CUDA(cudaMemsetAsync(pz + nc_, 0xFF, nr_, st));
    PP_CUDA(cudaMemsetAsync(ovf, 0, 4, st));
  }, 0);
  if (im.colmin_blocks + im.rowmin_blocks == 0) return;
  const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP);
  const int nmp = im.n_mp;
  const int64_t cbk = im.colmin_blocks, all = im.colmin_blocks + im.rowmin_blocks;
  PP_REQUIRE(all < (int64_t(1) << 31), "too many minima blocks");
  step(7, 0.0, [c, mf, nmp, cbk, all](cudaStream_t st) {
    mp_minima_kernel<<<static_cast<unsigned>(all), 256, 0, st>>>(mf, nmp, cbk);
    check_launch(c);
  }, 1);
}

// row-sharded all-gathers, NCCL groups of <= 256
template <class T> void PlanBuilder<T>::emit_gathers(const CopyList &list) {
  pp_context *c = ctx;
  const int NR = mem.NR;
  for (size_t g0 = 0; g0 < list.size(); g0 += 256) {
    CopyList part(list.begin() + static_cast<long>(g0), list.begin() + static_cast<long>(std::min(list.size(), g0 + 256)));
    double bytes = 0.0;
    for (const auto &x : part) bytes += static_cast<double>(std::get<2>(x)) * NR;
    step(15, bytes, [c, part](cudaStream_t st) {
      PP_REQUIRE(c->comm, "row-sharded plan without a communicator (virtual ranks run through pp_vgroup)");
      group_start();
      for (const auto &x : part) all_gather(c, std::get<0>(x), std::get<1>(x), std::get<2>(x), st);
      group_end();
    }, 0);
    P->gather_lists.push_back(part); // the k-th collective step (virtual ranks copy these blocks themselves)
  }
}

// programmatic dependent launch: the kernel is scheduled while its
// predecessor drains and waits in griddepcontrol.wait (minplus.cuh)
template <class... Args>
static void launch_pdl(void (*fn)(Args...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PP_CUDA(cudaLaunchKernelEx(&cfg, fn, args...));
}

static void (*mp_fold_fn(int jb))(const MpFold *, int, int64_t, int64_t) {
  return jb == 7 ? mp_fold_kernel<7> : jb == 6 ? mp_fold_kernel<6> : jb == 5 ? mp_fold_kernel<5> : jb == 4 ? mp_fold_kernel<4>
                                                                                                          : mp_fold_kernel<3>;
}

// per-wave plans: the launches of every effective wave
template <class T> void PlanBuilder<T>::emit_waves(const Image &im) {
  if (use_fused) return;
  pp_context *c = ctx;
  unsigned char *dimg = db + off_image;
  size_t next_run = 0;
  for (size_t wi = 0; wi < im.waves.size(); ++wi) {
    const auto &wr = im.waves[wi];
    if constexpr (std::is_same_v<T, int32_t>) {
      if (next_run < run_img.size() && run_img[next_run].w0 == static_cast<int>(wi) + 1) { // a chain run starts here
        const RunImg rn = run_img[next_run++];
        const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP) + rn.p0;
        const int64_t pb = rn.prep_blocks;
        const int n = rn.n, R = rn.R, jb = rn.jb;
        const unsigned grid = static_cast<unsigned>((rn.nu + R - 1) / R);
        step(6, 0.0, [c, mf, n, pb](cudaStream_t st) { // every fold's B'' (and missing column minima)
          mp_prep_kernel<<<static_cast<unsigned>(pb), 256, 0, st>>>(mf, n);
          check_launch(c);
        }, 1);
        step(17, rn.cells, [c, mf, n, R, grid, jb](cudaStream_t st) {
          mp_chain_launch(jb, R)<<<grid, kMpThreads, kMpChainSmem, st>>>(mf, n, R);
          check_launch(c);
        }, 1);
      }
    }
    emit_gathers(wr.gathers);
    if (wr.nmm > 0) { // merges feeding large folds' t2 (independent of this wave's folds)
      const MpMerge *mm = reinterpret_cast<const MpMerge *>(dimg + im.oMM) + wr.mm0;
      const int nmm = wr.nmm;
      const int64_t mb = wr.mm_blocks;
      PP_REQUIRE(mb < (int64_t(1) << 31), "wave too large");
      step(9, wr.mm_cells, [c, mm, nmm, mb](cudaStream_t st) {
        mp_merge_kernel<<<static_cast<unsigned>(mb), 256, 0, st>>>(mm, nmm);
        check_launch(c);
      }, 1);
    }
    for (const auto &grp : wr.mg64) { // large FP64 folds of this wave, per launch group: prep -> tile fold
      const Mp64Fold *mf = reinterpret_cast<const Mp64Fold *>(dimg + im.oM64) + grp.p0;
      const int np = grp.np;
      const int64_t pb = grp.prep_blocks, tiles = grp.tiles;
      PP_REQUIRE(pb < (int64_t(1) << 31) && tiles < (int64_t(1) << 31), "wave too large");
      step(6, 0.0, [c, mf, np, pb](cudaStream_t st) {
        mp64_prep_kernel<<<static_cast<unsigned>(pb), 256, 0, st>>>(mf, np);
        check_launch(c);
      }, 1);
      step(18, grp.cells, [c, mf, np, tiles](cudaStream_t st) {
        mp64_fold_kernel<<<static_cast<unsigned>(tiles), kMp64Threads, kMp64Smem, st>>>(mf, np);
        check_launch(c);
      }, 1);
    }
    for (const auto &grp : wr.mg) { // large fixed-point folds of this wave, per launch group: prep -> stream-K fold
      const MpFold *mf = reinterpret_cast<const MpFold *>(dimg + im.oMP) + grp.p0;
      const int np = grp.np;
      const int64_t pb = grp.prep_blocks, units = grp.units;
      // wide launches: whole tiles round-robin (no split tiles, operand blocks shared in L2)
      const int64_t dp = grp.tiles >= 4 * int64_t(ctx->sms) ? grp.tiles : 0;
      PP_REQUIRE(pb < (int64_t(1) << 31), "wave too large");
      const unsigned G = static_cast<unsigned>(std::min<int64_t>(units, int64_t(ctx->sms)));
      const auto fold = mp_fold_fn(grp.jb);
      // prep -> fold -> prep ... chained by programmatic dependent launches
      step(6, 0.0, [c, mf, np, pb](cudaStream_t st) {
        launch_pdl(mp_prep_kernel, static_cast<unsigned>(pb), 256, 0, st, mf, np);
        check_launch(c);
      }, 1);
      step(8, grp.cells, [c, mf, np, units, G, fold, dp](cudaStream_t st) {
        launch_pdl(fold, G, kMpThreads, kMpSmem, st, mf, np, units, dp);
        check_launch(c);
      }, 1);
    }
    const int64_t grid = wr.ftiles + wr.mblocks;
    if (!grid) continue;
    PP_REQUIRE(grid < (int64_t(1) << 31), "wave too large for one launch");
    const FoldDesc<T> *f = reinterpret_cast<const FoldDesc<T> *>(dimg + im.oF) + wr.f0;
    const MergeDesc<T> *m = reinterpret_cast<const MergeDesc<T> *>(dimg + im.oM) + wr.m0;
    const int nf = wr.nf, nm = wr.nm;
    const int64_t ft = wr.ftiles;
    step(1, wr.cells, [c, f, nf, ft, m, nm, grid](cudaStream_t st) {
      wave_kernel<T><<<static_cast<unsigned>(grid), kFoldThreads, 0, st>>>(f, nf, ft, m, nm);
      check_launch(c);
    }, 1);
  }
}

// finish (unwind + cost re-sum + results) arguments, shared by finish_kernel
// and the fused kernel's last phase
template <class T> FinishArgs PlanBuilder<T>::finish_args(const Image &im) const {
  const unsigned char *dimg = db + off_image;
  FinishArgs fa{};
  fa.blk_val = sb + im.oBV;
  fa.blk_idx = reinterpret_cast<const int64_t *>(sb + im.oBI);
  fa.nblk = nblk;
  fa.nodes = reinterpret_cast<const EnumNode *>(dimg + im.oN);
  fa.k = K;
  fa.node_layer = reinterpret_cast<const int32_t *>(dimg + im.oL);
  fa.indices = reinterpret_cast<int32_t *>(db + off_image + im.oIdx);
  fa.digits = fa.indices + t.nl;
  fa.final_cost = reinterpret_cast<double *>(db + off_image + im.oFC);
  fa.cost = fa.final_cost + 1;
  fa.peer = mem.shard ? reinterpret_cast<const unsigned char *const *>(dimg + im.oPeer) : nullptr;
  fa.shift = t.shift;
  fa.recs = reinterpret_cast<const UnwindRec *>(dimg + im.oR);
  fa.chain_nodes = reinterpret_cast<const int32_t *>(dimg + im.oCN);
  fa.n_rec = static_cast<int>(s.node_ops);
  fa.group_begin = reinterpret_cast<const int32_t *>(dimg + im.oG);
  fa.n_groups = im.nG;
  fa.terms = reinterpret_cast<double *>(sb + im.oT);
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
  fa.dev_res = db + off_image + P->res_off;
  fa.res_bytes = (P->res_bytes + 3) & ~size_t(3);
  return fa;
}

// One cooperative (and optionally clustered) launch for the whole plan.
template <class T>
void PlanBuilder<T>::emit_fused(const Image &im, const BuildArgs &ba, bool split_build, const FinishArgs &fa) {
  pp_context *c = ctx;
  const unsigned char *dimg = db + off_image;
  FusedArgs<T> fz{};
  fz.has_build = bp != nullptr && !early && !split_build;
  fz.build = ba;
  fz.xcells = fz.has_build ? t.xcells : 0;
  fz.waves = reinterpret_cast<const FusedWave<T> *>(dimg + im.oFW);
  fz.n_waves = static_cast<int32_t>(im.n_phases);
  fz.en = fa.nodes, fz.ee = reinterpret_cast<const EnumEdge *>(dimg + im.oE), fz.k = K;
  fz.m = static_cast<int>(s.final_edges.size());
  fz.space = space, fz.per_thread = per_thread;
  fz.blk_val = sb + im.oBV, fz.blk_idx = reinterpret_cast<int64_t *>(sb + im.oBI), fz.nblk = nblk;
  fz.fin = fa;
  fz.stamps = reinterpret_cast<uint64_t *>(sb + im.oST);
  fz.stage = kn.stage;
  if (!ctx->gbar.p) { // per context: its launches are ordered on ctx->stream
    ctx->gbar.alloc(64);
    PP_CUDA(cudaMemsetAsync(ctx->gbar.p, 0, ctx->gbar.bytes(), ctx->stream));
  }
  fz.gbar = kn.grid_barrier ? ctx->gbar.p : nullptr;
  fz.build_ctr = kn.build_dynamic ? reinterpret_cast<unsigned long long *>(ctx->gbar.p + 32) : nullptr;
  fz.trace = im.oTR ? reinterpret_cast<uint64_t *>(sb + im.oTR - 1) : nullptr;
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
    // carveout at what two co-resident blocks need (the rest stays L1, which
    // the table build and the wave folds lean on).  Function attributes are
    // per device: tracked per device under a lock (several contexts / threads)
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
  const int per_sm = kn.blocks_per_sm > 0 ? std::min(kn.blocks_per_sm, occ) : occ;
  // cooperative + cluster launch: the grid is whole clusters, all co-resident
  const int nc = std::max(1, kn.cluster);
  std::array<cudaLaunchAttribute, 2> attr{};
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
    q.attrs = attr.data();
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
  step(10, static_cast<double>(bp ? t.ncells + t.xcells : 0), [c, fz, grid, attr, dyn, nc, fused_fn](cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    auto at = attr;
    cfg.attrs = at.data();
    cfg.numAttrs = nc > 1 ? 2 : 1;
    PP_CUDA(cudaLaunchKernelEx(&cfg, fused_fn, fz));
    check_launch(c);
  }, 1);
}

template <class T> void PlanBuilder<T>::emit_steps(const Image &im) {
  P->steps.clear();
  P->step_kind.clear();
  P->step_work.clear();
  P->gather_lists.clear();
  launches = 0;
  const BuildArgs ba = build_args(im);
  // fused plans may build their tables in a separate launch before the DP
  // kernel (PARPLAN_SPLIT_BUILD): the DP kernel then runs without the K1/K2 code
  const bool split_build = use_fused && bp && bp->grid > 0 && !early && kn.split_build;
  emit_table_build(ba, split_build);
  emit_minima(im);
  emit_waves(im);
  emit_gathers(im.final_gathers);
  if (mem.shard && mp.any_opt) { // every rank sees any rank's optimistic-cap overflow (fetch reruns them all)
    pp_context *c = ctx;
    int32_t *ovf = reinterpret_cast<int32_t *>(db + off_image + im.oOvf);
    step(20, 4.0, [c, ovf](cudaStream_t st) {
      PP_REQUIRE(c->comm, "row-sharded plan without a communicator (virtual ranks run through pp_vgroup)");
      all_reduce_max(c, ovf, 1, st);
    }, 0);
    P->gather_lists.push_back(CopyList{{ovf, ovf, 4}}); // kind 20: the flag word (virtual ranks OR it on the host)
  }
  const FinishArgs fa = finish_args(im);
  P->nblk_dbg = nblk;
  P->ngroups_dbg = im.nG;
  if (use_fused) {
    emit_fused(im, ba, split_build, fa);
  } else {
    pp_context *c = ctx;
    const EnumNode *en = fa.nodes;
    const EnumEdge *ee = reinterpret_cast<const EnumEdge *>(db + off_image + im.oE);
    const int k = K, m = static_cast<int>(s.final_edges.size()), nb = nblk;
    const int64_t sp = space, pt = per_thread;
    A *bv = reinterpret_cast<A *>(sb + im.oBV);
    int64_t *bi = reinterpret_cast<int64_t *>(sb + im.oBI);
    step(2, static_cast<double>(space), [c, en, k, ee, m, sp, pt, bv, bi, nb](cudaStream_t st) {
      enum_kernel<T><<<nb, kEnumThreads, 0, st>>>(en, k, ee, m, sp, pt, bv, bi);
      check_launch(c);
    }, 1);
    step(3, 0.0, [c, fa](cudaStream_t st) {
      finish_kernel<T><<<1, kFinishThreads, 0, st>>>(fa);
      check_launch(c);
    }, 1);
  }
  // results reach the host by zero-copy stores at the end of the finish phase
  // (FinishArgs::host_res), so no D2H copy node follows
  P->launches_per_run = launches + (early ? 1 : 0);
}

} // namespace pp
