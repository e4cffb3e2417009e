// mp_plan.hpp — the large-fold plan of one prepared plan (plan.cu): which folds
// take the U16x2 min-plus kernels (span certificate, optimistic or proven
// operand caps and JB), the mp_chain runs, the per-wave launch groups and the
// scratch layout; and which FP64 folds take the mp64 kernels.  Pure host
// logic over the symbolic schedule and the tables' span statistics.
#pragma once

#include "minplus.cuh"
#include "minplus64.cuh"
#include "tables.hpp"

#include <algorithm>
#include <array>
#include <functional>
#include <type_traits>
#include <vector>

namespace pp {

inline size_t mp_align256(size_t x) { return (x + 255) & ~size_t(255); }

struct MinplusPlan {
  struct In {
    const Schedule &s;
    const Tables &t;
    const std::vector<int32_t> &rows, &cols; // configs of each table's source / destination node
    std::function<int(int)> nu_eff;          // rows of a table this rank works on
    bool shard;                              // row-sharded plan
    bool conservative;                       // proven caps only (after an optimistic overflow, on request)
    bool no_minplus;                         // kernel policy: generic folds only
    int sms;
    bool chains;                             // mp_chain runs (PARPLAN_MP_CHAIN)
    int chain_min;                           // shortest run worth a chain launch
    const std::vector<int> &prod_wave;       // wave writing each table (0: original)
  };
  struct Layout {
    size_t ra, cb, A, B, cnt; // A, B: per-wave section; cnt, ra, cb: persistent section
    int nchunks, tiles_i, tiles_k;
  };
  struct Run { // mp_chain run: consecutive one-fold waves chained through t1
    int w0 = 0;
    std::vector<int> ops;
    int R = 1;
  };
  // per op
  std::vector<char> large, fold_opt, large64;
  std::vector<int> fold_jb, mp_group, run_of, mp64_group;
  std::vector<int64_t> fold_m; // bound on a fold's minima (cap - 1)
  std::vector<Layout> mpl;
  std::vector<std::array<size_t, 2>> mp64_off; // A, B in the per-wave section
  // per table
  std::vector<int> mp_consumer, mp_consumer2, mp_producer; // large fold reading it as t1 / t2, writing it
  std::vector<char> mp_merge_out;                          // written by an mp_merge
  // per wave: JB of each launch group
  std::vector<std::vector<int>> wave_group_jb;
  std::vector<Run> runs;
  // sections: per-wave operand blocks; persistent = stream-K part slots | tile
  // counters (0 at rest) | ra, cb (0xFF.. before use) | chain B''
  size_t bytes = 0, part = 0, cnt = 0, ra = 0, cb = 0, chainb = 0;
  bool any_opt = false; // some large fold runs with an optimistic cap (the overflow flag matters)
  size_t pbytes() const { return part + cnt + ra + cb + chainb; }

  template <class T> void build(const In &in);
};

template <class T> void MinplusPlan::build(const In &in) {
  const Schedule &s = in.s;
  const Tables &t = in.t;
  const std::vector<int32_t> &rows = in.rows, &cols = in.cols;
  const std::vector<int> &prod_wave = in.prod_wave;
  const auto &nu_eff = in.nu_eff;
  const bool shard = in.shard, conservative = in.conservative;
  const int E_total = static_cast<int>(s.esrc.size());
  const size_t n_ops = s.ops.size();
  large.assign(n_ops, 0), fold_opt.assign(n_ops, 0), large64.assign(n_ops, 0);
  fold_jb.assign(n_ops, 0), mp_group.assign(n_ops, 0), run_of.assign(n_ops, -1), mp64_group.assign(n_ops, 0);
  fold_m.assign(n_ops, 0);
  mpl.assign(n_ops, Layout{});
  mp64_off.assign(n_ops, {0, 0});
  mp_consumer.assign(static_cast<size_t>(E_total), -1), mp_consumer2.assign(static_cast<size_t>(E_total), -1);
  mp_producer.assign(static_cast<size_t>(E_total), -1);
  mp_merge_out.assign(static_cast<size_t>(E_total), 0);
  wave_group_jb.assign(static_cast<size_t>(s.n_waves) + 1, {});
  // Span bounds per table (rows: max over rows of max-min; cols likewise),
  // propagated through the log: fold R(out) <= R(t2), K(out) <= K(t1);
  // merge R = R1 + R2, K = K1 + K2.  The proven cap of a fold is
  // min(rowspan(w + t1), colspan(t2)) + 1 (minplus.cuh).
  if constexpr (std::is_same_v<T, int32_t>) {
    std::vector<int64_t> R(static_cast<size_t>(E_total), 0), Kc(static_cast<size_t>(E_total), 0);
    for (int e = 0; e < t.ne; ++e) {
      R[static_cast<size_t>(e)] = t.row_span[static_cast<size_t>(e)];
      Kc[static_cast<size_t>(e)] = t.col_span[static_cast<size_t>(e)];
    }
    for (size_t oi = 0; oi < s.ops.size(); ++oi) {
      const Op &op = s.ops[oi];
      const size_t a = static_cast<size_t>(op.e1), b2 = static_cast<size_t>(op.e2), o = static_cast<size_t>(op.ne);
      if (op.type) {
        R[o] = R[a] + R[b2];
        Kc[o] = Kc[a] + Kc[b2];
        continue;
      }
      R[o] = R[b2];
      Kc[o] = Kc[a];
      const int nu = rows[a], nw = t.counts[static_cast<size_t>(op.removed)], nv = cols[b2];
      // every minimum <= min(rowspan(w + t1), colspan(t2)) (minplus.cuh: cap)
      fold_m[oi] = std::min(t.node_span[static_cast<size_t>(op.removed)] + R[a], Kc[b2]);
      fold_jb[oi] = fold_m[oi] < 32768 ? mp_jbits(fold_m[oi]) : 0;
      // optimistic JB 6 (cap 511, checked in the epilogue) unless conservative
      if (!conservative) fold_opt[oi] = 1, fold_jb[oi] = nw >= kMpWideNw ? kMpOptJBWide : kMpOptJB;
      large[oi] = nu >= 64 && nv >= 64 && nw >= 64 && fold_jb[oi] > 0 && !in.no_minplus;
      any_opt = any_opt || (large[oi] && fold_opt[oi]);
      if (large[oi] && nu_eff(op.e1) > 0) {
        mp_consumer[a] = static_cast<int>(oi);
        mp_consumer2[b2] = static_cast<int>(oi);
        mp_producer[o] = static_cast<int>(oi);
      }
    }
    for (const Op &op : s.ops) // merges feeding a large fold's t2 run as mp_merge (with its column minima)
      if (op.type && !shard && mp_consumer2[static_cast<size_t>(op.ne)] >= 0) mp_merge_out[static_cast<size_t>(op.ne)] = 1;
    auto take = [&](size_t &at, size_t bytes) {
      const size_t o = at;
      at += mp_align256(bytes);
      return o;
    };
    // chain runs (minplus.cuh: mp_chain): consecutive one-fold waves whose
    // folds chain through t1 and whose t2 exist before the run
    if (!shard && in.chains) {
      Run cur;
      auto close = [&] {
        if (static_cast<int>(cur.ops.size()) >= in.chain_min) runs.push_back(cur);
        cur = Run{};
      };
      for (int w = 1; w <= s.n_waves; ++w) {
        const int x0 = s.wave_begin[static_cast<size_t>(w)], x1 = s.wave_begin[static_cast<size_t>(w) + 1];
        const int oi = s.exec[static_cast<size_t>(x0)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        const bool ok = x1 - x0 == 1 && large[static_cast<size_t>(oi)] && !op.type && fold_jb[static_cast<size_t>(oi)] >= 5 &&
                        cols[static_cast<size_t>(op.e2)] <= kMpChainCols &&
                        t.counts[static_cast<size_t>(op.removed)] <= kMpChainNw &&
                        rows[static_cast<size_t>(op.e1)] <= kMpChainRows * in.sms;
        if (!ok) {
          close();
          continue;
        }
        const bool extends = !cur.ops.empty() && op.e1 == s.ops[static_cast<size_t>(cur.ops.back())].ne &&
                             prod_wave[static_cast<size_t>(op.e2)] < cur.w0;
        if (!extends) {
          close();
          cur.w0 = w;
        }
        cur.ops.push_back(oi);
      }
      close();
      for (size_t r = 0; r < runs.size(); ++r)
        for (int oi : runs[r].ops) {
          run_of[static_cast<size_t>(oi)] = static_cast<int>(r);
          // the run computes its row minima itself and feeds no column minima:
          // consumers of its outputs run their own minima passes
          mp_producer[static_cast<size_t>(s.ops[static_cast<size_t>(oi)].ne)] = -1;
        }
      for (Run &run : runs) {
        run.R = (rows[static_cast<size_t>(s.ops[static_cast<size_t>(run.ops[0])].e1)] + in.sms - 1) / in.sms;
        for (int oi : run.ops) {
          const Op &op = s.ops[static_cast<size_t>(oi)];
          Layout &L = mpl[static_cast<size_t>(oi)];
          L.nchunks = (t.counts[static_cast<size_t>(op.removed)] + kMpChunk - 1) / kMpChunk;
          L.tiles_i = L.tiles_k = 1;
          L.B = take(chainb, static_cast<size_t>(L.nchunks) * kMpChunk * kMpChainCols * 2);
          L.cb = take(cb, static_cast<size_t>(cols[static_cast<size_t>(op.e2)]) * 4);
          L.ra = take(ra, 4);
        }
      }
    }
    // per wave, in launch groups of at most kMpGroupBytes of operand blocks
    // (a wide wave — 471 folds of config 5 — would need 45 GB at C = 4096):
    // the operand blocks and tile counters (restored after every use) of one
    // group are reused by the next group / wave
    constexpr size_t kMpGroupBytes = size_t(2) << 30;
    for (int w = 1; w <= s.n_waves; ++w) {
      size_t off = 0, coff = 0;
      int g = 0;
      wave_group_jb[static_cast<size_t>(w)].assign(1, kMpOptJBWide);
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        if (!large[static_cast<size_t>(oi)] || run_of[static_cast<size_t>(oi)] >= 0) continue;
        const Op &op = s.ops[static_cast<size_t>(oi)];
        Layout &L = mpl[static_cast<size_t>(oi)];
        const int nu = nu_eff(op.e1), nw = t.counts[static_cast<size_t>(op.removed)],
                  nv = cols[static_cast<size_t>(op.e2)];
        if (nu == 0) continue; // no rows of this fold on this rank
        L.tiles_i = (nu + kMpTile - 1) / kMpTile;
        L.tiles_k = (nv + kMpTile - 1) / kMpTile;
        L.nchunks = (nw + kMpChunk - 1) / kMpChunk;
        const size_t need = mp_align256(static_cast<size_t>(L.tiles_i) * L.nchunks * kMpStageA) +
                            mp_align256(static_cast<size_t>(L.tiles_k) * L.nchunks * kMpStageB);
        if (off > 0 && off + need > kMpGroupBytes) { // close the group
          bytes = std::max(bytes, off);
          cnt = std::max(cnt, coff);
          off = coff = 0;
          ++g;
          wave_group_jb[static_cast<size_t>(w)].push_back(kMpOptJBWide);
        }
        mp_group[static_cast<size_t>(oi)] = g;
        int &gjb = wave_group_jb[static_cast<size_t>(w)].back();
        gjb = std::min(gjb, fold_jb[static_cast<size_t>(oi)]);
        L.A = take(off, static_cast<size_t>(L.tiles_i) * L.nchunks * kMpStageA);
        L.B = take(off, static_cast<size_t>(L.tiles_k) * L.nchunks * kMpStageB);
        L.cnt = take(coff, static_cast<size_t>(L.tiles_i) * L.tiles_k * 4);
        L.ra = take(ra, static_cast<size_t>(nu) * 4);
        L.cb = take(cb, static_cast<size_t>(nv) * 4);
      }
      bytes = std::max(bytes, off);
      cnt = std::max(cnt, coff);
    }
    if (bytes) part = static_cast<size_t>(in.sms) * kMpTileCells * 4;
  }
  // ---- large FP64 folds (minplus64.cuh): per wave, launch groups of operand blocks
  if constexpr (std::is_same_v<T, double>) {
    constexpr size_t kGroupBytes = size_t(2) << 30;
    for (int w = 1; w <= s.n_waves; ++w) {
      size_t off = 0;
      int g = 0;
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        if (op.type || in.no_minplus) continue;
        const int nu = nu_eff(op.e1), nw = t.counts[static_cast<size_t>(op.removed)], nv = cols[static_cast<size_t>(op.e2)];
        // below ~512 rows / columns a wave holds too few 64x64 tiles: the generic kernels win
        if (nu < kMp64MinSide || nv < kMp64MinSide || nw < kMp64Chunk * 2) continue;
        large64[static_cast<size_t>(oi)] = 1;
        const int nch = (nw + kMp64Chunk - 1) / kMp64Chunk;
        const size_t a = mp_align256(static_cast<size_t>((nu + kMp64Tile - 1) / kMp64Tile) * nch * kMp64StageA);
        const size_t b = mp_align256(static_cast<size_t>((nv + kMp64Tile - 1) / kMp64Tile) * nch * kMp64StageA);
        if (off > 0 && off + a + b > kGroupBytes) {
          bytes = std::max(bytes, off);
          off = 0;
          ++g;
        }
        mp64_group[static_cast<size_t>(oi)] = g;
        mp64_off[static_cast<size_t>(oi)] = {off, off + a};
        off += a + b;
      }
      bytes = std::max(bytes, off);
    }
  }
}

} // namespace pp
