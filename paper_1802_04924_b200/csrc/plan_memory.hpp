// plan_memory.hpp — the host-side layout stages of a prepared plan (plan.cu):
//
//   MemoryPlan         shapes of every table (rows = configs of its source
//                      node, cols = of its destination), the row-sharded block
//                      arithmetic (shard.hpp), and a liveness plan for the
//                      derived tables, their argmin tables and the all-gather
//                      targets
//   EffectiveSchedule  the fused kernel's schedule after merge absorption: an
//                      edge elimination (Eq. 3) whose operand comes from a fold
//                      is done in that fold's epilogue, so merge-only waves
//                      disappear and later folds move up
//
// Pure host logic over the symbolic schedule (scheduler.hpp).
#pragma once

#include "scheduler.hpp"
#include "shard.hpp"

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <iterator>
#include <map>
#include <utility>
#include <vector>

namespace pp {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// First-fit offset allocator with coalescing; derived tables are released
// after the wave that consumes them (never reused inside that wave).
class OffsetPlanner {
public:
  size_t alloc(size_t bytes) {
    bytes = align256(bytes);
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
    bytes = align256(bytes);
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

// Row sharding (pp_context_attach_comm): every derived table is split by rows
// into NR blocks of blk rows; rank RK computes and stores rows [RK*blk, ...).
// Original tables are replicated.  A fold needs its t2 in full: a derived t2 is
// all-gathered first (the re-association points), and so are the final edges;
// argmin tables stay on their ranks (the unwind reads them through peer bases).
struct MemoryPlan {
  int E_total = 0, NR = 1, RK = 0;
  bool shard = false;
  std::vector<int32_t> rows, cols; // per table id
  bool keep_all = true;            // no liveness reuse of derived tables (<= 4 GiB)
  std::vector<size_t> tab_off;     // derived table -> offset in the derived section
  std::vector<size_t> am_off;      // fold op -> offset of its argmin table
  std::vector<size_t> gat_off;     // derived table -> all-gather target (SIZE_MAX: none)
  std::vector<int> prod_wave;      // wave writing each table (0: original)
  size_t tab_end = 0, am_bytes = 0, gat_bytes = 0;

  int nrows(int id) const { return rows[static_cast<size_t>(id)]; }
  int ncols(int id) const { return cols[static_cast<size_t>(id)]; }
  int blk(int id) const { return shard_blk(nrows(id), NR); }
  int lr0(int id) const { return shard_first(nrows(id), NR, RK); }
  int lrows(int id) const { return shard_rows(nrows(id), NR, RK); }
  // rows of a fold's t1 / a merge's operands this rank works on
  int nu_eff(int id) const { return shard ? lrows(id) : nrows(id); }
  size_t cells(int id) const { return static_cast<size_t>(nrows(id)) * ncols(id); }
  // storage of a derived table on this rank
  size_t store_cells(int id) const { return shard ? static_cast<size_t>(blk(id)) * ncols(id) : cells(id); }
  // all-gather target (NR padded blocks)
  size_t full_cells(int id) const { return static_cast<size_t>(NR) * blk(id) * ncols(id); }

  // counts: configs per layer; ne: original edges; elem: bytes per table cell
  void build(const Schedule &s, const std::vector<int32_t> &counts, int ne, size_t elem, int nranks, int rank) {
    NR = nranks > 1 ? nranks : 1;
    RK = NR > 1 ? rank : 0;
    shard = NR > 1;
    E_total = static_cast<int>(s.esrc.size());
    rows.assign(static_cast<size_t>(E_total), 0);
    cols.assign(static_cast<size_t>(E_total), 0);
    for (int id = 0; id < E_total; ++id) {
      rows[static_cast<size_t>(id)] = counts[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])];
      cols[static_cast<size_t>(id)] = counts[static_cast<size_t>(s.edst[static_cast<size_t>(id)])];
    }
    size_t derived_total = 0;
    for (const Op &op : s.ops) derived_total += align256(store_cells(op.ne) * elem);
    keep_all = derived_total <= (size_t(4) << 30);
    OffsetPlanner tab_plan;
    tab_off.assign(static_cast<size_t>(E_total), 0);
    am_off.assign(s.ops.size(), 0);
    gat_off.assign(static_cast<size_t>(E_total), SIZE_MAX);
    prod_wave.assign(static_cast<size_t>(E_total), 0);
    am_bytes = gat_bytes = 0;
    for (int w = 1; w <= s.n_waves; ++w) {
      const int x0 = s.wave_begin[static_cast<size_t>(w)], x1 = s.wave_begin[static_cast<size_t>(w) + 1];
      for (int x = x0; x < x1; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        tab_off[static_cast<size_t>(op.ne)] = tab_plan.alloc(store_cells(op.ne) * elem);
        prod_wave[static_cast<size_t>(op.ne)] = w;
        if (op.type) continue;
        am_off[static_cast<size_t>(oi)] = am_bytes;
        am_bytes += align256(store_cells(op.ne) * 2);
        if (shard && op.e2 >= ne) { // derived t2: gathered in full before the fold
          gat_off[static_cast<size_t>(op.e2)] = gat_bytes;
          gat_bytes += align256(full_cells(op.e2) * elem);
        }
      }
      if (!keep_all)
        for (int x = x0; x < x1; ++x) {
          const Op &op = s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])];
          for (int in : {op.e1, op.e2})
            if (in >= ne) tab_plan.release(tab_off[static_cast<size_t>(in)], store_cells(in) * elem);
        }
    }
    if (shard)
      for (int id : s.final_edges)
        if (id >= ne && gat_off[static_cast<size_t>(id)] == SIZE_MAX) {
          gat_off[static_cast<size_t>(id)] = gat_bytes;
          gat_bytes += align256(full_cells(id) * elem);
        }
    tab_end = tab_plan.end();
  }
};

// An edge elimination (Eq. 3, out = a + b) whose operand a comes from a fold F
// (or from merges already absorbed into F) while b is ready before F runs is
// folded into F's epilogue: F writes ((v + b1) + b2)..., one IEEE add per merge
// in the reference's order (a single add is commutative, so which operand F
// produced does not matter).  Needs every derived table kept (no memory reuse
// across the reordered waves).  Without absorption the effective schedule is
// the symbolic one.
struct EffectiveSchedule {
  int n_waves = 0;
  std::vector<int> begin, exec;                       // surviving ops grouped by effective wave
  std::vector<int> out_table, op_wave;                // per op: table it writes last, effective wave
  std::vector<int> tab_wave;                          // per table: effective wave writing it (0: original)
  std::vector<std::vector<std::pair<int, int>>> epi;  // per fold: (table, table or -1) per absorbed merge
  std::vector<char> absorbed;                         // per op: done in a fold's epilogue

  void build(const Schedule &s, const std::vector<int> &prod_wave, bool absorb, size_t max_epi) {
    const int n_ops = static_cast<int>(s.ops.size());
    const int E_total = static_cast<int>(prod_wave.size());
    n_waves = s.n_waves;
    begin.assign(s.wave_begin.begin(), s.wave_begin.end());
    exec.assign(s.exec.begin(), s.exec.end());
    out_table.assign(static_cast<size_t>(n_ops), 0);
    op_wave.assign(static_cast<size_t>(n_ops), 0);
    epi.assign(static_cast<size_t>(n_ops), {});
    absorbed.assign(static_cast<size_t>(n_ops), 0);
    tab_wave = prod_wave;
    for (int oi = 0; oi < n_ops; ++oi) out_table[static_cast<size_t>(oi)] = s.ops[static_cast<size_t>(oi)].ne;
    for (int oi = 0; oi < n_ops; ++oi) op_wave[static_cast<size_t>(oi)] = s.ops[static_cast<size_t>(oi)].wave;
    if (!absorb) return;
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
          if (F < 0 || out_table[static_cast<size_t>(F)] != mine || epi[static_cast<size_t>(F)].size() >= max_epi) continue;
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
    n_waves = 0;
    for (int oi = 0; oi < n_ops; ++oi)
      if (!absorbed[static_cast<size_t>(oi)]) n_waves = std::max(n_waves, op_wave[static_cast<size_t>(oi)]);
    std::vector<std::vector<int>> by(static_cast<size_t>(n_waves) + 1);
    for (int w = 1; w <= s.n_waves; ++w)
      for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = s.exec[static_cast<size_t>(x)];
        if (!absorbed[static_cast<size_t>(oi)]) by[static_cast<size_t>(op_wave[static_cast<size_t>(oi)])].push_back(oi);
      }
    begin.assign(static_cast<size_t>(n_waves) + 2, 0);
    exec.clear();
    for (int w = 1; w <= n_waves; ++w) {
      begin[static_cast<size_t>(w)] = static_cast<int>(exec.size());
      exec.insert(exec.end(), by[static_cast<size_t>(w)].begin(), by[static_cast<size_t>(w)].end());
    }
    begin[static_cast<size_t>(n_waves) + 1] = static_cast<int>(exec.size());
  }
};

} // namespace pp
