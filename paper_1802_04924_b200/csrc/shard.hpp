// shard.hpp — the row-sharded plan's layout arithmetic (plan.cu), shared with
// pp_shard_layout (the C ABI, host-testable without a GPU).
//
// * A derived table of `rows` rows (configs of its source node) is split into
//   NR blocks of blk = ceil(rows / NR) rows; rank RK owns rows
//   [min(rows, RK*blk), min(rows, (RK+1)*blk)).  Storage and all-gathers use
//   the padded block (blk rows per rank), so plan memory layouts are identical
//   on every rank up to the argmin tables (the distributed unwind relies on it).
// * A fold whose t2 is a derived table needs it in full: that table is
//   all-gathered before the fold's wave (the re-association points); the final
//   edges are all-gathered before the enumeration.  Original tables are
//   replicated.
// * K1 is sharded by edge: rank q builds the edges whose first build block lies
//   in [q*EB/NR, (q+1)*EB/NR) of the EB edge blocks (whole edges).
#pragma once

#include "scheduler.hpp"

#include <algorithm>
#include <cstdint>
#include <vector>

namespace pp {

inline int shard_blk(int rows, int NR) { return (rows + NR - 1) / NR; }
inline int shard_first(int rows, int NR, int RK) { return std::min(rows, RK * shard_blk(rows, NR)); }
inline int shard_rows(int rows, int NR, int RK) {
  return std::max(0, std::min(rows, (RK + 1) * shard_blk(rows, NR)) - shard_first(rows, NR, RK));
}

// (wave, table id) of every all-gather, in execution order: derived t2 of folds
// (before the fold's wave), then the derived final edges (wave n_waves + 1)
inline std::vector<std::pair<int, int>> shard_gathers(const Schedule &s, int n_original_edges) {
  std::vector<std::pair<int, int>> out;
  for (int w = 1; w <= s.n_waves; ++w)
    for (int x = s.wave_begin[static_cast<size_t>(w)]; x < s.wave_begin[static_cast<size_t>(w) + 1]; ++x) {
      const Op &op = s.ops[static_cast<size_t>(s.exec[static_cast<size_t>(x)])];
      if (!op.type && op.e2 >= n_original_edges) out.emplace_back(w, op.e2);
    }
  for (int id : s.final_edges)
    if (id >= n_original_edges) out.emplace_back(s.n_waves + 1, id);
  return out;
}

// first edge of every rank's K1 share (NR + 1 entries; the last is ne), from
// the edges' first build blocks (ascending) and the total edge blocks
inline std::vector<int> shard_edges(const std::vector<int64_t> &blk_begin, int64_t eblocks, int NR) {
  const int ne = static_cast<int>(blk_begin.size());
  std::vector<int> first(static_cast<size_t>(NR) + 1, ne);
  for (int q = 0, e = 0; q < NR; ++q) {
    const int64_t want = eblocks * q / NR;
    while (e < ne && blk_begin[static_cast<size_t>(e)] < want) ++e;
    first[static_cast<size_t>(q)] = e;
  }
  return first;
}

} // namespace pp
