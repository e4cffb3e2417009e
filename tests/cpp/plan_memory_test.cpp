// Host-only checks of the prepared plan's layout stages (csrc/plan_memory.hpp),
// on random series-parallel schedules from the symbolic scheduler.  Built and
// run by tests/test_plan_layout.py (g++, no GPU):
//
//   MemoryPlan   derived tables never share memory while both are live (also
//                under liveness reuse, forced by > 4 GiB of derived tables);
//                argmin slots are disjoint; row blocks cover every row once;
//                sharded plans have a gather target for every derived t2 of a
//                fold and every derived final edge
//   EffectiveSchedule  every surviving op's operands are written in an earlier
//                effective wave; every merge is done exactly once (absorbed
//                into one fold's epilogue, or kept); waves never increase
#include "plan_memory.hpp"
#include "scheduler.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using namespace pp;

static int failures = 0;
#define CHECK(cond, ...)                                                                                               \
  do {                                                                                                                 \
    if (!(cond)) {                                                                                                     \
      ++failures;                                                                                                      \
      std::fprintf(stderr, "FAIL %s:%d %s: ", __FILE__, __LINE__, #cond);                                              \
      std::fprintf(stderr, __VA_ARGS__);                                                                               \
      std::fprintf(stderr, "\n");                                                                                      \
    }                                                                                                                  \
  } while (0)

// a chain of nodes with random diamonds (u -> a -> v, u -> b -> v) and
// parallel shortcut edges, layers numbered in topological order
static void random_graph(std::mt19937_64 &rng, int n, std::vector<int> &es, std::vector<int> &ed, int &layers) {
  es.clear(), ed.clear();
  int cur = 0;
  layers = 1;
  for (int i = 0; i < n; ++i) {
    const int kind = static_cast<int>(rng() % 10);
    if (kind < 3) { // diamond
      const int a = layers++, b = layers++, v = layers++;
      es.insert(es.end(), {cur, cur, a, b}), ed.insert(ed.end(), {a, b, v, v});
      cur = v;
    } else if (kind < 4 && cur > 0) { // parallel edge to a fresh node
      const int v = layers++;
      es.insert(es.end(), {cur, cur}), ed.insert(ed.end(), {v, v});
      cur = v;
    } else {
      const int v = layers++;
      es.push_back(cur), ed.push_back(v);
      cur = v;
    }
  }
}

int main(int argc, char **argv) {
  const int seeds = argc > 1 ? std::atoi(argv[1]) : 200;
  int checked = 0;
  for (int seed = 0; seed < seeds; ++seed) {
    std::mt19937_64 rng(static_cast<uint64_t>(seed) * 7919u + 1u);
    std::vector<int> es, ed;
    int nl = 0;
    random_graph(rng, 5 + static_cast<int>(rng() % 60), es, ed, nl);
    std::vector<int> rank(static_cast<size_t>(nl));
    for (int l = 0; l < nl; ++l) rank[static_cast<size_t>(l)] = l;
    const Schedule s = build_schedule(nl, es, ed, rank);
    const int ne = static_cast<int>(es.size());
    const int E = static_cast<int>(s.esrc.size());
    // config counts: small, or huge (forces liveness reuse past 4 GiB)
    const bool huge = seed % 3 == 0;
    std::vector<int32_t> counts(static_cast<size_t>(nl));
    for (auto &c : counts) c = huge ? 20000 + static_cast<int32_t>(rng() % 20000) : 1 + static_cast<int32_t>(rng() % 300);
    for (int NR : {1, 3}) {
      for (int RK = 0; RK < NR; ++RK) {
        MemoryPlan m;
        m.build(s, counts, ne, 4, NR, RK);
        ++checked;
        // lifetimes of derived tables: [producing wave, last consuming wave]
        std::vector<int> last(static_cast<size_t>(E), 0);
        for (const Op &op : s.ops)
          for (int in : {op.e1, op.e2}) last[static_cast<size_t>(in)] = std::max(last[static_cast<size_t>(in)], op.wave);
        for (int id : s.final_edges) last[static_cast<size_t>(id)] = s.n_waves + 1;
        for (const Op &a : s.ops)
          for (const Op &b : s.ops) {
            if (a.ne >= b.ne) continue;
            const size_t ba = align256(m.store_cells(a.ne) * 4), bb = align256(m.store_cells(b.ne) * 4);
            const size_t oa = m.tab_off[static_cast<size_t>(a.ne)], ob = m.tab_off[static_cast<size_t>(b.ne)];
            const bool overlap_mem = oa < ob + bb && ob < oa + ba && ba > 0 && bb > 0;
            // live ranges (a table stays until the wave after its last consumer is planned)
            const int a0 = m.prod_wave[static_cast<size_t>(a.ne)], a1 = last[static_cast<size_t>(a.ne)];
            const int b0 = m.prod_wave[static_cast<size_t>(b.ne)], b1 = last[static_cast<size_t>(b.ne)];
            const bool overlap_time = a0 <= b1 && b0 <= a1;
            CHECK(!(overlap_mem && overlap_time), "seed %d NR %d: tables %d [%d,%d] and %d [%d,%d] share memory", seed,
                  NR, a.ne, a0, a1, b.ne, b0, b1);
          }
        if (huge && NR == 1) CHECK(!m.keep_all, "seed %d: > 4 GiB of derived tables but keep_all", seed);
        // argmin slots disjoint
        std::vector<std::pair<size_t, size_t>> am;
        for (size_t oi = 0; oi < s.ops.size(); ++oi)
          if (!s.ops[oi].type) am.emplace_back(m.am_off[oi], align256(m.store_cells(s.ops[oi].ne) * 2));
        std::sort(am.begin(), am.end());
        for (size_t k = 1; k < am.size(); ++k)
          CHECK(am[k - 1].first + am[k - 1].second <= am[k].first, "seed %d: argmin slots overlap", seed);
        // row blocks
        for (int id = 0; id < E; ++id) {
          CHECK(m.lr0(id) + m.lrows(id) <= m.nrows(id), "seed %d: row block past the rows", seed);
          CHECK(m.blk(id) * NR >= m.nrows(id), "seed %d: blocks do not cover the rows", seed);
        }
        if (NR > 1) {
          for (const Op &op : s.ops)
            if (!op.type && op.e2 >= ne)
              CHECK(m.gat_off[static_cast<size_t>(op.e2)] != SIZE_MAX, "seed %d: derived t2 %d has no gather target",
                    seed, op.e2);
          for (int id : s.final_edges)
            if (id >= ne) CHECK(m.gat_off[static_cast<size_t>(id)] != SIZE_MAX, "seed %d: final edge %d not gathered", seed, id);
        }
      }
      if (NR == 1) { // sum of row blocks over ranks
        for (int id = 0; id < E; ++id) {
          int tot = 0;
          for (int RK = 0; RK < 3; ++RK) {
            MemoryPlan m3;
            m3.build(s, counts, ne, 4, 3, RK);
            tot += m3.lrows(id);
          }
          CHECK(tot == counts[static_cast<size_t>(s.esrc[static_cast<size_t>(id)])], "seed %d: row blocks of %d sum to %d",
                seed, id, tot);
        }
      }
    }
    // effective schedule (merge absorption)
    MemoryPlan m;
    m.build(s, counts, ne, 4, 1, 0);
    EffectiveSchedule eff;
    eff.build(s, m.prod_wave, true, 4);
    CHECK(eff.n_waves <= s.n_waves, "seed %d: absorption added waves", seed);
    int absorbed_merges = 0, epi_entries = 0;
    for (size_t oi = 0; oi < s.ops.size(); ++oi) {
      if (s.ops[oi].type && eff.absorbed[oi]) ++absorbed_merges;
      if (!s.ops[oi].type) {
        CHECK(!eff.absorbed[oi], "seed %d: a fold was absorbed", seed);
        for (const auto &ab : eff.epi[oi]) epi_entries += ab.second >= 0 ? 2 : 1;
      }
    }
    // a single epilogue term absorbs one merge, a pair (epi, epi2) two: the
    // merge writing the host's table and the merge of the pair's operands
    CHECK(absorbed_merges == epi_entries, "seed %d: %d absorbed merges vs %d epilogue operands", seed, absorbed_merges,
          epi_entries);
    for (int w = 1; w <= eff.n_waves; ++w)
      for (int x = eff.begin[static_cast<size_t>(w)]; x < eff.begin[static_cast<size_t>(w) + 1]; ++x) {
        const int oi = eff.exec[static_cast<size_t>(x)];
        const Op &op = s.ops[static_cast<size_t>(oi)];
        CHECK(eff.op_wave[static_cast<size_t>(oi)] == w, "seed %d: op %d listed in wave %d", seed, oi, w);
        for (int in : {op.e1, op.e2})
          CHECK(eff.tab_wave[static_cast<size_t>(in)] < w, "seed %d: op %d (wave %d) reads table %d of wave %d", seed, oi,
                w, in, eff.tab_wave[static_cast<size_t>(in)]);
        for (const auto &ab : eff.epi[static_cast<size_t>(oi)]) {
          CHECK(eff.tab_wave[static_cast<size_t>(ab.first)] < w, "seed %d: epilogue operand %d not ready", seed, ab.first);
          if (ab.second >= 0)
            CHECK(eff.tab_wave[static_cast<size_t>(ab.second)] < w, "seed %d: epilogue operand %d not ready", seed,
                  ab.second);
        }
      }
  }
  std::printf("%d layouts checked, %d failures\n", checked, failures);
  return failures ? 1 : 0;
}
