/* parplan/planner.hpp — the elimination planner (Eq. 2, Eq. 3, Algorithm 1).
 *
 * Drop-in for /root/reference/proj/include/parplan/planner.hpp:
 *   NodeElimRecord / EdgeElimRecord / EliminationRecord (:28-45)
 *   ReducedGraph step API (:51-245)
 *   enumerate_final (:251-304), unwind (:306-319)
 *   PlanResult / plan_with_tables / plan (:321-371)
 *
 * Every elimination, enumeration and plan executes in libparplan_cuda.so on
 * the B200: the symbolic scheduler reproduces the reference's elimination
 * order exactly, folds / merges run as device kernels, and results (tables,
 * argmins, indices, costs) are bit-identical to the reference.  ReducedGraph
 * keeps its tables on the device; edge_table() and log() copy to host vectors
 * on access (cached), so the reference's reference-returning accessors work.
 */
#pragma once

#include "parplan/cost.hpp"

#include <map>
#include <optional>
#include <variant>

namespace parplan {

struct NodeElimRecord {
  int removed = -1;
  int in_edge = -1, out_edge = -1, new_edge = -1;
  int src = -1, dst = -1;
  std::vector<std::vector<int>> argmin; // [src config][dst config]
};

struct EdgeElimRecord {
  int e1 = -1, e2 = -1, new_edge = -1;
  int src = -1, dst = -1;
};

using EliminationRecord = std::variant<NodeElimRecord, EdgeElimRecord>;

/// A computation graph under elimination; device-resident tables.
class ReducedGraph {
public:
  struct EdgeRec {
    int id, src, dst;
    bool alive;
  };

  ReducedGraph(const ComputationGraph &graph, const CostTables &tables)
      : graph_(&graph), tables_(&tables), g_(runtime::native(graph)),
        t_(detail::upload_tables(tables, graph, g_.get())) {
    pp_reduced *r = nullptr;
    runtime::check(pp_reduced_create(runtime::context(), g_.get(), t_.get(), &r));
    rg_.reset(r);
  }

  const ComputationGraph &graph() const { return *graph_; }
  const CostTables &tables() const { return *tables_; }

  bool node_alive(int l) const {
    int32_t a = 0;
    runtime::check(pp_reduced_node_alive(rg_.get(), l, &a));
    return a != 0;
  }
  int live_node_count() const { return counts()[2]; }
  int live_edge_count() const { return counts()[3]; }
  std::vector<int> live_nodes() const {
    std::vector<int> out;
    for (int l = 0; l < graph_->layer_count(); ++l)
      if (node_alive(l)) out.push_back(l);
    return out;
  }
  std::vector<EdgeRec> live_edges() const {
    std::vector<EdgeRec> out;
    for (int id = 0; id < counts()[0]; ++id) {
      const EdgeRec e = edge_rec(id);
      if (e.alive) out.push_back(e);
    }
    return out;
  }
  const std::vector<std::vector<double>> &edge_table(int id) const {
    auto it = table_cache_.find(id);
    if (it != table_cache_.end()) return it->second;
    int32_t s, d, a, rows, cols;
    runtime::check(pp_reduced_edge(rg_.get(), id, &s, &d, &a, &rows, &cols));
    std::vector<double> flat(static_cast<size_t>(rows) * static_cast<size_t>(cols));
    runtime::check(pp_reduced_edge_table(rg_.get(), id, flat.data()));
    std::vector<std::vector<double>> m(static_cast<size_t>(rows));
    for (int i = 0; i < rows; ++i)
      m[static_cast<size_t>(i)].assign(flat.begin() + static_cast<long>(i) * cols,
                                       flat.begin() + static_cast<long>(i + 1) * cols);
    return table_cache_.emplace(id, std::move(m)).first->second;
  }
  const std::vector<double> &node_table(int l) const { return tables_->node[static_cast<size_t>(l)]; }

  const std::vector<EliminationRecord> &log() const {
    const int n = counts()[1];
    for (int r = static_cast<int>(log_.size()); r < n; ++r) {
      pp_record rec;
      runtime::check(pp_reduced_log_record(rg_.get(), r, &rec));
      if (rec.type == 0) {
        NodeElimRecord nr{rec.removed, rec.e1, rec.e2, rec.new_edge, rec.src, rec.dst, {}};
        const int rows = tables_->config_count(rec.src), cols = tables_->config_count(rec.dst);
        std::vector<int32_t> flat(static_cast<size_t>(rows) * static_cast<size_t>(cols));
        runtime::check(pp_reduced_argmin(rg_.get(), r, flat.data()));
        nr.argmin.resize(static_cast<size_t>(rows));
        for (int i = 0; i < rows; ++i)
          nr.argmin[static_cast<size_t>(i)].assign(flat.begin() + static_cast<long>(i) * cols,
                                                   flat.begin() + static_cast<long>(i + 1) * cols);
        log_.emplace_back(std::move(nr));
      } else {
        log_.emplace_back(EdgeElimRecord{rec.e1, rec.e2, rec.new_edge, rec.src, rec.dst});
      }
    }
    return log_;
  }

  /// Eq. 2 on the lowest-topological-rank node with one in- and one out-edge.
  bool node_elimination() {
    int32_t acted = 0;
    runtime::check(pp_reduced_node_elimination(rg_.get(), &acted));
    return acted != 0;
  }

  /// Eq. 3 on the lexicographically smallest parallel pair (src, dst, e1, e2).
  bool edge_elimination() {
    int32_t acted = 0;
    runtime::check(pp_reduced_edge_elimination(rg_.get(), &acted));
    return acted != 0;
  }

  /// Eliminations to a fixpoint, node eliminations first.
  void reduce() { runtime::check(pp_reduced_reduce(rg_.get())); }

  pp_reduced *native() const { return rg_.get(); }

private:
  std::array<int32_t, 4> counts() const {
    std::array<int32_t, 4> c{};
    runtime::check(pp_reduced_counts(rg_.get(), &c[0], &c[1], &c[2], &c[3]));
    return c;
  }
  EdgeRec edge_rec(int id) const {
    int32_t s, d, a, r, c;
    runtime::check(pp_reduced_edge(rg_.get(), id, &s, &d, &a, &r, &c));
    return EdgeRec{id, s, d, a != 0};
  }

  const ComputationGraph *graph_;
  const CostTables *tables_;
  runtime::GraphHandle g_;
  runtime::TablesHandle t_;
  runtime::ReducedHandle rg_;
  mutable std::map<int, std::vector<std::vector<double>>> table_cache_;
  mutable std::vector<EliminationRecord> log_;
};

/// Cheapest joint assignment of the remaining nodes (ascending layer order);
/// ties resolve to the lexicographically smallest index tuple.
inline std::pair<std::vector<int>, double> enumerate_final(const ReducedGraph &rg,
                                                           int k_bound = kDefaultFinalGraphBound) {
  const int k = rg.live_node_count();
  std::vector<int32_t> idx(static_cast<size_t>(std::max(k, 1)));
  double cost = 0.0;
  runtime::check(pp_reduced_enumerate_final(rg.native(), k_bound, idx.data(), &cost));
  return {std::vector<int>(idx.begin(), idx.begin() + k), cost};
}

/// Replays the log backwards (planner.hpp:306-319).
inline void unwind(const std::vector<EliminationRecord> &log, std::vector<int> &indices) {
  for (auto it = log.rbegin(); it != log.rend(); ++it)
    if (const auto *ne = std::get_if<NodeElimRecord>(&*it))
      indices[static_cast<size_t>(ne->removed)] =
          ne->argmin[static_cast<size_t>(indices[static_cast<size_t>(ne->src)])]
                    [static_cast<size_t>(indices[static_cast<size_t>(ne->dst)])];
}

struct PlanResult {
  Strategy strategy;
  std::vector<int> indices;
  double cost = 0.0;
  int final_graph_nodes = 0;
  int node_eliminations = 0;
  int edge_eliminations = 0;

  int eliminations() const { return node_eliminations + edge_eliminations; }
};

namespace detail {
inline PlanResult finish_plan(const std::vector<int32_t> &idx, const pp_plan_result &res,
                              const std::vector<std::vector<Config>> &catalog) {
  PlanResult r;
  r.indices.assign(idx.begin(), idx.end());
  r.cost = res.cost;
  r.final_graph_nodes = res.final_graph_nodes;
  r.node_eliminations = res.node_eliminations;
  r.edge_eliminations = res.edge_eliminations;
  r.strategy.resize(idx.size());
  for (size_t l = 0; l < idx.size(); ++l)
    r.strategy[l] = catalog[l][static_cast<size_t>(idx[l])];
  return r;
}
} // namespace detail

/// Reduce + enumerate_final + unwind on the device; cost re-read from the
/// input tables in the canonical order (bit-identical to evaluate_strategy).
inline PlanResult plan_with_tables(const ComputationGraph &graph, const CostTables &tables,
                                   int k_bound = kDefaultFinalGraphBound) {
  auto g = runtime::native(graph);
  auto t = detail::upload_tables(tables, graph, g.get());
  std::vector<int32_t> idx(static_cast<size_t>(graph.layer_count()));
  pp_plan_result res{};
  runtime::check(pp_plan_with_tables(runtime::context(), g.get(), t.get(), k_bound, idx.data(), &res));
  return detail::finish_plan(idx, res, tables.catalog);
}

/// build_cost_tables + plan_with_tables, entirely on the device.
inline PlanResult plan(const ComputationGraph &graph, const DeviceGraph &devices,
                       int k_bound = kDefaultFinalGraphBound) {
  auto g = runtime::native(graph);
  const pp_device_desc d = runtime::device_desc(devices);
  std::vector<int32_t> idx(static_cast<size_t>(graph.layer_count()));
  pp_plan_result res{};
  runtime::check(pp_plan(runtime::context(), g.get(), &d, k_bound, idx.data(), &res));
  // the chosen configs from the library's catalogs (already enumerated for the tables)
  std::vector<int64_t> cfg(static_cast<size_t>(graph.layer_count()) * 4);
  runtime::check(pp_graph_configs_at(g.get(), devices.count(), idx.data(), cfg.data()));
  PlanResult r;
  r.indices.assign(idx.begin(), idx.end());
  r.cost = res.cost;
  r.final_graph_nodes = res.final_graph_nodes;
  r.node_eliminations = res.node_eliminations;
  r.edge_eliminations = res.edge_eliminations;
  r.strategy.resize(idx.size());
  for (size_t l = 0; l < idx.size(); ++l)
    r.strategy[l] = Config{cfg[4 * l], cfg[4 * l + 1], cfg[4 * l + 2], cfg[4 * l + 3]};
  return r;
}

} // namespace parplan
