// scheduler.hpp — symbolic elimination scheduler (host).
//
// The reference picks its next elimination from the TOPOLOGY alone
// (planner.hpp:114-127: lowest-topological-rank live node with exactly one
// in-edge and one out-edge; planner.hpp:167-188: otherwise the
// lexicographically smallest (src, dst, e1, e2) parallel pair), never from
// table values.  So the whole elimination log — record sequence, new edge
// ids, and the producer/consumer DAG — is computed here before any arithmetic,
// in O((N + E) log N) instead of the reference's O(E^2) rescans, and the
// device then executes the numeric work in dependency waves.
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <utility>
#include <vector>

namespace pp {

struct Op {
  int type = 0;     // 0 node elimination (Eq. 2), 1 edge elimination (Eq. 3)
  int removed = -1; // node ops: the eliminated layer
  int e1 = -1, e2 = -1, ne = -1;
  int u = -1, v = -1; // endpoints of the new edge
  int wave = 0;       // 1-based dependency wave
};

class Scheduler {
public:
  // n layers, original edges (src, dst) in id order, topo rank per layer
  Scheduler(int n_layers, const std::vector<int> &esrc, const std::vector<int> &edst, const std::vector<int> &rank);

  bool node_step(Op *out); // planner.hpp:114-163
  bool edge_step(Op *out); // planner.hpp:167-206
  void reduce(std::vector<Op> *ops);

  int edges_total() const { return static_cast<int>(src_.size()); }
  int edge_src(int id) const { return src_[static_cast<size_t>(id)]; }
  int edge_dst(int id) const { return dst_[static_cast<size_t>(id)]; }
  bool edge_alive(int id) const { return alive_e_[static_cast<size_t>(id)]; }
  bool node_alive(int l) const { return alive_n_[static_cast<size_t>(l)]; }
  int live_nodes() const { return live_nodes_; }
  int live_edges() const { return live_edges_; }
  std::vector<int> live_node_list() const;
  std::vector<int> live_edge_list() const;
  int edge_wave(int id) const { return wave_[static_cast<size_t>(id)]; }

private:
  int new_edge(int u, int v, int wave);
  void drop_edge(int id);
  void refresh(int layer);

  std::vector<int> rank_;
  std::vector<int> src_, dst_, wave_;
  std::vector<char> alive_e_, alive_n_;
  std::vector<std::set<int>> in_, out_;
  std::set<std::pair<int, int>> eligible_;          // (topo rank, layer)
  std::map<std::pair<int, int>, std::set<int>> by_ends_; // (src, dst) -> live ids
  std::set<std::pair<int, int>> parallel_;          // keys holding >= 2 ids
  int live_nodes_ = 0, live_edges_ = 0;
};

// Full schedule of a graph: the log in reference order plus its wave layout.
struct Schedule {
  std::vector<Op> ops;          // reduce() log order (planner.hpp:209-217)
  std::vector<int> exec;        // op indices grouped by wave (stable)
  std::vector<int> wave_begin;  // [n_waves + 1] offsets into exec
  std::vector<int> final_nodes; // live layers after reduce, ascending
  std::vector<int> final_edges; // live edge ids after reduce, ascending
  std::vector<int> esrc, edst;  // endpoints of every edge id (original + new)
  int n_waves = 0;
  int node_ops = 0, edge_ops = 0;
};

Schedule build_schedule(int n_layers, const std::vector<int> &esrc, const std::vector<int> &edst,
                        const std::vector<int> &rank);

} // namespace pp
