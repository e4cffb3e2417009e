// scheduler.cpp — see scheduler.hpp.
#include "scheduler.hpp"

#include <algorithm>

namespace pp {

Scheduler::Scheduler(int n, const std::vector<int> &esrc, const std::vector<int> &edst, const std::vector<int> &rank)
    : rank_(rank), alive_n_(static_cast<size_t>(n), 1), in_(static_cast<size_t>(n)), out_(static_cast<size_t>(n)) {
  live_nodes_ = n;
  for (size_t e = 0; e < esrc.size(); ++e) new_edge(esrc[e], edst[e], 0);
  for (int l = 0; l < n; ++l) refresh(l);
}

int Scheduler::new_edge(int u, int v, int wave) { // planner.hpp:220-227: id = edges_.size()
  const int id = static_cast<int>(src_.size());
  src_.push_back(u);
  dst_.push_back(v);
  wave_.push_back(wave);
  alive_e_.push_back(1);
  in_[static_cast<size_t>(v)].insert(id);
  out_[static_cast<size_t>(u)].insert(id);
  auto &ids = by_ends_[{u, v}];
  ids.insert(id);
  if (ids.size() >= 2) parallel_.insert({u, v});
  ++live_edges_;
  return id;
}

void Scheduler::drop_edge(int id) { // planner.hpp:229-236
  const int u = src_[static_cast<size_t>(id)], v = dst_[static_cast<size_t>(id)];
  alive_e_[static_cast<size_t>(id)] = 0;
  in_[static_cast<size_t>(v)].erase(id);
  out_[static_cast<size_t>(u)].erase(id);
  auto it = by_ends_.find({u, v});
  it->second.erase(id);
  if (it->second.size() < 2) parallel_.erase({u, v});
  if (it->second.empty()) by_ends_.erase(it);
  --live_edges_;
}

void Scheduler::refresh(int l) {
  const auto key = std::make_pair(rank_[static_cast<size_t>(l)], l);
  const bool ok = alive_n_[static_cast<size_t>(l)] && in_[static_cast<size_t>(l)].size() == 1 &&
                  out_[static_cast<size_t>(l)].size() == 1;
  if (ok)
    eligible_.insert(key);
  else
    eligible_.erase(key);
}

bool Scheduler::node_step(Op *op) {
  if (eligible_.empty()) return false;
  const int w = eligible_.begin()->second;
  eligible_.erase(eligible_.begin());
  const int e1 = *in_[static_cast<size_t>(w)].begin();
  const int e2 = *out_[static_cast<size_t>(w)].begin();
  const int u = src_[static_cast<size_t>(e1)], v = dst_[static_cast<size_t>(e2)];
  const int wave = std::max(wave_[static_cast<size_t>(e1)], wave_[static_cast<size_t>(e2)]) + 1;
  const int ne = new_edge(u, v, wave);
  drop_edge(e1);
  drop_edge(e2);
  alive_n_[static_cast<size_t>(w)] = 0;
  --live_nodes_;
  // u keeps one out-edge (e1 -> ne) and v one in-edge (e2 -> ne): degrees and
  // therefore eligibility of u and v are unchanged.
  *op = Op{0, w, e1, e2, ne, u, v, wave};
  return true;
}

bool Scheduler::edge_step(Op *op) {
  if (parallel_.empty()) return false;
  const auto key = *parallel_.begin(); // smallest (src, dst)
  const auto &ids = by_ends_[key];
  auto it = ids.begin();
  const int a = *it++, b = *it; // two smallest ids under that key
  const int wave = std::max(wave_[static_cast<size_t>(a)], wave_[static_cast<size_t>(b)]) + 1;
  const int ne = new_edge(key.first, key.second, wave);
  drop_edge(a);
  drop_edge(b);
  refresh(key.first);
  refresh(key.second);
  *op = Op{1, -1, a, b, ne, key.first, key.second, wave};
  return true;
}

void Scheduler::reduce(std::vector<Op> *ops) { // planner.hpp:209-217
  Op op;
  for (;;) {
    if (node_step(&op) || edge_step(&op)) {
      ops->push_back(op);
      continue;
    }
    break;
  }
}

std::vector<int> Scheduler::live_node_list() const {
  std::vector<int> out;
  for (size_t l = 0; l < alive_n_.size(); ++l)
    if (alive_n_[l]) out.push_back(static_cast<int>(l));
  return out;
}

std::vector<int> Scheduler::live_edge_list() const {
  std::vector<int> out;
  for (size_t e = 0; e < alive_e_.size(); ++e)
    if (alive_e_[e]) out.push_back(static_cast<int>(e));
  return out;
}

Schedule build_schedule(int n, const std::vector<int> &esrc, const std::vector<int> &edst,
                        const std::vector<int> &rank) {
  Scheduler s(n, esrc, edst, rank);
  Schedule out;
  s.reduce(&out.ops);
  for (const Op &op : out.ops) {
    out.n_waves = std::max(out.n_waves, op.wave);
    (op.type ? out.edge_ops : out.node_ops)++;
  }
  out.wave_begin.assign(static_cast<size_t>(out.n_waves) + 2, 0);
  for (const Op &op : out.ops) ++out.wave_begin[static_cast<size_t>(op.wave) + 1];
  for (size_t w = 1; w < out.wave_begin.size(); ++w) out.wave_begin[w] += out.wave_begin[w - 1];
  // wave_begin[w] = first exec slot of wave w (waves are 1-based; slot 0 empty)
  out.exec.assign(out.ops.size(), 0);
  std::vector<int> fill(out.wave_begin.begin(), out.wave_begin.end());
  for (size_t k = 0; k < out.ops.size(); ++k) out.exec[static_cast<size_t>(fill[static_cast<size_t>(out.ops[k].wave)]++)] = static_cast<int>(k);
  out.final_nodes = s.live_node_list();
  out.final_edges = s.live_edge_list();
  for (int id = 0; id < s.edges_total(); ++id) {
    out.esrc.push_back(s.edge_src(id));
    out.edst.push_back(s.edge_dst(id));
  }
  return out;
}

} // namespace pp
