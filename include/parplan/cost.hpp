/* parplan/cost.hpp — cost model, cost tables, strategy evaluation.
 *
 * Drop-in for /root/reference/proj/include/parplan/cost.hpp:
 *   layer_flops / parameter_bytes (:28-55), compute_cost / sync_cost (:57-94),
 *   TransferProfile / transfer_profile / transfer_cost (:96-137),
 *   CostTables (:148-168), build_cost_tables (:170-206),
 *   detail::strategy_indices / total_cost_by_index, evaluate_strategy,
 *   CostBreakdown / evaluate_components (:208-293).
 *
 * build_cost_tables runs on the B200: one launch of the node-cost fill (K2)
 * and the xfer-table builder (K1) in libparplan_cuda.so, then the tables are
 * copied into the reference's nested-vector CostTables.  The single-pair
 * functions (compute_cost, sync_cost, transfer_profile) evaluate the same
 * formulas (geometry.hpp) for one config pair on the host, as the reference
 * API does; no table or plan is ever built on the host.
 */
#pragma once

#include "parplan/geometry.hpp"
#include "parplan/partition.hpp"
#include "parplan/runtime.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <utility>

namespace parplan {

namespace detail {
inline std::array<i64, 7> params_of(const LayerKind &k) {
  std::array<i64, 7> p{};
  kind_params(k, p.data());
  return p;
}
} // namespace detail

inline i64 layer_flops(const LayerKind &kind, const TensorShape &out, const TensorShape &in) {
  const auto p = detail::params_of(kind);
  const auto o = detail::dims_of(out), i = detail::dims_of(in);
  return geo::layer_flops(static_cast<int>(kind.index()), p.data(), o.data(), i.data());
}

inline double parameter_bytes(const LayerKind &kind, const TensorShape &out, const TensorShape &in) {
  const auto p = detail::params_of(kind);
  const auto o = detail::dims_of(out), i = detail::dims_of(in);
  return geo::parameter_bytes(static_cast<int>(kind.index()), p.data(), o.data(), i.data());
}

inline double compute_cost(const LayerKind &kind, const TensorShape &out, const TensorShape &in, const Config &config,
                           const DeviceGraph &devices) {
  const i64 flops = layer_flops(kind, out, in);
  if (flops == 0) return 0.0;
  const Placement pl = place(config, devices);
  double slowest = devices.compute_rate(pl.device(0));
  for (i64 p = 1; p < config.total(); ++p) slowest = std::min(slowest, devices.compute_rate(pl.device(p)));
  return geo::compute_seconds(flops, config.total(), slowest);
}

inline double sync_cost(const LayerKind &kind, const TensorShape &out, const TensorShape &in, const Config &config,
                        const DeviceGraph &devices) {
  const double param = parameter_bytes(kind, out, in);
  if (param == 0.0) return 0.0;
  if (config.total() / config.channel == 1) return 0.0;
  const Placement pl = place(config, devices);
  const double shard = param / static_cast<double>(config.channel);
  double t = 0.0;
  for (i64 p = 1; p < config.total(); ++p) t += 2.0 * shard / devices.bandwidth(pl.device(p), 0);
  return t;
}

struct TransferProfile {
  double seconds = 0.0;
  double bytes = 0.0;
};

/// Bottleneck transfer time of one edge under (c_src, c_dst): per device-pair
/// bytes, max over pairs of bytes / bandwidth (all links concurrent).
inline TransferProfile transfer_profile(const ComputationGraph &graph, const Edge &edge, const Config &c_src,
                                        const Config &c_dst, const DeviceGraph &devices) {
  const Placement src_pl = place(c_src, devices);
  const Placement dst_pl = place(c_dst, devices);
  const auto sshape = detail::dims_of(graph.edge_shape(edge));
  const auto cs = detail::dims_of(c_src);
  std::map<std::pair<int, int>, double> pair_bytes;
  for (i64 q = 0; q < c_dst.total(); ++q) {
    const Region need = required_input_region(graph, edge, c_dst, q);
    if (need.empty()) continue;
    for (i64 p = 0; p < c_src.total(); ++p) {
      if (src_pl.device(p) == dst_pl.device(q)) continue;
      i64 lo[4], hi[4];
      geo::owned_box(sshape.data(), cs.data(), p, lo, hi);
      i64 vol = 1;
      for (int d = 0; d < 4; ++d) vol *= std::max<i64>(0, std::min(hi[d], need.hi[static_cast<size_t>(d)]) -
                                                             std::max(lo[d], need.lo[static_cast<size_t>(d)]));
      if (vol > 0) pair_bytes[{src_pl.device(p), dst_pl.device(q)}] += kBytesPerElement * static_cast<double>(vol);
    }
  }
  TransferProfile out;
  for (const auto &[pair, bytes] : pair_bytes) {
    out.bytes += bytes;
    out.seconds = std::max(out.seconds, bytes / devices.bandwidth(pair.first, pair.second));
  }
  return out;
}

inline double transfer_cost(const ComputationGraph &graph, const Edge &edge, const Config &c_src, const Config &c_dst,
                            const DeviceGraph &devices) {
  return transfer_profile(graph, edge, c_src, c_dst, devices).seconds;
}

/// node[l][i] = compute + sync of layer l under its i-th config; xfer[e][i][j]
/// = transfer time of edge e between its endpoints' i-th / j-th configs.
struct CostTables {
  std::vector<std::vector<Config>> catalog;
  std::vector<std::vector<double>> node;
  std::vector<std::vector<double>> compute;
  std::vector<std::vector<double>> sync;
  std::vector<std::vector<std::vector<double>>> xfer;

  int config_count(int layer) const { return static_cast<int>(catalog[static_cast<size_t>(layer)].size()); }

  int config_index(int layer, const Config &c) const {
    const auto &cat = catalog[static_cast<size_t>(layer)];
    auto it = std::lower_bound(cat.begin(), cat.end(), c);
    return it == cat.end() || !(*it == c) ? -1 : static_cast<int>(it - cat.begin());
  }
};

namespace detail {

/// Copies device tables into the reference's nested-vector layout.
inline CostTables download_tables(pp_tables *t, const ComputationGraph &graph, bool with_split) {
  const int n = graph.layer_count();
  std::vector<int32_t> counts(static_cast<size_t>(n));
  int64_t xcells = 0;
  runtime::check(pp_tables_counts(t, counts.data(), &xcells));
  int64_t total = 0;
  for (int32_t c : counts) total += c;
  std::vector<int64_t> cfg(static_cast<size_t>(total) * 4);
  std::vector<double> node(static_cast<size_t>(total)), comp(static_cast<size_t>(total)),
      syn(static_cast<size_t>(total)), xf(static_cast<size_t>(xcells));
  runtime::check(pp_tables_download(t, cfg.data(), node.data(), with_split ? comp.data() : nullptr,
                                    with_split ? syn.data() : nullptr, xf.data()));
  CostTables out;
  out.catalog.resize(static_cast<size_t>(n));
  out.node.resize(static_cast<size_t>(n));
  if (with_split) {
    out.compute.resize(static_cast<size_t>(n));
    out.sync.resize(static_cast<size_t>(n));
  }
  size_t k = 0;
  for (int l = 0; l < n; ++l)
    for (int c = 0; c < counts[static_cast<size_t>(l)]; ++c, ++k) {
      out.catalog[static_cast<size_t>(l)].push_back({cfg[4 * k], cfg[4 * k + 1], cfg[4 * k + 2], cfg[4 * k + 3]});
      out.node[static_cast<size_t>(l)].push_back(node[k]);
      if (with_split) {
        out.compute[static_cast<size_t>(l)].push_back(comp[k]);
        out.sync[static_cast<size_t>(l)].push_back(syn[k]);
      }
    }
  out.xfer.resize(static_cast<size_t>(graph.edge_count()));
  size_t x = 0;
  for (const Edge &e : graph.edges()) {
    auto &m = out.xfer[static_cast<size_t>(e.id)];
    m.assign(static_cast<size_t>(counts[static_cast<size_t>(e.src)]),
             std::vector<double>(static_cast<size_t>(counts[static_cast<size_t>(e.dst)])));
    for (auto &row : m)
      for (double &v : row) v = xf[x++];
  }
  return out;
}

/// Uploads host CostTables (hand-built, generated, measured) to the device.
inline runtime::TablesHandle upload_tables(const CostTables &t, const ComputationGraph &graph, pp_graph *g) {
  const int n = graph.layer_count();
  if (t.node.size() != static_cast<size_t>(n) || t.xfer.size() != static_cast<size_t>(graph.edge_count()))
    throw InputError("cost tables do not match the graph");
  std::vector<int32_t> counts;
  std::vector<int64_t> cfg;
  std::vector<double> node, xf;
  for (int l = 0; l < n; ++l) {
    const auto &nd = t.node[static_cast<size_t>(l)];
    counts.push_back(static_cast<int32_t>(nd.size()));
    node.insert(node.end(), nd.begin(), nd.end());
    for (size_t c = 0; c < nd.size(); ++c) {
      const Config cc = l < static_cast<int>(t.catalog.size()) && c < t.catalog[static_cast<size_t>(l)].size()
                            ? t.catalog[static_cast<size_t>(l)][c]
                            : Config{};
      cfg.insert(cfg.end(), {cc.sample, cc.channel, cc.height, cc.width});
    }
  }
  for (const Edge &e : graph.edges()) {
    const auto &m = t.xfer[static_cast<size_t>(e.id)];
    if (m.size() != static_cast<size_t>(counts[static_cast<size_t>(e.src)]))
      throw InputError("xfer table of edge " + std::to_string(e.id) + " has the wrong shape");
    for (const auto &row : m) {
      if (row.size() != static_cast<size_t>(counts[static_cast<size_t>(e.dst)]))
        throw InputError("xfer table of edge " + std::to_string(e.id) + " has the wrong shape");
      xf.insert(xf.end(), row.begin(), row.end());
    }
  }
  pp_tables *out = nullptr;
  runtime::check(pp_tables_upload(runtime::context(), g, counts.data(), cfg.data(), node.data(), xf.data(), &out));
  return runtime::TablesHandle(out);
}

} // namespace detail

/// Catalogs + node costs (K2) + xfer tables (K1), built on the B200.
inline CostTables build_cost_tables(const ComputationGraph &graph, const DeviceGraph &devices) {
  auto g = runtime::native(graph);
  const pp_device_desc d = runtime::device_desc(devices);
  pp_tables *t = nullptr;
  runtime::check(pp_tables_build(runtime::context(), g.get(), &d, &t));
  runtime::TablesHandle h(t);
  return detail::download_tables(t, graph, true);
}

namespace detail {

inline std::vector<int> strategy_indices(const ComputationGraph &graph, const CostTables &tables,
                                         const Strategy &strategy) {
  if (strategy.size() != static_cast<size_t>(graph.layer_count()))
    throw InputError("strategy covers " + std::to_string(strategy.size()) + " layers, graph has " +
                     std::to_string(graph.layer_count()));
  std::vector<int> idx(strategy.size());
  for (int l = 0; l < graph.layer_count(); ++l) {
    idx[static_cast<size_t>(l)] = tables.config_index(l, strategy[static_cast<size_t>(l)]);
    if (idx[static_cast<size_t>(l)] < 0)
      throw InputError("config " + to_string(strategy[static_cast<size_t>(l)]) + " is not valid for layer '" +
                       graph.layer(l).id + "'");
  }
  return idx;
}

/// The pinned summation order: nodes by layer index, then xfer by edge id.
inline double total_cost_by_index(const ComputationGraph &graph, const CostTables &tables, const std::vector<int> &idx) {
  double t = 0.0;
  for (int l = 0; l < graph.layer_count(); ++l)
    t += tables.node[static_cast<size_t>(l)][static_cast<size_t>(idx[static_cast<size_t>(l)])];
  for (const Edge &e : graph.edges())
    t += tables.xfer[static_cast<size_t>(e.id)][static_cast<size_t>(idx[static_cast<size_t>(e.src)])]
                    [static_cast<size_t>(idx[static_cast<size_t>(e.dst)])];
  return t;
}

} // namespace detail

inline double evaluate_strategy(const ComputationGraph &graph, const CostTables &tables, const Strategy &strategy) {
  return detail::total_cost_by_index(graph, tables, detail::strategy_indices(graph, tables, strategy));
}

struct CostBreakdown {
  double total = 0.0;
  double node_total = 0.0;
  double xfer_total = 0.0;
  std::vector<double> per_layer_node;
  std::vector<double> per_layer_compute;
  std::vector<double> per_layer_sync;
  std::vector<double> per_edge_xfer;
};

inline CostBreakdown evaluate_components(const ComputationGraph &graph, const CostTables &tables,
                                         const Strategy &strategy) {
  const auto idx = detail::strategy_indices(graph, tables, strategy);
  CostBreakdown b;
  const bool split = !tables.compute.empty();
  for (int l = 0; l < graph.layer_count(); ++l) {
    const auto li = static_cast<size_t>(l), ci = static_cast<size_t>(idx[li]);
    b.per_layer_node.push_back(tables.node[li][ci]);
    if (split) {
      b.per_layer_compute.push_back(tables.compute[li][ci]);
      b.per_layer_sync.push_back(tables.sync[li][ci]);
    }
    b.node_total += tables.node[li][ci];
  }
  for (const Edge &e : graph.edges()) {
    const double x = tables.xfer[static_cast<size_t>(e.id)][static_cast<size_t>(idx[static_cast<size_t>(e.src)])]
                                [static_cast<size_t>(idx[static_cast<size_t>(e.dst)])];
    b.per_edge_xfer.push_back(x);
    b.xfer_total += x;
  }
  b.total = detail::total_cost_by_index(graph, tables, idx);
  return b;
}

} // namespace parplan
