/* parplan/io.hpp — the reference's JSON file formats (proj/include/parplan/io.hpp):
 *
 *   network   {"batch", "layers": [{"id", "kind", "inputs", <kind fields>}]}  (:80-183)
 *   devices   {"devices": [{"id", "flops"}], "links": [{"src", "dst",
 *              "bandwidth"}], "default_bandwidth"}                             (:185-229)
 *   strategy  {"cost_seconds", "layers": {id: config}, "eliminations",
 *              "final_graph_nodes"}                                            (:231-281)
 *   measured  {"node_costs": {layer id: [s...]},
 *              "xfer_costs": {edge index: [[s...]...]}}                        (:283-348)
 *
 * Same entry points, field defaults and InputError messages as the reference;
 * the JSON type is nlohmann::ordered_json (header-only, third party, from the
 * image: see tests/cpp/Makefile for the include path).  Measured costs
 * overlay the host CostTables; plan_with_tables uploads them as given.
 */
#pragma once

#include "parplan/cost.hpp"

#include <fstream>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

namespace parplan {

using json = nlohmann::ordered_json;

namespace detail {

// Typed access to one JSON object with the reference's error wording.
class JsonFields {
public:
  JsonFields(const json &obj, std::string where) : obj_(obj), where_(std::move(where)) {}

  bool has(const std::string &key) const { return obj_.contains(key); }

  template <typename T> T need(const std::string &key) const {
    if (!has(key)) throw InputError(where_ + ": missing field '" + key + "'");
    return as<T>(key);
  }
  template <typename T> T get(const std::string &key, T dflt) const { return has(key) ? as<T>(key) : dflt; }

  // square "<base>" or per-axis "<base>_h" / "<base>_w" (per-axis wins)
  std::pair<i64, i64> axes(const std::string &base, i64 dflt) const {
    const i64 both = get<i64>(base, dflt);
    return {get<i64>(base + "_h", both), get<i64>(base + "_w", both)};
  }

  const std::string &where() const { return where_; }

private:
  template <typename T> T as(const std::string &key) const {
    try {
      return obj_.at(key).get<T>();
    } catch (const nlohmann::json::exception &) {
      throw InputError(where_ + ": field '" + key + "' has the wrong type");
    }
  }
  const json &obj_;
  std::string where_;
};

inline json read_json(const std::string &path) {
  std::ifstream in(path);
  if (!in) throw InputError("cannot open '" + path + "'");
  try {
    return json::parse(in);
  } catch (const nlohmann::json::exception &e) {
    throw InputError("'" + path + "': " + e.what());
  }
}

inline Dim dim_from_name(const std::string &name, const std::string &where) {
  for (Dim d : kAllDims)
    if (name == dim_name(d)) return d;
  throw InputError(where + ": unknown dimension '" + name + "'");
}

inline LayerKind kind_from_json(const JsonFields &f) {
  const std::string kind = f.need<std::string>("kind");
  if (kind == "input") return Input{f.need<i64>("channel"), f.need<i64>("height"), f.need<i64>("width")};
  if (kind == "conv2d" || kind == "pool2d") {
    const auto [kh, kw] = f.axes("kernel", 1);
    const auto [sh, sw] = f.axes("stride", 1);
    const auto [ph, pw] = f.axes("pad", 0);
    if (kind == "pool2d") return Pool2D{kh, kw, sh, sw, ph, pw};
    return Conv2D{f.need<i64>("out_channels"), kh, kw, sh, sw, ph, pw};
  }
  if (kind == "fully_connected") return FullyConnected{f.need<i64>("out_channels")};
  if (kind == "flatten") return Flatten{};
  if (kind == "concat") return Concat{dim_from_name(f.get<std::string>("axis", "channel"), f.where())};
  if (kind == "softmax") return Softmax{};
  throw InputError(f.where() + ": unknown kind '" + kind + "'");
}

// kind-specific fields of one layer, per-axis form (io.hpp:137-183)
inline void kind_to_json(const LayerKind &k, json &lj) {
  auto window = [&](i64 kh, i64 kw, i64 sh, i64 sw, i64 ph, i64 pw) {
    lj["kernel_h"] = kh, lj["kernel_w"] = kw;
    lj["stride_h"] = sh, lj["stride_w"] = sw;
    lj["pad_h"] = ph, lj["pad_w"] = pw;
  };
  if (const auto *in = std::get_if<Input>(&k)) {
    lj["channel"] = in->channel, lj["height"] = in->height, lj["width"] = in->width;
  } else if (const auto *c = std::get_if<Conv2D>(&k)) {
    lj["out_channels"] = c->out_channels;
    window(c->kernel_h, c->kernel_w, c->stride_h, c->stride_w, c->pad_h, c->pad_w);
  } else if (const auto *p = std::get_if<Pool2D>(&k)) {
    window(p->kernel_h, p->kernel_w, p->stride_h, p->stride_w, p->pad_h, p->pad_w);
  } else if (const auto *fc = std::get_if<FullyConnected>(&k)) {
    lj["out_channels"] = fc->out_channels;
  } else if (const auto *cc = std::get_if<Concat>(&k)) {
    lj["axis"] = dim_name(cc->axis);
  }
}

// a non-negative measured cost (NaN fails the test too, as in the reference)
inline bool cost_ok(double v) { return v >= 0; }

} // namespace detail

// ---- network files ----------------------------------------------------------

/// `batch_override` > 0 replaces the file's batch size (default 32).
inline ComputationGraph parse_network(const json &j, i64 batch_override = 0) {
  const detail::JsonFields top(j, "network");
  const i64 batch = batch_override > 0 ? batch_override : top.get<i64>("batch", 32);
  if (!j.contains("layers") || !j.at("layers").is_array()) throw InputError("network: missing 'layers' array");
  std::vector<Layer> layers;
  std::vector<std::vector<std::string>> inputs;
  for (const json &lj : j.at("layers")) {
    const std::string id = detail::JsonFields(lj, "network layer").need<std::string>("id");
    const detail::JsonFields f(lj, "layer '" + id + "'");
    layers.push_back({id, detail::kind_from_json(f)});
    inputs.push_back(f.get<std::vector<std::string>>("inputs", {}));
  }
  return ComputationGraph::create(std::move(layers), inputs, batch);
}

inline ComputationGraph parse_network_file(const std::string &path, i64 batch_override = 0) {
  return parse_network(detail::read_json(path), batch_override);
}

inline json emit_network(const ComputationGraph &g) {
  json layers = json::array();
  for (int l = 0; l < g.layer_count(); ++l) {
    json lj;
    lj["id"] = g.layer(l).id;
    lj["kind"] = kind_name(g.layer(l).kind);
    json ins = json::array();
    for (int e : g.in_edges(l)) ins.push_back(g.layer(g.edge(e).src).id);
    lj["inputs"] = std::move(ins);
    detail::kind_to_json(g.layer(l).kind, lj);
    layers.push_back(std::move(lj));
  }
  return json{{"batch", g.batch()}, {"layers", std::move(layers)}};
}

// ---- device files -----------------------------------------------------------

/// Device ids must be dense 0..n-1 (any order); links are ordered pairs and
/// pairs without one use default_bandwidth.
inline DeviceGraph parse_device_graph(const json &j) {
  if (!j.contains("devices") || !j.at("devices").is_array() || j.at("devices").empty())
    throw InputError("device file: missing non-empty 'devices' array");
  const json &devs = j.at("devices");
  const i64 n = static_cast<i64>(devs.size());
  std::vector<double> rates(static_cast<size_t>(n), 0.0);
  std::vector<char> seen(static_cast<size_t>(n), 0);
  for (const json &dj : devs) {
    const i64 id = detail::JsonFields(dj, "device").need<i64>("id");
    if (id < 0 || id >= n)
      throw InputError("device id " + std::to_string(id) + " out of range (ids must be dense 0.." +
                       std::to_string(n - 1) + ")");
    if (seen[static_cast<size_t>(id)]) throw InputError("duplicate device id " + std::to_string(id));
    seen[static_cast<size_t>(id)] = 1;
    rates[static_cast<size_t>(id)] = detail::JsonFields(dj, "device " + std::to_string(id)).need<double>("flops");
  }
  const double dflt = detail::JsonFields(j, "device file").get<double>("default_bandwidth", kDefaultBandwidth);
  std::vector<double> bw(static_cast<size_t>(n * n), dflt);
  if (j.contains("links"))
    for (const json &lj : j.at("links")) {
      const detail::JsonFields f(lj, "link");
      const i64 src = f.need<i64>("src"), dst = f.need<i64>("dst");
      if (src < 0 || src >= n || dst < 0 || dst >= n)
        throw InputError("link " + std::to_string(src) + "->" + std::to_string(dst) + " references unknown device");
      bw[static_cast<size_t>(src * n + dst)] = f.need<double>("bandwidth");
    }
  return DeviceGraph(std::move(rates), std::move(bw));
}

inline DeviceGraph parse_device_file(const std::string &path) { return parse_device_graph(detail::read_json(path)); }

// ---- strategy files ---------------------------------------------------------

inline json config_json(const Config &c) {
  return json{{"sample", c.sample}, {"channel", c.channel}, {"height", c.height}, {"width", c.width}};
}

inline json strategy_json(const ComputationGraph &graph, const Strategy &strategy, double cost, int eliminations,
                          int final_graph_nodes) {
  json layers = json::object();
  for (int l = 0; l < graph.layer_count(); ++l) layers[graph.layer(l).id] = config_json(strategy[static_cast<size_t>(l)]);
  return json{{"cost_seconds", cost},
              {"layers", std::move(layers)},
              {"eliminations", eliminations},
              {"final_graph_nodes", final_graph_nodes}};
}

/// Every graph layer must appear; unknown ids are rejected; absent
/// dimensions default to 1.
inline Strategy parse_strategy(const json &j, const ComputationGraph &graph) {
  if (!j.contains("layers") || !j.at("layers").is_object()) throw InputError("strategy: missing 'layers' object");
  const size_t n = static_cast<size_t>(graph.layer_count());
  Strategy s(n);
  std::vector<char> covered(n, 0);
  for (const auto &[id, cj] : j.at("layers").items()) {
    const int l = graph.index_of(id);
    if (l < 0) throw InputError("strategy names unknown layer '" + id + "'");
    const detail::JsonFields f(cj, "strategy for layer '" + id + "'");
    s[static_cast<size_t>(l)] = Config{f.get<i64>("sample", 1), f.get<i64>("channel", 1), f.get<i64>("height", 1),
                                       f.get<i64>("width", 1)};
    covered[static_cast<size_t>(l)] = 1;
  }
  for (size_t l = 0; l < n; ++l)
    if (!covered[l]) throw InputError("strategy missing layer '" + graph.layer(static_cast<int>(l)).id + "'");
  return s;
}

inline Strategy parse_strategy_file(const std::string &path, const ComputationGraph &graph) {
  return parse_strategy(detail::read_json(path), graph);
}

// ---- measured costs ---------------------------------------------------------

/// Overlays measured node / transfer costs (entries in catalog order; edge
/// keys are decimal edge indices).  Unnamed layers and edges keep their
/// analytic values; any override drops the compute/sync split.
inline void apply_measured_costs(const json &j, const ComputationGraph &graph, CostTables &tables) {
  bool changed = false;
  if (j.contains("node_costs"))
    for (const auto &[id, vj] : j.at("node_costs").items()) {
      const int l = graph.index_of(id);
      if (l < 0) throw InputError("cost file names unknown layer '" + id + "'");
      std::vector<double> v = vj.get<std::vector<double>>();
      std::vector<double> &cur = tables.node[static_cast<size_t>(l)];
      if (v.size() != cur.size())
        throw InputError("cost file: layer '" + id + "' has " + std::to_string(v.size()) + " node costs, catalog has " +
                         std::to_string(cur.size()));
      for (double x : v)
        if (!detail::cost_ok(x)) throw InputError("cost file: layer '" + id + "' has a negative cost");
      cur = std::move(v);
      changed = true;
    }
  if (j.contains("xfer_costs"))
    for (const auto &[key, mj] : j.at("xfer_costs").items()) {
      int e = -1; // std::stoi semantics, the whole key consumed
      try {
        size_t used = 0;
        const int v = std::stoi(key, &used);
        if (used == key.size()) e = v;
      } catch (const std::exception &) {
      }
      if (e < 0 || e >= graph.edge_count()) throw InputError("cost file names unknown edge '" + key + "'");
      std::vector<std::vector<double>> m = mj.get<std::vector<std::vector<double>>>();
      std::vector<std::vector<double>> &cur = tables.xfer[static_cast<size_t>(e)];
      if (m.size() != cur.size()) throw InputError("cost file: edge " + key + " row count mismatch");
      for (size_t i = 0; i < m.size(); ++i) {
        if (m[i].size() != cur[i].size()) throw InputError("cost file: edge " + key + " column count mismatch");
        for (double x : m[i])
          if (!detail::cost_ok(x)) throw InputError("cost file: edge " + key + " has a negative cost");
      }
      cur = std::move(m);
      changed = true;
    }
  if (changed) {
    tables.compute.clear();
    tables.sync.clear();
  }
}

inline void apply_measured_costs_file(const std::string &path, const ComputationGraph &graph, CostTables &tables) {
  apply_measured_costs(detail::read_json(path), graph, tables);
}

} // namespace parplan
