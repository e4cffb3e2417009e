// generators.cpp — seeded instance generators (oracle.hpp:98-185).
//
// random_series_parallel_graph: series-parallel topology (chains plus
// two-branch diamonds) drawn with std::mt19937_64 in the reference's order,
// then dyadic table values k/64, k = rng() % 641, in the pinned fill order
// (nodes by layer, then xfer by edge id, row-major).  The config-5 variant
// keeps the draw order and replaces the catalogs by C dummy configs
// {1,1,1,i+1}.  Host code: generation is part of fixture construction, and the
// tables are uploaded to the device like any other CostTables.
#include "internal.hpp"
#include "tables.hpp"

#include <random>

namespace pp {

struct Instance {
  parplan::ComputationGraph graph;
  std::vector<int32_t> counts;
  std::vector<int64_t> configs;
  std::vector<double> node, xfer;
};

// oracle.hpp:130-157 — returns the graph; rng continues for the tables.
static parplan::ComputationGraph sp_topology(std::mt19937_64 &rng, int n, double bp) {
  std::vector<parplan::Layer> layers;
  std::vector<std::vector<std::string>> inputs;
  auto add = [&](parplan::LayerKind k, std::vector<std::string> in) {
    std::string id = "n" + std::to_string(layers.size());
    layers.push_back({id, std::move(k)});
    inputs.push_back(std::move(in));
    return id;
  };
  auto chance = [&](double p) { return static_cast<double>(rng() % 1000) / 1000.0 < p; };
  std::string tip = add(parplan::Input{4, 1, 1}, {});
  int count = 1;
  while (count < n) {
    if (n - count >= 3 && chance(bp)) {
      const std::string a = add(parplan::Softmax{}, {tip});
      const std::string b = add(parplan::Softmax{}, {tip});
      tip = add(parplan::Concat{parplan::Dim::Channel}, {a, b});
      count += 3;
    } else {
      tip = add(parplan::Softmax{}, {tip});
      count += 1;
    }
  }
  return parplan::ComputationGraph::create(std::move(layers), inputs, 8);
}

static Instance make_instance(uint64_t seed, int n, int maxc, double bp, int ndev, int fixed_c) {
  if (n < 1) throw parplan::InputError("random graph needs at least one node");
  if (fixed_c <= 0 && maxc < 1) throw parplan::InputError("random graph needs at least one config per layer");
  if (fixed_c <= 0 && ndev < 1) throw parplan::InputError("random graph needs at least one device");
  std::mt19937_64 rng(seed);
  Instance in{sp_topology(rng, n, bp), {}, {}, {}, {}};
  const auto &g = in.graph;
  auto dyadic = [&] { return static_cast<double>(rng() % 641) / 64.0; };
  for (int l = 0; l < g.layer_count(); ++l) {
    if (fixed_c > 0) {
      in.counts.push_back(fixed_c);
      for (int i = 0; i < fixed_c; ++i) in.configs.insert(in.configs.end(), {1, 1, 1, i + 1});
    } else {
      auto cat = parplan::enumerate_configs(g.layer(l).kind, g.shape(l), ndev);
      if (static_cast<int>(cat.size()) > maxc) cat.resize(static_cast<size_t>(maxc));
      in.counts.push_back(static_cast<int32_t>(cat.size()));
      for (const auto &c : cat) in.configs.insert(in.configs.end(), {c.sample, c.channel, c.height, c.width});
    }
    for (int i = 0; i < in.counts.back(); ++i) in.node.push_back(dyadic());
  }
  for (const parplan::Edge &e : g.edges()) {
    const size_t cells = static_cast<size_t>(in.counts[static_cast<size_t>(e.src)]) * in.counts[static_cast<size_t>(e.dst)];
    for (size_t k = 0; k < cells; ++k) in.xfer.push_back(dyadic());
  }
  return in;
}

} // namespace pp

using pp::guard;

extern "C" {

pp_status pp_graph_series_parallel(uint64_t seed, int32_t node_count, double bp, pp_graph **out) {
  return guard([&] {
    PP_REQUIRE(out, "null argument");
    if (node_count < 1) throw parplan::InputError("random graph needs at least one node");
    std::mt19937_64 rng(seed);
    *out = new pp_graph(pp::sp_topology(rng, node_count, bp));
  });
}

pp_status pp_random_instance(pp_context *ctx, uint64_t seed, int32_t node_count, int32_t max_configs, double bp,
                             int32_t device_count, int32_t configs_override, pp_graph **graph, pp_tables **tables) {
  pp_graph *g = nullptr;
  pp::Instance inst;
  if (configs_override > 0) // config 5: the same draw order, int32 units (k/64 -> k) streamed to the device
    return guard([&] {
      PP_REQUIRE(ctx && graph && tables, "null argument");
      if (node_count < 1) throw parplan::InputError("random graph needs at least one node");
      std::mt19937_64 rng(seed);
      auto gp = std::make_unique<pp_graph>(pp::sp_topology(rng, node_count, bp));
      *tables = pp::tables_fixed_streamed(ctx, gp->impl, configs_override, 6, 640, [&](int32_t *dst, size_t n) {
        for (size_t k = 0; k < n; ++k) dst[k] = static_cast<int32_t>(rng() % 641);
      });
      *graph = gp.release();
    });
  pp_status st = guard([&] {
    PP_REQUIRE(ctx && graph && tables, "null argument");
    inst = pp::make_instance(seed, node_count, max_configs, bp, device_count, configs_override);
    g = new pp_graph(inst.graph);
  });
  if (st != PP_OK) return st;
  st = pp_tables_upload(ctx, g, inst.counts.data(), inst.configs.data(), inst.node.data(), inst.xfer.data(), tables);
  if (st != PP_OK) {
    pp_graph_destroy(g);
    return st;
  }
  *graph = g;
  return PP_OK;
}

} // extern "C"
