// graph_api.cpp — host half of the C ABI: graphs, catalogs, the symbolic
// schedule, error reporting.  No CUDA here; all of it works without a GPU.
#include "internal.hpp"
#include "shard.hpp"

#include "parplan/models.hpp"

#include <cstring>
#include <list>
#include <mutex>

namespace pp {

static thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }

Graph::Graph(parplan::ComputationGraph cg) : g(std::move(cg)) {
  nl = g.layer_count();
  ne = g.edge_count();
  kind.resize(static_cast<size_t>(nl));
  params.resize(static_cast<size_t>(nl) * 7);
  shape.resize(static_cast<size_t>(nl) * 4);
  rank.resize(static_cast<size_t>(nl));
  for (int l = 0; l < nl; ++l) {
    kind[static_cast<size_t>(l)] = static_cast<int32_t>(g.layer(l).kind.index());
    parplan::detail::kind_params(g.layer(l).kind, &params[static_cast<size_t>(l) * 7]);
    const auto s = parplan::detail::dims_of(g.shape(l));
    std::memcpy(&shape[static_cast<size_t>(l) * 4], s.data(), 4 * sizeof(int64_t));
    rank[static_cast<size_t>(l)] = g.topo_rank(l);
  }
  for (const parplan::Edge &e : g.edges()) {
    esrc.push_back(e.src);
    edst.push_back(e.dst);
    epos.push_back(e.dst_input_pos);
    band_offset.push_back(parplan::detail::concat_band_offset(g, e));
  }
}

const Schedule &Graph::schedule() {
  std::lock_guard<std::mutex> lock(lazy);
  if (!sched) sched = std::make_unique<Schedule>(build_schedule(nl, esrc, edst, rank));
  return *sched;
}

const Graph::Catalogs &Graph::catalogs(int devices) const {
  std::lock_guard<std::mutex> lock(lazy);
  auto it = catalog_cache.find(devices);
  if (it != catalog_cache.end()) return it->second;
  Catalogs c;
  enumerate_catalogs(*this, devices, &c.counts, &c.configs);
  c.configs32.assign(c.configs.begin(), c.configs.end());
  return catalog_cache.emplace(devices, std::move(c)).first->second;
}

void enumerate_catalogs(const Graph &g, int devices, std::vector<int32_t> *counts, std::vector<int64_t> *configs) {
  counts->clear();
  configs->clear();
  for (int l = 0; l < g.nl; ++l) {
    const auto cat = parplan::enumerate_configs(g.g.layer(l).kind, g.g.shape(l), devices);
    counts->push_back(static_cast<int32_t>(cat.size()));
    for (const auto &c : cat) {
      configs->push_back(c.sample);
      configs->push_back(c.channel);
      configs->push_back(c.height);
      configs->push_back(c.width);
    }
  }
}

} // namespace pp

using pp::guard;

extern "C" {

const char *pp_last_error(void) { return pp::g_last_error.c_str(); }
int pp_abi_version(void) { return PP_ABI_VERSION; }

namespace {
// Content-addressed cache of the most recent graphs: the key is the whole
// descriptor, so a hit is exactly an equal graph (memoised pure functions of an
// immutable value).  Strong references, least recently used evicted.
struct GraphCache {
  std::mutex mu;
  std::list<std::pair<std::string, std::shared_ptr<pp::Graph>>> lru;
  static constexpr size_t kMax = 16;
};
GraphCache &graph_cache() {
  static GraphCache c;
  return c;
}
std::string desc_key(const pp_graph_desc *d) {
  std::string k;
  auto put = [&](const void *p, size_t n) { k.append(static_cast<const char *>(p), n); };
  put(&d->n_layers, sizeof d->n_layers);
  put(&d->n_edges, sizeof d->n_edges);
  put(&d->batch, sizeof d->batch);
  for (int l = 0; l < d->n_layers; ++l) {
    const char *id = d->ids && d->ids[l] ? d->ids[l] : "";
    k.append(id);
    k.push_back('\0');
  }
  put(d->kind, sizeof(int32_t) * static_cast<size_t>(d->n_layers));
  put(d->params, sizeof(int64_t) * 7 * static_cast<size_t>(d->n_layers));
  put(d->edge_src, sizeof(int32_t) * static_cast<size_t>(d->n_edges));
  put(d->edge_dst, sizeof(int32_t) * static_cast<size_t>(d->n_edges));
  k.push_back(d->ids ? 'i' : 'n');
  return k;
}
} // namespace

pp_status pp_graph_create(const pp_graph_desc *d, pp_graph **out) {
  return guard([&] {
    PP_REQUIRE(d && out, "pp_graph_create: null argument");
    PP_REQUIRE(d->n_layers >= 0 && d->n_edges >= 0, "pp_graph_create: negative sizes");
    PP_REQUIRE(d->n_layers == 0 || (d->kind && d->params), "pp_graph_create: null layer arrays");
    PP_REQUIRE(d->n_edges == 0 || (d->edge_src && d->edge_dst), "pp_graph_create: null edge arrays");
    const std::string key = desc_key(d);
    GraphCache &cache = graph_cache();
    {
      std::lock_guard<std::mutex> lock(cache.mu);
      for (auto it = cache.lru.begin(); it != cache.lru.end(); ++it)
        if (it->first == key) {
          cache.lru.splice(cache.lru.begin(), cache.lru, it);
          *out = new pp_graph(cache.lru.front().second);
          return;
        }
    }
    std::vector<parplan::Layer> layers;
    std::vector<std::vector<std::string>> inputs(static_cast<size_t>(d->n_layers));
    for (int l = 0; l < d->n_layers; ++l) {
      std::string id = d->ids ? std::string(d->ids[l] ? d->ids[l] : "") : "n" + std::to_string(l);
      layers.push_back({std::move(id), parplan::detail::kind_from_params(d->kind[l], d->params + 7 * l)});
    }
    int prev = 0;
    for (int e = 0; e < d->n_edges; ++e) {
      const int s = d->edge_src[e], t = d->edge_dst[e];
      PP_REQUIRE(s >= 0 && s < d->n_layers && t >= 0 && t < d->n_layers,
                 "edge " + std::to_string(e) + " references an undeclared layer");
      PP_REQUIRE(t >= prev, "edges must be listed in destination order (the reference's dense edge ids)");
      prev = t;
      inputs[static_cast<size_t>(t)].push_back(layers[static_cast<size_t>(s)].id);
    }
    auto g = std::make_shared<pp::Graph>(parplan::ComputationGraph::create(std::move(layers), inputs, d->batch));
    {
      std::lock_guard<std::mutex> lock(cache.mu);
      cache.lru.emplace_front(key, g);
      if (cache.lru.size() > GraphCache::kMax) cache.lru.pop_back();
    }
    *out = new pp_graph(std::move(g));
  });
}

pp_status pp_graph_configs_at(const pp_graph *g, int32_t devices, const int32_t *indices, int64_t *configs) {
  return guard([&] {
    PP_REQUIRE(g && indices && configs, "pp_graph_configs_at: null argument");
    const pp::Graph::Catalogs &c = g->impl.catalogs(devices);
    int64_t off = 0;
    for (int l = 0; l < g->impl.nl; ++l) {
      const int32_t n = c.counts[static_cast<size_t>(l)];
      PP_REQUIRE(indices[l] >= 0 && indices[l] < n, "config index out of range");
      std::memcpy(configs + 4 * l, &c.configs[static_cast<size_t>(4 * (off + indices[l]))], 4 * sizeof(int64_t));
      off += n;
    }
  });
}

pp_status pp_graph_builtin(const char *name, int64_t batch, pp_graph **out) {
  return guard([&] {
    PP_REQUIRE(name && out, "pp_graph_builtin: null argument");
    *out = new pp_graph(parplan::builtin_model(name, batch));
  });
}

pp_status pp_graph_destroy(pp_graph *g) {
  delete g;
  return PP_OK;
}

pp_status pp_graph_size(const pp_graph *g, int32_t *nl, int32_t *ne) {
  return guard([&] {
    PP_REQUIRE(g, "null graph");
    if (nl) *nl = g->impl.nl;
    if (ne) *ne = g->impl.ne;
  });
}

pp_status pp_graph_layers(const pp_graph *g, int32_t *kind, int64_t *params, int64_t *shapes, int32_t *topo) {
  return guard([&] {
    PP_REQUIRE(g, "null graph");
    const auto &G = g->impl;
    if (kind) std::memcpy(kind, G.kind.data(), G.kind.size() * sizeof(int32_t));
    if (params) std::memcpy(params, G.params.data(), G.params.size() * sizeof(int64_t));
    if (shapes) std::memcpy(shapes, G.shape.data(), G.shape.size() * sizeof(int64_t));
    if (topo)
      for (int r = 0; r < G.nl; ++r) topo[r] = G.g.topo_order()[static_cast<size_t>(r)];
  });
}

pp_status pp_graph_edges(const pp_graph *g, int32_t *src, int32_t *dst, int32_t *pos) {
  return guard([&] {
    PP_REQUIRE(g, "null graph");
    const auto &G = g->impl;
    for (int e = 0; e < G.ne; ++e) {
      if (src) src[e] = G.esrc[static_cast<size_t>(e)];
      if (dst) dst[e] = G.edst[static_cast<size_t>(e)];
      if (pos) pos[e] = G.epos[static_cast<size_t>(e)];
    }
  });
}

pp_status pp_graph_layer_id(const pp_graph *g, int32_t l, char *buf, int32_t cap) {
  return guard([&] {
    PP_REQUIRE(g && buf && cap > 0, "pp_graph_layer_id: bad argument");
    PP_REQUIRE(l >= 0 && l < g->impl.nl, "layer index out of range");
    const std::string &id = g->impl.g.layer(l).id;
    const size_t n = std::min(id.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, id.data(), n);
    buf[n] = 0;
  });
}

pp_status pp_graph_catalogs(const pp_graph *g, int32_t devices, int32_t *counts, int64_t *configs) {
  return guard([&] {
    PP_REQUIRE(g && counts, "pp_graph_catalogs: null argument");
    std::vector<int32_t> c;
    std::vector<int64_t> cfg;
    pp::enumerate_catalogs(g->impl, devices, &c, &cfg);
    std::memcpy(counts, c.data(), c.size() * sizeof(int32_t));
    if (configs) std::memcpy(configs, cfg.data(), cfg.size() * sizeof(int64_t));
  });
}

pp_status pp_graph_schedule(const pp_graph *g, int32_t *n, pp_record *recs, int32_t *n_waves) {
  return guard([&] {
    PP_REQUIRE(g && n, "pp_graph_schedule: null argument");
    const pp::Schedule &s = const_cast<pp_graph *>(g)->impl.schedule();
    *n = static_cast<int32_t>(s.ops.size());
    if (n_waves) *n_waves = s.n_waves;
    if (recs)
      for (size_t k = 0; k < s.ops.size(); ++k) {
        const pp::Op &o = s.ops[k];
        recs[k] = pp_record{o.type, o.removed, o.e1, o.e2, o.ne, o.u, o.v, o.wave};
      }
  });
}

pp_status pp_shard_layout(const pp_graph *g, const int32_t *counts, int32_t nranks, int32_t rank, int32_t *n_tables,
                          int32_t *blk, int32_t *first, int32_t *local_rows, int32_t *n_gathers, int32_t *gather_wave,
                          int32_t *gather_table) {
  return guard([&] {
    PP_REQUIRE(g && counts && n_tables && n_gathers, "pp_shard_layout: null argument");
    PP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / world size");
    const pp::Schedule &s = const_cast<pp_graph *>(g)->impl.schedule();
    const int E = static_cast<int>(s.esrc.size());
    *n_tables = E;
    for (int id = 0; id < E; ++id) {
      const int rows = counts[s.esrc[static_cast<size_t>(id)]];
      if (blk) blk[id] = pp::shard_blk(rows, nranks);
      if (first) first[id] = pp::shard_first(rows, nranks, rank);
      if (local_rows) local_rows[id] = pp::shard_rows(rows, nranks, rank);
    }
    const auto gs = pp::shard_gathers(s, g->impl.ne);
    *n_gathers = static_cast<int32_t>(gs.size());
    for (size_t k = 0; k < gs.size(); ++k) {
      if (gather_wave) gather_wave[k] = gs[k].first;
      if (gather_table) gather_table[k] = gs[k].second;
    }
  });
}

} // extern "C"
