// ref_driver.cpp — exposes the REAL reference planner (compiled from the
// read-only headers under /root/reference/proj/include) through the same
// orc_* C entry points as the plain-C restatement (parplan_oracle.h).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into
// oracle/_ref/libparplan_ref.so (git-ignored, shipped to the GPU box as a
// prebuilt file).  Used to pin the restatement and as the bench's CPU
// reference arm; never linked into the product.
//
// This file contains no reference code: it only calls the reference API
// (graph.hpp, cost.hpp, planner.hpp, oracle.hpp, models.hpp).
#include "parplan/cost.hpp"
#include "parplan/graph.hpp"
#include "parplan/models.hpp"
#include "parplan/oracle.hpp"
#include "parplan/partition.hpp"
#include "parplan/planner.hpp"

#include "parplan_oracle.h"

#include <cstring>
#include <memory>
#include <optional>
#include <random>

using namespace parplan;

namespace {

thread_local std::string g_err;

struct Inst {
  ComputationGraph graph;
  std::optional<DeviceGraph> devices;
  CostTables tables;
  bool have_tables = false;
  std::unique_ptr<ReducedGraph> rg;
};

LayerKind make_kind(int kind, const int64_t *p) {
  switch (kind) {
  case ORC_INPUT:
    return Input{p[0], p[1], p[2]};
  case ORC_CONV:
    return Conv2D{p[0], p[1], p[2], p[3], p[4], p[5], p[6]};
  case ORC_POOL:
    return Pool2D{p[0], p[1], p[2], p[3], p[4], p[5]};
  case ORC_FC:
    return FullyConnected{p[0]};
  case ORC_FLATTEN:
    return Flatten{};
  case ORC_CONCAT:
    return Concat{static_cast<Dim>(p[0])};
  default:
    return Softmax{};
  }
}

void kind_params(const LayerKind &k, int64_t *p) {
  std::memset(p, 0, 7 * sizeof(int64_t));
  if (auto *x = std::get_if<Input>(&k)) p[0] = x->channel, p[1] = x->height, p[2] = x->width;
  if (auto *x = std::get_if<Conv2D>(&k))
    p[0] = x->out_channels, p[1] = x->kernel_h, p[2] = x->kernel_w, p[3] = x->stride_h, p[4] = x->stride_w,
    p[5] = x->pad_h, p[6] = x->pad_w;
  if (auto *x = std::get_if<Pool2D>(&k))
    p[0] = x->kernel_h, p[1] = x->kernel_w, p[2] = x->stride_h, p[3] = x->stride_w, p[4] = x->pad_h, p[5] = x->pad_w;
  if (auto *x = std::get_if<FullyConnected>(&k)) p[0] = x->out_channels;
  if (auto *x = std::get_if<Concat>(&k)) p[0] = static_cast<int64_t>(x->axis);
}

Config cfg(const int64_t *c) { return Config{c[0], c[1], c[2], c[3]}; }

template <class F> int guard(F &&f) {
  try {
    f();
    return 0;
  } catch (const LimitError &e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception &e) {
    g_err = e.what();
    return 1;
  }
}

Inst *wrap(ComputationGraph g) {
  auto *i = new Inst;
  i->graph = std::move(g);
  return i;
}

} // namespace

extern "C" {

const char *orc_error(void) { return g_err.c_str(); }
int orc_kind(void) { return 1; }

orc_instance *orc_graph(int nl, int ne, int64_t batch, const int32_t *kind, const int64_t *params,
                        const int32_t *esrc, const int32_t *edst, const char *const *ids) {
  Inst *out = nullptr;
  guard([&] {
    std::vector<Layer> layers;
    std::vector<std::vector<std::string>> inputs(static_cast<size_t>(nl));
    for (int l = 0; l < nl; ++l)
      layers.push_back({ids ? std::string(ids[l]) : "n" + std::to_string(l), make_kind(kind[l], params + 7 * l)});
    for (int e = 0; e < ne; ++e) {
      if (esrc[e] < 0 || esrc[e] >= nl || edst[e] < 0 || edst[e] >= nl)
        throw InputError("edge references an undeclared layer");
      inputs[static_cast<size_t>(edst[e])].push_back(layers[static_cast<size_t>(esrc[e])].id);
    }
    out = wrap(ComputationGraph::create(layers, inputs, batch));
  });
  return reinterpret_cast<orc_instance *>(out);
}

orc_instance *orc_builtin(const char *model, int64_t batch) {
  Inst *out = nullptr;
  guard([&] { out = wrap(builtin_model(model, batch)); });
  return reinterpret_cast<orc_instance *>(out);
}

orc_instance *orc_random(uint64_t seed, int n, int maxc, double bp, int ndev) {
  Inst *out = nullptr;
  guard([&] {
    RandomGraphSpec spec{seed, n, maxc, bp, ndev};
    auto inst = random_series_parallel_graph(spec);
    out = wrap(std::move(inst.graph));
    out->tables = std::move(inst.tables);
    out->have_tables = true;
  });
  return reinterpret_cast<orc_instance *>(out);
}

// Config-5 generator: the reference generator's draw order with
// C-sized dummy catalogs {1,1,1,i+1}; built on the reference types.
orc_instance *orc_synthetic(uint64_t seed, int n, int C, double bp) {
  Inst *out = nullptr;
  guard([&] {
    std::mt19937_64 rng(seed);
    auto chance = [&](double p) { return static_cast<double>(rng() % 1000) / 1000.0 < p; };
    std::vector<Layer> layers;
    std::vector<std::vector<std::string>> inputs;
    auto add = [&](LayerKind k, std::vector<std::string> in) {
      std::string id = "n" + std::to_string(layers.size());
      layers.push_back({id, std::move(k)});
      inputs.push_back(std::move(in));
      return id;
    };
    std::string tip = add(Input{4, 1, 1}, {});
    int count = 1;
    while (count < n) {
      if (n - count >= 3 && chance(bp)) {
        auto a = add(Softmax{}, {tip});
        auto b = add(Softmax{}, {tip});
        tip = add(Concat{Dim::Channel}, {a, b});
        count += 3;
      } else {
        tip = add(Softmax{}, {tip});
        count += 1;
      }
    }
    out = wrap(ComputationGraph::create(std::move(layers), inputs, 8));
    auto dyadic = [&] { return static_cast<double>(rng() % 641) / 64.0; };
    const auto &g = out->graph;
    auto &t = out->tables;
    t.catalog.resize(static_cast<size_t>(g.layer_count()));
    t.node.resize(static_cast<size_t>(g.layer_count()));
    for (int l = 0; l < g.layer_count(); ++l) {
      for (int i = 0; i < C; ++i) t.catalog[static_cast<size_t>(l)].push_back(Config{1, 1, 1, i + 1});
      for (int i = 0; i < C; ++i) t.node[static_cast<size_t>(l)].push_back(dyadic());
    }
    t.xfer.resize(static_cast<size_t>(g.edge_count()));
    for (const Edge &e : g.edges()) {
      auto &m = t.xfer[static_cast<size_t>(e.id)];
      m.assign(static_cast<size_t>(C), std::vector<double>(static_cast<size_t>(C)));
      for (auto &row : m)
        for (double &v : row) v = dyadic();
    }
    out->have_tables = true;
  });
  return reinterpret_cast<orc_instance *>(out);
}

void orc_free(orc_instance *p) { delete reinterpret_cast<Inst *>(p); }

int orc_build_tables(orc_instance *p, int nd, const double *rates, const double *bw) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] {
    i->devices.emplace(std::vector<double>(rates, rates + nd),
                       std::vector<double>(bw, bw + static_cast<size_t>(nd) * static_cast<size_t>(nd)));
    i->rg.reset();
    i->tables = build_cost_tables(i->graph, *i->devices);
    i->have_tables = true;
  });
}

int orc_set_tables(orc_instance *p, const int32_t *ncfg, const int64_t *configs, const double *node,
                   const double *xfer) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] {
    i->rg.reset();
    CostTables t;
    const auto &g = i->graph;
    size_t oc = 0, on = 0, ox = 0;
    t.catalog.resize(static_cast<size_t>(g.layer_count()));
    t.node.resize(static_cast<size_t>(g.layer_count()));
    for (int l = 0; l < g.layer_count(); ++l) {
      for (int c = 0; c < ncfg[l]; ++c) {
        t.catalog[static_cast<size_t>(l)].push_back(cfg(configs + 4 * oc));
        ++oc;
        t.node[static_cast<size_t>(l)].push_back(node[on++]);
      }
    }
    t.xfer.resize(static_cast<size_t>(g.edge_count()));
    for (const Edge &e : g.edges()) {
      auto &m = t.xfer[static_cast<size_t>(e.id)];
      m.assign(static_cast<size_t>(ncfg[e.src]), std::vector<double>(static_cast<size_t>(ncfg[e.dst])));
      for (auto &row : m)
        for (double &v : row) v = xfer[ox++];
    }
    i->tables = std::move(t);
    i->have_tables = true;
  });
}

int orc_n_layers(const orc_instance *p) { return reinterpret_cast<const Inst *>(p)->graph.layer_count(); }
int orc_n_edges(const orc_instance *p) { return reinterpret_cast<const Inst *>(p)->graph.edge_count(); }
void orc_edges(const orc_instance *p, int32_t *s, int32_t *d, int32_t *pos) {
  for (const Edge &e : reinterpret_cast<const Inst *>(p)->graph.edges()) {
    if (s) s[e.id] = e.src;
    if (d) d[e.id] = e.dst;
    if (pos) pos[e.id] = e.dst_input_pos;
  }
}
void orc_shapes(const orc_instance *p, int64_t *o) {
  const auto &g = reinterpret_cast<const Inst *>(p)->graph;
  for (int l = 0; l < g.layer_count(); ++l) {
    const auto &s = g.shape(l);
    o[4 * l] = s.sample, o[4 * l + 1] = s.channel, o[4 * l + 2] = s.height, o[4 * l + 3] = s.width;
  }
}
void orc_topo(const orc_instance *p, int32_t *o) {
  const auto &t = reinterpret_cast<const Inst *>(p)->graph.topo_order();
  for (size_t k = 0; k < t.size(); ++k) o[k] = t[k];
}
int orc_config_count(const orc_instance *p, int l) {
  auto *i = reinterpret_cast<const Inst *>(p);
  return i->have_tables ? i->tables.config_count(l) : -1;
}
void orc_catalog(const orc_instance *p, int l, int64_t *o) {
  const auto &c = reinterpret_cast<const Inst *>(p)->tables.catalog[static_cast<size_t>(l)];
  for (size_t k = 0; k < c.size(); ++k)
    o[4 * k] = c[k].sample, o[4 * k + 1] = c[k].channel, o[4 * k + 2] = c[k].height, o[4 * k + 3] = c[k].width;
}
static void copy_vec(const std::vector<double> &v, double *o) { std::memcpy(o, v.data(), v.size() * sizeof(double)); }
void orc_node(const orc_instance *p, int l, double *o) {
  copy_vec(reinterpret_cast<const Inst *>(p)->tables.node[static_cast<size_t>(l)], o);
}
void orc_compute(const orc_instance *p, int l, double *o) {
  auto &t = reinterpret_cast<const Inst *>(p)->tables;
  if (static_cast<size_t>(l) < t.compute.size()) copy_vec(t.compute[static_cast<size_t>(l)], o);
}
void orc_sync(const orc_instance *p, int l, double *o) {
  auto &t = reinterpret_cast<const Inst *>(p)->tables;
  if (static_cast<size_t>(l) < t.sync.size()) copy_vec(t.sync[static_cast<size_t>(l)], o);
}
void orc_xfer(const orc_instance *p, int e, double *o) {
  const auto &m = reinterpret_cast<const Inst *>(p)->tables.xfer[static_cast<size_t>(e)];
  size_t k = 0;
  for (const auto &row : m)
    for (double v : row) o[k++] = v;
}
int orc_layer(const orc_instance *p, int l, int64_t *params, char *id, int cap) {
  const auto &L = reinterpret_cast<const Inst *>(p)->graph.layer(l);
  if (params) kind_params(L.kind, params);
  if (id && cap > 0) {
    std::strncpy(id, L.id.c_str(), static_cast<size_t>(cap) - 1);
    id[cap - 1] = 0;
  }
  return static_cast<int>(L.kind.index());
}

int orc_transfer_profile(const orc_instance *p, int e, const int64_t *cs, const int64_t *cd, int nd,
                         const double *bw, double *sec, double *bytes) {
  auto *i = reinterpret_cast<const Inst *>(p);
  return guard([&] {
    DeviceGraph d(std::vector<double>(static_cast<size_t>(nd), kDefaultComputeRate),
                  std::vector<double>(bw, bw + static_cast<size_t>(nd) * static_cast<size_t>(nd)));
    auto prof = transfer_profile(i->graph, i->graph.edge(e), cfg(cs), cfg(cd), d);
    *sec = prof.seconds;
    *bytes = prof.bytes;
  });
}

int orc_owned_region(const int64_t *shape, const int64_t *c, int64_t part, int64_t *o) {
  return guard([&] {
    Region r = owned_region(TensorShape{shape[0], shape[1], shape[2], shape[3]}, cfg(c), part);
    for (int d = 0; d < 4; ++d) o[d] = r.lo[static_cast<size_t>(d)], o[4 + d] = r.hi[static_cast<size_t>(d)];
  });
}

int orc_required_region(const orc_instance *p, int e, const int64_t *dc, int64_t part, int64_t *o) {
  auto *i = reinterpret_cast<const Inst *>(p);
  return guard([&] {
    Region r = required_input_region(i->graph, i->graph.edge(e), cfg(dc), part);
    for (int d = 0; d < 4; ++d) o[d] = r.lo[static_cast<size_t>(d)], o[4 + d] = r.hi[static_cast<size_t>(d)];
  });
}

int orc_enumerate_configs(int kind, const int64_t *shape, int nd, int64_t *out, int cap) {
  int n = -1;
  guard([&] {
    int64_t zeros[7] = {1, 1, 1, 1, 1, 1, 1};
    auto v = enumerate_configs(make_kind(kind, zeros), TensorShape{shape[0], shape[1], shape[2], shape[3]}, nd);
    n = static_cast<int>(v.size());
    for (int k = 0; k < n && k < cap; ++k)
      out[4 * k] = v[static_cast<size_t>(k)].sample, out[4 * k + 1] = v[static_cast<size_t>(k)].channel,
              out[4 * k + 2] = v[static_cast<size_t>(k)].height, out[4 * k + 3] = v[static_cast<size_t>(k)].width;
  });
  return n;
}

int orc_plan(orc_instance *p, int kb, int32_t *indices, double *cost, int32_t *stats) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] {
    auto r = plan_with_tables(i->graph, i->tables, kb);
    for (int l = 0; l < i->graph.layer_count(); ++l) indices[l] = r.indices[static_cast<size_t>(l)];
    *cost = r.cost;
    stats[0] = r.final_graph_nodes, stats[1] = r.node_eliminations, stats[2] = r.edge_eliminations;
  });
}

int orc_reduce(orc_instance *p) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] {
    i->rg = std::make_unique<ReducedGraph>(i->graph, i->tables);
    i->rg->reduce();
  });
}

int orc_rg_init(orc_instance *p) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] { i->rg = std::make_unique<ReducedGraph>(i->graph, i->tables); });
}
int orc_rg_node(orc_instance *p) {
  auto *i = reinterpret_cast<Inst *>(p);
  return i->rg ? (i->rg->node_elimination() ? 1 : 0) : -1;
}
int orc_rg_edge(orc_instance *p) {
  auto *i = reinterpret_cast<Inst *>(p);
  return i->rg ? (i->rg->edge_elimination() ? 1 : 0) : -1;
}
int orc_rg_edges_total(const orc_instance *p) {
  auto *i = reinterpret_cast<const Inst *>(p);
  if (!i->rg) return 0;
  int n = 0; // ids are dense: the largest id of any record + 1, or the original count
  n = i->graph.edge_count();
  for (const auto &rec : i->rg->log())
    n = std::max(n, 1 + std::visit([](const auto &r) { return r.new_edge; }, rec));
  return n;
}
int orc_rg_edge_info(const orc_instance *p, int e, int32_t *info3) {
  auto *i = reinterpret_cast<const Inst *>(p);
  if (!i->rg) return 1;
  for (const auto &er : i->rg->live_edges())
    if (er.id == e) {
      info3[0] = er.src, info3[1] = er.dst, info3[2] = 1;
      return 0;
    }
  // dead edge: recover endpoints from the graph or the log
  if (e < i->graph.edge_count()) {
    info3[0] = i->graph.edge(e).src, info3[1] = i->graph.edge(e).dst, info3[2] = 0;
    return 0;
  }
  for (const auto &rec : i->rg->log()) {
    int ne = std::visit([](const auto &r) { return r.new_edge; }, rec);
    if (ne == e) {
      std::visit([&](const auto &r) { info3[0] = r.src, info3[1] = r.dst; }, rec);
      info3[2] = 0;
      return 0;
    }
  }
  return 1;
}

int orc_log_size(const orc_instance *p) {
  auto *i = reinterpret_cast<const Inst *>(p);
  return i->rg ? static_cast<int>(i->rg->log().size()) : 0;
}

int orc_log_record(const orc_instance *p, int r, int32_t *o) {
  const auto &rec = reinterpret_cast<const Inst *>(p)->rg->log()[static_cast<size_t>(r)];
  if (auto *n = std::get_if<NodeElimRecord>(&rec)) {
    o[0] = 0, o[1] = n->removed, o[2] = n->in_edge, o[3] = n->out_edge, o[4] = n->new_edge, o[5] = n->src,
    o[6] = n->dst;
  } else {
    auto &e = std::get<EdgeElimRecord>(rec);
    o[0] = 1, o[1] = -1, o[2] = e.e1, o[3] = e.e2, o[4] = e.new_edge, o[5] = e.src, o[6] = e.dst;
  }
  return 0;
}

int orc_log_argmin(const orc_instance *p, int r, int32_t *o) {
  const auto &rec = reinterpret_cast<const Inst *>(p)->rg->log()[static_cast<size_t>(r)];
  auto *n = std::get_if<NodeElimRecord>(&rec);
  if (!n) return 1;
  size_t k = 0;
  for (const auto &row : n->argmin)
    for (int v : row) o[k++] = v;
  return 0;
}

int orc_edge_table_dims(const orc_instance *p, int e, int32_t *d) {
  auto *i = reinterpret_cast<const Inst *>(p);
  if (!i->rg) return 1;
  const auto &t = i->rg->edge_table(e);
  d[0] = static_cast<int32_t>(t.size());
  d[1] = t.empty() ? 0 : static_cast<int32_t>(t[0].size());
  return 0;
}

int orc_edge_table(const orc_instance *p, int e, double *o) {
  auto *i = reinterpret_cast<const Inst *>(p);
  if (!i->rg) return 1;
  size_t k = 0;
  for (const auto &row : i->rg->edge_table(e))
    for (double v : row) o[k++] = v;
  return 0;
}

int orc_live_nodes(const orc_instance *p, int32_t *o) {
  auto *i = reinterpret_cast<const Inst *>(p);
  if (!i->rg) {
    if (o)
      for (int l = 0; l < i->graph.layer_count(); ++l) o[l] = l;
    return i->graph.layer_count();
  }
  auto v = i->rg->live_nodes();
  if (o)
    for (size_t k = 0; k < v.size(); ++k) o[k] = v[k];
  return static_cast<int>(v.size());
}

int orc_enumerate_final(orc_instance *p, int kb, int32_t *idx, double *cost) {
  auto *i = reinterpret_cast<Inst *>(p);
  return guard([&] {
    if (!i->rg) i->rg = std::make_unique<ReducedGraph>(i->graph, i->tables);
    auto [v, c] = enumerate_final(*i->rg, kb);
    for (size_t k = 0; k < v.size(); ++k) idx[k] = v[k];
    *cost = c;
  });
}

double orc_total_cost(const orc_instance *p, const int32_t *idx) {
  auto *i = reinterpret_cast<const Inst *>(p);
  std::vector<int> v(idx, idx + i->graph.layer_count());
  return detail::total_cost_by_index(i->graph, i->tables, v);
}

int orc_brute(const orc_instance *p, uint64_t budget, int32_t *indices, double *cost, uint64_t *visited) {
  auto *i = reinterpret_cast<const Inst *>(p);
  return guard([&] {
    auto r = brute_force_plan(i->graph, i->tables, budget);
    for (size_t k = 0; k < r.indices.size(); ++k) indices[k] = r.indices[k];
    *cost = r.cost;
    *visited = r.visited;
  });
}

// One Eq. 2 fold through the reference's ReducedGraph on a 3-node chain
// (u -> w -> v) with the given tables.
void orc_fold(int nu, int nw, int nv, const double *w, const double *t1, const double *t2, double *out,
              int32_t *am) {
  guard([&] {
    auto g = ComputationGraph::create({{"u", Input{1, 1, 1}}, {"w", Softmax{}}, {"v", Softmax{}}},
                                      {{}, {"u"}, {"w"}}, 1);
    CostTables t;
    auto cat = [](int n) {
      std::vector<Config> c;
      for (int i = 0; i < n; ++i) c.push_back(Config{1, 1, 1, i + 1});
      return c;
    };
    t.catalog = {cat(nu), cat(nw), cat(nv)};
    t.node = {std::vector<double>(static_cast<size_t>(nu)), std::vector<double>(w, w + nw),
              std::vector<double>(static_cast<size_t>(nv))};
    t.xfer.resize(2);
    t.xfer[0].assign(static_cast<size_t>(nu), std::vector<double>(static_cast<size_t>(nw)));
    t.xfer[1].assign(static_cast<size_t>(nw), std::vector<double>(static_cast<size_t>(nv)));
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nw; ++j) t.xfer[0][static_cast<size_t>(i)][static_cast<size_t>(j)] = t1[i * nw + j];
    for (int j = 0; j < nw; ++j)
      for (int k = 0; k < nv; ++k) t.xfer[1][static_cast<size_t>(j)][static_cast<size_t>(k)] = t2[j * nv + k];
    ReducedGraph rg(g, t);
    rg.node_elimination();
    const auto &rec = std::get<NodeElimRecord>(rg.log()[0]);
    const auto &tab = rg.edge_table(rec.new_edge);
    for (int i = 0; i < nu; ++i)
      for (int k = 0; k < nv; ++k) {
        out[i * nv + k] = tab[static_cast<size_t>(i)][static_cast<size_t>(k)];
        am[i * nv + k] = rec.argmin[static_cast<size_t>(i)][static_cast<size_t>(k)];
      }
  });
}

} // extern "C"
