// plan_api.cu — C ABI for planning: plan / plan_with_tables, the ReducedGraph
// step API, and the brute-force search.
#include "dp.hpp"

#include <cstdio>
#include <cstring>

using namespace pp;

struct pp_reduced {
  pp_context *ctx = nullptr;
  Graph *g = nullptr;
  Tables *t = nullptr;
  std::unique_ptr<Scheduler> sched;
  std::vector<Op> log;
  std::vector<const void *> tab; // device table per edge id
  std::vector<int32_t> rows, cols;
  std::vector<DBuf<unsigned char>> owned;      // derived tables
  std::vector<DBuf<uint16_t>> argmin;          // per log record
};

namespace {

const void *node_table(const Tables &t, int l) {
  return t.mode == kFP64 ? static_cast<const void *>(t.node.p + t.cat_off[static_cast<size_t>(l)])
                         : static_cast<const void *>(t.node32.p + t.cat_off[static_cast<size_t>(l)]);
}

const void *xfer_table(const Tables &t, int e) {
  return t.mode == kFP64 ? static_cast<const void *>(t.xfer64.p + t.xoff[static_cast<size_t>(e)])
                         : static_cast<const void *>(t.xfer32.p + t.xoff[static_cast<size_t>(e)]);
}

size_t elem_size(const Tables &t) { return t.mode == kFP64 ? 8 : 4; }

void apply(pp_reduced *rg, const Op &op) {
  Tables &t = *rg->t;
  const int nu = rg->rows[static_cast<size_t>(op.e1)];
  const int nv = op.type ? rg->cols[static_cast<size_t>(op.e1)] : rg->cols[static_cast<size_t>(op.e2)];
  const int nw = op.type ? 0 : t.counts[static_cast<size_t>(op.removed)];
  DBuf<unsigned char> out(static_cast<size_t>(nu) * nv * elem_size(t));
  DBuf<uint16_t> am;
  if (!op.type) {
    PP_REQUIRE(nw <= 65535, "argmin index exceeds 16 bits");
    am.alloc(static_cast<size_t>(nu) * nv);
  }
  run_single_op(rg->ctx, t.mode, op, rg->tab[static_cast<size_t>(op.e1)], rg->tab[static_cast<size_t>(op.e2)],
                op.type ? nullptr : node_table(t, op.removed), out.p, am.p, nu, nw, nv);
  rg->tab.push_back(out.p);
  rg->rows.push_back(nu);
  rg->cols.push_back(nv);
  rg->owned.push_back(std::move(out));
  rg->argmin.push_back(std::move(am));
  rg->log.push_back(op);
}

} // namespace

extern "C" {

pp_status pp_reduced_create(pp_context *ctx, const pp_graph *g, pp_tables *t, pp_reduced **out) {
  return guard([&] {
    PP_REQUIRE(ctx && g && t && out, "pp_reduced_create: null argument");
    Graph &G = const_cast<pp_graph *>(g)->impl;
    PP_REQUIRE(t->impl.nl == G.nl && t->impl.ne == G.ne, "tables do not match the graph");
    auto rg = std::make_unique<pp_reduced>();
    rg->ctx = ctx;
    rg->g = &G;
    rg->t = &t->impl;
    rg->sched = std::make_unique<Scheduler>(G.nl, G.esrc, G.edst, G.rank);
    for (int e = 0; e < G.ne; ++e) {
      rg->tab.push_back(xfer_table(t->impl, e));
      rg->rows.push_back(t->impl.counts[static_cast<size_t>(G.esrc[static_cast<size_t>(e)])]);
      rg->cols.push_back(t->impl.counts[static_cast<size_t>(G.edst[static_cast<size_t>(e)])]);
    }
    rg->owned.resize(static_cast<size_t>(G.ne));
    *out = rg.release();
  });
}

pp_status pp_reduced_destroy(pp_reduced *rg) {
  delete rg;
  return PP_OK;
}

pp_status pp_reduced_node_elimination(pp_reduced *rg, int32_t *acted) {
  return guard([&] {
    PP_REQUIRE(rg && acted, "null argument");
    Op op;
    *acted = rg->sched->node_step(&op) ? 1 : 0;
    if (*acted) apply(rg, op);
  });
}

pp_status pp_reduced_edge_elimination(pp_reduced *rg, int32_t *acted) {
  return guard([&] {
    PP_REQUIRE(rg && acted, "null argument");
    Op op;
    *acted = rg->sched->edge_step(&op) ? 1 : 0;
    if (*acted) apply(rg, op);
  });
}

pp_status pp_reduced_reduce(pp_reduced *rg) {
  return guard([&] {
    PP_REQUIRE(rg, "null argument");
    Op op;
    for (;;) {
      if (rg->sched->node_step(&op) || rg->sched->edge_step(&op)) {
        apply(rg, op);
        continue;
      }
      break;
    }
  });
}

pp_status pp_reduced_counts(const pp_reduced *rg, int32_t *edges_total, int32_t *log_size, int32_t *live_nodes,
                            int32_t *live_edges) {
  return guard([&] {
    PP_REQUIRE(rg, "null argument");
    if (edges_total) *edges_total = rg->sched->edges_total();
    if (log_size) *log_size = static_cast<int32_t>(rg->log.size());
    if (live_nodes) *live_nodes = rg->sched->live_nodes();
    if (live_edges) *live_edges = rg->sched->live_edges();
  });
}

pp_status pp_reduced_edge(const pp_reduced *rg, int32_t id, int32_t *src, int32_t *dst, int32_t *alive, int32_t *rows,
                          int32_t *cols) {
  return guard([&] {
    PP_REQUIRE(rg, "null argument");
    PP_REQUIRE(id >= 0 && id < rg->sched->edges_total(), "edge id out of range");
    if (src) *src = rg->sched->edge_src(id);
    if (dst) *dst = rg->sched->edge_dst(id);
    if (alive) *alive = rg->sched->edge_alive(id);
    if (rows) *rows = rg->rows[static_cast<size_t>(id)];
    if (cols) *cols = rg->cols[static_cast<size_t>(id)];
  });
}

pp_status pp_reduced_node_alive(const pp_reduced *rg, int32_t layer, int32_t *alive) {
  return guard([&] {
    PP_REQUIRE(rg && alive, "null argument");
    PP_REQUIRE(layer >= 0 && layer < rg->g->nl, "layer out of range");
    *alive = rg->sched->node_alive(layer);
  });
}

pp_status pp_reduced_edge_table(pp_reduced *rg, int32_t id, double *out) {
  return guard([&] {
    PP_REQUIRE(rg && out, "null argument");
    PP_REQUIRE(id >= 0 && id < static_cast<int32_t>(rg->tab.size()), "edge id out of range");
    download_table(rg->ctx, rg->t->mode, rg->t->shift, rg->tab[static_cast<size_t>(id)],
                   static_cast<int64_t>(rg->rows[static_cast<size_t>(id)]) * rg->cols[static_cast<size_t>(id)], out);
  });
}

pp_status pp_reduced_log_record(const pp_reduced *rg, int32_t r, pp_record *out) {
  return guard([&] {
    PP_REQUIRE(rg && out, "null argument");
    PP_REQUIRE(r >= 0 && r < static_cast<int32_t>(rg->log.size()), "record index out of range");
    const Op &o = rg->log[static_cast<size_t>(r)];
    *out = pp_record{o.type, o.removed, o.e1, o.e2, o.ne, o.u, o.v, o.wave};
  });
}

pp_status pp_reduced_argmin(pp_reduced *rg, int32_t r, int32_t *out) {
  return guard([&] {
    PP_REQUIRE(rg && out, "null argument");
    PP_REQUIRE(r >= 0 && r < static_cast<int32_t>(rg->log.size()), "record index out of range");
    const Op &o = rg->log[static_cast<size_t>(r)];
    PP_REQUIRE(o.type == 0, "edge records carry no argmin");
    download_argmin(rg->ctx, rg->argmin[static_cast<size_t>(r)].p,
                    static_cast<int64_t>(rg->rows[static_cast<size_t>(o.ne)]) * rg->cols[static_cast<size_t>(o.ne)], out);
  });
}

pp_status pp_reduced_enumerate_final(pp_reduced *rg, int32_t k_bound, int32_t *idx, double *cost) {
  return guard([&] {
    PP_REQUIRE(rg && idx && cost, "null argument");
    const std::vector<int> nodes = rg->sched->live_node_list();
    const int k = static_cast<int>(nodes.size());
    if (k > k_bound)
      throw parplan::LimitError("final graph has " + std::to_string(k) + " nodes, exceeding the enumeration bound of " +
                                std::to_string(k_bound) + " (graph is not reducible enough)");
    std::vector<int> pos(static_cast<size_t>(rg->g->nl), -1);
    std::vector<const void *> nt;
    std::vector<int32_t> counts;
    for (int d = 0; d < k; ++d) {
      pos[static_cast<size_t>(nodes[static_cast<size_t>(d)])] = d;
      nt.push_back(node_table(*rg->t, nodes[static_cast<size_t>(d)]));
      counts.push_back(rg->t->counts[static_cast<size_t>(nodes[static_cast<size_t>(d)])]);
    }
    std::vector<const void *> et;
    std::vector<int32_t> ps, pd, ec;
    for (int id : rg->sched->live_edge_list()) {
      et.push_back(rg->tab[static_cast<size_t>(id)]);
      ps.push_back(pos[static_cast<size_t>(rg->sched->edge_src(id))]);
      pd.push_back(pos[static_cast<size_t>(rg->sched->edge_dst(id))]);
      ec.push_back(rg->cols[static_cast<size_t>(id)]);
    }
    run_enumerate(rg->ctx, rg->t->mode, rg->t->shift, nt, counts, et, ps, pd, ec, idx, cost);
  });
}

pp_status pp_brute_force(pp_context *ctx, const pp_graph *g, pp_tables *tp, uint64_t budget, int32_t *indices,
                         double *cost, uint64_t *visited) {
  return guard([&] {
    PP_REQUIRE(ctx && g && tp && indices && cost, "pp_brute_force: null argument");
    const Graph &G = g->impl;
    const Tables &t = tp->impl;
    PP_REQUIRE(t.nl == G.nl && t.ne == G.ne, "tables do not match the graph");
    long double space = 1.0L;
    for (int32_t c : t.counts) space *= static_cast<long double>(c);
    if (space > static_cast<long double>(budget)) { // oracle.hpp:56-63
      char buf[64];
      if (space < 1e15L)
        std::snprintf(buf, sizeof buf, "%llu", static_cast<unsigned long long>(space));
      else
        std::snprintf(buf, sizeof buf, "%g", static_cast<double>(space));
      throw parplan::LimitError(std::string("strategy space has ") + buf +
                                " strategies, exceeding the exhaustive-search budget of " + std::to_string(budget));
    }
    std::vector<const void *> nt, et;
    std::vector<int32_t> counts, ps, pd, ec;
    for (int l = 0; l < G.nl; ++l) {
      nt.push_back(node_table(t, l));
      counts.push_back(t.counts[static_cast<size_t>(l)]);
    }
    for (int e = 0; e < G.ne; ++e) {
      et.push_back(xfer_table(t, e));
      ps.push_back(G.esrc[static_cast<size_t>(e)]);
      pd.push_back(G.edst[static_cast<size_t>(e)]);
      ec.push_back(t.counts[static_cast<size_t>(G.edst[static_cast<size_t>(e)])]);
    }
    run_enumerate(ctx, t.mode, t.shift, nt, counts, et, ps, pd, ec, indices, cost);
    if (visited) *visited = static_cast<uint64_t>(space);
  });
}

} // extern "C"
