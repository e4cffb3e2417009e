/*
 * parplan_oracle.h — CPU restatement of the reference planner (TEST INFRASTRUCTURE ONLY).
 *
 * This header and parplan_oracle.c restate, in plain C11, the algorithm of the
 * reference `parplan` headers (/root/reference/proj/include/parplan/ *.hpp):
 * graph creation + min-heap Kahn order, shape inference, config enumeration,
 * partition regions, the analytic cost model, cost-table construction, the
 * node/edge elimination dynamic program, final enumeration, unwind, the
 * brute-force search and the seeded instance generators.  Every function cites
 * the reference file:line it follows.
 *
 * It is the CHECKER for the CUDA product (libparplan_cuda.so): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product never links, calls or falls back to it.
 *
 * Parity pinning: tests/test_oracle_pin.py checks this restatement against
 * (a) the reference's own known-answer tests (restated as golden vectors in
 * tests/golden/kat.json), and (b) the real reference compiled from
 * /root/reference into oracle/_ref/libparplan_ref.so (oracle/Makefile), which
 * exports the same orc_* entry points, on every builtin and on seeded graphs.
 */
#ifndef PARPLAN_ORACLE_H
#define PARPLAN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layer kinds in reference variant order (graph.hpp:66-68). */
enum { ORC_INPUT = 0, ORC_CONV = 1, ORC_POOL = 2, ORC_FC = 3, ORC_FLATTEN = 4, ORC_CONCAT = 5, ORC_SOFTMAX = 6 };
#define ORC_NPARAM 7

typedef struct orc_instance orc_instance;

/* Last error message of this thread ("" if none). */
const char *orc_error(void);
/* 0 = restatement (port), 1 = compiled reference. */
int orc_kind(void);

/* ---- construction ----------------------------------------------------- */
/* Graph from flat arrays: params[l*7..] per kind (see product header
 * include/parplan_c.h for the layout), inputs given as (edge_src, edge_dst) in
 * creation order (layers ascending, then input position). ids may be NULL. */
orc_instance *orc_graph(int n_layers, int n_edges, int64_t batch, const int32_t *kind, const int64_t *params,
                        const int32_t *edge_src, const int32_t *edge_dst, const char *const *ids);
orc_instance *orc_builtin(const char *model, int64_t batch);
/* oracle.hpp:121-185 */
orc_instance *orc_random(uint64_t seed, int node_count, int max_configs, double branch_probability, int device_count);
/* SURVEY §9 config-5 generator: oracle.hpp draw order, catalogs {1,1,1,i+1}, i<C. */
orc_instance *orc_synthetic(uint64_t seed, int node_count, int configs, double branch_probability);
void orc_free(orc_instance *);

/* cost.hpp:170-206 with DeviceGraph(rates, bw) (graph.hpp:193-214). Returns 0 ok. */
int orc_build_tables(orc_instance *, int n_devices, const double *rates, const double *bw);
/* Inject hand-built tables: ncfg[l], configs (4 per config, layer-major),
 * node (flattened per layer), xfer (flattened per edge, row-major [src][dst]). */
int orc_set_tables(orc_instance *, const int32_t *ncfg, const int64_t *configs, const double *node, const double *xfer);

/* ---- accessors ---------------------------------------------------------- */
int orc_n_layers(const orc_instance *);
int orc_n_edges(const orc_instance *);
void orc_edges(const orc_instance *, int32_t *src, int32_t *dst, int32_t *pos);
void orc_shapes(const orc_instance *, int64_t *out4);
void orc_topo(const orc_instance *, int32_t *order);
int orc_config_count(const orc_instance *, int layer);
void orc_catalog(const orc_instance *, int layer, int64_t *out4);
void orc_node(const orc_instance *, int layer, double *out);
void orc_compute(const orc_instance *, int layer, double *out);
void orc_sync(const orc_instance *, int layer, double *out);
void orc_xfer(const orc_instance *, int edge, double *out);
/* Layer kind + params (7) + id; returns kind. */
int orc_layer(const orc_instance *, int layer, int64_t *params, char *id, int id_cap);

/* ---- single-call cost functions (cost.hpp:60-137) ----------------------- */
int orc_transfer_profile(const orc_instance *, int edge, const int64_t *c_src, const int64_t *c_dst, int n_devices,
                         const double *bw, double *seconds, double *bytes);
/* partition.hpp:213-232 / :283-350 ; out = lo[4], hi[4] */
int orc_owned_region(const int64_t *shape, const int64_t *config, int64_t part, int64_t *out8);
int orc_required_region(const orc_instance *, int edge, const int64_t *dst_config, int64_t part, int64_t *out8);
/* partition.hpp:174-204 ; returns count, writes up to cap configs */
int orc_enumerate_configs(int kind, const int64_t *shape, int device_count, int64_t *out4, int cap);

/* ---- planning (planner.hpp) --------------------------------------------- */
/* plan_with_tables (:339-366). stats = {final_nodes, node_elims, edge_elims}. 0 ok, 2 LimitError, 1 error. */
int orc_plan(orc_instance *, int k_bound, int32_t *indices, double *cost, int32_t *stats);
/* reduce only (:209-217), then log access */
int orc_reduce(orc_instance *);
/* ReducedGraph step API (:57-206): init, one node / edge elimination
 * (returns 1 acted, 0 none), edge ids created so far, {src,dst,alive}. */
int orc_rg_init(orc_instance *);
int orc_rg_node(orc_instance *);
int orc_rg_edge(orc_instance *);
int orc_rg_edges_total(const orc_instance *);
int orc_rg_edge_info(const orc_instance *, int edge, int32_t *info3);
int orc_log_size(const orc_instance *);
/* rec = {type(0 node,1 edge), removed, e1(in_edge), e2(out_edge), new_edge, src, dst} */
int orc_log_record(const orc_instance *, int r, int32_t *rec7);
int orc_log_argmin(const orc_instance *, int r, int32_t *out);
/* table of (possibly derived) edge id after reduce */
int orc_edge_table_dims(const orc_instance *, int edge, int32_t *dims2);
int orc_edge_table(const orc_instance *, int edge, double *out);
/* live_nodes of the reduced graph */
int orc_live_nodes(const orc_instance *, int32_t *out);
/* enumerate_final (:256-304) on the reduced graph */
int orc_enumerate_final(orc_instance *, int k_bound, int32_t *idx, double *cost);
/* total_cost_by_index (cost.hpp:235-246) */
double orc_total_cost(const orc_instance *, const int32_t *indices);
/* brute_force_plan (oracle.hpp:52-93). 0 ok, 2 LimitError */
int orc_brute(const orc_instance *, uint64_t budget, int32_t *indices, double *cost, uint64_t *visited);

/* One Eq. 2 fold on raw tables (planner.hpp:139-155): out[nu*nv], argmin[nu*nv]. */
void orc_fold(int nu, int nw, int nv, const double *w, const double *t1, const double *t2, double *out, int32_t *argmin);

#ifdef __cplusplus
}
#endif
#endif
