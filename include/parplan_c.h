/*
 * parplan_c.h — the C ABI of libparplan_cuda.so, the B200 (sm_100a) planner.
 *
 * This is the drop-in boundary.  The reference `parplan` is a header-only
 * C++20 library with no FFI of its own; its hot path is four calls
 * (citations relative to /root/reference/proj/include/parplan/):
 *
 *   ComputationGraph::create           graph.hpp:123-125, :263-360
 *   build_cost_tables                  cost.hpp:170-206
 *   ReducedGraph (step API) / reduce   planner.hpp:55-245
 *   enumerate_final / unwind           planner.hpp:256-319
 *   plan_with_tables / plan            planner.hpp:339-371
 *   brute_force_plan                   oracle.hpp:52-93
 *
 * Every one of them maps onto an entry point below.  The C++ drop-in headers in
 * include/parplan/ *.hpp keep the reference API (same namespace, types and
 * signatures) and call through this ABI; a Python/ctypes or any other FFI
 * binds it directly.
 *
 * Conventions
 *   - every function returns a pp_status; on failure pp_last_error() holds a
 *     message matching the reference exception text (InputError -> PP_ERR_INPUT,
 *     LimitError -> PP_ERR_LIMIT);
 *   - plain pointers and sizes only; arrays are caller-allocated;
 *   - a pp_context owns one CUDA device + stream and is single-threaded; every
 *     call is synchronous from the caller's point of view;
 *   - there is no CPU fallback: calls that compute tables or plans fail with
 *     PP_ERR_CUDA when no usable sm_100 device is present.  Graph construction,
 *     catalog enumeration and the symbolic elimination schedule are host logic
 *     and work without a GPU.
 */
#ifndef PARPLAN_C_H
#define PARPLAN_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 1

typedef enum pp_status {
  PP_OK = 0,
  PP_ERR_INPUT = 1,    /* parplan::InputError (base.hpp:38-41) */
  PP_ERR_LIMIT = 2,    /* parplan::LimitError (base.hpp:45-48) */
  PP_ERR_CUDA = 3,     /* no device / CUDA failure */
  PP_ERR_INTERNAL = 4, /* bug */
} pp_status;

/* Layer kinds, in the order of the reference LayerKind variant (graph.hpp:66-68). */
enum {
  PP_KIND_INPUT = 0,
  PP_KIND_CONV2D = 1,
  PP_KIND_POOL2D = 2,
  PP_KIND_FULLY_CONNECTED = 3,
  PP_KIND_FLATTEN = 4,
  PP_KIND_CONCAT = 5,
  PP_KIND_SOFTMAX = 6,
};

/* Per-layer parameter block: PP_NPARAM int64 values.
 *   input:           {channel, height, width}                       (graph.hpp:33-37)
 *   conv2d:          {out_channels, kh, kw, sh, sw, ph, pw}         (graph.hpp:39-44)
 *   pool2d:          {kh, kw, sh, sw, ph, pw}                       (graph.hpp:46-50)
 *   fully_connected: {out_channels}                                 (graph.hpp:52-54)
 *   concat:          {axis}  0 sample, 1 channel, 2 height, 3 width (graph.hpp:60-62)
 *   flatten/softmax: {}                                                              */
#define PP_NPARAM 7

/* Precision policy of the elimination DP.
 *   AUTO:  exact fixed point (int32 units of 2^-s) when the host certificate
 *          proves every sum exact (dyadic tables, e.g. the seeded generators),
 *          FP64 otherwise (analytic tables).  Both are bit-identical to the
 *          reference's FP64 arithmetic.
 *   FP64:  always FP64. */
enum { PP_PRECISION_AUTO = 0, PP_PRECISION_FP64 = 1 };

typedef struct pp_context pp_context;
typedef struct pp_graph pp_graph;
typedef struct pp_tables pp_tables;
typedef struct pp_reduced pp_reduced;
typedef struct pp_prepared pp_prepared;

/* A computation graph as flat arrays (ComputationGraph::create inputs).
 * Edges are listed in creation order: by destination layer ascending, then by
 * input position — exactly the dense edge ids the reference assigns
 * (graph.hpp:305-318). */
typedef struct pp_graph_desc {
  int32_t n_layers;
  int32_t n_edges;
  int64_t batch;
  const char *const *ids; /* [n_layers] layer ids; NULL -> "n<i>" */
  const int32_t *kind;    /* [n_layers] PP_KIND_* */
  const int64_t *params;  /* [n_layers * PP_NPARAM] */
  const int32_t *edge_src;
  const int32_t *edge_dst;
} pp_graph_desc;

/* DeviceGraph(rates, bandwidth) (graph.hpp:193-214): modelled devices. */
typedef struct pp_device_desc {
  int32_t count;
  const double *compute_rates; /* [count] flop/s */
  const double *bandwidth;     /* [count*count] bytes/s, row-major [from][to] */
} pp_device_desc;

typedef struct pp_plan_result {
  double cost; /* evaluate_strategy on the input tables (planner.hpp:364) */
  int32_t final_graph_nodes;
  int32_t node_eliminations;
  int32_t edge_eliminations;
  int32_t precision; /* 0 fixed-point int32, 1 FP64 (what the DP ran in) */
  int32_t waves;     /* dependency waves the schedule executed in */
  int32_t launches;  /* kernel launches issued by this call */
  double device_ms;  /* CUDA-event time of the device work of this call */
  int64_t h2d_bytes; /* host->device bytes the call copied (descriptor image) */
  int64_t d2h_bytes; /* device->host bytes (indices + cost) */
} pp_plan_result;

/* One elimination record (planner.hpp:32-45). type 0 = node, 1 = edge. */
typedef struct pp_record {
  int32_t type;
  int32_t removed; /* node records: eliminated layer; -1 for edge records */
  int32_t e1;      /* node: in_edge;  edge: lower id */
  int32_t e2;      /* node: out_edge; edge: higher id */
  int32_t new_edge;
  int32_t src;
  int32_t dst;
  int32_t wave; /* dependency wave (1-based) the op executes in */
} pp_record;

/* ---- library ---------------------------------------------------------- */
const char *pp_last_error(void);
int pp_abi_version(void);
/* number of usable CUDA devices (0 on a machine without a GPU) */
pp_status pp_device_count(int32_t *count);

/* ---- context ---------------------------------------------------------- */
pp_status pp_context_create(int32_t device, pp_context **out);
/* Same, but every call is ordered on the caller's cudaStream_t (e.g. a
 * PyTorch stream), so the caller's CUDA events time the planner's work. */
pp_status pp_context_create_on_stream(int32_t device, void *cuda_stream, pp_context **out);
pp_status pp_context_stream(const pp_context *ctx, void **cuda_stream);
pp_status pp_context_destroy(pp_context *ctx);
pp_status pp_context_set_precision(pp_context *ctx, int32_t policy);
/* Bit mask.  0 (default): large certified fixed-point folds use the U16x2
 * min-plus kernels (optimistic operand caps, checked on the device; a plan
 * whose check fires is re-run with proven caps), plans without them one fused
 * cooperative kernel.  Bit 0: every fold uses the generic tiled kernel (parity
 * checks); bit 1: one launch per wave instead of the fused kernel; bit 2:
 * proven min-plus operand caps only. */
pp_status pp_context_set_kernel_policy(pp_context *ctx, int32_t policy);
/* Multi-GPU: one process per GPU.  Rank 0 creates a 128-byte NCCL unique id,
 * the caller broadcasts it (e.g. torch.distributed), every rank attaches.  A
 * context with nranks > 1 row-shards every plan: derived tables are split by
 * the rows of their source configs, folds compute only local rows, derived t2
 * operands are all-gathered over NVLink at re-association points, and the final
 * tables + argmins are all-gathered so every rank returns the same plan.
 * NCCL is loaded at run time (libnccl.so.2); no link-time dependency. */
pp_status pp_comm_unique_id(void *id128);
pp_status pp_context_attach_comm(pp_context *ctx, int32_t nranks, int32_t rank, const void *id128);
/* Virtual ranks: n contexts on ONE device run a row-sharded plan through the
 * multi-GPU code path (row blocks of c_u, all-gathers of derived t2 at
 * re-association points and of the final edges, the distributed unwind that
 * reads each record's argmin row from its owner rank), each all-gather being
 * one device-to-device copy per rank block.  Results equal the single-GPU
 * plan bit for bit.  pp_vgroup_plan: give exactly one of dev (build_cost_tables
 * + plan on every rank, planner.hpp:368-371) and t (plan_with_tables,
 * planner.hpp:339-364; the tables are shared by the ranks). */
typedef struct pp_vgroup pp_vgroup;
pp_status pp_vgroup_create(int32_t device, int32_t nranks, pp_vgroup **out);
pp_status pp_vgroup_plan(pp_vgroup *group, const pp_graph *g, const pp_device_desc *dev, pp_tables *t,
                         int32_t k_bound, int32_t *indices, pp_plan_result *res);
pp_status pp_vgroup_destroy(pp_vgroup *group);
/* Host-only (no GPU): the row-sharded layout a context with nranks ranks uses
 * for this graph and per-layer config counts — for every table id of the
 * elimination log (originals then derived): rows per rank block, this rank's
 * first row and row count; and every all-gather as (wave, table id): derived t2
 * before its fold's wave, then derived final edges at wave n_waves + 1.  Call
 * with NULL arrays to get n_tables / n_gathers. */
pp_status pp_shard_layout(const pp_graph *g, const int32_t *counts, int32_t nranks, int32_t rank, int32_t *n_tables,
                          int32_t *blk, int32_t *first, int32_t *local_rows, int32_t *n_gathers, int32_t *gather_wave,
                          int32_t *gather_table);
/* One-shot plans draw on grow-only device pools (no cudaMalloc on the steady
 * state path); this returns them to the device (e.g. after one very large plan). */
pp_status pp_context_release_pools(pp_context *ctx);
/* kernel launches issued on this context since creation */
pp_status pp_context_launch_count(const pp_context *ctx, int64_t *launches);

/* ---- graph (host) ------------------------------------------------------ */
pp_status pp_graph_create(const pp_graph_desc *desc, pp_graph **out);
/* builtin_model (models.hpp:141-165): lenet5, alexnet, vgg16, inception_chain[(k)] */
pp_status pp_graph_builtin(const char *name, int64_t batch, pp_graph **out);
pp_status pp_graph_destroy(pp_graph *g);
pp_status pp_graph_size(const pp_graph *g, int32_t *n_layers, int32_t *n_edges);
/* any output pointer may be NULL */
pp_status pp_graph_layers(const pp_graph *g, int32_t *kind, int64_t *params, int64_t *shapes4, int32_t *topo_order);
pp_status pp_graph_edges(const pp_graph *g, int32_t *src, int32_t *dst, int32_t *dst_input_pos);
/* copies layer i's id into buf (NUL-terminated, truncated to cap) */
pp_status pp_graph_layer_id(const pp_graph *g, int32_t layer, char *buf, int32_t cap);
/* enumerate_configs (partition.hpp:174-204) for every layer: counts[n_layers];
 * configs may be NULL (size query), else [sum(counts) * 4]. */
pp_status pp_graph_catalogs(const pp_graph *g, int32_t device_count, int32_t *counts, int64_t *configs);
/* The chosen config of every layer (4 int64 each: sample, channel, height,
 * width) for per-layer catalog indices — PlanResult::strategy (planner.hpp:325-334)
 * without copying the catalogs.  Catalogs are cached per (graph, device count);
 * graphs created from equal descriptors share those caches and the schedule. */
pp_status pp_graph_configs_at(const pp_graph *g, int32_t device_count, const int32_t *indices, int64_t *configs);
/* The symbolic elimination schedule (planner.hpp:111-217) computed by the
 * O((N+E) log N) host scheduler: the exact record sequence reduce() logs.
 * records may be NULL (size query). */
pp_status pp_graph_schedule(const pp_graph *g, int32_t *n_records, pp_record *records, int32_t *n_waves);

/* ---- seeded instances (oracle.hpp:98-185) ------------------------------- */
/* Series-parallel topology of random_series_parallel_graph for `seed`
 * (std::mt19937_64, the reference's draw order), without tables. */
pp_status pp_graph_series_parallel(uint64_t seed, int32_t node_count, double branch_probability, pp_graph **out);
/* random_series_parallel_graph (graph + dyadic tables, uploaded).  With
 * configs_override > 0 every catalog is C dummy configs {1,1,1,i+1} instead
 * of the truncated enumeration (the config-5 sweep generator). */
pp_status pp_random_instance(pp_context *ctx, uint64_t seed, int32_t node_count, int32_t max_configs,
                             double branch_probability, int32_t device_count, int32_t configs_override,
                             pp_graph **graph, pp_tables **tables);

/* ---- cost tables (device) ----------------------------------------------- */
/* build_cost_tables (cost.hpp:170-206): K2 node-cost fill + K1 xfer builder. */
pp_status pp_tables_build(pp_context *ctx, const pp_graph *g, const pp_device_desc *dev, pp_tables **out);
/* Hand-built / measured / generated tables (CostTables fields, flattened):
 * counts[n_layers]; configs [sum*4] (may be NULL); node [sum];
 * xfer: per edge id, row-major [count(src)][count(dst)], concatenated. */
pp_status pp_tables_upload(pp_context *ctx, const pp_graph *g, const int32_t *counts, const int64_t *configs,
                           const double *node, const double *xfer, pp_tables **out);
/* Seeded synthetic tables generated on the device (config-5 sweep at sizes the
 * host generator cannot feed): catalogs {1,1,1,i+1} i<configs, values
 * k/64, k = splitmix64(seed, table, cell) % 641. */
pp_status pp_tables_synthetic(pp_context *ctx, const pp_graph *g, int32_t configs, uint64_t seed, pp_tables **out);
/* FP64 variant (values (k + u) / 64 with a 53-bit fraction u: rejected by the
 * fixed-point certificate, like measured costs): exercises the FP64 large-table
 * fold (minplus64.cuh). */
pp_status pp_tables_synthetic64(pp_context *ctx, const pp_graph *g, int32_t configs, uint64_t seed, pp_tables **out);
pp_status pp_tables_destroy(pp_tables *t);
/* counts[n_layers]; xfer_cells = sum over edges of count(src)*count(dst) */
pp_status pp_tables_counts(const pp_tables *t, int32_t *counts, int64_t *xfer_cells);
/* Downloads the CostTables fields. Any pointer may be NULL. compute/sync are
 * zero for uploaded tables (the reference leaves them empty). */
pp_status pp_tables_download(pp_tables *t, int64_t *configs, double *node, double *compute, double *sync, double *xfer);
/* device time of the build call that produced t (ms), 0 for uploads */
pp_status pp_tables_build_ms(const pp_tables *t, double *ms);

/* ---- planning (device) -------------------------------------------------- */
/* plan() (planner.hpp:368-371): tables + reduce + enumerate_final + unwind.
 * indices[n_layers] receives the config index per layer.  A call repeated on
 * the same context with an equal graph, device description, k_bound, kernel
 * policy and knobs replays a prepared plan the context keeps (at most 4, LRU;
 * freed by pp_context_release_pools / pp_context_destroy): the descriptor image
 * is uploaded and the tables and the search rerun on the device every call.
 * PARPLAN_PLAN_CACHE=0 disables it. */
pp_status pp_plan(pp_context *ctx, const pp_graph *g, const pp_device_desc *dev, int32_t k_bound, int32_t *indices,
                  pp_plan_result *res);
/* plan_with_tables() (planner.hpp:339-366) */
pp_status pp_plan_with_tables(pp_context *ctx, const pp_graph *g, pp_tables *t, int32_t k_bound, int32_t *indices,
                              pp_plan_result *res);
/* Prepared plans — for callers that re-plan the same graph: the host work
 * (catalogs, the symbolic schedule, the memory plan, every launch descriptor)
 * runs once in prepare; launch enqueues only device work (one CUDA graph:
 * K1/K2 when built from a device graph, one wave kernel per dependency wave,
 * K5, unwind + cost re-sum, and the D2H of the result), optionally preceded by
 * the H2D of the descriptor image (upload_inputs != 0); fetch waits and
 * returns what pp_plan returns.  Give exactly one of dev / t. */
pp_status pp_plan_prepare(pp_context *ctx, const pp_graph *g, const pp_device_desc *dev, pp_tables *t, int32_t k_bound,
                          pp_prepared **out);
pp_status pp_plan_launch(pp_prepared *p, int32_t upload_inputs);
pp_status pp_plan_fetch(pp_prepared *p, int32_t *indices, pp_plan_result *res);
pp_status pp_plan_destroy(pp_prepared *p);
/* Runs the prepared device work once with a CUDA event between launches and
 * reports, per step: device ms, kind and algorithmic work (table cells for
 * K1/K2; sum of nu*nw*nv fold cells plus merge cells for folds; candidates for
 * K5; bytes for collectives).  n_steps receives the count.  Kinds: 0 K1/K2
 * tables, 1 wave of K3/K4 folds and merges, 2 K5 enumeration, 3 unwind + cost
 * re-sum, 5 min-plus memsets, 6 mp_prep / mp64_prep, 7 mp_minima, 8 mp_fold,
 * 9 mp_merge, 10 fused kernel (expanded into its phases: 11 tables, 12 wave,
 * 13 enumerate, 14 finish, 16 chain segment, then 10 for the residual),
 * 15 all-gather, 17 mp_chain, 18 mp64_fold, 19 K1 edge-range broadcast,
 * 20 all-reduce of the optimistic-cap overflow flag (row-sharded plans). */
pp_status pp_plan_profile(pp_prepared *p, int32_t cap, double *step_ms, int32_t *step_kind, double *step_work,
                          int32_t *n_steps);

/* evaluate_strategy by index (cost.hpp:235-255), computed on the device from the
 * device-resident tables in the pinned summation order. */
pp_status pp_tables_total_cost(pp_tables *t, const int32_t *indices, double *cost);

/* Batched evaluate_strategy / evaluate_components totals (cost.hpp:235-293) for
 * n strategies given as config indices indices[n][n_layers]: cost[s] summed in
 * the reference's order (nodes by layer, then edges by id), optionally the node
 * and transfer totals (each summed from 0.0 in the same order).  One device
 * thread per strategy; the `compare` sweeps of SURVEY §8f. */
pp_status pp_tables_evaluate_batch(pp_tables *t, int64_t n, const int32_t *indices, double *cost, double *node_total,
                                   double *xfer_total);
/* brute_force_plan (oracle.hpp:52-93) on the device; LimitError text matches. */
pp_status pp_brute_force(pp_context *ctx, const pp_graph *g, pp_tables *t, uint64_t budget, int32_t *indices,
                         double *cost, uint64_t *visited);

/* ---- ReducedGraph step API (planner.hpp:55-245) ------------------------- */
pp_status pp_reduced_create(pp_context *ctx, const pp_graph *g, pp_tables *t, pp_reduced **out);
pp_status pp_reduced_destroy(pp_reduced *rg);
pp_status pp_reduced_node_elimination(pp_reduced *rg, int32_t *acted);
pp_status pp_reduced_edge_elimination(pp_reduced *rg, int32_t *acted);
pp_status pp_reduced_reduce(pp_reduced *rg);
/* edges_total = original + created edge ids so far */
pp_status pp_reduced_counts(const pp_reduced *rg, int32_t *edges_total, int32_t *log_size, int32_t *live_nodes,
                            int32_t *live_edges);
pp_status pp_reduced_edge(const pp_reduced *rg, int32_t id, int32_t *src, int32_t *dst, int32_t *alive,
                          int32_t *rows, int32_t *cols);
pp_status pp_reduced_node_alive(const pp_reduced *rg, int32_t layer, int32_t *alive);
/* FP64 copy of edge id's table, row-major [rows*cols] */
pp_status pp_reduced_edge_table(pp_reduced *rg, int32_t id, double *out);
pp_status pp_reduced_log_record(const pp_reduced *rg, int32_t r, pp_record *out);
/* argmin of node record r, row-major [rows(src)*cols(dst)] */
pp_status pp_reduced_argmin(pp_reduced *rg, int32_t r, int32_t *out);
/* enumerate_final (planner.hpp:256-304): idx[live_nodes] ascending layer order */
pp_status pp_reduced_enumerate_final(pp_reduced *rg, int32_t k_bound, int32_t *idx, double *cost);

#ifdef __cplusplus
}
#endif
#endif /* PARPLAN_C_H */
