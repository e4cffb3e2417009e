// dp.hpp — device DP entry points used by the C ABI (plan_api.cu).
#pragma once

#include "tables.hpp"

#include <vector>

namespace pp {

// plan_with_tables (t given) or plan (dev given: K1/K2 first) on the device:
// waves of K3/K4, K5, unwind, cost re-sum — one-shot, from the context pools.
void run_plan(pp_context *ctx, Graph &g, Tables *t, const pp_device_desc *dev, int k_bound, int32_t *indices,
              pp_plan_result *res);

// K5 over an explicit node/edge list (ReducedGraph::enumerate_final, brute force).
void run_enumerate(pp_context *ctx, int mode, int shift, const std::vector<const void *> &node_tabs,
                   const std::vector<int32_t> &counts, const std::vector<const void *> &edge_tabs,
                   const std::vector<int32_t> &eps, const std::vector<int32_t> &epd, const std::vector<int32_t> &ecols,
                   int32_t *digits, double *cost);

// One fold (op.type 0) or merge (op.type 1), synchronously.
void run_single_op(pp_context *ctx, int mode, const Op &op, const void *t1, const void *t2, const void *w, void *out,
                   uint16_t *am, int nu, int nw, int nv);

void download_table(pp_context *ctx, int mode, int shift, const void *src, int64_t n, double *out);
void download_argmin(pp_context *ctx, const uint16_t *src, int64_t n, int32_t *out);

} // namespace pp
