// tables.hpp — device-resident cost tables (CostTables, cost.hpp:148-168).
#pragma once

#include <functional>

#include "device.hpp"

#include <cstdint>
#include <vector>

namespace pp {

enum Mode : int { kFixed = 0, kFP64 = 1 };

struct Tables {
  pp_context *ctx = nullptr;
  int nl = 0, ne = 0;
  std::vector<int> esrc, edst;
  std::vector<int32_t> counts;
  std::vector<int64_t> cat_off; // per layer, prefix over counts
  std::vector<int64_t> configs; // host copy, 4 per config
  std::vector<int64_t> xoff;    // per edge, offset (cells) into the xfer arena
  int64_t xcells = 0, ncells = 0;
  int mode = kFP64;
  int shift = 0;         // fixed point: value = units * 2^-shift
  bool analytic = false; // compute/sync split available
  // FP64 storage
  DBuf<double> node, compute, sync, xfer64;
  // fixed-point storage (int32 units)
  DBuf<int32_t> node32, xfer32;
  // fixed point: per-original-table bounds used by the fold-kernel selector
  std::vector<int64_t> node_span;           // max - min per layer (units)
  std::vector<int64_t> row_span, col_span;  // per edge: max over rows of (row max - row min), same for columns
  std::vector<int64_t> absmax_node, absmax_edge;
  double build_ms = 0.0;

  int64_t xfer_bytes() const { return xcells * (mode == kFP64 ? 8 : 4); }
};

// ---- K1/K2 launch descriptors ------------------------------------------------

struct LayerDev {
  int64_t shape[4];
  int64_t in_shape[4];
  int64_t params[7];
  int64_t cat_off;
  int32_t kind;
  int32_t count;
};

struct EdgeDev {
  int64_t sshape[4];
  int64_t dshape[4];
  int64_t params[7];
  int64_t band;
  int64_t cat_u, cat_v;
  int64_t out_off;
  int64_t cells;
  int64_t blk_begin;
  int32_t kind;
  int32_t nu, nv;
  int32_t pad;
};

struct BuildArgs {
  const LayerDev *layers;
  const EdgeDev *edges;
  const int32_t *cfg; // 4 per config (degrees <= device count)
  const double *rates;
  const double *bw; // D*D
  double *node, *compute, *sync, *xfer;
  int64_t ncells;
  int32_t nl, ne, D;
  int32_t node_blocks;
  double bw_uniform; // > 0 when every off-diagonal bandwidth is this value
  int64_t edge_block0; // first edge block of this launch (row-sharded plans build an edge range per rank)
};

struct BuildPlan {
  std::vector<LayerDev> L;
  std::vector<EdgeDev> E;
  int64_t node_blocks = 0, grid = 0;
  double bw_uniform = 0.0;
  int D = 0;
  std::vector<double> rates, bw; // the device graph, for plans that embed it
  const std::vector<int32_t> *cfg32 = nullptr; // catalogs as the kernels read them (the graph's cache)
};

// Fills t's layout (catalogs, offsets; FP64 analytic mode, no allocation) and
// the K1/K2 launch descriptors for graph g on devices dev.
BuildPlan plan_build(Tables &t, const Graph &g, const pp_device_desc *dev, bool host_configs = true);
void launch_build(pp_context *ctx, cudaStream_t st, const BuildArgs &a, int64_t grid);

// Decides fixed point vs FP64 for host tables and fills the span bounds.
// Returns true when every value is k * 2^-s (s <= 24) and every possible sum
// of one entry per table stays below 2^31 units (the exactness certificate).
bool certify_fixed_point(const std::vector<double> &node, const std::vector<int64_t> &node_off,
                         const std::vector<double> &xfer, const std::vector<int64_t> &xoff,
                         const std::vector<int32_t> &counts, const std::vector<int> &esrc,
                         const std::vector<int> &edst, int *shift);

// fixed-C fixed-point tables streamed from a host generator (generators.cpp)
pp_tables *tables_fixed_streamed(pp_context *ctx, const Graph &g, int32_t C, int shift, int64_t vmax,
                                 const std::function<void(int32_t *, size_t)> &gen);
void compute_spans_fixed(Tables &t, const std::vector<int32_t> &node_units, const std::vector<int32_t> &xfer_units);

} // namespace pp

struct pp_tables {
  pp::Tables impl;
};
