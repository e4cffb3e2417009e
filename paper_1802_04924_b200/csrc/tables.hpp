// tables.hpp — device-resident cost tables (CostTables, cost.hpp:148-168).
#pragma once

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

// Decides fixed point vs FP64 for host tables and fills the span bounds.
// Returns true when every value is k * 2^-s (s <= 24) and every possible sum
// of one entry per table stays below 2^31 units (the exactness certificate).
bool certify_fixed_point(const std::vector<double> &node, const std::vector<int64_t> &node_off,
                         const std::vector<double> &xfer, const std::vector<int64_t> &xoff,
                         const std::vector<int32_t> &counts, const std::vector<int> &esrc,
                         const std::vector<int> &edst, int *shift);

void compute_spans_fixed(Tables &t, const std::vector<int32_t> &node_units, const std::vector<int32_t> &xfer_units);

} // namespace pp

struct pp_tables {
  pp::Tables impl;
};
