/* parplan/runtime.hpp — glue between the reference-compatible C++ API and the
 * C ABI of libparplan_cuda.so (include/parplan_c.h).
 *
 * Not part of the reference API.  It owns the process-wide default planner
 * context (device = $PARPLAN_DEVICE or 0), maps pp_status codes back to the
 * reference's exceptions (InputError / LimitError, base.hpp:38-48), and
 * marshals ComputationGraph / DeviceGraph / CostTables into the flat ABI
 * structures.  Link with -lparplan_cuda.
 */
#pragma once

#include "parplan/graph.hpp"
#include "parplan_c.h"

#include <cstdlib>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace parplan {

/// A CUDA failure or a missing device (the planner has no CPU fallback).
class DeviceError : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

namespace runtime {

inline void check(pp_status st) {
  if (st == PP_OK) return;
  const std::string msg = pp_last_error();
  if (st == PP_ERR_INPUT) throw InputError(msg);
  if (st == PP_ERR_LIMIT) throw LimitError(msg);
  if (st == PP_ERR_CUDA) throw DeviceError(msg);
  throw std::runtime_error(msg);
}

/// The process-wide planner context (created on first use).
inline pp_context *context() {
  static std::once_flag once;
  static pp_context *ctx = nullptr;
  std::call_once(once, [] {
    const char *env = std::getenv("PARPLAN_DEVICE");
    check(pp_context_create(env ? std::atoi(env) : 0, &ctx));
  });
  return ctx;
}

struct GraphDeleter {
  void operator()(pp_graph *g) const { pp_graph_destroy(g); }
};
struct TablesDeleter {
  void operator()(pp_tables *t) const { pp_tables_destroy(t); }
};
struct ReducedDeleter {
  void operator()(pp_reduced *r) const { pp_reduced_destroy(r); }
};
using GraphHandle = std::unique_ptr<pp_graph, GraphDeleter>;
using TablesHandle = std::unique_ptr<pp_tables, TablesDeleter>;
using ReducedHandle = std::unique_ptr<pp_reduced, ReducedDeleter>;

/// The graph as the ABI sees it (ComputationGraph::create inputs, flattened).
inline GraphHandle native(const ComputationGraph &g) {
  const int n = g.layer_count();
  std::vector<const char *> ids;
  std::vector<int32_t> kind;
  std::vector<int64_t> params(static_cast<size_t>(n) * 7);
  std::vector<int32_t> src, dst;
  for (int l = 0; l < n; ++l) {
    ids.push_back(g.layer(l).id.c_str());
    kind.push_back(static_cast<int32_t>(g.layer(l).kind.index()));
    detail::kind_params(g.layer(l).kind, &params[static_cast<size_t>(l) * 7]);
  }
  for (const Edge &e : g.edges()) {
    src.push_back(e.src);
    dst.push_back(e.dst);
  }
  pp_graph_desc d{n, g.edge_count(), g.batch(), ids.data(), kind.data(), params.data(), src.data(), dst.data()};
  pp_graph *out = nullptr;
  check(pp_graph_create(&d, &out));
  return GraphHandle(out);
}

inline pp_device_desc device_desc(const DeviceGraph &d) {
  return pp_device_desc{d.count(), d.rates().data(), d.bandwidths().data()};
}

} // namespace runtime
} // namespace parplan
