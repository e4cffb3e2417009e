// internal.hpp — shared internals of libparplan_cuda.so (not installed).
#pragma once

#include "parplan_c.h"
#include "scheduler.hpp"

#include "parplan/graph.hpp"
#include "parplan/partition.hpp"

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace pp {

// ---- errors -----------------------------------------------------------------

struct Error : std::runtime_error {
  pp_status code;
  Error(pp_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(pp_status c, const std::string &m) { throw Error(c, m); }

void set_last_error(const std::string &m);

// Runs f, mapping exceptions to status codes + the thread-local message.
template <class F> pp_status guard(F &&f) {
  try {
    f();
    set_last_error("");
    return PP_OK;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.code;
  } catch (const parplan::LimitError &e) {
    set_last_error(e.what());
    return PP_ERR_LIMIT;
  } catch (const parplan::InputError &e) {
    set_last_error(e.what());
    return PP_ERR_INPUT;
  } catch (const std::bad_alloc &) {
    set_last_error("out of host memory");
    return PP_ERR_INTERNAL;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return PP_ERR_INTERNAL;
  }
}

#define PP_REQUIRE(cond, msg)                                                                                         \
  do {                                                                                                                 \
    if (!(cond)) ::pp::fail(PP_ERR_INPUT, msg);                                                                        \
  } while (0)

// ---- graph ------------------------------------------------------------------

// A validated ComputationGraph plus the flat views the kernels consume.
struct Graph {
  parplan::ComputationGraph g;
  int nl = 0, ne = 0;
  std::vector<int32_t> kind;
  std::vector<int64_t> params; // 7 per layer
  std::vector<int64_t> shape;  // 4 per layer
  std::vector<int> esrc, edst, epos, rank;
  std::vector<int64_t> band_offset; // per edge, Concat destinations
  std::unique_ptr<Schedule> sched;  // lazily built, topology-only
  // enumerate_configs of every layer for a device count (pure function of the
  // immutable graph and D): counts, configs (4 x int64), configs (4 x int32)
  struct Catalogs {
    std::vector<int32_t> counts;
    std::vector<int64_t> configs;
    std::vector<int32_t> configs32;
  };
  mutable std::map<int, Catalogs> catalog_cache;
  mutable std::mutex lazy; // the schedule and catalog caches (a graph may be shared across threads)

  explicit Graph(parplan::ComputationGraph cg);
  const Schedule &schedule();
  const Catalogs &catalogs(int devices) const;
};

// Catalogs of every layer (enumerate_configs) flattened: counts + 4 int64 each.
void enumerate_catalogs(const Graph &g, int devices, std::vector<int32_t> *counts, std::vector<int64_t> *configs);

} // namespace pp

// A handle on an immutable graph.  Handles created from equal descriptors
// share one pp::Graph (graph_api.cpp: content-addressed cache), so repeated
// plans of the same network skip shape inference, catalogs and the schedule.
struct pp_graph {
  std::shared_ptr<pp::Graph> own;
  pp::Graph &impl;
  explicit pp_graph(parplan::ComputationGraph cg) : own(std::make_shared<pp::Graph>(std::move(cg))), impl(*own) {}
  explicit pp_graph(std::shared_ptr<pp::Graph> g) : own(std::move(g)), impl(*own) {}
};
