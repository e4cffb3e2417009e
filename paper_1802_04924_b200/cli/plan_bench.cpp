// plan_bench — per-call latency of the drop-in C++ API, as a reference caller
// pays it: every timed call builds the model graph and runs
// parplan::plan(graph, DeviceGraph::uniform(D)) (planner.hpp:368-371; the
// reference's acceptance C5 times exactly this, acceptance.cpp:292-303), so the
// drop-in's pp_graph, catalogs and schedule are rebuilt per call, unlike the
// cached-graph pp_plan number of bench.py.  Graphs equal to a recent one share
// its host work (content-addressed cache in the library): "dropin_plan" is the
// repeated call, "dropin_plan_cold" a graph never seen before (a new batch size
// per call).  Also times acceptance C4's pair
// (brute_force_plan vs plan_with_tables on host CostTables, lenet5@4).
//
//   plan_bench [runs=20] [warmup=3]   -> one JSON object per line on stdout
#include "parplan/models.hpp"
#include "parplan/oracle.hpp"
#include "parplan/planner.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

using namespace parplan;
using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

static void stats(const char *label, const std::string &workload, std::vector<double> v, double cost) {
  std::sort(v.begin(), v.end());
  double sum = 0.0;
  for (double x : v) sum += x;
  std::printf("{\"kind\": \"%s\", \"workload\": \"%s\", \"runs\": %zu, \"median_ms\": %.6f, \"mean_ms\": %.6f, "
              "\"min_ms\": %.6f, \"max_ms\": %.6f, \"cost\": \"%a\"}\n",
              label, workload.c_str(), v.size(), v[v.size() / 2], sum / static_cast<double>(v.size()), v.front(),
              v.back(), cost);
  std::fflush(stdout);
}

int main(int argc, char **argv) {
  const int runs = argc > 1 ? std::atoi(argv[1]) : 20;
  const int warmup = argc > 2 ? std::atoi(argv[2]) : 3;
  struct W {
    std::string name;
    int modules; // inception_chain modules; 0: by name
    int devices;
  };
  const std::vector<W> ws = {{"inception_chain", 12, 16}, {"inception_chain", 12, 64}, {"inception_chain", 13, 16},
                             {"vgg16", 0, 16},            {"alexnet", 0, 4},            {"lenet5", 0, 4}};
  for (const W &w : ws) {
    auto build = [&] {
      return w.modules ? models::inception_chain(32, w.modules) : builtin_model(w.name, 32);
    };
    const std::string label = (w.modules ? "inception_chain(" + std::to_string(w.modules) + ")" : w.name) + "@" +
                              std::to_string(w.devices);
    std::vector<double> t;
    double cost = 0.0;
    for (int k = 0; k < warmup + runs; ++k) {
      const auto t0 = Clock::now();
      const ComputationGraph g = build();
      const DeviceGraph d = DeviceGraph::uniform(w.devices);
      const PlanResult p = plan(g, d);
      const double dt = ms_since(t0);
      cost = p.cost;
      if (k >= warmup) t.push_back(dt);
    }
    stats("dropin_plan", label, t, cost);
    // cold: a graph the library has not seen (batch 33, 34, ...: new shapes, so
    // no content-cache hit — shape inference, catalogs and the schedule per call)
    std::vector<double> tc;
    for (int k = 0; k < runs; ++k) {
      const int64_t batch = 33 + static_cast<int64_t>(w.devices) * 1000 + k;
      const auto t0 = Clock::now();
      const ComputationGraph g =
          w.modules ? models::inception_chain(batch, w.modules) : builtin_model(w.name, batch);
      const PlanResult p = plan(g, DeviceGraph::uniform(w.devices));
      tc.push_back(ms_since(t0));
      (void)p;
    }
    stats("dropin_plan_cold", label, tc, 0.0);
  }
  { // acceptance C4's pair on host CostTables (acceptance.cpp:258-268)
    const ComputationGraph g = models::lenet5(32);
    const CostTables tables = build_cost_tables(g, DeviceGraph::uniform(4));
    std::vector<double> tb, tp;
    double cb = 0.0, cp = 0.0;
    for (int k = 0; k < warmup + runs; ++k) {
      auto t0 = Clock::now();
      const auto b = brute_force_plan(g, tables);
      const double db = ms_since(t0);
      t0 = Clock::now();
      const auto p = plan_with_tables(g, tables);
      const double dp = ms_since(t0);
      cb = b.cost, cp = p.cost;
      if (k >= warmup) tb.push_back(db), tp.push_back(dp);
    }
    stats("brute_force_plan", "lenet5@4", tb, cb);
    stats("plan_with_tables", "lenet5@4", tp, cp);
  }
  return 0;
}
