// parplan — command-line front end of the GPU planner, a drop-in for the
// reference CLI (proj/tools/parplan_main.cpp): subcommands plan / brute /
// eval / compare / emit-model, the same options, JSON documents, text
// reports and exit codes (0 ok, 2 input or usage error, 3 limit error).
// Tables, plans and the brute force run on the B200 through the drop-in
// headers (libparplan_cuda.so); argument parsing is self-contained (the
// reference uses CLI11, which this image lacks).
#include "parplan/parplan.hpp"

#include <chrono>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace {

using namespace parplan;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- argument parsing ---------------------------------------------------------

struct Options {
  std::string model, network_file, device_file, cost_file, out_file, strategy_file;
  int devices = 1;
  i64 batch = 32;
  int k_bound = kDefaultFinalGraphBound;
  u64 budget = kDefaultBruteForceBudget;
  bool json = false, bytes = false;
  std::set<std::string> given; // options present on the command line
};

struct Command {
  std::string name, help;
  bool graph_exclusive = true; // --model and --network exclude each other
  std::vector<std::string> extra;  // subcommand-specific valued options
  std::vector<std::string> required;
};

const std::vector<Command> &commands() {
  static const std::vector<Command> c = {
      {"plan", "find the minimum-cost parallelization strategy", true, {"--k-bound"}, {}},
      {"brute", "exhaustive search over all joint configurations", true, {"--budget"}, {}},
      {"eval", "evaluate a strategy file's cost", true, {"--strategy"}, {"--strategy"}},
      {"compare", "cost table over data/model/owt baselines and the optimum", true, {"--k-bound"}, {}},
      {"emit-model", "write a builtin model as network JSON", false, {}, {}},
  };
  return c;
}

const std::vector<std::string> kValued = {"--model", "--network", "--devices", "--device-file",
                                          "--batch", "--cost-file", "--out"};
const std::vector<std::string> kFlags = {"--json", "--bytes"};

void usage(std::ostream &os, const Command *cmd) {
  if (!cmd) {
    os << "layer-wise parallelization planner for CNN computation graphs on modeled device clusters\n"
          "usage: parplan <plan|brute|eval|compare|emit-model> [options]\n";
    for (const Command &c : commands()) os << "  " << c.name << "  " << c.help << "\n";
    return;
  }
  os << "usage: parplan " << cmd->name << " [options]\n  " << cmd->help << "\n"
     << "  --model NAME        builtin model (lenet5, alexnet, vgg16, inception_chain[(K)])\n"
     << "  --network FILE      network JSON file\n"
     << "  --devices N         number of identical modeled devices\n"
     << "  --device-file FILE  device JSON file\n"
     << "  --batch N           batch size (default 32)\n"
     << "  --cost-file FILE    measured cost JSON overriding the analytic tables\n"
     << "  --out FILE          write the strategy JSON to this file\n"
     << "  --json              machine-readable output on stdout\n"
     << "  --bytes             also report raw cross-device bytes\n";
  for (const std::string &x : cmd->extra) os << "  " << x << " VALUE\n";
}

template <class I> I parse_int(const std::string &opt, const std::string &v) {
  try {
    size_t used = 0;
    const long long x = std::stoll(v, &used);
    if (used != v.size()) throw UsageError(opt + ": invalid number '" + v + "'");
    return static_cast<I>(x);
  } catch (const std::logic_error &) {
    throw UsageError(opt + ": invalid number '" + v + "'");
  }
}

// Returns the parsed command, or nullptr after printing help.
const Command *parse(int argc, char **argv, Options &o) {
  if (argc < 2) throw UsageError("a subcommand is required");
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    usage(std::cout, nullptr);
    return nullptr;
  }
  const Command *cmd = nullptr;
  for (const Command &c : commands())
    if (c.name == sub) cmd = &c;
  if (!cmd) throw UsageError("unknown subcommand '" + sub + "'");
  auto is = [](const std::vector<std::string> &v, const std::string &x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], val;
    bool has_val = false;
    if (const size_t eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos)
      val = a.substr(eq + 1), a = a.substr(0, eq), has_val = true;
    if (a == "-h" || a == "--help") {
      usage(std::cout, cmd);
      return nullptr;
    }
    if (is(kFlags, a)) {
      if (has_val) throw UsageError(a + " takes no value");
      (a == "--json" ? o.json : o.bytes) = true;
      o.given.insert(a);
      continue;
    }
    if (!is(kValued, a) && !is(cmd->extra, a)) throw UsageError("unknown option '" + a + "' for '" + cmd->name + "'");
    if (!has_val) {
      if (i + 1 >= argc) throw UsageError(a + " needs a value");
      val = argv[++i];
    }
    o.given.insert(a);
    if (a == "--model") o.model = val;
    else if (a == "--network") o.network_file = val;
    else if (a == "--devices") o.devices = parse_int<int>(a, val);
    else if (a == "--device-file") o.device_file = val;
    else if (a == "--batch") {
      o.batch = parse_int<i64>(a, val);
      if (o.batch <= 0) throw UsageError("--batch: value must be positive");
    } else if (a == "--cost-file") o.cost_file = val;
    else if (a == "--out") o.out_file = val;
    else if (a == "--k-bound") o.k_bound = parse_int<int>(a, val);
    else if (a == "--budget") o.budget = parse_int<u64>(a, val);
    else if (a == "--strategy") o.strategy_file = val;
  }
  if (cmd->graph_exclusive && o.given.count("--model") && o.given.count("--network"))
    throw UsageError("--model excludes --network");
  if (o.given.count("--devices") && o.given.count("--device-file")) throw UsageError("--devices excludes --device-file");
  for (const std::string &r : cmd->required)
    if (!o.given.count(r)) throw UsageError(r + " is required");
  return cmd;
}

// ---- subcommands --------------------------------------------------------------

ComputationGraph load_graph(const Options &o) {
  if (!o.network_file.empty()) return parse_network_file(o.network_file, o.given.count("--batch") ? o.batch : 0);
  if (!o.model.empty()) return builtin_model(o.model, o.batch);
  throw InputError("one of --model or --network is required");
}

DeviceGraph load_devices(const Options &o) {
  return o.device_file.empty() ? DeviceGraph::uniform(o.devices) : parse_device_file(o.device_file);
}

CostTables load_tables(const ComputationGraph &g, const DeviceGraph &d, const Options &o) {
  CostTables t = build_cost_tables(g, d);
  if (!o.cost_file.empty()) apply_measured_costs_file(o.cost_file, g, t);
  return t;
}

void write_doc(const std::string &path, const json &doc) {
  std::ofstream out(path);
  if (!out) throw InputError("cannot write '" + path + "'");
  out << doc.dump(2) << "\n";
}

int plan_like(const Options &o, bool brute) {
  const ComputationGraph g = load_graph(o);
  const DeviceGraph d = load_devices(o);
  const CostTables t = load_tables(g, d, o);
  const auto t0 = std::chrono::steady_clock::now();
  Strategy s;
  double cost = 0.0;
  int elims = 0, final_nodes = 0;
  u64 visited = 0;
  if (brute) {
    BruteForceResult r = brute_force_plan(g, t, o.budget);
    s = std::move(r.strategy), cost = r.cost, visited = r.visited;
    final_nodes = g.layer_count();
  } else {
    PlanResult r = plan_with_tables(g, t, o.k_bound);
    s = std::move(r.strategy), cost = r.cost;
    elims = r.eliminations(), final_nodes = r.final_graph_nodes;
  }
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  json doc = strategy_json(g, s, cost, elims, final_nodes);
  if (brute) doc["strategies_visited"] = visited;
  if (!o.out_file.empty()) write_doc(o.out_file, doc);
  if (o.json) {
    std::cout << doc.dump(2) << "\n";
  } else {
    Report rep = make_report(brute ? "brute-force optimal" : "optimal", g, t, s, d, o.bytes);
    rep.planning_ms = ms, rep.final_graph_nodes = final_nodes, rep.eliminations = elims;
    render_report(std::cout, rep);
  }
  return 0;
}

int eval(const Options &o) {
  const ComputationGraph g = load_graph(o);
  const DeviceGraph d = load_devices(o);
  const CostTables t = load_tables(g, d, o);
  const Strategy s = parse_strategy_file(o.strategy_file, g);
  for (int l = 0; l < g.layer_count(); ++l)
    if (t.config_index(l, s[static_cast<size_t>(l)]) < 0)
      throw InputError("config " + to_string(s[static_cast<size_t>(l)]) + " is not valid for layer '" + g.layer(l).id +
                       "'");
  const Report rep = make_report(o.strategy_file, g, t, s, d, o.bytes);
  if (o.json)
    std::cout << report_json(rep).dump(2) << "\n";
  else
    render_report(std::cout, rep);
  return 0;
}

int compare(const Options &o) {
  const ComputationGraph g = load_graph(o);
  const DeviceGraph d = load_devices(o);
  const CostTables t = load_tables(g, d, o);
  std::vector<std::pair<std::string, Strategy>> rows;
  for (BaselineKind k : {BaselineKind::Data, BaselineKind::Model, BaselineKind::Owt})
    rows.emplace_back(baseline_name(k), baseline_strategy(k, g, d));
  rows.emplace_back("optimal", plan_with_tables(g, t, o.k_bound).strategy);
  std::vector<Report> reps;
  json out = json::array();
  for (const auto &[name, s] : rows) {
    Report rep = make_report(name, g, t, s, d, o.bytes);
    json rj;
    rj["strategy"] = name;
    rj["cost_seconds"] = rep.total;
    rj["node_seconds"] = rep.node_total;
    rj["transfer_seconds"] = rep.xfer_total;
    if (rep.has_split) {
      rj["compute_seconds"] = rep.compute_total;
      rj["sync_seconds"] = rep.sync_total;
      rj["communication_seconds"] = rep.sync_total + rep.xfer_total;
    }
    if (o.bytes) {
      rj["transfer_bytes"] = rep.xfer_bytes;
      rj["sync_bytes"] = rep.sync_bytes;
      rj["communication_bytes"] = rep.xfer_bytes + rep.sync_bytes;
    }
    out.push_back(std::move(rj));
    reps.push_back(std::move(rep));
  }
  if (o.json) {
    std::cout << out.dump(2) << "\n";
    return 0;
  }
  const bool split = reps.front().has_split;
  std::cout << std::left << std::setw(10) << "strategy" << std::right << std::setw(16) << "total s" << std::setw(16)
            << "node s" << std::setw(16) << "transfer s";
  if (split) std::cout << std::setw(16) << "comm s";
  if (o.bytes) std::cout << std::setw(18) << "comm bytes";
  std::cout << "\n" << std::scientific << std::setprecision(6);
  for (const Report &r : reps) {
    std::cout << std::left << std::setw(10) << r.label << std::right << std::setw(16) << r.total << std::setw(16)
              << r.node_total << std::setw(16) << r.xfer_total;
    if (r.has_split) std::cout << std::setw(16) << r.sync_total + r.xfer_total;
    if (o.bytes) std::cout << std::setw(18) << r.xfer_bytes + r.sync_bytes;
    std::cout << "\n";
  }
  return 0;
}

int emit_model(const Options &o) {
  if (o.model.empty()) throw InputError("emit-model requires --model");
  const json doc = emit_network(load_graph(o));
  if (!o.out_file.empty())
    write_doc(o.out_file, doc);
  else
    std::cout << doc.dump(2) << "\n";
  return 0;
}

} // namespace

int main(int argc, char **argv) {
  Options o;
  const Command *cmd = nullptr;
  try {
    cmd = parse(argc, argv, o);
  } catch (const UsageError &e) {
    std::cerr << "error: " << e.what() << "\n";
    usage(std::cerr, nullptr);
    return 2;
  }
  if (!cmd) return 0; // help printed
  try {
    const std::map<std::string, std::function<int()>> run = {
        {"plan", [&] { return plan_like(o, false); }},
        {"brute", [&] { return plan_like(o, true); }},
        {"eval", [&] { return eval(o); }},
        {"compare", [&] { return compare(o); }},
        {"emit-model", [&] { return emit_model(o); }},
    };
    return run.at(cmd->name)();
  } catch (const LimitError &e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception &e) { // InputError, CUDA errors, I/O
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
