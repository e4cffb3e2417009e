"""Small, ncu-friendly workloads (one process, one GPU).

  python tools/profile_run.py search   # plan(inception_chain(12)@16): K1/K2, 16 waves, K5, finish
  python tools/profile_run.py minplus [C] [layers]  # config-5 graph, int32 min-plus waves
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "search"
ctx = P.Context(0)
if mode == "search":
    g = P.builtin_model("inception_chain", 32)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(16), ctx=ctx)
    for _ in range(3):
        prep.launch()
        r = prep.fetch()
    print("search", r.cost, r.device_ms)
else:
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    g = P.series_parallel_graph(1, n, 0.3)
    t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
    r = P.plan_with_tables(g, t)
    print("minplus", C, n, r.cost, r.device_ms)
