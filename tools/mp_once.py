"""One prepared min-plus plan on the config-5 graph at C configs, launched
twice (for ncu launch lists / captures).  python tools/mp_once.py C"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = P.series_parallel_graph(1, 1000, 0.3)
ctx = P.Context(0)
t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
prep = P.PreparedPlan(g, tables=t, ctx=ctx)
for _ in range(2):
    prep.launch()
    r = prep.fetch()
print(f"C={C} cost={r.cost} device_ms={r.device_ms:.2f}")
