"""Min-plus plan (config-5 graph) device time under the current env knobs."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
C = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
ctx = P.Context(0)
g = P.series_parallel_graph(1, n, 0.3)
t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
prep = P.PreparedPlan(g, tables=t, ctx=ctx)
for _ in range(2): prep.launch(); r = prep.fetch()
ms = []
for _ in range(3):
    prep.launch(); r = prep.fetch(); ms.append(r.device_ms)
agg = collections.Counter()
for k, m, w in prep.profile(): agg[k] += m
print("plan ms", round(min(ms), 2), {k: round(v, 2) for k, v in agg.items()}, "cost", r.cost)
