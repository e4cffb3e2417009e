"""Median device time of the standalone K1/K2 table build (CostTables.build_ms)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
out = {}
for spec in (sys.argv[1:] or ["inception_chain@16", "inception_chain@64", "vgg16@16"]):
    m, D = spec.split("@")
    g = P.builtin_model(m, 32)
    ms = []
    for _ in range(15):
        t = P.build_cost_tables(g, P.DeviceGraph.uniform(int(D)), ctx)
        ms.append(t.build_ms)
    out[spec] = round(statistics.median(ms[3:]) * 1000, 1)
print(out)
