"""Builds the cost tables of one model a few times (ncu target for K1/K2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
m, D = (sys.argv[1] if len(sys.argv) > 1 else "inception_chain@16").split("@")
ctx = P.Context(0)
g = P.builtin_model(m, 32)
for _ in range(3):
    t = P.build_cost_tables(g, P.DeviceGraph.uniform(int(D)), ctx)
