import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
D = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = P.Context(0)
g = P.builtin_model("inception_chain", 32)
for _ in range(2):
    t = P.build_cost_tables(g, P.DeviceGraph.uniform(D), ctx)
print("k1 ms", t.build_ms)
