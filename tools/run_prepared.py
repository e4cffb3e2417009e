"""Launch a prepared plan a few times (a target for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
m, D = (sys.argv[1] if len(sys.argv) > 1 else "inception_chain@16").split("@")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = P.Context(0)
prep = P.PreparedPlan(P.builtin_model(m, 32), devices=P.DeviceGraph.uniform(int(D)), ctx=ctx)
for _ in range(n):
    prep.launch(); prep.fetch()
print("ok", m, D)
