"""Host-side stage times of one-shot pp_plan calls (PARPLAN_TRACE=2)."""
import os
import sys

os.environ.setdefault("PARPLAN_TRACE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

g = P.builtin_model(sys.argv[1] if len(sys.argv) > 1 else "inception_chain", 32)
dev = P.DeviceGraph.uniform(int(sys.argv[2]) if len(sys.argv) > 2 else 16)
ctx = P.Context(0)
for _ in range(8):
    r = P.plan(g, dev, ctx=ctx)
print(r.cost, r.device_ms)
