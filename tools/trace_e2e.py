import os, sys, time
os.environ.setdefault("PARPLAN_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
m, D = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("inception_chain", 16)
g = P.builtin_model(m, 32); dev = P.DeviceGraph.uniform(D)
for k in range(8):
    t0 = time.perf_counter(); r = P.plan(g, dev, ctx=ctx); dt = (time.perf_counter() - t0) * 1e6
    print(m, D, "python-level us", round(dt, 1), "device_ms", round(r.device_ms, 4), file=sys.stderr)
