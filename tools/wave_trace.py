"""PARPLAN_WAVE_TRACE timeline of one fused run (stderr), per model."""
import os, sys
os.environ.setdefault("PARPLAN_WAVE_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
for m, D in [(a.split("@")[0], int(a.split("@")[1])) for a in (sys.argv[1:] or ["inception_chain@16"])]:
    g = P.builtin_model(m, 32)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(5): prep.launch(); prep.fetch()
    print(m, D, flush=True)
    prep.profile()
    sys.stderr.flush()
