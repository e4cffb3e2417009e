"""Median python-level e2e of P.plan() under env knob settings, interleaved in one process."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_04924_b200 as P
knob = sys.argv[1] if len(sys.argv) > 1 else "PARPLAN_EARLY_BUILD"
vals = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1"]
ctx = P.Context(0)
g = P.builtin_model("inception_chain", 32); dev = P.DeviceGraph.uniform(16)
res = {v: [] for v in vals}
for v in vals:
    os.environ[knob] = v
    for _ in range(5): P.plan(g, dev, ctx=ctx)
for rnd in range(40):
    for v in vals:
        os.environ[knob] = v
        t0 = time.perf_counter(); r = P.plan(g, dev, ctx=ctx); res[v].append((time.perf_counter() - t0) * 1e6)
print(knob, {v: round(float(np.median(x)), 1) for v, x in res.items()})
