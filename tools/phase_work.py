"""Per-phase device time and work (cells) of prepared I64 and I16 plans (profile())."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
for D in (64, 16):
    prep = P.PreparedPlan(P.builtin_model("inception_chain", 32), devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(3): prep.launch(); prep.fetch()
    for k, ms, w in prep.profile():
        print(D, k, round(ms*1e3, 1), "us", int(w), "cells", f"{w/(ms*1e-3):.3e}/s" if ms > 0 else "")
