"""Prepared LeNet5@4, I16 and I64 plans, launched a few times (ncu target: build_tables_kernel vs dp_fused_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
for m, D in [("lenet5", 4), ("inception_chain", 16), ("inception_chain", 64)]:
    prep = P.PreparedPlan(P.builtin_model(m, 32), devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(3): prep.launch(); prep.fetch()
