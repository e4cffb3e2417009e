"""Randomised sweep of row-sharded plans on virtual ranks against one GPU:
synthetic config-5-style instances (series-parallel graphs, C configs per
layer, the large-fold U16 path with optimistic caps) and builtin models on
random device counts.  python tools/sharded_sweep.py [instances=60]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
ctx = P.Context(0)
groups = {k: P.VirtualRanks(k) for k in (2, 3, 4, 5)}
bad = 0
for i in range(n):
    k = 2 + i % 4
    if i % 3 == 2:
        model = ["alexnet", "vgg16", "inception_chain(3)", "inception_chain"][i % 4]
        D = [2, 4, 8, 16, 6][i % 5]
        g = P.builtin_model(model, 32)
        one = P.plan(g, P.DeviceGraph.uniform(D), ctx=ctx)
        r = groups[k].plan(g, devices=P.DeviceGraph.uniform(D))
        what = f"{model}@{D}"
    else:
        C = [64, 96, 130, 200, 257, 300][i % 6]
        nodes = 30 + (i * 17) % 150
        g, t = P.synthetic_instance(i, nodes, C, 0.3 + 0.1 * (i % 3), ctx=ctx)
        one = P.plan_with_tables(g, t)
        r = groups[k].plan(g, tables=t)
        what = f"synthetic seed {i} n={nodes} C={C}"
    ok = list(r.indices) == list(one.indices) and r.cost == one.cost
    bad += not ok
    print(f"{'OK ' if ok else 'BAD'} ranks={k} {what} cost={one.cost}", flush=True)
print(f"{n} sharded plans, {bad} mismatches against one GPU")
