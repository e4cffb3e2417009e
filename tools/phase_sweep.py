import collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
ctx = P.Context(0)
res = {}
for m, D in [("inception_chain", 16), ("vgg16", 16), ("alexnet", 4), ("inception_chain", 64)]:
    g = P.builtin_model(m, 32)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(3): prep.launch(); prep.fetch()
    agg = collections.OrderedDict()
    for _ in range(5):
        for k, ms, w in prep.profile():
            agg[k] = agg.get(k, 0.0) + ms / 5
    res[f"{m}@{D}"] = {k: round(v * 1000, 1) for k, v in agg.items()}
print(os.environ.get("PARPLAN_FUSED_BLOCKS_PER_SM", "occ"), json.dumps(res))
