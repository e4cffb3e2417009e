"""A/B of fused-kernel knobs in one process: interleaved runs, median per-phase us."""
import collections, json, os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_04924_b200 as P

knobs = {"PARPLAN_PANEL": ["0", "1"], "PARPLAN_STAGE": ["0", "1"], "PARPLAN_FUSED_BLOCKS_PER_SM": ["1", "0"]}
if len(sys.argv) > 1:
    knobs = json.loads(sys.argv[1])
models = [("inception_chain", 16), ("vgg16", 16), ("alexnet", 4)]
combos = [dict(zip(knobs, v)) for v in itertools.product(*knobs.values())]
ctx = P.Context(0)
res = collections.defaultdict(lambda: collections.defaultdict(list))
preps = {}
for ci, c in enumerate(combos):
    for k, v in c.items():
        os.environ[k] = v
    for m, D in models:
        g = P.builtin_model(m, 32)
        preps[(ci, m)] = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=ctx)
for rnd in range(5):
    for ci in range(len(combos)):
        for m, D in models:
            prep = preps[(ci, m)]
            for _ in range(2): prep.launch(); prep.fetch()
            agg = collections.Counter()
            for k, ms, w in prep.profile():
                agg[k] += ms
            res[ci][m].append((agg["fused.wave"] * 1000, sum(agg.values()) * 1000))
for ci, c in enumerate(combos):
    row = {m: "wave %.1f total %.1f" % tuple(np.median(np.array(v), axis=0)) for m, v in res[ci].items()}
    print(json.dumps(c), json.dumps(row))
