"""Per-phase device time of one plan(inception_chain(12)@D) search (fused and per-wave executors)."""
import collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P

D = int(sys.argv[1]) if len(sys.argv) > 1 else 16
model = sys.argv[2] if len(sys.argv) > 2 else "inception_chain"
g = P.builtin_model(model, 32)
out = {}
for pol in ("auto", "unfused"):
    ctx = P.Context(0)
    ctx.set_kernel_policy(pol)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(5):
        prep.launch(); prep.fetch()
    agg = collections.OrderedDict()
    for _ in range(5):
        for k, ms, w in prep.profile():
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1; a[1] += ms / 5
    out[pol] = {k: {"n": v[0] // 5, "ms": round(v[1], 4)} for k, v in agg.items()}
print(json.dumps(out))
