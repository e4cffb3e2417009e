"""Small workloads for compute-sanitizer (tests/test_gpu_sanitizer.py).

  python tools/sanitize_run.py fused      # fused plan kernel: I16, VGG@16, inception_chain(3)@8
  python tools/sanitize_run.py minplus    # U16 min-plus plan (prep, stream-K fold, merges, minima)
  python tools/sanitize_run.py vranks     # row-sharded plan on 2 virtual ranks (gathers, peer unwind)
Each result is checked against the reference goldens / the generic fold.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_04924_b200 as P  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))


def gold(model, D):
    return next(c for c in GOLD["builtins"] if c["model"] == model and c["devices"] == D)


def check(r, g):
    assert [int(x) for x in r.indices] == g["indices"] and float(r.cost).hex() == g["cost"], (r.cost, g["cost_repr"])


mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
ctx = P.Context(0)
if mode == "fused":
    for model, D in (("inception_chain", 16), ("vgg16", 16), ("inception_chain(3)", 4)):
        check(P.plan(P.builtin_model(model, 32), P.DeviceGraph.uniform(D), ctx=ctx), gold(model, D))
elif mode == "minplus":
    g, t = P.synthetic_instance(1, 60, 200, 0.4, ctx=ctx)
    a = P.plan_with_tables(g, t)
    ctx.set_kernel_policy("generic")
    b = P.plan_with_tables(g, t)
    assert list(a.indices) == list(b.indices) and a.cost == b.cost
elif mode == "vranks":
    r = P.VirtualRanks(2).plan(P.builtin_model("inception_chain(3)", 32), devices=P.DeviceGraph.uniform(4))
    check(r, gold("inception_chain(3)", 4))
    g, t = P.synthetic_instance(1, 40, 130, 0.4, ctx=ctx)
    one = P.plan_with_tables(g, t)
    two = P.VirtualRanks(2).plan(g, tables=t)
    assert list(one.indices) == list(two.indices) and one.cost == two.cost
print(mode, "ok")
