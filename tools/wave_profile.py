"""Per-wave device time of the fused plan kernel, with each wave's work."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_04924_b200 as P

def describe(g, D):
    cnt = [len(c) for c in g.catalogs(D)]
    ops, nw = g.schedule()
    s, d, _ = g.edges()
    waves = [[] for _ in range(nw)]
    for (typ, removed, e1, e2, ne, u, v, w) in ops:
        waves[w - 1].append((typ, removed, u, v))
    return cnt, waves

ctx = P.Context(0)
for m, D in [("inception_chain", 16), ("vgg16", 16)]:
    g = P.builtin_model(m, 32)
    cnt, waves = describe(g, D)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=ctx)
    for _ in range(3): prep.launch(); prep.fetch()
    acc = None
    for _ in range(10):
        wv = [ms for k, ms, w in prep.profile() if k == "fused.wave"]
        acc = np.array(wv) if acc is None else acc + np.array(wv)
    acc /= 10
    print(m, D, "waves", len(waves), "total us", round(acc.sum() * 1000, 1))
    for i, (t, ops) in enumerate(zip(acc, waves)):
        desc = []
        for typ, removed, u, v in ops:
            desc.append(("N" if typ == 0 else "E") + f"{removed}:{cnt[u] if u >= 0 else -1}x{cnt[removed] if typ == 0 else 0}x{cnt[v] if v >= 0 else -1}")
        print(f"  w{i:2d} {t*1000:6.1f} us  {' '.join(desc[:6])}{' ...' if len(desc) > 6 else ''} ({len(ops)} ops)")
