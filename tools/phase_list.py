"""Per-phase device time of the fused plan kernel (median of runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_04924_b200 as P
ctx = P.Context(0)
for arg in sys.argv[1:] or ["inception_chain@16", "vgg16@16"]:
    m, D = arg.split("@")
    prep = P.PreparedPlan(P.builtin_model(m, 32), devices=P.DeviceGraph.uniform(int(D)), ctx=ctx)
    for _ in range(3): prep.launch(); prep.fetch()
    runs = [prep.profile() for _ in range(7)]
    names = [(k, w) for k, _, w in runs[0]]
    ms = np.median(np.array([[x for _, x, _ in r] for r in runs]), axis=0)
    print(arg, " ".join(f"{k}:{v * 1000:.1f}" for (k, w), v in zip(names, ms)))
