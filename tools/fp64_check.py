"""FP64 (uncertified) large-table folds: the config-5 topology with random
non-dyadic tables (values (k + u) / 64, u in [0, 1) irrational-ish) uploaded as
FP64, planned on the device; per-kernel profile.  python tools/fp64_check.py C nodes"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = P.series_parallel_graph(1, n, 0.3)
rng = np.random.default_rng(5)
es, ed, _ = g.edges()
node = [(rng.integers(0, 641, C) + rng.random(C)) / 64.0 for _ in range(g.n_layers)]
xfer = [(rng.integers(0, 641, (C, C)) + rng.random((C, C))) / 64.0 for _ in range(g.n_edges)]
cat = [np.tile([1, 1, 1, 1], (C, 1)) for _ in range(g.n_layers)]
ctx = P.Context(0)
t = P.upload_cost_tables(g, cat, node, xfer, ctx)
del xfer
prep = P.PreparedPlan(g, tables=t, ctx=ctx)
prep.launch()
r = prep.fetch()
prof = prep.profile()
by = {}
for k, ms, w in prof:
    by[k] = by.get(k, 0.0) + ms
fold_kinds = ("mp64_fold", "fused.wave", "fused.chain") if any(k == "mp64_fold" for k, _, _ in prof) else ("wave", "fused.wave", "fused.chain")
cells = sum(w for k, _, w in prof if k in fold_kinds)
fold_ms = sum(ms for k, ms, _ in prof if k in fold_kinds) or 1e-9
prep.launch()
r2 = prep.fetch()
print(f"C={C} n={n} precision={r.precision} cost={r.cost!r} plan_ms={r2.device_ms:.2f} fold_ms={fold_ms:.2f} "
      f"cells/s={cells / (fold_ms * 1e-3):.3e} by={ {k: round(v, 2) for k, v in by.items()} }", flush=True)
ctx.set_kernel_policy("generic")
b = P.plan_with_tables(g, t)
print(f"matches_generic={list(b.indices) == list(r.indices) and b.cost == r.cost} generic_ms={b.device_ms:.2f}")
