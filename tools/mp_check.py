"""Min-plus plan on the config-5 graph at C configs: U16 path vs the generic
int32 tiled fold (bit-exact indices + cost), plus the per-kernel profile.
  python tools/mp_check.py C [C ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P  # noqa: E402

for C in [int(x) for x in sys.argv[1:]] or [1024]:
    g = P.series_parallel_graph(1, 1000, 0.3)
    fast = P.Context(0)
    t = P.synthetic_cost_tables(g, C, seed=1, ctx=fast)
    prep = P.PreparedPlan(g, tables=t, ctx=fast)
    prep.launch()
    r = prep.fetch()
    prof = prep.profile()
    by = {}
    for k, ms, w in prof:
        by[k] = by.get(k, 0.0) + ms
    cells = sum(w for k, _, w in prof if k in ("mp_fold", "mp_chain"))
    fold_ms = by.get("mp_fold", 0.0) + by.get("mp_chain", 0.0)
    t0 = time.time()
    prep.launch()
    r2 = prep.fetch()
    plan_ms = r2.device_ms
    peak = 148 * 128 * 1965e6
    print(f"C={C} cost={r.cost} plan_ms={plan_ms:.2f} fold_ms={fold_ms:.2f} fold_frac={cells / (fold_ms * 1e-3) / peak:.3f} "
          f"plan_frac={cells / (plan_ms * 1e-3) / peak:.3f} by={ {k: round(v, 2) for k, v in by.items()} }", flush=True)
    del prep
    if "--generic" in sys.argv or C <= 2048:
        fast.set_kernel_policy("generic")  # the same device tables through the generic int32 fold
        b = P.plan_with_tables(g, t)
        fast.set_kernel_policy("auto")
        print(f"C={C} matches_generic={list(b.indices) == list(r.indices) and b.cost == r.cost} "
              f"generic_ms={b.device_ms:.1f}", flush=True)
    del t
