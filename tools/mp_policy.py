"""Config-5 min-plus plan at C configs under a kernel policy (auto / conservative): device ms and per-kernel profile.  python tools/mp_policy.py C policy"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04924_b200 as P
C = int(sys.argv[1]); pol = sys.argv[2]
g = P.series_parallel_graph(1, 1000, 0.3)
ctx = P.Context(0)
ctx.set_kernel_policy(pol)
t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
prep = P.PreparedPlan(g, tables=t, ctx=ctx)
for _ in range(2):
    prep.launch(); r = prep.fetch()
by = {}
for k, ms, w in prep.profile(): by[k] = by.get(k, 0.0) + ms
print(C, pol, os.environ.get("PARPLAN_MP_CHAIN", "1"), round(r.device_ms, 1), {k: round(v, 1) for k, v in by.items()}, r.cost)
