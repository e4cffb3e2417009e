"""Randomised parity sweep (a one-off validation, heavier than the test suite):
random series-parallel instances in the reference's generator order, planned by
the fused kernel, the per-wave executor and the generic policy, against each
other and against the C restatement of the reference (oracle/, the checker).
Large diamond-heavy instances overflow the generator's channel counts (4 * 2^k)
and leave layers with no config; the library rejects those (InputError) and the
sweep reports and skips them.
  python tools/random_sweep.py [seeds=300]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

import paper_1802_04924_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
fused, unfused, generic = P.Context(0), P.Context(0), P.Context(0)
unfused.set_kernel_policy("unfused")
generic.set_kernel_policy("generic")
bad = skipped = 0
for seed in range(n):
    nodes = 5 + (seed * 37) % 400
    mc = 2 + seed % 6
    bp = 0.2 + 0.1 * (seed % 5)
    D = 2 + seed % 7
    try:
        g, t = P.random_series_parallel_graph(seed, nodes, mc, bp, D, ctx=fused)
    except P.ParplanError as exc:
        print("generator error seed", seed, nodes, mc, bp, D, exc, flush=True)
        skipped += 1
        continue
    cat, node, _, _, xfer = t.download()
    res = [P.plan_with_tables(g, t)]
    for c in (unfused, generic):
        res.append(P.plan_with_tables(g, P.upload_cost_tables(g, cat, node, xfer, c)))
    want = O.Instance.random(seed, nodes, mc, bp, D, "port").plan() if hasattr(O.Instance, "random") else None
    ok = all(list(r.indices) == list(res[0].indices) and r.cost == res[0].cost for r in res)
    if want is not None:
        ok = ok and list(res[0].indices) == list(want.indices) and res[0].cost == want.cost
    if not ok:
        bad += 1
        print("MISMATCH seed", seed, nodes, mc, bp, D, [r.cost for r in res], want and want.cost, flush=True)
print(f"{n} instances ({skipped} rejected by the generator), {bad} mismatches against each other and the oracle")
