import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1802_04924_b200 as P, oracle as O
want = O.Instance.builtin("inception_chain", 32, "port").build_tables(16).plan()
for ext in (False, True):
    s = torch.cuda.Stream(); torch.cuda.set_stream(s)
    ctx = P.Context(0, stream=s.cuda_stream if ext else None)
    g = P.builtin_model("inception_chain", 32); dev = P.DeviceGraph.uniform(16)
    prep = P.PreparedPlan(g, devices=dev, ctx=ctx)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for k in range(3):
        flush.zero_(); prep.launch(); r = prep.fetch()
        print("prep", ext, k, r.cost == want.cost, list(r.indices) == list(want.indices))
    for k in range(3):
        flush.zero_(); torch.cuda.synchronize()
        res = P.plan(g, dev, ctx=ctx)
        print("plan", ext, k, res.cost == want.cost, list(res.indices) == list(want.indices), res.cost, want.cost)
    prep.launch(); r = prep.fetch(); print("prep-after", r.cost == want.cost)
