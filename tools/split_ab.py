"""A/B: prepared I16 plan with the table build inside the fused kernel vs a
separate build launch (PARPLAN_SPLIT_BUILD=1), and one-shot e2e."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_04924_b200 as P  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for model, D in [("inception_chain", 16), ("inception_chain", 64), ("vgg16", 16)]:
    g = P.builtin_model(model, 32)
    dev = P.DeviceGraph.uniform(D)
    prep = P.PreparedPlan(g, devices=dev, ctx=ctx)
    ms = []
    for k in range(40):
        flush.zero_()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        prep.launch()
        s1.record(stream)
        prep.fetch()
        s1.synchronize()
        if k >= 5:
            ms.append(s0.elapsed_time(s1))
    e2e = []
    for k in range(40):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.plan(g, dev, ctx=ctx)
        if k >= 5:
            e2e.append((time.perf_counter() - t0) * 1e3)
    print(f"{os.environ.get('PARPLAN_SPLIT_BUILD', '0')} {model}@{D} device {statistics.median(ms):.4f} ms  e2e {statistics.median(e2e):.4f} ms", flush=True)
