"""torchrun worker: row-sharded plans on N GPUs == single-GPU plans (bit-exact).

    torchrun --standalone --nproc-per-node 2 tests/mgpu_worker.py
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_04924_b200 as P  # noqa: E402
from paper_1802_04924_b200 import distributed as PD  # noqa: E402


def main():
    rank, size = PD.world()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shard_ctx = P.Context(local)
    PD.attach(shard_ctx)
    solo = P.Context(local)  # no communicator: the reference result
    fails = []

    def check(name, a, b):
        if list(a.indices) != list(b.indices) or a.cost != b.cost:
            fails.append(name)

    for model, D in [("alexnet", 4), ("vgg16", 16), ("inception_chain", 16), ("inception_chain", 64)]:
        g = P.builtin_model(model, 32)
        dev = P.DeviceGraph.uniform(D)
        check(f"{model}@{D}", P.plan(g, dev, ctx=shard_ctx), P.plan(g, dev, ctx=solo))
    for C, n in [(96, 200), (256, 300), (700, 60)]:
        g = P.series_parallel_graph(7, n, 0.4)
        ts = P.synthetic_cost_tables(g, C, seed=5, ctx=shard_ctx)
        t1 = P.synthetic_cost_tables(g, C, seed=5, ctx=solo)
        a, b = P.plan_with_tables(g, ts), P.plan_with_tables(g, t1)
        check(f"synthetic C={C} n={n}", a, b)
        prep = P.PreparedPlan(g, tables=ts, ctx=shard_ctx)
        kinds = [k for k, _, _ in prep.profile()]
        if "allgather" not in kinds:
            fails.append(f"no all-gather in sharded plan C={C}")
        prep.launch()
        check(f"prepared sharded C={C}", prep.fetch(), b)
    # optimistic operand caps overflow on some rank: all ranks re-plan with proven caps
    import numpy as np

    m = 96
    layers = [P.Layer("u", "input", [4, 1, 1])] + [P.Layer(f"n{i}", "softmax") for i in range(1, 3)]
    g = P.ComputationGraph.create(layers, [[]] + [[layers[i - 1].id] for i in range(1, 3)], 8)
    x1 = np.full((m, m), 2000 / 64.0)
    x1[np.arange(m), np.arange(m)] = 0.0
    x2 = np.full((m, m), 2000 / 64.0)
    x2[(np.arange(m) + 1) % m, np.arange(m)] = 0.0
    rng = np.random.default_rng(7)
    node = [rng.integers(0, 64, m) / 64.0, np.zeros(m), rng.integers(0, 64, m) / 64.0]
    cat = [np.tile([1, 1, 1, 1], (m, 1)) for _ in range(3)]
    want = P.plan_with_tables(g, P.upload_cost_tables(g, cat, node, [x1, x2], solo))
    ts = P.upload_cost_tables(g, cat, node, [x1, x2], shard_ctx)
    check("overflow one-shot", P.plan_with_tables(g, ts), want)
    prep = P.PreparedPlan(g, tables=ts, ctx=shard_ctx)
    prep.launch()
    check("overflow prepared", prep.fetch(), want)
    for seed in range(20):
        g, t = P.random_series_parallel_graph(seed, 10 + 9 * seed, 3, 0.4, 4, ctx=shard_ctx)
        cat, node, _, _, xfer = t.download()
        t1 = P.upload_cost_tables(g, cat, node, xfer, solo)
        check(f"random seed {seed}", P.plan_with_tables(g, t), P.plan_with_tables(g, t1))
    ok = torch.tensor([0 if not fails else 1], device="cuda")
    dist.all_reduce(ok)
    print(f"rank {rank}/{size}: {'OK' if not fails else 'FAIL ' + ', '.join(fails)}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if ok.item() else 0)


if __name__ == "__main__":
    main()
