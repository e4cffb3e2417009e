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
