"""Multi-process paths.

* CPU (gloo, world_size 2): the sweep sharding, the global argmin all-gather
  and the max-over-ranks reduction of paper_1802_04924_b200.distributed.
* GPU (>= 2 B200s; skipped on a single-GPU box): row-sharded plans over NCCL
  equal single-GPU plans bit for bit (tests/mgpu_worker.py under torchrun).
"""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, size, port, q):
    sys.path.insert(0, ROOT)
    from paper_1802_04924_b200 import distributed as PD

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    items = list(range(11))
    mine = PD.shard(items, rank, size)
    # a fake sweep: cost = (i - 6)^2 with a deliberate tie at i = 4 and i = 8
    local = [((i - 6) ** 2 if i not in (4, 8) else 1, i, f"plan{i}") for i, _ in mine]
    best = PD.global_best(local)
    mx = PD.max_over_ranks(float(rank + 1))
    q.put((rank, [i for i, _ in mine], best, mx))
    dist.barrier()
    dist.destroy_process_group()


def test_sweep_sharding_and_global_argmin_gloo():
    size, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    covered = sorted(i for _, part, _, _ in out for i in part)
    assert covered == list(range(11))
    for _, _, best, mx in out:
        assert best == (0, 6, "plan6")
        assert mx == 2.0


@pytest.mark.gpu
def test_row_sharded_plans_match_single_gpu():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", f"--nproc-per-node={n}",
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert p.stdout.count(": OK") == n


# ---- virtual ranks: the row-sharded plan path on one B200 ------------------------

GOLD = None


def _gold():
    global GOLD
    if GOLD is None:
        import json

        GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))
    return GOLD


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("case", [("inception_chain", 16), ("inception_chain", 64), ("vgg16", 16),
                                  ("inception_chain(3)", 4), ("alexnet", 4)], ids=lambda c: f"{c[0]}@{c[1]}")
def test_virtual_ranks_builtin_match_reference(gpu, n, case):
    """n virtual ranks (row blocks, K1/K2 on every rank, all-gathers at the
    re-association points, distributed unwind) vs the reference golden."""
    import paper_1802_04924_b200 as P

    model, D = case
    gold = next(c for c in _gold()["builtins"] if c["model"] == model and c["devices"] == D)
    vr = P.VirtualRanks(n)
    r = vr.plan(P.builtin_model(model, 32), devices=P.DeviceGraph.uniform(D))
    assert [int(x) for x in r.indices] == gold["indices"]
    assert float(r.cost).hex() == gold["cost"]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("C", [256, 700])
def test_virtual_ranks_config5_match_single_gpu(gpu, n, C):
    """Config-5 graph (U16 min-plus folds, row-sharded, optimistic operand caps
    with the overflow flag OR-ed over the ranks): the same indices and cost as
    one GPU; at C = 256 also the real reference."""
    import json

    import paper_1802_04924_b200 as P

    g, t = P.synthetic_instance(1, 1000 if C == 256 else 300, C, 0.3, ctx=gpu.ctx)
    one = P.plan_with_tables(g, t)
    r = P.VirtualRanks(n).plan(g, tables=t)
    assert list(r.indices) == list(one.indices) and r.cost == one.cost
    if C == 256:
        gold = next(c for c in _gold()["synthetic"] if c["configs"] == 256)
        assert [int(x) for x in r.indices] == gold["indices"] and float(r.cost).hex() == gold["cost"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,C", [(2, 600), (4, 600), (2, 1100)])
def test_virtual_ranks_fp64_large_folds_match_single_gpu(gpu, n, C):
    """Uncertified FP64 tables, row-sharded (at C=1100 on 2 ranks each rank's
    550 rows still take the mp64 fold): same IEEE result and argmins as one GPU."""
    import paper_1802_04924_b200 as P

    g = P.series_parallel_graph(3, 40, 0.4)
    ctx = P.Context(0)
    t = P.synthetic_cost_tables64(g, C, seed=9, ctx=ctx)
    one = P.plan_with_tables(g, t)
    assert one.precision == "fp64"
    r = P.VirtualRanks(n).plan(g, tables=t)
    assert list(r.indices) == list(one.indices) and r.cost == one.cost


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_virtual_ranks_optimistic_cap_overflow_reruns(gpu, n):
    """Every fold minimum is 2000 units, above the optimistic operand cap: some
    rank's device check fires, the flag is OR-ed over the ranks (kind-20 step)
    and every rank re-plans with proven caps -- the generic fold's result."""
    import numpy as np

    import paper_1802_04924_b200 as P

    m = 96
    layers = [P.Layer("u", "input", [4, 1, 1])] + [P.Layer(f"n{i}", "softmax") for i in range(1, 3)]
    g = P.ComputationGraph.create(layers, [[]] + [[layers[i - 1].id] for i in range(1, 3)], 8)
    t1 = np.full((m, m), 2000 / 64.0)
    t1[np.arange(m), np.arange(m)] = 0.0
    t2 = np.full((m, m), 2000 / 64.0)
    t2[(np.arange(m) + 1) % m, np.arange(m)] = 0.0
    rng = np.random.default_rng(7)
    node = [rng.integers(0, 64, m) / 64.0, np.zeros(m), rng.integers(0, 64, m) / 64.0]
    cat = [np.tile([1, 1, 1, 1], (m, 1)) for _ in range(3)]
    slow = P.Context(0)
    slow.set_kernel_policy("generic")
    want = P.plan_with_tables(g, P.upload_cost_tables(g, cat, node, [t1, t2], slow))
    tf = P.upload_cost_tables(g, cat, node, [t1, t2], gpu.ctx)
    r = P.VirtualRanks(n).plan(g, tables=tf)
    assert list(r.indices) == list(want.indices) and r.cost == want.cost


@pytest.mark.gpu
def test_mgpu_plan_without_torch():
    """bin/mgpu_plan: NCCL unique id handed to forked per-GPU processes through a
    pipe (no torch.distributed, no MPI); the row-sharded I64 plan equals the
    reference golden."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import json

    exe = os.path.join(ROOT, "paper_1802_04924_b200", "bin", "mgpu_plan")
    p = subprocess.run([exe, "2", "inception_chain", "64"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    rows = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    gold = next(c for c in _gold()["builtins"] if c["model"] == "inception_chain" and c["devices"] == 64)
    assert rows and all(r["cost"] == gold["cost"] for r in rows)


# ---- the row-sharded layout, host only (shard.hpp via pp_shard_layout) -----------

def _restated_layout(g, counts, nranks, rank):
    """Python restatement of the row-block arithmetic and the all-gather schedule."""
    import numpy as np

    recs, n_waves = g.schedule()
    es, ed, _ = g.edges()
    src = list(es)
    for rec in recs:  # derived edge ids are assigned in log order (planner.hpp:220-227)
        assert rec[4] == len(src)
        src.append(rec[5])
    blk, first, local = [], [], []
    for s in src:
        rows = int(counts[s])
        b = -(-rows // nranks)
        f = min(rows, rank * b)
        blk.append(b)
        first.append(f)
        local.append(max(0, min(rows, (rank + 1) * b) - f))
    ne = g.n_edges
    gathers = []
    for w in range(1, n_waves + 1):
        for rec in recs:  # a wave's records in log order
            if rec[7] == w and rec[0] == 0 and rec[3] >= ne:
                gathers.append((w, rec[3]))
    consumed = {rec[2] for rec in recs} | {rec[3] for rec in recs}
    gathers += [(n_waves + 1, e) for e in range(ne, len(src)) if e not in consumed]
    return np.array(blk), np.array(first), np.array(local), gathers


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
@pytest.mark.parametrize("graph", ["inception_chain", "vgg16", "series_parallel"])
def test_shard_layout_matches_restatement(graph, nranks):
    import numpy as np

    sys.path.insert(0, ROOT)
    import paper_1802_04924_b200 as P

    g = P.series_parallel_graph(3, 300, 0.4) if graph == "series_parallel" else P.builtin_model(graph, 32)
    counts = np.random.default_rng(nranks).integers(1, 700, g.n_layers).astype(np.int32)
    covered = None
    for rank in range(nranks):
        blk, first, local, gathers = P.shard_layout(g, counts, nranks, rank)
        rb, rf, rl, rg = _restated_layout(g, counts, nranks, rank)
        assert (blk == rb).all() and (first == rf).all() and (local == rl).all()
        assert gathers == rg
        covered = local.copy() if covered is None else covered + local
    # the ranks' row blocks tile every table exactly
    recs, _ = g.schedule()
    es, _, _ = g.edges()
    src = list(es) + [rec[5] for rec in recs]
    assert (covered == counts[np.array(src)]).all()
