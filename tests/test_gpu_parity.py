"""CUDA path vs the CPU oracle on the BASELINE configs (bit-exact).

Tables: K1 xfer + K2 node costs against the restatement, compared as IEEE bit
patterns.  Plans: indices, cost (bit-exact), elimination counts, the full
log and every argmin table through the ReducedGraph step API.
"""
import numpy as np
import pytest

import oracle as O
from impls import bits

pytestmark = pytest.mark.gpu

BUILTINS = [("lenet5", 1), ("lenet5", 2), ("lenet5", 4), ("alexnet", 4), ("vgg16", 4), ("vgg16", 16),
            ("inception_chain(3)", 2), ("inception_chain(3)", 8), ("inception_chain", 16)]


# device counts whose degree sets mix factors that do not divide one another
# (2 vs 3): K1's identity-dimension closed forms fall back to the x loop there
ODD_D = [("lenet5", 3), ("alexnet", 6), ("inception_chain(3)", 12), ("vgg16", 6)]


@pytest.mark.parametrize("model,D", BUILTINS + ODD_D)
def test_tables_bit_exact(gpu, model, D):
    g = gpu.builtin(model, 32)
    t = gpu.build_tables(g, D)
    cat, node, xfer = gpu.tables(t)
    comp, sync = gpu.analytic_split(t)
    ref = O.Instance.builtin(model, 32, "port").build_tables(D)
    for l in range(ref.n_layers):
        assert (cat[l] == ref.catalog(l)).all()
        assert (bits(node[l]) == bits(ref.node(l))).all(), f"node table of layer {l}"
        assert (bits(comp[l]) == bits(ref.compute(l))).all()
        assert (bits(sync[l]) == bits(ref.sync(l))).all()
    for e in range(ref.n_edges):
        assert (bits(xfer[e]) == bits(ref.xfer(e))).all(), f"xfer table of edge {e}"


@pytest.mark.parametrize("model,D", BUILTINS)
def test_plan_matches_oracle(gpu, model, D):
    g = gpu.builtin(model, 32)
    idx, cost, stats = gpu.plan(g, D)
    want = O.Instance.builtin(model, 32, "port").build_tables(D).plan()
    assert list(idx) == list(want.indices)
    assert cost == want.cost
    assert stats == (want.final_graph_nodes, want.node_eliminations, want.edge_eliminations)


@pytest.mark.parametrize("model,D", [("alexnet", 4), ("vgg16", 16), ("inception_chain", 16)])
def test_log_and_argmins(gpu, model, D):
    g = gpu.builtin(model, 32)
    t = gpu.build_tables(g, D)
    rg = gpu.reduced(g, t)
    rg.reduce()
    ref = O.Instance.builtin(model, 32, "port").build_tables(D).reduce()
    assert rg.log() == ref.log()
    for r, rec in enumerate(ref.log()):
        if rec[0] == 0:
            assert (rg.argmin(r) == ref.log_argmin(r)).all(), f"argmin of record {r}"
        assert (bits(rg.edge_table(rec[4])) == bits(ref.edge_table(rec[4]))).all(), f"table of edge {rec[4]}"


def test_nonuniform_devices(gpu):
    rng = np.random.default_rng(7)
    D = 8
    rates = rng.uniform(5e12, 2e13, D)
    bw = rng.uniform(5e9, 5e10, D * D)
    g = gpu.builtin("inception_chain(2)", 16)
    t = gpu.build_tables(g, D, rates=rates, bw=bw)
    _, node, xfer = gpu.tables(t)
    ref = O.Instance.builtin("inception_chain(2)", 16, "port").build_tables(D, rates, bw)
    assert all((bits(a) == bits(b)).all() for a, b in zip(node, ref.nodes()))
    assert all((bits(a) == bits(b)).all() for a, b in zip(xfer, ref.xfers()))
    idx, cost, _ = gpu.plan_with_tables(g, t)
    want = ref.plan()
    assert list(idx) == list(want.indices) and cost == want.cost


@pytest.mark.parametrize("C", [4, 16, 64])
def test_synthetic_config5_fixed_point(gpu, C):
    """config-5 generator (N=1000, bp=0.3, seed 1): exact int32 fixed-point DP."""
    g, t = gpu.synthetic(1, 1000, C)
    idx, cost, stats = gpu.plan_with_tables(g, t)
    ref = O.Instance.synthetic(1, 1000, C, 0.3, "port")
    want = ref.plan()
    assert list(idx) == list(want.indices)
    assert cost == want.cost
    assert stats == (want.final_graph_nodes, want.node_eliminations, want.edge_eliminations)


def test_fp64_and_fixed_point_agree(gpu):
    import paper_1802_04924_b200 as P

    inst = O.Instance.synthetic(3, 300, 24, 0.3, "port")
    g = gpu._graph_of(inst)
    ctx64 = P.Context(0, precision="fp64")
    t_fix = P.upload_cost_tables(g, inst.catalogs(), inst.nodes(), inst.xfers(), gpu.ctx)
    t_64 = P.upload_cost_tables(g, inst.catalogs(), inst.nodes(), inst.xfers(), ctx64)
    a = P.plan_with_tables(g, t_fix)
    b = P.plan_with_tables(g, t_64)
    assert a.precision == "fixed" and b.precision == "fp64"
    assert list(a.indices) == list(b.indices) and a.cost == b.cost == inst.plan().cost


def test_prepared_plan_and_profile(gpu):
    import paper_1802_04924_b200 as P

    g = P.builtin_model("inception_chain", 32)
    dev = P.DeviceGraph.uniform(16)
    prep = P.PreparedPlan(g, devices=dev, ctx=gpu.ctx)
    want = O.Instance.builtin("inception_chain", 32, "port").build_tables(16).plan()
    for upload in (True, False, False):
        prep.launch(upload)
        r = prep.fetch()
        assert list(r.indices) == list(want.indices) and r.cost == want.cost
    prof = prep.profile()
    kinds = [k for k, _, _ in prof]
    # one phase per wave, except chain segments (several waves, one phase)
    phases = kinds.count("fused.wave") + kinds.count("fused.chain")
    # the table build: its own launch (default) or the fused kernel's first phase
    assert kinds[0] in ("tables", "fused.tables") and 1 <= phases <= r.waves and kinds[-1] == "fused"
    assert sum(w for k, _, w in prof if k in ("fused.wave", "fused.chain")) > 0


def test_library_generators_match_reference_draw_order(gpu):
    import paper_1802_04924_b200 as P

    for seed in range(40):
        n, mc, bp = 1 + seed % 9, 1 + seed % 4, 0.35 * (seed % 3)
        g, t = P.random_series_parallel_graph(seed, n, mc, bp, 4, ctx=gpu.ctx)
        ref = O.Instance.random(seed, n, mc, bp, 4, "port")
        cat, node, _, _, xfer = t.download()
        assert all((bits(a) == bits(b)).all() for a, b in zip(node, ref.nodes()))
        assert all((bits(a) == bits(b)).all() for a, b in zip(xfer, ref.xfers()))
        r = P.plan_with_tables(g, t)
        assert r.cost == ref.plan().cost
    g = P.series_parallel_graph(1, 1000, 0.3)
    ref = O.Instance.synthetic(1, 1000, 2, 0.3, "port")
    assert g.n_layers == ref.n_layers and (np.stack(g.edges()) == np.stack(ref.edges())).all()


def test_device_synthetic_tables(gpu):
    import paper_1802_04924_b200 as P

    g = P.series_parallel_graph(5, 200, 0.3)
    t = P.synthetic_cost_tables(g, 48, seed=9, ctx=gpu.ctx)
    cat, node, _, _, xfer = t.download()
    assert all(((v * 64) == np.floor(v * 64)).all() and v.min() >= 0 and v.max() <= 10 for v in node + xfer)
    # the same tables through the host upload path and the FP64 path agree
    inst_nodes, inst_xfer = node, xfer
    ctx64 = P.Context(0, precision="fp64")
    t64 = P.upload_cost_tables(g, cat, inst_nodes, inst_xfer, ctx64)
    a, b = P.plan_with_tables(g, t), P.plan_with_tables(g, t64)
    assert a.precision == "fixed" and b.precision == "fp64"
    assert list(a.indices) == list(b.indices) and a.cost == b.cost


@pytest.mark.parametrize("model,D", [("alexnet", 4), ("vgg16", 16), ("inception_chain", 16), ("inception_chain", 64)])
def test_fused_and_per_wave_executors_agree(gpu, model, D):
    """One cooperative kernel for the whole plan vs one launch per wave."""
    import paper_1802_04924_b200 as P

    g = P.builtin_model(model, 32)
    dev = P.DeviceGraph.uniform(D)
    fused = P.Context(0)
    split = P.Context(0)
    split.set_kernel_policy("unfused")
    pf = P.PreparedPlan(g, devices=dev, ctx=fused)
    ps = P.PreparedPlan(g, devices=dev, ctx=split)
    assert [k for k, _, _ in pf.profile()][-1] == "fused"
    assert "wave" in [k for k, _, _ in ps.profile()]
    pf.launch()
    ps.launch()
    a, b = pf.fetch(), ps.fetch()
    assert list(a.indices) == list(b.indices) and a.cost == b.cost
    c = P.plan(g, dev, ctx=fused)
    assert list(c.indices) == list(a.indices) and c.cost == a.cost


def test_fused_random_graphs(gpu):
    import paper_1802_04924_b200 as P

    split = P.Context(0)
    split.set_kernel_policy("unfused")
    for seed in range(30):
        g, t = P.random_series_parallel_graph(seed, 5 + seed * 7, 3, 0.4, 4, ctx=gpu.ctx)
        cat, node, _, _, xfer = t.download()
        t2 = P.upload_cost_tables(g, cat, node, xfer, split)
        a, b = P.plan_with_tables(g, t), P.plan_with_tables(g, t2)
        assert list(a.indices) == list(b.indices) and a.cost == b.cost


def _seq_sum(vals):
    t = 0.0
    for v in vals:
        t += float(v)
    return t


@pytest.mark.parametrize("source", ["lenet5@4", "alexnet@4", "inception_chain(2)@4", "random", "synthetic"])
def test_evaluate_batch_matches_oracle(gpu, source):
    """Batched evaluate_strategy: every total bit-equal to the
    oracle's in-order sums (nodes by layer, then edges by id)."""
    import paper_1802_04924_b200 as P

    rng = np.random.default_rng(7)
    if source == "random":
        g, t = P.random_series_parallel_graph(11, 8, 4, 0.3, 4, ctx=gpu.ctx)
        ref = O.Instance.random(11, 8, 4, 0.3, 4, "port")
    elif source == "synthetic":
        g = P.series_parallel_graph(3, 40, 0.3)
        ref = O.Instance.synthetic(3, 40, 24, 0.3, "port")
        t = P.upload_cost_tables(g, ref.catalogs(), ref.nodes(), ref.xfers(), ctx=gpu.ctx)
    else:
        model, D = source.split("@")
        g = P.builtin_model(model, 32)
        t = P.build_cost_tables(g, P.DeviceGraph.uniform(int(D)), gpu.ctx)
        ref = O.Instance.builtin(model, 32, "port").build_tables(int(D))
    counts = [len(x) for x in ref.nodes()]
    ix = np.stack([rng.integers(0, c, size=300) for c in counts], axis=1).astype(np.int32)
    cost, node, xfer = t.evaluate_batch(ix)
    nodes, xfers = ref.nodes(), ref.xfers()
    src, dst, _ = g.edges()
    for s in range(0, 300, 7):
        row = ix[s]
        assert cost[s] == ref.total_cost(row)
        assert node[s] == _seq_sum(nodes[l][row[l]] for l in range(len(counts)))
        assert xfer[s] == _seq_sum(xfers[e][row[src[e]]][row[dst[e]]] for e in range(len(src)))
    with pytest.raises(P.InputError):
        bad = ix.copy()
        bad[0, 0] = counts[0]
        t.evaluate_batch(bad)


# fused-kernel knobs (read per prepare): every setting must give the oracle's
# plan — the hand-rolled barrier vs grid.sync(), dynamic vs static build chunks,
# chain segments and merge absorption off, the early table build off
KNOBS = [{"PARPLAN_GRID_BARRIER": "0"}, {"PARPLAN_BUILD_DYNAMIC": "0"}, {"PARPLAN_CHAINS": "0"},
         {"PARPLAN_SPLIT_BUILD": "0"}, {"PARPLAN_SPLIT_BUILD": "0", "PARPLAN_BUILD_DYNAMIC": "0"},
         {"PARPLAN_MERGE_FUSE": "0"}, {"PARPLAN_EARLY_BUILD": "0"}, {"PARPLAN_STAGE": "0", "PARPLAN_PANEL": "0"},
         # narrow waves on the first thread-block cluster (cluster barriers between
         # consecutive narrow waves; the staging-visibility rule of plan.cu's `seen`)
         {"PARPLAN_NARROW_ITEMS": "64", "PARPLAN_CLUSTER": "1"}, {"PARPLAN_NARROW_ITEMS": "64", "PARPLAN_CLUSTER": "2"},
         {"PARPLAN_NARROW_ITEMS": "256", "PARPLAN_CLUSTER": "4"}, {"PARPLAN_NARROW_ITEMS": "64", "PARPLAN_CHAINS": "0"}]


@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_fused_knobs_match_oracle(gpu, knobs, monkeypatch):
    import paper_1802_04924_b200 as P

    for name, value in knobs.items():
        monkeypatch.setenv(name, value)
    for model, D in [("alexnet", 4), ("vgg16", 16), ("inception_chain", 16)]:
        g = P.builtin_model(model, 32)
        want = O.Instance.builtin(model, 32, "port").build_tables(D).plan()
        prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(D), ctx=gpu.ctx)
        for _ in range(2):  # the counters and barrier words are rearmed by each launch
            prep.launch()
            r = prep.fetch()
            assert list(r.indices) == list(want.indices) and r.cost == want.cost
        r = P.plan(g, P.DeviceGraph.uniform(D), ctx=gpu.ctx)
        assert list(r.indices) == list(want.indices) and r.cost == want.cost


def test_repeated_plan_calls_through_the_plan_cache(gpu):
    """pp_plan keeps a prepared plan for a repeated (graph, devices, k_bound,
    policy) call: the third and later calls replay it.  Interleaved device
    counts, fresh graph objects (content-addressed) and a policy change must
    each give the oracle's plan."""
    import paper_1802_04924_b200 as P

    ctx = P.Context(0)
    want = {D: O.Instance.builtin("inception_chain", 32, "port").build_tables(D).plan() for D in (8, 16)}
    for k in range(5):
        for D in (16, 8):
            g = P.builtin_model("inception_chain", 32)  # a new pp_graph per call
            r = P.plan(g, P.DeviceGraph.uniform(D), ctx=ctx)
            assert list(r.indices) == list(want[D].indices) and r.cost == want[D].cost, (k, D)
    ctx.set_kernel_policy("unfused")
    g = P.builtin_model("inception_chain", 32)
    for _ in range(3):
        r = P.plan(g, P.DeviceGraph.uniform(16), ctx=ctx)
        assert list(r.indices) == list(want[16].indices) and r.cost == want[16].cost
    # a different bandwidth is a different key (the tables change)
    fast = P.DeviceGraph.uniform(16, bandwidth=2.5e10)
    want_fast = None
    for _ in range(3):
        r = P.plan(g, fast, ctx=ctx)
        want_fast = want_fast or r
        assert list(r.indices) == list(want_fast.indices) and r.cost == want_fast.cost
    ctx.release_pools()
    r = P.plan(g, P.DeviceGraph.uniform(16), ctx=ctx)
    assert list(r.indices) == list(want[16].indices) and r.cost == want[16].cost


def test_plan_cache_eviction_keeps_results(gpu):
    """Six keys through a four-entry plan cache, twice round: evicted plans are
    rebuilt and every call still returns its key's first (uncached) result."""
    import paper_1802_04924_b200 as P

    ctx = P.Context(0)
    g = P.builtin_model("inception_chain(3)", 32)
    devs = [P.DeviceGraph.uniform(8, bandwidth=1.25e10 * (1 + k)) for k in range(6)]
    first = [P.plan(g, d, ctx=ctx) for d in devs]
    for _ in range(2):
        for d, f in zip(devs, first):
            for _ in range(3):
                r = P.plan(g, d, ctx=ctx)
                assert list(r.indices) == list(f.indices) and r.cost == f.cost
