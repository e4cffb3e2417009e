"""The S16x2 min-plus fold (minplus.cuh) against the generic tiled fold and
the CPU oracle: values, argmins (lowest-index ties), padding at sizes that are
not multiples of the 128x128 tile / 32-j chunk, split-j CTAs, tie-heavy data."""
import numpy as np
import pytest

import oracle as O
from impls import bits

pytestmark = pytest.mark.gpu


def _chain(P, n):
    layers = [P.Layer("u", "input", [4, 1, 1])] + [P.Layer(f"n{i}", "softmax") for i in range(1, n)]
    inputs = [[]] + [[layers[i - 1].id] for i in range(1, n)]
    return P.ComputationGraph.create(layers, inputs, 8)


def _tables(rng, counts, edges, hi):
    node = [rng.integers(0, hi, c) / 64.0 for c in counts]
    xfer = [rng.integers(0, hi, (counts[s], counts[d])) / 64.0 for s, d in edges]
    return node, xfer


@pytest.mark.parametrize("sizes,hi", [((300, 200, 257), 641), ((129, 70, 1000), 3), ((64, 64, 64), 2),
                                      ((1024, 96, 512), 641), ((130, 2048, 66), 5)])
def test_fold_matches_generic_and_oracle(gpu, sizes, hi):
    import paper_1802_04924_b200 as P

    rng = np.random.default_rng(sum(sizes) + hi)
    nu, nw, nv = sizes
    g = _chain(P, 3)
    counts = [nu, nw, nv]
    node, xfer = _tables(rng, counts, [(0, 1), (1, 2)], hi)
    cat = [np.tile([1, 1, 1, 1], (c, 1)) for c in counts]
    fast = P.Context(0)
    slow = P.Context(0)
    slow.set_kernel_policy("generic")
    ra = P.ReducedGraph(g, P.upload_cost_tables(g, cat, node, xfer, fast))
    tf = P.upload_cost_tables(g, cat, node, xfer, fast)
    ts = P.upload_cost_tables(g, cat, node, xfer, slow)
    pf = P.PreparedPlan(g, tables=tf, ctx=fast)
    kinds = [k for k, _, _ in pf.profile()]
    assert "mp_fold" in kinds, kinds
    a = P.plan_with_tables(g, tf)
    b = P.plan_with_tables(g, ts)
    assert list(a.indices) == list(b.indices) and a.cost == b.cost
    # the fold's table and argmin (step API uses the generic kernel) vs the oracle
    want_t, want_am = O.fold(node[1], xfer[0], xfer[1])
    ra.node_elimination()
    assert (bits(ra.edge_table(2)) == bits(want_t)).all()
    assert (ra.argmin(0) == want_am).all()
    # the plan's unwound middle index equals the oracle argmin at the chosen endpoints
    assert a.indices[1] == want_am[a.indices[0], a.indices[2]]


@pytest.mark.parametrize("C", [96, 200, 512])
def test_synthetic_graph_fast_vs_generic(gpu, C):
    import paper_1802_04924_b200 as P

    g = P.series_parallel_graph(11, 120, 0.4)
    fast = P.Context(0)
    slow = P.Context(0)
    slow.set_kernel_policy("generic")
    tf = P.synthetic_cost_tables(g, C, seed=3, ctx=fast)
    cat, node, _, _, xfer = tf.download()
    ts = P.upload_cost_tables(g, cat, node, xfer, slow)
    a = P.plan_with_tables(g, tf)
    b = P.plan_with_tables(g, ts)
    assert list(a.indices) == list(b.indices) and a.cost == b.cost
    prof = P.PreparedPlan(g, tables=tf, ctx=fast).profile()
    assert sum(w for k, _, w in prof if k == "mp_fold") > 0


@pytest.mark.parametrize("policy", ["auto", "conservative"])
def test_optimistic_cap_overflow_reruns_exactly(gpu, policy):
    """Every fold minimum is 2000 units, above the optimistic JB-5 operand cap
    (1022): the device check fires and the plan is re-run with the proven cap
    (min(rowspan, colspan) + 1 = 2001, JB 4) — same result as the generic fold."""
    import paper_1802_04924_b200 as P

    n = 96
    g = _chain(P, 3)
    t1 = np.full((n, n), 2000 / 64.0)
    t1[np.arange(n), np.arange(n)] = 0.0
    t2 = np.full((n, n), 2000 / 64.0)
    t2[(np.arange(n) + 1) % n, np.arange(n)] = 0.0
    rng = np.random.default_rng(7)
    node = [rng.integers(0, 64, n) / 64.0, np.zeros(n), rng.integers(0, 64, n) / 64.0]
    cat = [np.tile([1, 1, 1, 1], (n, 1)) for _ in range(3)]
    fast, slow = P.Context(0), P.Context(0)
    fast.set_kernel_policy(policy)
    slow.set_kernel_policy("generic")
    tf = P.upload_cost_tables(g, cat, node, [t1, t2], fast)
    ts = P.upload_cost_tables(g, cat, node, [t1, t2], slow)
    assert "mp_fold" in [k for k, _, _ in P.PreparedPlan(g, tables=tf, ctx=fast).profile()]
    b = P.plan_with_tables(g, ts)
    for _ in range(2):  # one-shot, then prepared (graph) plans
        a = P.plan_with_tables(g, tf)
        assert list(a.indices) == list(b.indices) and a.cost == b.cost
        pp = P.PreparedPlan(g, tables=tf, ctx=fast)
        pp.launch()
        c = pp.fetch()
        assert list(c.indices) == list(b.indices) and c.cost == b.cost


# ---- FP64 large-table fold (minplus64.cuh) -------------------------------------------


def test_fp64_large_fold_matches_generic(gpu):
    """Non-dyadic (uncertified) FP64 tables: the 64x64-tile FP64 fold vs the
    generic tiled fold — same IEEE sums in the reference's order, same argmins."""
    import paper_1802_04924_b200 as P

    g = P.series_parallel_graph(3, 40, 0.4)
    ctx = P.Context(0)
    t = P.synthetic_cost_tables64(g, 600, seed=9, ctx=ctx)
    prof = P.PreparedPlan(g, tables=t, ctx=ctx).profile()
    assert "mp64_fold" in [k for k, _, _ in prof]
    a = P.plan_with_tables(g, t)
    assert a.precision == "fp64"
    ctx.set_kernel_policy("generic")
    b = P.plan_with_tables(g, t)
    assert list(a.indices) == list(b.indices) and a.cost == b.cost


def test_fp64_large_fold_matches_fixed_point_on_dyadic_tables(gpu):
    """The same dyadic tables planned in FP64 (precision forced) through the
    FP64 large fold and in exact int32 through the U16 kernels: identical plans
    (every FP64 sum of k/64 values is exact here)."""
    import paper_1802_04924_b200 as P

    g, t32 = P.synthetic_instance(4, 60, 520, 0.4, ctx=gpu.ctx)
    cat, node, _, _, xfer = t32.download()
    c64 = P.Context(0)
    c64.set_precision("fp64")
    t64 = P.upload_cost_tables(g, cat, node, xfer, c64)
    assert "mp64_fold" in [k for k, _, _ in P.PreparedPlan(g, tables=t64, ctx=c64).profile()]
    a, b = P.plan_with_tables(g, t32), P.plan_with_tables(g, t64)
    assert a.precision == "fixed" and b.precision == "fp64"
    assert list(a.indices) == list(b.indices) and a.cost == b.cost


@pytest.mark.parametrize("C,n", [(300, 40), (1000, 12), (130, 60)])
def test_chain_runs_match_generic(gpu, C, n):
    """A pure chain (one fold per wave, all t2 original): the whole run goes to
    mp_chain (rows per CTA = ceil(C / 148), odd column counts, a last partial
    row block) — same plan as the generic fold, and the C=300 tie-heavy variant."""
    import paper_1802_04924_b200 as P

    g = _chain(P, n)
    rng = np.random.default_rng(C + n)
    hi = 5 if C == 300 else 641  # C=300: values in [0, 4] -> many exact ties
    counts = [C] * n
    node, xfer = _tables(rng, counts, [(i, i + 1) for i in range(n - 1)], hi)
    cat = [np.tile([1, 1, 1, 1], (c, 1)) for c in counts]
    fast, slow = P.Context(0), P.Context(0)
    slow.set_kernel_policy("generic")
    tf = P.upload_cost_tables(g, cat, node, xfer, fast)
    ts = P.upload_cost_tables(g, cat, node, xfer, slow)
    kinds = [k for k, _, _ in P.PreparedPlan(g, tables=tf, ctx=fast).profile()]
    assert "mp_chain" in kinds, kinds
    a, b = P.plan_with_tables(g, tf), P.plan_with_tables(g, ts)
    assert list(a.indices) == list(b.indices) and a.cost == b.cost
