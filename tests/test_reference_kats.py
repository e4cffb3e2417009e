"""The reference's own known-answer and property tests, restated once and run
on every implementation (``impl`` = port | reference | gpu, see impls.py).

Sources (relative to /root/reference/proj/tests/):
  test_planner.cpp   :27-350   Eq. 2 / Eq. 3 KATs, reduction counts, final
                               enumeration, unwind, plan-level checks, theorems
  test_oracle.cpp    :23-166   brute force, generator, 120-seed oracle equality
  test_cost_model.cpp:23-295   cost formulas and transfer KATs
On the gpu parameter every table, fold, merge, enumeration and plan below runs
through libparplan_cuda.so on the B200.
"""
import numpy as np
import pytest

from impls import InputErr, LimitErr

ONES, TWO = [1, 1, 1, 1], [2, 1, 1, 1]


def chain_fixture(impl):
    """u -> w -> v with two configs everywhere; only w has node cost (test_planner.cpp:27-40)."""
    g = impl.graph([("u", "input", [4, 1, 1]), ("w", "softmax", []), ("v", "softmax", [])], [[], ["u"], ["w"]], 8)
    t = impl.set_tables(g, [[ONES, TWO]] * 3, [[0, 0], [1, 2], [0, 0]], [[[0, 5], [5, 0]], [[0, 5], [5, 0]]])
    return g, t


def diamond(impl, xfer):
    g = impl.graph([("a", "input", [2, 1, 1]), ("b", "softmax", []), ("c", "softmax", []), ("j", "concat", [1])],
                   [[], ["a"], ["a"], ["b", "c"]], 4)
    t = impl.set_tables(g, [[ONES, TWO]] * 4, [[0, 0]] * 4, xfer)
    return g, t


def test_node_elimination_folds_middle_node(impl):  # test_planner.cpp:44-60
    g, t = chain_fixture(impl)
    rg = impl.reduced(g, t)
    assert rg.node_elimination()
    assert not rg.node_elimination()
    assert rg.live_node_count() == 2
    live = rg.live_edges()
    assert len(live) == 1
    assert rg.edge_table(live[0][0]).tolist() == [[1.0, 6.0], [6.0, 2.0]]
    rec = rg.log()[0]
    assert rec[0] == 0 and rec[1] == 1
    assert rg.argmin(0).tolist() == [[0, 0], [0, 1]]


def test_two_in_edges_not_eligible(impl):  # test_planner.cpp:62-71
    g = impl.graph([("a", "input", [2, 1, 1]), ("b", "input", [2, 1, 1]), ("j", "concat", [1])],
                   [[], [], ["a", "b"]], 4)
    t = impl.build_tables(g, 2)
    rg = impl.reduced(g, t)
    assert not rg.node_elimination()
    assert rg.live_node_count() == 3


def test_edge_elimination_adds_entrywise(impl):  # test_planner.cpp:73-102
    g, t = diamond(impl, [[[1, 2], [3, 4]], [[10, 20], [30, 40]], [[0, 1000], [1000, 0]], [[0, 1000], [1000, 0]]])
    rg = impl.reduced(g, t)
    assert rg.node_elimination() and rg.node_elimination()
    assert not rg.node_elimination()
    assert rg.edge_elimination()
    assert not rg.edge_elimination()
    live = rg.live_edges()
    assert len(live) == 1
    assert rg.edge_table(live[0][0]).tolist() == [[11.0, 22.0], [33.0, 44.0]]


def test_zero_parallel_edge_is_identity(impl):  # test_planner.cpp:104-122
    g, t = diamond(impl, [[[1, 2], [3, 4]], [[0, 0], [0, 0]], [[0, 1000], [1000, 0]], [[0, 0], [0, 0]]])
    rg = impl.reduced(g, t)
    rg.reduce()
    live = rg.live_edges()
    assert len(live) == 1
    assert rg.edge_table(live[0][0]).tolist() == [[1, 2], [3, 4]]


def _counts(log):
    n = sum(1 for r in log if r[0] == 0)
    return n, len(log) - n


def test_vgg16_needs_node_eliminations_only(impl):  # test_planner.cpp:124-137
    g = impl.builtin("vgg16", 32)
    t = impl.build_tables(g, 4)
    rg = impl.reduced(g, t)
    rg.reduce()
    assert rg.live_node_count() == 2
    assert _counts(rg.log()) == (19, 0)


def test_inception_needs_both_rules(impl):  # test_planner.cpp:138-149
    g = impl.builtin("inception_chain(3)", 8)
    t = impl.build_tables(g, 2)
    rg = impl.reduced(g, t)
    rg.reduce()
    assert rg.live_node_count() == 2
    n, e = _counts(rg.log())
    assert n > 0 and e > 0


def test_single_node_fixpoint(impl):  # test_planner.cpp:150-157
    g = impl.graph([("in", "input", [3, 4, 4])], [[]], 2)
    t = impl.build_tables(g, 2)
    rg = impl.reduced(g, t)
    rg.reduce()
    assert rg.live_node_count() == 1
    assert rg.log() == []


def test_each_elimination_removes_one_edge(impl):  # test_planner.cpp:160-172
    g = impl.builtin("inception_chain(2)", 8)
    t = impl.build_tables(g, 2)
    rg = impl.reduced(g, t)
    edges = rg.live_edge_count()
    while rg.node_elimination() or rg.edge_elimination():
        assert rg.live_edge_count() == edges - 1
        edges = rg.live_edge_count()


def test_final_single_node(impl):  # test_planner.cpp:175-184
    g = impl.graph([("in", "input", [4, 1, 1])], [[]], 8)
    t = impl.set_tables(g, [[ONES, TWO, [4, 1, 1, 1]]], [[3, 1, 2]], [])
    rg = impl.reduced(g, t)
    idx, cost = rg.enumerate_final()
    assert list(idx) == [1] and cost == 1.0


def test_final_two_nodes(impl):  # test_planner.cpp:185-192
    g, t = chain_fixture(impl)
    rg = impl.reduced(g, t)
    rg.reduce()
    idx, cost = rg.enumerate_final()
    assert len(idx) == 2 and cost == 1.0


def test_k_bound_limit_error(impl):  # test_planner.cpp:193-219
    layers = [(f"s{i}", "input", [2, 1, 1]) for i in range(6)] + [(f"j{i}", "concat", [1]) for i in range(6)]
    inputs = [[] for _ in range(6)] + [[f"s{i}", f"s{(i + 1) % 6}"] for i in range(6)]
    g = impl.graph(layers, inputs, 4)
    t = impl.build_tables(g, 2)
    rg = impl.reduced(g, t)
    rg.reduce()
    assert rg.live_node_count() == 12
    with pytest.raises(LimitErr) as e:
        rg.enumerate_final(8)
    assert "12" in str(e.value)
    idx, cost = rg.enumerate_final(12)  # 3^12 candidates
    assert len(idx) == 12
    with pytest.raises(LimitErr):
        impl.plan_with_tables(g, t, 8)


def test_unwind_restores_nodes(impl):  # test_planner.cpp:222-232 via plan_with_tables
    g, t = chain_fixture(impl)
    idx, cost, stats = impl.plan_with_tables(g, t)
    assert list(idx) == [0, 0, 0] and cost == 1.0
    rg = impl.reduced(g, t)
    rg.reduce()
    am = rg.argmin(0)
    assert am[0][0] == 0 and am[1][1] == 1  # {0,-1,0} -> 0, {1,-1,1} -> 1


def test_plan_reports_exact_table_cost(impl):  # test_planner.cpp:234-244
    g = impl.builtin("vgg16", 32)
    t = impl.build_tables(g, 4)
    idx, cost, stats = impl.plan_with_tables(g, t)
    assert len(idx) == 21 and stats[0] == 2
    assert cost == impl.evaluate(g, t, idx)


def test_one_device_all_ones(impl):  # test_planner.cpp:246-257
    g = impl.builtin("lenet5", 32)
    idx, cost, _ = impl.plan(g, 1)
    assert list(idx) == [0] * 6
    t = impl.build_tables(g, 1)
    _, node, xfer = impl.tables(t)
    s = 0.0
    for v in node:
        s += v[0]
    assert cost == s
    assert all((x == 0).all() for x in xfer)


def test_planning_is_deterministic(impl):  # test_planner.cpp:259-266
    g = impl.builtin("inception_chain(4)", 16)
    a = impl.plan(g, 4)
    b = impl.plan(g, 4)
    assert list(a[0]) == list(b[0]) and a[1] == b[1]


def _reduced_min(rg):
    """exhaustive minimum over the live part of a reduced graph (test_planner.cpp:277-313)."""
    return rg.enumerate_final(64)[1]


def test_theorem1_node_elimination_preserves_optimum(impl):  # test_planner.cpp:268-314
    for seed in range(50):
        g, t = impl.random(seed, 4 + seed % 3, 3, 0.6, 4)
        _, before, _ = impl.brute(g, t)
        rg = impl.reduced(g, t)
        if not rg.node_elimination():
            continue
        assert _reduced_min(rg) == before


def test_theorem2_edge_elimination_preserves_costs(impl):  # test_planner.cpp:316-350
    for seed in range(100, 130):
        g, t = impl.random(seed, 4, 3, 1.0, 4)
        rg = impl.reduced(g, t)
        assert rg.node_elimination() and rg.node_elimination()
        nodes = rg.live_nodes()
        assert len(nodes) == 2
        node = impl.tables(t)[1]

        def scan():
            costs = []
            live = rg.live_edges()
            tabs = [rg.edge_table(e[0]) for e in live]
            for i in range(len(node[nodes[0]])):
                for k in range(len(node[nodes[1]])):
                    c = node[nodes[0]][i] + node[nodes[1]][k]
                    for tab in tabs:
                        c += tab[i][k]
                    costs.append(c)
            return costs

        before = scan()
        assert rg.edge_elimination()
        assert scan() == before


# ---- test_oracle.cpp --------------------------------------------------------

def test_brute_single_layer(impl):  # test_oracle.cpp:23-35
    g = impl.graph([("in", "input", [4, 1, 1]), ("s", "softmax", [])], [[], ["in"]], 8)
    t = impl.set_tables(g, [[ONES], [ONES, [1, 2, 1, 1], TWO]], [[0], [3, 1, 2]], [[[0, 0, 0]]])
    idx, cost, visited = impl.brute(g, t)
    assert cost == 1.0 and list(idx) == [0, 1] and visited == 3


def test_brute_visits_whole_space(impl):  # test_oracle.cpp:37-45
    g = impl.builtin("lenet5", 4)
    t = impl.build_tables(g, 2)
    cat, _, _ = impl.tables(t)
    _, _, visited = impl.brute(g, t)
    assert visited == int(np.prod([len(c) for c in cat]))


def test_brute_budget(impl):  # test_oracle.cpp:47-56
    g = impl.builtin("vgg16", 32)
    t = impl.build_tables(g, 4)
    with pytest.raises(LimitErr) as e:
        impl.brute(g, t)
    assert "budget" in str(e.value)


def test_brute_tie_break(impl):  # test_oracle.cpp:57-66
    g = impl.graph([("in", "input", [4, 1, 1]), ("s", "softmax", [])], [[], ["in"]], 8)
    t = impl.set_tables(g, [[ONES, TWO], [ONES, TWO]], [[1, 1], [1, 1]], [[[0, 0], [0, 0]]])
    idx, _, _ = impl.brute(g, t)
    assert list(idx) == [0, 0]


def test_every_instance_reduces_to_two(impl):  # test_oracle.cpp:117-125
    for seed in range(100):
        g, t = impl.random(seed, 3 + seed % 10, 3, 0.5, 4)
        rg = impl.reduced(g, t)
        rg.reduce()
        assert rg.live_node_count() <= 2


def test_planner_matches_brute_force_120_seeds(impl):  # test_oracle.cpp:127-140
    for seed in range(120):
        g, t = impl.random(seed, 1 + seed % 8, 1 + seed % 4, 0.35 * (seed % 3), 4)
        _, bf, _ = impl.brute(g, t)
        idx, cost, _ = impl.plan_with_tables(g, t)
        assert cost == bf
        assert impl.evaluate(g, t, idx) == bf


# ---- test_cost_model.cpp (through table construction) ----------------------

def test_fc_compute_cost(impl):  # test_cost_model.cpp:33-39
    g = impl.graph([("in", "input", [512, 7, 7]), ("fc", "fully_connected", [4096])], [[], ["in"]], 32)
    t = impl.build_tables(g, 1)
    _, node, _ = impl.tables(t)
    assert node[1][0] == 1.9730006016e-3


def test_sync_cost_parameter_server(impl):  # test_cost_model.cpp:84-109
    g = impl.graph([("in", "input", [512, 7, 7]), ("fc", "fully_connected", [4096])], [[], ["in"]], 32)
    t = impl.build_tables(g, 2, bw=np.full(4, 1e10))
    cat, _, _ = impl.tables(t)
    comp, sync = impl.analytic_split(t)
    k = [list(c) for c in cat[1]].index(TWO)
    assert sync[1][k] == 0.0822083584
    t4 = impl.build_tables(g, 4, bw=np.full(16, 1e10))
    cat4, _, _ = impl.tables(t4)
    comp4, sync4 = impl.analytic_split(t4)
    assert sync4[1][[list(c) for c in cat4[1]].index([1, 4, 1, 1])] == 0.0
    param = 4.0 * 25088 * 4096
    per = 2.0 * (param / 2.0) / 1e10
    assert sync4[1][[list(c) for c in cat4[1]].index([2, 2, 1, 1])] == per + per + per


def test_halo_transfer(impl):  # test_cost_model.cpp:118-128
    g = impl.graph([("in", "input", [1, 8, 8]), ("c1", "conv2d", [1, 3, 3, 1, 1, 1, 1]),
                    ("c2", "conv2d", [1, 3, 3, 1, 1, 1, 1])], [[], ["in"], ["c1"]], 1)
    t = impl.build_tables(g, 2, bw=np.full(4, 1e10))
    cat, _, xfer = impl.tables(t)
    i = [list(c) for c in cat[1]].index([1, 1, 2, 1])
    j = [list(c) for c in cat[2]].index([1, 1, 2, 1])
    assert xfer[1][i][j] == 32.0 / 1e10


def test_channel_parallel_fc_transfer(impl):  # test_cost_model.cpp:137-143
    g = impl.graph([("in", "input", [512, 7, 7]), ("fc", "fully_connected", [4096])], [[], ["in"]], 32)
    t = impl.build_tables(g, 2, bw=np.full(4, 1e10))
    cat, _, xfer = impl.tables(t)
    i = [list(c) for c in cat[0]].index([1, 2, 1, 1])
    j = [list(c) for c in cat[1]].index([1, 2, 1, 1])
    assert xfer[0][i][j] == (4.0 * 32.0 * 25088.0 / 2.0) / 1e10


def test_owned_only_requirements_move_nothing(impl):  # test_cost_model.cpp:130-136
    g = impl.graph([("in", "input", [512, 7, 7]), ("fc", "fully_connected", [4096]), ("sm", "softmax", [])],
                   [[], ["in"], ["fc"]], 32)
    t = impl.build_tables(g, 2, bw=np.full(4, 1e10))
    cat, _, xfer = impl.tables(t)
    for c in (TWO, [1, 2, 1, 1]):
        i = [list(x) for x in cat[1]].index(c)
        j = [list(x) for x in cat[2]].index(c)
        assert xfer[1][i][j] == 0.0


def test_nonuniform_bandwidth_uses_pair_quotients(impl):
    """Per-pair bandwidths take the pair-walking K1 path (cost.hpp:119-130)."""
    D = 4
    bw = np.array([[0, 1e10, 2e10, 3e10], [5e9, 0, 1e10, 7e9], [4e10, 2e9, 0, 1e10], [1e10, 1e10, 3e9, 0]]).reshape(-1)
    g = impl.builtin("lenet5", 8)
    t = impl.build_tables(g, D, rates=np.array([1e13, 5e12, 2e13, 1e13]), bw=bw)
    cat, node, xfer = impl.tables(t)
    ref = get_port_tables("lenet5", 8, D, np.array([1e13, 5e12, 2e13, 1e13]), bw)
    assert all((a.view(np.int64) == b.view(np.int64)).all() for a, b in zip(node, ref[1]))
    assert all((a.view(np.int64) == b.view(np.int64)).all() for a, b in zip(xfer, ref[2]))


def get_port_tables(model, batch, D, rates, bw):
    import oracle as O

    inst = O.Instance.builtin(model, batch, "port").build_tables(D, rates, bw)
    return inst.catalogs(), inst.nodes(), inst.xfers()


def test_graph_errors(impl):  # test_graph.cpp:60-112
    with pytest.raises(InputErr) as e:
        impl.graph([("in", "input", [1, 4, 4]), ("c", "softmax", [])], [[], ["ghost"]], 1)
    assert "ghost" in str(e.value)
    with pytest.raises(InputErr):
        impl.graph([("x", "input", [1, 4, 4]), ("x", "softmax", [])], [[], ["x"]], 1)
    with pytest.raises(InputErr):
        impl.graph([("in", "input", [2, 4, 4]), ("a", "softmax", []), ("b", "softmax", [])], [[], ["b"], ["a"]], 1)
    with pytest.raises(InputErr):
        impl.graph([("in", "input", [3, 4, 4]), ("c", "conv2d", [4, 7, 7, 1, 1, 0, 0])], [[], ["in"]], 1)
    with pytest.raises(InputErr):
        impl.builtin("resnet50", 8)
    with pytest.raises(InputErr):
        impl.builtin("inception_chain(0)", 8)
