"""One interface over the three implementations the parity tests compare:

* ``gpu``       — the product, libparplan_cuda.so through its C ABI;
* ``port``      — the plain-C restatement in oracle/ (CPU checker);
* ``reference`` — the real reference compiled from /root/reference into
                  oracle/_ref (CPU checker; absent -> tests skip it).

The reference's own unit tests (proj/tests/test_planner.cpp, test_oracle.cpp,
...) are restated once against this interface and run on every implementation,
so the same known-answer tests pin the oracle (CPU, every round) and the CUDA
path (B200).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402


class LimitErr(Exception):
    pass


class InputErr(Exception):
    pass


class OracleImpl:
    """graph and tables share one orc_instance."""

    def __init__(self, kind: str):
        self.kind = kind
        self.name = kind

    def _wrap(self, fn, *a, **k):
        try:
            return fn(*a, **k)
        except O.OracleLimitError as e:
            raise LimitErr(str(e)) from None
        except O.OracleError as e:
            raise InputErr(str(e)) from None

    def graph(self, layers, inputs, batch):
        """layers: [(id, kind_name, params)], inputs: [[id, ...]]"""
        ids = [l[0] for l in layers]
        index = {}
        for i, x in enumerate(ids):
            index.setdefault(x, i)
        kinds = [O.KINDS[l[1]] for l in layers]
        params = np.zeros((len(layers), 7), np.int64)
        for i, l in enumerate(layers):
            params[i, : len(l[2])] = l[2]
        src, dst = [], []
        for i, ins in enumerate(inputs):
            for n in ins:
                if n not in index:
                    raise InputErr(f"layer '{ids[i]}' references undeclared layer '{n}'")
                src.append(index[n])
                dst.append(i)
        return self._wrap(O.Instance.graph, kinds, params, src, dst, batch, ids, kind=self.kind)

    def builtin(self, name, batch=32):
        return self._wrap(O.Instance.builtin, name, batch, self.kind)

    def random(self, seed, n, maxc, bp, ndev):
        inst = O.Instance.random(seed, n, maxc, bp, ndev, self.kind)
        return inst, inst

    def synthetic(self, seed, n, C, bp=0.3):
        inst = O.Instance.synthetic(seed, n, C, bp, self.kind)
        return inst, inst

    def build_tables(self, g, D, rates=None, bw=None):
        return self._wrap(g.build_tables, D, rates, bw)

    def set_tables(self, g, catalogs, node, xfer):
        return g.set_tables(catalogs, node, xfer)

    def tables(self, t):
        return t.catalogs(), t.nodes(), t.xfers()

    def analytic_split(self, t):
        n = t.n_layers
        return [t.compute(l) for l in range(n)], [t.sync(l) for l in range(n)]

    def plan_with_tables(self, g, t, k=8):
        p = self._wrap(t.plan, k)
        return p.indices, p.cost, (p.final_graph_nodes, p.node_eliminations, p.edge_eliminations)

    def plan(self, g, D):
        t = self.build_tables(g, D)
        return self.plan_with_tables(g, t)

    def evaluate(self, g, t, idx):
        return t.total_cost(idx)

    def brute(self, g, t, budget=10_000_000):
        return self._wrap(t.brute, budget)

    def reduced(self, g, t):
        return OracleRG(self, t)


class OracleRG:
    def __init__(self, impl, inst):
        self.impl, self.i = impl, inst.rg_init()

    def node_elimination(self):
        return self.i.node_elimination()

    def edge_elimination(self):
        return self.i.edge_elimination()

    def reduce(self):
        while self.i.node_elimination() or self.i.edge_elimination():
            pass

    def live_edges(self):
        return self.i.live_edges()

    def live_nodes(self):
        return list(self.i.live_nodes())

    def live_node_count(self):
        return len(self.i.live_nodes())

    def live_edge_count(self):
        return len(self.i.live_edges())

    def edge_table(self, e):
        return self.i.edge_table(e)

    def log(self):
        return self.i.log()

    def argmin(self, r):
        return self.i.log_argmin(r)

    def enumerate_final(self, k=8):
        return self.impl._wrap(self.i.enumerate_final, k)


class GpuImpl:
    name = "gpu"

    def __init__(self):
        import paper_1802_04924_b200 as P

        self.P = P
        self.ctx = P.default_context()

    def _wrap(self, fn, *a, **k):
        P = self.P
        try:
            return fn(*a, **k)
        except P.LimitError as e:
            raise LimitErr(str(e)) from None
        except P.InputError as e:
            raise InputErr(str(e)) from None

    def graph(self, layers, inputs, batch):
        P = self.P
        ls = [P.Layer(l[0], l[1], list(l[2])) for l in layers]
        return self._wrap(P.ComputationGraph.create, ls, inputs, batch)

    def builtin(self, name, batch=32):
        return self._wrap(self.P.builtin_model, name, batch)

    def _graph_of(self, inst):
        k, p, _ = zip(*[inst.layer(l) for l in range(inst.n_layers)])
        s, d, _ = inst.edges()
        names = {v: k for k, v in O.KINDS.items()}
        layers = [(f"n{l}", names[k[l]], list(p[l])) for l in range(inst.n_layers)]
        inputs = [[] for _ in range(inst.n_layers)]
        for e in range(len(s)):
            inputs[d[e]].append(f"n{s[e]}")
        return self.graph(layers, inputs, 8)

    def random(self, seed, n, maxc, bp, ndev):
        inst = O.Instance.random(seed, n, maxc, bp, ndev, "port")
        g = self._graph_of(inst)
        return g, self.set_tables(g, inst.catalogs(), inst.nodes(), inst.xfers())

    def synthetic(self, seed, n, C, bp=0.3):
        inst = O.Instance.synthetic(seed, n, C, bp, "port")
        g = self._graph_of(inst)
        return g, self.set_tables(g, inst.catalogs(), inst.nodes(), inst.xfers())

    def build_tables(self, g, D, rates=None, bw=None):
        P = self.P
        dev = P.DeviceGraph.uniform(D) if rates is None and bw is None else P.DeviceGraph(
            np.asarray(rates if rates is not None else np.full(D, 1e13), np.float64),
            np.asarray(bw if bw is not None else np.full(D * D, 1.25e10), np.float64))
        return self._wrap(P.build_cost_tables, g, dev, self.ctx)

    def set_tables(self, g, catalogs, node, xfer):
        return self._wrap(self.P.upload_cost_tables, g, catalogs, node, xfer, self.ctx)

    def tables(self, t):
        cat, node, _, _, xfer = t.download()
        return cat, node, xfer

    def analytic_split(self, t):
        _, _, comp, sync, _ = t.download()
        return comp, sync

    def plan_with_tables(self, g, t, k=8):
        p = self._wrap(self.P.plan_with_tables, g, t, k)
        return p.indices, p.cost, (p.final_graph_nodes, p.node_eliminations, p.edge_eliminations)

    def plan(self, g, D):
        P = self.P
        p = self._wrap(P.plan, g, P.DeviceGraph.uniform(D), 8, self.ctx)
        return p.indices, p.cost, (p.final_graph_nodes, p.node_eliminations, p.edge_eliminations)

    def evaluate(self, g, t, idx):
        return t.total_cost(idx)

    def brute(self, g, t, budget=10_000_000):
        return self._wrap(self.P.brute_force_plan, g, t, budget)

    def reduced(self, g, t):
        return GpuRG(self, self.P.ReducedGraph(g, t))


class GpuRG:
    def __init__(self, impl, rg):
        self.impl, self.rg = impl, rg

    def node_elimination(self):
        return self.rg.node_elimination()

    def edge_elimination(self):
        return self.rg.edge_elimination()

    def reduce(self):
        self.rg.reduce()

    def live_edges(self):
        return self.rg.live_edges()

    def live_nodes(self):
        return self.rg.live_nodes()

    def live_node_count(self):
        return self.rg.live_node_count()

    def live_edge_count(self):
        return self.rg.live_edge_count()

    def edge_table(self, e):
        return self.rg.edge_table(e)

    def log(self):
        return [r[:7] for r in self.rg.log()]

    def argmin(self, r):
        return self.rg.argmin(r)

    def enumerate_final(self, k=8):
        return self.impl._wrap(self.rg.enumerate_final, k)


def oracle_kinds():
    return ["port"] + (["reference"] if O.available("reference") else [])


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64).view(np.int64)
