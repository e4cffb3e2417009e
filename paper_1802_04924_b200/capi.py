"""ctypes binding of libparplan_cuda.so (include/parplan_c.h) with a thin
Pythonic mirror of the reference ``parplan`` API.

Names follow the reference (citations relative to
/root/reference/proj/include/parplan/): ``ComputationGraph`` / ``builtin_model``
(graph.hpp, models.hpp), ``DeviceGraph.uniform`` (graph.hpp:208), ``CostTables`` /
``build_cost_tables`` (cost.hpp:148-206), ``ReducedGraph`` (planner.hpp:55-245),
``enumerate_final`` (:256), ``plan_with_tables`` / ``plan`` (:339-371),
``brute_force_plan`` (oracle.hpp:52).  Errors map to ``InputError`` /
``LimitError`` with the reference's messages.

There is no fallback: importing this module without the built CUDA library
raises, and every table/plan call needs an sm_100 GPU.
"""
from __future__ import annotations

import ctypes as C
import time
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libparplan_cuda.so")

KIND = {"input": 0, "conv2d": 1, "pool2d": 2, "fully_connected": 3, "flatten": 4, "concat": 5, "softmax": 6}
KIND_NAMES = {v: k for k, v in KIND.items()}
DIM = {"sample": 0, "channel": 1, "height": 2, "width": 3}


class ParplanError(RuntimeError):
    pass


class InputError(ParplanError):
    """parplan::InputError (base.hpp:38-41)."""


class LimitError(ParplanError):
    """parplan::LimitError (base.hpp:45-48)."""


class CudaError(ParplanError):
    """No usable sm_100 device, or a CUDA failure."""


class _Record(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("type", "removed", "e1", "e2", "new_edge", "src", "dst", "wave")]


class _PlanResult(C.Structure):
    _fields_ = [("cost", C.c_double), ("final_graph_nodes", C.c_int32), ("node_eliminations", C.c_int32),
                ("edge_eliminations", C.c_int32), ("precision", C.c_int32), ("waves", C.c_int32),
                ("launches", C.c_int32), ("device_ms", C.c_double), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64)]


class _GraphDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_edges", C.c_int32), ("batch", C.c_int64), ("ids", C.c_void_p),
                ("kind", C.c_void_p), ("params", C.c_void_p), ("edge_src", C.c_void_p), ("edge_dst", C.c_void_p)]


class _DeviceDesc(C.Structure):
    _fields_ = [("count", C.c_int32), ("compute_rates", C.c_void_p), ("bandwidth", C.c_void_p)]


_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)

_SIGS = {
    "pp_last_error": (C.c_char_p, []),
    "pp_abi_version": (C.c_int, []),
    "pp_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "pp_context_create": (C.c_int, [C.c_int32, _pp]),
    "pp_context_create_on_stream": (C.c_int, [C.c_int32, _vp, _pp]),
    "pp_context_stream": (C.c_int, [_vp, _pp]),
    "pp_plan_prepare": (C.c_int, [_vp, _vp, C.c_void_p, _vp, C.c_int32, _pp]),
    "pp_plan_launch": (C.c_int, [_vp, C.c_int32]),
    "pp_plan_fetch": (C.c_int, [_vp, _i32p, C.POINTER(_PlanResult)]),
    "pp_plan_destroy": (C.c_int, [_vp]),
    "pp_plan_profile": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, C.POINTER(C.c_int32)]),
    "pp_context_destroy": (C.c_int, [_vp]),
    "pp_context_set_precision": (C.c_int, [_vp, C.c_int32]),
    "pp_context_set_kernel_policy": (C.c_int, [_vp, C.c_int32]),
    "pp_comm_unique_id": (C.c_int, [C.c_char_p]),
    "pp_context_attach_comm": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_char_p]),
    "pp_context_launch_count": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "pp_vgroup_create": (C.c_int, [C.c_int32, C.c_int32, _pp]),
    "pp_context_release_pools": (C.c_int, [_vp]),
    "pp_shard_layout": (C.c_int, [_vp, _i32p, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p]),
    "pp_vgroup_plan": (C.c_int, [_vp, _vp, C.c_void_p, _vp, C.c_int32, _i32p, C.POINTER(_PlanResult)]),
    "pp_vgroup_destroy": (C.c_int, [_vp]),
    "pp_graph_create": (C.c_int, [C.POINTER(_GraphDesc), _pp]),
    "pp_graph_builtin": (C.c_int, [C.c_char_p, C.c_int64, _pp]),
    "pp_graph_destroy": (C.c_int, [_vp]),
    "pp_graph_size": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pp_graph_layers": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pp_graph_edges": (C.c_int, [_vp, _vp, _vp, _vp]),
    "pp_graph_layer_id": (C.c_int, [_vp, C.c_int32, C.c_char_p, C.c_int32]),
    "pp_graph_catalogs": (C.c_int, [_vp, C.c_int32, _i32p, _vp]),
    "pp_graph_schedule": (C.c_int, [_vp, C.POINTER(C.c_int32), _vp, C.POINTER(C.c_int32)]),
    "pp_graph_series_parallel": (C.c_int, [C.c_uint64, C.c_int32, C.c_double, _pp]),
    "pp_random_instance": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32, _pp,
                                     _pp]),
    "pp_tables_build": (C.c_int, [_vp, _vp, C.POINTER(_DeviceDesc), _pp]),
    "pp_tables_upload": (C.c_int, [_vp, _vp, _i32p, _vp, _f64p, _f64p, _pp]),
    "pp_tables_synthetic": (C.c_int, [_vp, _vp, C.c_int32, C.c_uint64, _pp]),
    "pp_tables_synthetic64": (C.c_int, [_vp, _vp, C.c_int32, C.c_uint64, _pp]),
    "pp_tables_destroy": (C.c_int, [_vp]),
    "pp_tables_counts": (C.c_int, [_vp, _vp, C.POINTER(C.c_int64)]),
    "pp_tables_download": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pp_tables_build_ms": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "pp_tables_total_cost": (C.c_int, [_vp, _i32p, C.POINTER(C.c_double)]),
    "pp_tables_evaluate_batch": (C.c_int, [_vp, C.c_int64, _i32p, _f64p, _f64p, _f64p]),
    "pp_plan": (C.c_int, [_vp, _vp, C.POINTER(_DeviceDesc), C.c_int32, _i32p, C.POINTER(_PlanResult)]),
    "pp_plan_with_tables": (C.c_int, [_vp, _vp, _vp, C.c_int32, _i32p, C.POINTER(_PlanResult)]),
    "pp_brute_force": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _i32p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "pp_reduced_create": (C.c_int, [_vp, _vp, _vp, _pp]),
    "pp_reduced_destroy": (C.c_int, [_vp]),
    "pp_reduced_node_elimination": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "pp_reduced_edge_elimination": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "pp_reduced_reduce": (C.c_int, [_vp]),
    "pp_reduced_counts": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pp_reduced_edge": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "pp_reduced_node_alive": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_int32)]),
    "pp_reduced_edge_table": (C.c_int, [_vp, C.c_int32, _f64p]),
    "pp_reduced_log_record": (C.c_int, [_vp, C.c_int32, C.POINTER(_Record)]),
    "pp_reduced_argmin": (C.c_int, [_vp, C.c_int32, _i32p]),
    "pp_reduced_enumerate_final": (C.c_int, [_vp, C.c_int32, _i32p, C.POINTER(C.c_double)]),
}

EXPORTED = tuple(_SIGS)

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """The loaded CUDA library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (the planner has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.pp_abi_version() != 1:
            raise ImportError("libparplan_cuda ABI mismatch")
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().pp_last_error().decode()
    if rc == 1:
        raise InputError(msg)
    if rc == 2:
        raise LimitError(msg)
    if rc == 3:
        raise CudaError(msg)
    raise ParplanError(msg)


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(lib().pp_comm_unique_id(buf))
    return buf.raw


def device_count() -> int:
    n = C.c_int32()
    _check(lib().pp_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------

class Context:
    """One CUDA device + stream (pp_context)."""

    def __init__(self, device: int = 0, precision: str = "auto", stream: Optional[int] = None):
        """stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
        to order every planner call on, so the caller's CUDA events time it."""
        h = C.c_void_p()
        if stream is None:
            _check(lib().pp_context_create(device, C.byref(h)))
        else:
            _check(lib().pp_context_create_on_stream(device, C.c_void_p(stream), C.byref(h)))
        self.h = h
        self.device = device
        if precision != "auto":
            self.set_precision(precision)

    def set_precision(self, precision: str) -> None:
        _check(lib().pp_context_set_precision(self.h, {"auto": 0, "fp64": 1}[precision]))

    def set_kernel_policy(self, policy: str) -> None:
        """'auto': U16x2 min-plus for large certified folds (optimistic operand caps,
        checked on the device), one fused cooperative kernel for plans without them;
        'generic': tiled fold only; 'unfused': one launch per wave; 'conservative':
        min-plus with proven caps only; '+'-joined combinations ('generic+unfused')."""
        bits = {"auto": 0, "generic": 1, "unfused": 2, "generic_unfused": 3, "conservative": 4}
        _check(lib().pp_context_set_kernel_policy(self.h, sum(bits[p] for p in policy.split("+"))))

    def release_pools(self) -> None:
        """Return the one-shot plan pools (grow-only) to the device."""
        _check(lib().pp_context_release_pools(self.h))

    def attach_comm(self, nranks: int, rank: int, unique_id: bytes) -> None:
        """Join an NCCL communicator: plans on this context are row-sharded across ranks."""
        _check(lib().pp_context_attach_comm(self.h, nranks, rank, unique_id))

    @property
    def launches(self) -> int:
        n = C.c_int64()
        _check(lib().pp_context_launch_count(self.h, C.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().pp_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("PARPLAN_DEVICE", "0")))
    return _default_ctx


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------

@dataclass
class Layer:
    """Layer{id, kind} (graph.hpp:94-97); params = the PP_NPARAM block."""
    id: str
    kind: str
    params: Sequence[int] = ()


def conv(out_channels, kernel, stride=1, pad=0):  # models.hpp:52-54
    return ("conv2d", [out_channels, kernel, kernel, stride, stride, pad, pad])


def pool(kernel, stride, pad=0):
    return ("pool2d", [kernel, kernel, stride, stride, pad, pad])


class ComputationGraph:
    """Validated DAG with inferred shapes (ComputationGraph::create)."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle
        nl, ne = C.c_int32(), C.c_int32()
        _check(lib().pp_graph_size(self.h, C.byref(nl), C.byref(ne)))
        self.n_layers, self.n_edges = nl.value, ne.value

    @classmethod
    def create(cls, layers: Sequence[Layer], inputs: Sequence[Sequence[str]], batch: int) -> "ComputationGraph":
        n = len(layers)
        if len(inputs) != n:
            raise InputError("one input list per layer required")
        kind = np.array([KIND[l.kind] for l in layers], np.int32)
        params = np.zeros((n, 7), np.int64)
        for i, l in enumerate(layers):
            p = list(l.params)
            if l.kind == "concat" and p and isinstance(p[0], str):
                p = [DIM[p[0]]]
            params[i, : len(p)] = p
        index = {}
        for i, l in enumerate(layers):
            index.setdefault(l.id, i)
        src, dst = [], []
        for i, ins in enumerate(inputs):
            for name in ins:
                if name not in index:
                    raise InputError(f"layer '{layers[i].id}' references undeclared layer '{name}'")
                src.append(index[name])
                dst.append(i)
        ids = (C.c_char_p * n)(*[l.id.encode() for l in layers])
        s = np.array(src, np.int32)
        d = np.array(dst, np.int32)
        desc = _GraphDesc(n, len(s), batch, C.cast(ids, C.c_void_p), _ptr(kind), _ptr(params), _ptr(s), _ptr(d))
        h = C.c_void_p()
        _check(lib().pp_graph_create(C.byref(desc), C.byref(h)))
        return cls(h)

    @classmethod
    def builtin(cls, name: str, batch: int = 32) -> "ComputationGraph":
        h = C.c_void_p()
        _check(lib().pp_graph_builtin(name.encode(), batch, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().pp_graph_destroy(self.h)
            self.h = None

    def layer_count(self) -> int:
        return self.n_layers

    def edge_count(self) -> int:
        return self.n_edges

    def kinds(self) -> np.ndarray:
        k = np.zeros(self.n_layers, np.int32)
        _check(lib().pp_graph_layers(self.h, _ptr(k), None, None, None))
        return k

    def params(self) -> np.ndarray:
        p = np.zeros((self.n_layers, 7), np.int64)
        _check(lib().pp_graph_layers(self.h, None, _ptr(p), None, None))
        return p

    def shapes(self) -> np.ndarray:
        s = np.zeros((self.n_layers, 4), np.int64)
        _check(lib().pp_graph_layers(self.h, None, None, _ptr(s), None))
        return s

    def topo_order(self) -> np.ndarray:
        t = np.zeros(self.n_layers, np.int32)
        _check(lib().pp_graph_layers(self.h, None, None, None, _ptr(t)))
        return t

    def edges(self):
        s, d, p = (np.zeros(self.n_edges, np.int32) for _ in range(3))
        _check(lib().pp_graph_edges(self.h, _ptr(s), _ptr(d), _ptr(p)))
        return s, d, p

    def layer_id(self, l: int) -> str:
        buf = C.create_string_buffer(256)
        _check(lib().pp_graph_layer_id(self.h, l, buf, 256))
        return buf.value.decode()

    def index_of(self, name: str) -> int:
        for l in range(self.n_layers):
            if self.layer_id(l) == name:
                return l
        return -1

    def catalogs(self, devices: int) -> list:
        counts = np.zeros(self.n_layers, np.int32)
        _check(lib().pp_graph_catalogs(self.h, devices, counts, None))
        cfg = np.zeros(int(counts.sum()) * 4, np.int64)
        _check(lib().pp_graph_catalogs(self.h, devices, counts, _ptr(cfg)))
        out, k = [], 0
        for c in counts:
            out.append(cfg[4 * k: 4 * (k + int(c))].reshape(-1, 4))
            k += int(c)
        return out

    def schedule(self):
        """The elimination log reduce() produces, from the symbolic scheduler."""
        n, w = C.c_int32(), C.c_int32()
        _check(lib().pp_graph_schedule(self.h, C.byref(n), None, C.byref(w)))
        recs = (_Record * max(n.value, 1))()
        _check(lib().pp_graph_schedule(self.h, C.byref(n), C.cast(recs, C.c_void_p), C.byref(w)))
        return [tuple(getattr(recs[i], f) for f, _ in _Record._fields_) for i in range(n.value)], w.value


def builtin_model(name: str, batch: int = 32) -> ComputationGraph:
    return ComputationGraph.builtin(name, batch)


@dataclass
class DeviceGraph:
    """DeviceGraph(rates, bandwidth) (graph.hpp:189-225)."""
    rates: np.ndarray
    bandwidth: np.ndarray  # [n*n] row-major

    @classmethod
    def uniform(cls, n: int, compute_rate: float = 1e13, bandwidth: float = 1.25e10) -> "DeviceGraph":
        if n < 1:
            raise InputError("device graph: need at least one device")
        return cls(np.full(n, float(compute_rate)), np.full(n * n, float(bandwidth)))

    def count(self) -> int:
        return len(self.rates)

    def _desc(self):
        self._r = np.ascontiguousarray(self.rates, np.float64)
        self._b = np.ascontiguousarray(self.bandwidth, np.float64).reshape(-1)
        return _DeviceDesc(len(self._r), _ptr(self._r), _ptr(self._b))


# ---------------------------------------------------------------------------
# tables and planning
# ---------------------------------------------------------------------------

class CostTables:
    """Device-resident cost tables (CostTables, cost.hpp:148-168)."""

    def __init__(self, ctx: Context, graph: ComputationGraph, handle: C.c_void_p):
        self.ctx, self.graph, self.h = ctx, graph, handle
        self.counts = np.zeros(graph.n_layers, np.int32)
        xc = C.c_int64()
        _check(lib().pp_tables_counts(self.h, _ptr(self.counts), C.byref(xc)))
        self.xfer_cells = xc.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().pp_tables_destroy(self.h)
            self.h = None

    @property
    def build_ms(self) -> float:
        ms = C.c_double()
        _check(lib().pp_tables_build_ms(self.h, C.byref(ms)))
        return ms.value

    def download(self):
        """(catalog, node, compute, sync, xfer) as lists like the reference fields."""
        n = int(self.counts.sum())
        cfg = np.zeros(4 * n, np.int64)
        node, comp, sync = (np.zeros(n) for _ in range(3))
        xf = np.zeros(self.xfer_cells)
        _check(lib().pp_tables_download(self.h, _ptr(cfg), _ptr(node), _ptr(comp), _ptr(sync), _ptr(xf)))
        offs = np.concatenate([[0], np.cumsum(self.counts)])
        split = lambda a: [a[offs[l]:offs[l + 1]] for l in range(len(self.counts))]
        catalog = [cfg.reshape(-1, 4)[offs[l]:offs[l + 1]] for l in range(len(self.counts))]
        s, d, _ = self.graph.edges()
        xfer, k = [], 0
        for e in range(self.graph.n_edges):
            r, c = int(self.counts[s[e]]), int(self.counts[d[e]])
            xfer.append(xf[k:k + r * c].reshape(r, c))
            k += r * c
        return catalog, split(node), split(comp), split(sync), xfer

    def total_cost(self, indices) -> float:
        c = C.c_double()
        _check(lib().pp_tables_total_cost(self.h, np.ascontiguousarray(indices, np.int32), C.byref(c)))
        return c.value

    def evaluate_batch(self, indices):
        """(cost, node_total, transfer_total) of many strategies, indices [n, n_layers]
        (batched evaluate_strategy / evaluate_components totals on the device)."""
        ix = np.ascontiguousarray(indices, np.int32)
        if ix.ndim != 2 or ix.shape[1] != len(self.counts):
            raise InputError("evaluate_batch: indices must be [n, n_layers]")
        n = ix.shape[0]
        cost, node, xfer = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(lib().pp_tables_evaluate_batch(self.h, n, ix, cost, node, xfer))
        return cost, node, xfer


def build_cost_tables(graph: ComputationGraph, devices: DeviceGraph, ctx: Optional[Context] = None) -> CostTables:
    ctx = ctx or default_context()
    h = C.c_void_p()
    d = devices._desc()
    _check(lib().pp_tables_build(ctx.h, graph.h, C.byref(d), C.byref(h)))
    return CostTables(ctx, graph, h)


def upload_cost_tables(graph: ComputationGraph, catalogs, node, xfer, ctx: Optional[Context] = None) -> CostTables:
    """Hand-built / measured tables (the reference tests' injected CostTables)."""
    ctx = ctx or default_context()
    counts = np.array([len(v) for v in node], np.int32)
    cfg = None
    if catalogs is not None:
        cfg = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int64).reshape(-1, 4) for c in catalogs]).reshape(-1))
    nd = np.ascontiguousarray(np.concatenate([np.asarray(v, np.float64).reshape(-1) for v in node]), np.float64)
    xs = [np.asarray(x, np.float64).reshape(-1) for x in xfer]
    xf = np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0), np.float64)
    h = C.c_void_p()
    _check(lib().pp_tables_upload(ctx.h, graph.h, counts, _ptr(cfg), nd, xf, C.byref(h)))
    return CostTables(ctx, graph, h)


def synthetic_cost_tables(graph: ComputationGraph, configs: int, seed: int, ctx: Optional[Context] = None) -> CostTables:
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().pp_tables_synthetic(ctx.h, graph.h, configs, seed, C.byref(h)))
    return CostTables(ctx, graph, h)


def series_parallel_graph(seed: int, node_count: int, bp: float = 0.3) -> ComputationGraph:
    """Topology of random_series_parallel_graph (oracle.hpp:130-157)."""
    h = C.c_void_p()
    _check(lib().pp_graph_series_parallel(seed, node_count, bp, C.byref(h)))
    return ComputationGraph(h)


def random_series_parallel_graph(seed: int, node_count: int = 6, max_configs: int = 3, bp: float = 0.3,
                                 device_count: int = 4, ctx: Optional[Context] = None):
    """oracle.hpp:121-185 -> (graph, device tables)."""
    ctx = ctx or default_context()
    g, t = C.c_void_p(), C.c_void_p()
    _check(lib().pp_random_instance(ctx.h, seed, node_count, max_configs, bp, device_count, 0, C.byref(g), C.byref(t)))
    graph = ComputationGraph(g)
    return graph, CostTables(ctx, graph, t)


def synthetic_cost_tables64(graph: ComputationGraph, configs: int, seed: int, ctx: Optional[Context] = None) -> CostTables:
    """FP64 config-5 tables (non-dyadic values; the FP64 large-table fold)."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().pp_tables_synthetic64(ctx.h, graph.h, configs, seed, C.byref(h)))
    return CostTables(ctx, graph, h)


def synthetic_instance(seed: int, node_count: int, configs: int, bp: float = 0.3, ctx: Optional[Context] = None):
    """Config-5 generator (reference draw order, C dummy configs per layer) -> (graph, device tables)."""
    ctx = ctx or default_context()
    g, t = C.c_void_p(), C.c_void_p()
    _check(lib().pp_random_instance(ctx.h, seed, node_count, 1, bp, 1, configs, C.byref(g), C.byref(t)))
    graph = ComputationGraph(g)
    return graph, CostTables(ctx, graph, t)


@dataclass
class PlanResult:
    """PlanResult (planner.hpp:325-334) + device accounting."""
    indices: np.ndarray
    cost: float
    final_graph_nodes: int
    node_eliminations: int
    edge_eliminations: int
    precision: str = "fp64"
    waves: int = 0
    launches: int = 0
    device_ms: float = 0.0
    strategy: list = field(default_factory=list)

    def eliminations(self) -> int:
        return self.node_eliminations + self.edge_eliminations


def _result(idx, r: _PlanResult) -> PlanResult:
    out = PlanResult(idx, r.cost, r.final_graph_nodes, r.node_eliminations, r.edge_eliminations,
                     "fp64" if r.precision == 1 else "fixed", r.waves, r.launches, r.device_ms)
    out.h2d_bytes, out.d2h_bytes = r.h2d_bytes, r.d2h_bytes
    return out


def plan_with_tables(graph: ComputationGraph, tables: CostTables, k_bound: int = 8) -> PlanResult:
    idx = np.zeros(graph.n_layers, np.int32)
    r = _PlanResult()
    _check(lib().pp_plan_with_tables(tables.ctx.h, graph.h, tables.h, k_bound, idx, C.byref(r)))
    return _result(idx, r)


def plan(graph: ComputationGraph, devices: DeviceGraph, k_bound: int = 8, ctx: Optional[Context] = None) -> PlanResult:
    ctx = ctx or default_context()
    idx = np.zeros(graph.n_layers, np.int32)
    r = _PlanResult()
    d = devices._desc()
    _check(lib().pp_plan(ctx.h, graph.h, C.byref(d), k_bound, idx, C.byref(r)))
    return _result(idx, r)


def shard_layout(graph: "ComputationGraph", counts, nranks: int, rank: int):
    """Host-only: the row-sharded layout (shard.hpp) -> (blk, first, local_rows)
    per table id of the log, and the all-gathers as [(wave, table id)]."""
    counts = np.ascontiguousarray(counts, np.int32)
    nt, ng = C.c_int32(), C.c_int32()
    _check(lib().pp_shard_layout(graph.h, counts, nranks, rank, C.byref(nt), None, None, None, C.byref(ng), None, None))
    blk, first, local = (np.zeros(nt.value, np.int32) for _ in range(3))
    gw, gt = np.zeros(max(ng.value, 1), np.int32), np.zeros(max(ng.value, 1), np.int32)
    _check(lib().pp_shard_layout(graph.h, counts, nranks, rank, C.byref(nt), _ptr(blk), _ptr(first), _ptr(local),
                                 C.byref(ng), _ptr(gw), _ptr(gt)))
    return blk, first, local, list(zip(gw[:ng.value].tolist(), gt[:ng.value].tolist()))


class VirtualRanks:
    """pp_vgroup: n contexts on one device run the row-sharded (multi-GPU) plan
    path; all-gathers are device-to-device copies, the unwind reads argmin rows
    from their owner rank.  Results equal the single-GPU plan bit for bit."""

    def __init__(self, nranks: int, device: int = 0):
        h = C.c_void_p()
        _check(lib().pp_vgroup_create(device, nranks, C.byref(h)))
        self.h, self.nranks = h, nranks

    def plan(self, graph: ComputationGraph, devices: Optional[DeviceGraph] = None,
             tables: Optional[CostTables] = None, k_bound: int = 8) -> PlanResult:
        idx = np.zeros(graph.n_layers, np.int32)
        r = _PlanResult()
        d = devices._desc() if devices is not None else None
        t0 = time.perf_counter()
        _check(lib().pp_vgroup_plan(self.h, graph.h, C.cast(C.pointer(d), C.c_void_p) if d is not None else None,
                                    tables.h if tables is not None else None, k_bound, idx, C.byref(r)))
        out = _result(idx, r)
        out.wall_ms = (time.perf_counter() - t0) * 1e3
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().pp_vgroup_destroy(self.h)
            self.h = None


class PreparedPlan:
    """pp_plan_prepare: host work once, then launch() = device work only."""

    def __init__(self, graph: ComputationGraph, devices: Optional[DeviceGraph] = None,
                 tables: Optional[CostTables] = None, k_bound: int = 8, ctx: Optional[Context] = None):
        self.ctx = tables.ctx if tables is not None else (ctx or default_context())
        self.graph, self.tables = graph, tables
        h = C.c_void_p()
        d = devices._desc() if devices is not None else None
        self._dev = devices
        _check(lib().pp_plan_prepare(self.ctx.h, graph.h, C.cast(C.pointer(d), C.c_void_p) if d is not None else None,
                                     tables.h if tables is not None else None, k_bound, C.byref(h)))
        self.h = h

    def launch(self, upload_inputs: bool = False) -> None:
        _check(lib().pp_plan_launch(self.h, 1 if upload_inputs else 0))

    def fetch(self) -> PlanResult:
        idx = np.zeros(self.graph.n_layers, np.int32)
        r = _PlanResult()
        _check(lib().pp_plan_fetch(self.h, idx, C.byref(r)))
        out = _result(idx, r)
        out.h2d_bytes, out.d2h_bytes = r.h2d_bytes, r.d2h_bytes
        return out

    def profile(self):
        """[(kind, device_ms, work)] for one run with events between launches."""
        n = C.c_int32()
        _check(lib().pp_plan_profile(self.h, 0, None, None, None, C.byref(n)))
        ms, kind, work = np.zeros(n.value), np.zeros(n.value, np.int32), np.zeros(n.value)
        _check(lib().pp_plan_profile(self.h, n.value, _ptr(ms), _ptr(kind), _ptr(work), C.byref(n)))
        names = {0: "tables", 1: "wave", 2: "enumerate", 3: "finish", 4: "d2h", 5: "memset", 6: "mp_prep",
                 7: "mp_minima", 8: "mp_fold", 9: "mp_merge", 10: "fused", 11: "fused.tables",
                 12: "fused.wave", 13: "fused.enumerate", 14: "fused.finish", 15: "allgather", 16: "fused.chain",
                 17: "mp_chain", 18: "mp64_fold", 19: "tables.broadcast", 20: "allreduce.ovf"}
        return [(names[int(k)], float(m), float(w)) for k, m, w in zip(kind, ms, work)]

    def __del__(self):
        if getattr(self, "h", None):
            lib().pp_plan_destroy(self.h)
            self.h = None


def brute_force_plan(graph: ComputationGraph, tables: CostTables, budget: int = 10_000_000):
    idx = np.zeros(graph.n_layers, np.int32)
    c = C.c_double()
    v = C.c_uint64()
    _check(lib().pp_brute_force(tables.ctx.h, graph.h, tables.h, budget, idx, C.byref(c), C.byref(v)))
    return idx, c.value, v.value


class ReducedGraph:
    """The step API of planner.hpp:55-245, executed on the device."""

    def __init__(self, graph: ComputationGraph, tables: CostTables):
        self.graph, self.tables = graph, tables
        h = C.c_void_p()
        _check(lib().pp_reduced_create(tables.ctx.h, graph.h, tables.h, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().pp_reduced_destroy(self.h)
            self.h = None

    def node_elimination(self) -> bool:
        a = C.c_int32()
        _check(lib().pp_reduced_node_elimination(self.h, C.byref(a)))
        return bool(a.value)

    def edge_elimination(self) -> bool:
        a = C.c_int32()
        _check(lib().pp_reduced_edge_elimination(self.h, C.byref(a)))
        return bool(a.value)

    def reduce(self) -> None:
        _check(lib().pp_reduced_reduce(self.h))

    def _counts(self):
        v = [C.c_int32() for _ in range(4)]
        _check(lib().pp_reduced_counts(self.h, *[C.byref(x) for x in v]))
        return [x.value for x in v]

    def live_node_count(self) -> int:
        return self._counts()[2]

    def live_edge_count(self) -> int:
        return self._counts()[3]

    def edge(self, eid: int):
        v = [C.c_int32() for _ in range(5)]
        _check(lib().pp_reduced_edge(self.h, eid, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)  # src, dst, alive, rows, cols

    def live_edges(self):
        total = self._counts()[0]
        out = []
        for e in range(total):
            s, d, a, _, _ = self.edge(e)
            if a:
                out.append((e, s, d))
        return out

    def live_nodes(self):
        out = []
        a = C.c_int32()
        for l in range(self.graph.n_layers):
            _check(lib().pp_reduced_node_alive(self.h, l, C.byref(a)))
            if a.value:
                out.append(l)
        return out

    def edge_table(self, eid: int) -> np.ndarray:
        _, _, _, r, c = self.edge(eid)
        o = np.zeros(r * c)
        _check(lib().pp_reduced_edge_table(self.h, eid, o))
        return o.reshape(r, c)

    def log(self):
        n = self._counts()[1]
        out = []
        rec = _Record()
        for r in range(n):
            _check(lib().pp_reduced_log_record(self.h, r, C.byref(rec)))
            out.append(tuple(getattr(rec, f) for f, _ in _Record._fields_))
        return out

    def argmin(self, r: int) -> np.ndarray:
        rec = self.log()[r]
        _, _, _, rows, cols = self.edge(rec[4])
        o = np.zeros(rows * cols, np.int32)
        _check(lib().pp_reduced_argmin(self.h, r, o))
        return o.reshape(rows, cols)

    def enumerate_final(self, k_bound: int = 8):
        n = self.live_node_count()
        o = np.zeros(max(n, 1), np.int32)
        c = C.c_double()
        _check(lib().pp_reduced_enumerate_final(self.h, k_bound, o, C.byref(c)))
        return o[:n], c.value


def enumerate_final(rg: ReducedGraph, k_bound: int = 8):
    return rg.enumerate_final(k_bound)
