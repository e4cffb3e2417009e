"""ctypes front end for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two shared libraries export the same ``orc_*`` C API (``parplan_oracle.h``):

* ``oracle/_build/libparplan_oracle.so`` — the plain-C restatement of the
  reference algorithm (``kind == "port"``);
* ``oracle/_ref/libparplan_ref.so`` — the real reference headers compiled from
  ``/root/reference`` by ``oracle/Makefile`` (``kind == "reference"``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
import this module.  The CUDA product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libparplan_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libparplan_ref.so")

KINDS = {"input": 0, "conv2d": 1, "pool2d": 2, "fully_connected": 3, "flatten": 4, "concat": 5, "softmax": 6}

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the checkers (the _ref target is skipped when /root/reference is absent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(RuntimeError):
    pass


class OracleLimitError(OracleError):
    pass


def _bind(lib: C.CDLL) -> C.CDLL:
    vp = C.c_void_p
    sig = {
        "orc_error": (C.c_char_p, []),
        "orc_kind": (C.c_int, []),
        "orc_graph": (vp, [C.c_int, C.c_int, C.c_int64, _i32p, _i64p, _i32p, _i32p, vp]),
        "orc_builtin": (vp, [C.c_char_p, C.c_int64]),
        "orc_random": (vp, [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_int]),
        "orc_synthetic": (vp, [C.c_uint64, C.c_int, C.c_int, C.c_double]),
        "orc_free": (None, [vp]),
        "orc_build_tables": (C.c_int, [vp, C.c_int, _f64p, _f64p]),
        "orc_set_tables": (C.c_int, [vp, _i32p, _i64p, _f64p, _f64p]),
        "orc_n_layers": (C.c_int, [vp]),
        "orc_n_edges": (C.c_int, [vp]),
        "orc_edges": (None, [vp, _i32p, _i32p, _i32p]),
        "orc_shapes": (None, [vp, _i64p]),
        "orc_topo": (None, [vp, _i32p]),
        "orc_config_count": (C.c_int, [vp, C.c_int]),
        "orc_catalog": (None, [vp, C.c_int, _i64p]),
        "orc_node": (None, [vp, C.c_int, _f64p]),
        "orc_compute": (None, [vp, C.c_int, _f64p]),
        "orc_sync": (None, [vp, C.c_int, _f64p]),
        "orc_xfer": (None, [vp, C.c_int, _f64p]),
        "orc_layer": (C.c_int, [vp, C.c_int, _i64p, C.c_char_p, C.c_int]),
        "orc_transfer_profile": (C.c_int, [vp, C.c_int, _i64p, _i64p, C.c_int, _f64p, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]),
        "orc_owned_region": (C.c_int, [_i64p, _i64p, C.c_int64, _i64p]),
        "orc_required_region": (C.c_int, [vp, C.c_int, _i64p, C.c_int64, _i64p]),
        "orc_enumerate_configs": (C.c_int, [C.c_int, _i64p, C.c_int, _i64p, C.c_int]),
        "orc_plan": (C.c_int, [vp, C.c_int, _i32p, C.POINTER(C.c_double), _i32p]),
        "orc_reduce": (C.c_int, [vp]),
        "orc_rg_init": (C.c_int, [vp]),
        "orc_rg_node": (C.c_int, [vp]),
        "orc_rg_edge": (C.c_int, [vp]),
        "orc_rg_edges_total": (C.c_int, [vp]),
        "orc_rg_edge_info": (C.c_int, [vp, C.c_int, _i32p]),
        "orc_log_size": (C.c_int, [vp]),
        "orc_log_record": (C.c_int, [vp, C.c_int, _i32p]),
        "orc_log_argmin": (C.c_int, [vp, C.c_int, _i32p]),
        "orc_edge_table_dims": (C.c_int, [vp, C.c_int, _i32p]),
        "orc_edge_table": (C.c_int, [vp, C.c_int, _f64p]),
        "orc_live_nodes": (C.c_int, [vp, C.c_void_p]),
        "orc_enumerate_final": (C.c_int, [vp, C.c_int, _i32p, C.POINTER(C.c_double)]),
        "orc_total_cost": (C.c_double, [vp, _i32p]),
        "orc_brute": (C.c_int, [vp, C.c_uint64, _i32p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
        "orc_fold": (None, [C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _i32p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_LIBS: dict[str, C.CDLL] = {}


def load(kind: str = "port") -> C.CDLL:
    path = PORT_SO if kind == "port" else REF_SO
    if kind not in _LIBS:
        if not os.path.exists(path):
            raise OracleError(f"checker library missing: {path} (run `make -C oracle`)")
        _LIBS[kind] = _bind(C.CDLL(path))
    return _LIBS[kind]


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


@dataclass
class Plan:
    indices: np.ndarray
    cost: float
    final_graph_nodes: int
    node_eliminations: int
    edge_eliminations: int


class Instance:
    """One graph (+ tables) inside a checker library."""

    def __init__(self, lib: C.CDLL, handle: int):
        if not handle:
            raise OracleError(lib.orc_error().decode())
        self.lib = lib
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_free(self.h)
            self.h = None

    def _check(self, rc: int):
        if rc == 2:
            raise OracleLimitError(self.lib.orc_error().decode())
        if rc:
            raise OracleError(self.lib.orc_error().decode())

    # -- construction ---------------------------------------------------
    @classmethod
    def builtin(cls, name: str, batch: int = 32, kind: str = "port") -> "Instance":
        lib = load(kind)
        return cls(lib, lib.orc_builtin(name.encode(), batch))

    @classmethod
    def graph(cls, kinds, params, edge_src, edge_dst, batch, ids=None, kind: str = "port") -> "Instance":
        lib = load(kind)
        k = np.ascontiguousarray(kinds, np.int32)
        p = np.ascontiguousarray(params, np.int64).reshape(-1)
        s = np.ascontiguousarray(edge_src, np.int32)
        d = np.ascontiguousarray(edge_dst, np.int32)
        idp = None
        if ids is not None:
            arr = (C.c_char_p * len(ids))(*[i.encode() for i in ids])
            idp = C.cast(arr, C.c_void_p)
        return cls(lib, lib.orc_graph(len(k), len(s), batch, k, p, s, d, idp))

    @classmethod
    def random(cls, seed, node_count=6, max_configs=3, bp=0.3, device_count=4, kind: str = "port") -> "Instance":
        lib = load(kind)
        return cls(lib, lib.orc_random(seed, node_count, max_configs, bp, device_count))

    @classmethod
    def synthetic(cls, seed, node_count, configs, bp=0.3, kind: str = "port") -> "Instance":
        lib = load(kind)
        return cls(lib, lib.orc_synthetic(seed, node_count, configs, bp))

    def build_tables(self, n_devices: int, rates=None, bw=None) -> "Instance":
        rates = np.full(n_devices, 1e13) if rates is None else np.ascontiguousarray(rates, np.float64)
        bw = np.full(n_devices * n_devices, 1.25e10) if bw is None else np.ascontiguousarray(bw, np.float64).reshape(-1)
        self._check(self.lib.orc_build_tables(self.h, n_devices, rates, bw))
        return self

    def set_tables(self, catalogs, node, xfer) -> "Instance":
        ncfg = np.array([len(c) for c in catalogs], np.int32)
        cfg = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int64).reshape(-1, 4) for c in catalogs]), np.int64)
        nd = np.ascontiguousarray(np.concatenate([np.asarray(v, np.float64).reshape(-1) for v in node]), np.float64)
        xs = [np.asarray(x, np.float64).reshape(-1) for x in xfer]
        xf = np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0), np.float64)
        self._check(self.lib.orc_set_tables(self.h, ncfg, cfg.reshape(-1), nd, xf))
        return self

    # -- accessors --------------------------------------------------------
    @property
    def n_layers(self) -> int:
        return self.lib.orc_n_layers(self.h)

    @property
    def n_edges(self) -> int:
        return self.lib.orc_n_edges(self.h)

    def edges(self):
        n = self.n_edges
        s, d, p = (np.zeros(n, np.int32) for _ in range(3))
        self.lib.orc_edges(self.h, s, d, p)
        return s, d, p

    def shapes(self) -> np.ndarray:
        o = np.zeros(4 * self.n_layers, np.int64)
        self.lib.orc_shapes(self.h, o)
        return o.reshape(-1, 4)

    def topo(self) -> np.ndarray:
        o = np.zeros(self.n_layers, np.int32)
        self.lib.orc_topo(self.h, o)
        return o

    def layer(self, l: int):
        p = np.zeros(7, np.int64)
        buf = C.create_string_buffer(128)
        k = self.lib.orc_layer(self.h, l, p, buf, 128)
        return k, p, buf.value.decode()

    def config_count(self, l: int) -> int:
        return self.lib.orc_config_count(self.h, l)

    def catalog(self, l: int) -> np.ndarray:
        o = np.zeros(4 * self.config_count(l), np.int64)
        self.lib.orc_catalog(self.h, l, o)
        return o.reshape(-1, 4)

    def node(self, l: int) -> np.ndarray:
        o = np.zeros(self.config_count(l), np.float64)
        self.lib.orc_node(self.h, l, o)
        return o

    def compute(self, l: int) -> np.ndarray:
        o = np.zeros(self.config_count(l), np.float64)
        self.lib.orc_compute(self.h, l, o)
        return o

    def sync(self, l: int) -> np.ndarray:
        o = np.zeros(self.config_count(l), np.float64)
        self.lib.orc_sync(self.h, l, o)
        return o

    def xfer(self, e: int) -> np.ndarray:
        s, d, _ = self.edges()
        o = np.zeros(self.config_count(int(s[e])) * self.config_count(int(d[e])), np.float64)
        self.lib.orc_xfer(self.h, e, o)
        return o.reshape(self.config_count(int(s[e])), self.config_count(int(d[e])))

    def catalogs(self):
        return [self.catalog(l) for l in range(self.n_layers)]

    def nodes(self):
        return [self.node(l) for l in range(self.n_layers)]

    def xfers(self):
        return [self.xfer(e) for e in range(self.n_edges)]

    # -- planning -----------------------------------------------------------
    def plan(self, k_bound: int = 8) -> Plan:
        idx = np.zeros(self.n_layers, np.int32)
        cost = C.c_double()
        st = np.zeros(3, np.int32)
        self._check(self.lib.orc_plan(self.h, k_bound, idx, C.byref(cost), st))
        return Plan(idx, cost.value, int(st[0]), int(st[1]), int(st[2]))

    def reduce(self) -> "Instance":
        self._check(self.lib.orc_reduce(self.h))
        return self

    # -- ReducedGraph step API ----------------------------------------------
    def rg_init(self) -> "Instance":
        self._check(self.lib.orc_rg_init(self.h))
        return self

    def node_elimination(self) -> bool:
        return self.lib.orc_rg_node(self.h) == 1

    def edge_elimination(self) -> bool:
        return self.lib.orc_rg_edge(self.h) == 1

    def live_edges(self):
        out = []
        info = np.zeros(3, np.int32)
        for e in range(self.lib.orc_rg_edges_total(self.h)):
            if self.lib.orc_rg_edge_info(self.h, e, info) == 0 and info[2]:
                out.append((e, int(info[0]), int(info[1])))
        return out

    def log(self):
        out = []
        rec = np.zeros(7, np.int32)
        for r in range(self.lib.orc_log_size(self.h)):
            self.lib.orc_log_record(self.h, r, rec)
            out.append(tuple(int(x) for x in rec))
        return out

    def log_argmin(self, r: int) -> np.ndarray:
        rec = self.log()[r]
        nu = self.config_count(rec[5])
        nv = self.config_count(rec[6])
        o = np.zeros(nu * nv, np.int32)
        self._check(self.lib.orc_log_argmin(self.h, r, o))
        return o.reshape(nu, nv)

    def edge_table(self, e: int) -> np.ndarray:
        d = np.zeros(2, np.int32)
        self._check(self.lib.orc_edge_table_dims(self.h, e, d))
        o = np.zeros(int(d[0]) * int(d[1]), np.float64)
        self._check(self.lib.orc_edge_table(self.h, e, o))
        return o.reshape(int(d[0]), int(d[1]))

    def live_nodes(self) -> np.ndarray:
        n = self.lib.orc_live_nodes(self.h, None)
        o = np.zeros(n, np.int32)
        self.lib.orc_live_nodes(self.h, o.ctypes.data_as(C.c_void_p))
        return o

    def enumerate_final(self, k_bound: int = 8):
        n = self.lib.orc_live_nodes(self.h, None)
        o = np.zeros(max(n, 1), np.int32)
        c = C.c_double()
        self._check(self.lib.orc_enumerate_final(self.h, k_bound, o, C.byref(c)))
        return o[:n], c.value

    def total_cost(self, indices) -> float:
        return self.lib.orc_total_cost(self.h, np.ascontiguousarray(indices, np.int32))

    def brute(self, budget: int = 10_000_000):
        idx = np.zeros(self.n_layers, np.int32)
        c = C.c_double()
        v = C.c_uint64()
        self._check(self.lib.orc_brute(self.h, budget, idx, C.byref(c), C.byref(v)))
        return idx, c.value, v.value

    def transfer_profile(self, e, c_src, c_dst, n_devices, bw=1.25e10):
        bwm = np.full(n_devices * n_devices, float(bw)) if np.isscalar(bw) else np.ascontiguousarray(bw, np.float64)
        s, b = C.c_double(), C.c_double()
        self._check(self.lib.orc_transfer_profile(self.h, e, np.asarray(c_src, np.int64), np.asarray(c_dst, np.int64),
                                                  n_devices, bwm, C.byref(s), C.byref(b)))
        return s.value, b.value

    def required_region(self, e, dst_config, part):
        o = np.zeros(8, np.int64)
        self._check(self.lib.orc_required_region(self.h, e, np.asarray(dst_config, np.int64), part, o))
        return o[:4], o[4:]


def enumerate_configs(kind: int, shape, devices: int, lib_kind: str = "port") -> np.ndarray:
    lib = load(lib_kind)
    sh = np.asarray(shape, np.int64)
    n = lib.orc_enumerate_configs(kind, sh, devices, np.zeros(4, np.int64), 0)
    o = np.zeros(4 * max(n, 1), np.int64)
    lib.orc_enumerate_configs(kind, sh, devices, o, n)
    return o[: 4 * n].reshape(-1, 4)


def owned_region(shape, config, part, lib_kind: str = "port"):
    lib = load(lib_kind)
    o = np.zeros(8, np.int64)
    if lib.orc_owned_region(np.asarray(shape, np.int64), np.asarray(config, np.int64), part, o):
        raise OracleError(lib.orc_error().decode())
    return o[:4], o[4:]


def fold(w, t1, t2, lib_kind: str = "port"):
    lib = load(lib_kind)
    w = np.ascontiguousarray(w, np.float64)
    t1 = np.ascontiguousarray(t1, np.float64)
    t2 = np.ascontiguousarray(t2, np.float64)
    nu, nw = t1.shape
    nv = t2.shape[1]
    out = np.zeros(nu * nv, np.float64)
    am = np.zeros(nu * nv, np.int32)
    lib.orc_fold(nu, nw, nv, w, t1.reshape(-1), t2.reshape(-1), out, am)
    return out.reshape(nu, nv), am.reshape(nu, nv)
