"""Pins the CPU oracle (the plain-C restatement, oracle/parplan_oracle.c) to the
REAL reference: compiled from /root/reference into oracle/_ref by
oracle/Makefile, and, where that is absent (GPU box), to the golden fixtures
tests/golden/reference_golden.json generated from it.  Bit-exact throughout."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from impls import bits

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
need_ref = pytest.mark.skipif(not O.available("reference"), reason="oracle/_ref not built (no /root/reference)")


def sha(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@need_ref
@pytest.mark.parametrize("model,D", [("lenet5", 1), ("lenet5", 4), ("alexnet", 4), ("vgg16", 4), ("vgg16", 8),
                                     ("inception_chain(3)", 2), ("inception_chain(3)", 8), ("inception_chain(4)", 16)])
def test_port_equals_reference_builtins(model, D):
    a = O.Instance.builtin(model, 32, "port").build_tables(D)
    b = O.Instance.builtin(model, 32, "reference").build_tables(D)
    assert (a.shapes() == b.shapes()).all() and (a.topo() == b.topo()).all()
    for l in range(a.n_layers):
        assert (a.catalog(l) == b.catalog(l)).all()
        assert (bits(a.node(l)) == bits(b.node(l))).all()
        assert (bits(a.compute(l)) == bits(b.compute(l))).all()
        assert (bits(a.sync(l)) == bits(b.sync(l))).all()
    for e in range(a.n_edges):
        assert (bits(a.xfer(e)) == bits(b.xfer(e))).all()
    pa, pb = a.plan(), b.plan()
    assert list(pa.indices) == list(pb.indices) and pa.cost == pb.cost
    a.reduce(), b.reduce()
    assert a.log() == b.log()
    for r, rec in enumerate(a.log()):
        if rec[0] == 0:
            assert (a.log_argmin(r) == b.log_argmin(r)).all()


@need_ref
def test_port_equals_reference_random_seeds():
    for seed in range(200):
        n, mc, bp = 1 + seed % 9, 1 + seed % 4, 0.35 * (seed % 3)
        a = O.Instance.random(seed, n, mc, bp, 4, "port")
        b = O.Instance.random(seed, n, mc, bp, 4, "reference")
        assert all((x == y).all() for x, y in zip(a.xfers(), b.xfers()))
        assert all((x == y).all() for x, y in zip(a.nodes(), b.nodes()))
        pa, pb = a.plan(), b.plan()
        assert list(pa.indices) == list(pb.indices) and pa.cost == pb.cost
        ba, bb = a.brute(), b.brute()
        assert (ba[0] == bb[0]).all() and ba[1] == bb[1] == pa.cost and ba[2] == bb[2]
        a.reduce(), b.reduce()
        assert a.log() == b.log()


@need_ref
def test_port_equals_reference_transfer_profile_nonuniform():
    rng = np.random.default_rng(3)
    D = 6
    bw = rng.uniform(1e9, 5e10, D * D)
    a = O.Instance.builtin("alexnet", 8, "port")
    b = O.Instance.builtin("alexnet", 8, "reference")
    for e in range(a.n_edges):
        for cs, cd in [([1, 1, 1, 1], [2, 1, 1, 1]), ([2, 1, 1, 1], [1, 2, 1, 1]), ([1, 2, 1, 1], [1, 1, 2, 1])]:
            try:
                sa = a.transfer_profile(e, cs, cd, D, bw)
            except O.OracleError:
                continue
            sb = b.transfer_profile(e, cs, cd, D, bw)
            assert sa == sb


@pytest.mark.parametrize("case", [c for c in GOLD["builtins"] if c["devices"] <= 16],
                         ids=lambda c: f"{c['model']}@{c['devices']}")
def test_port_matches_reference_golden(case):
    inst = O.Instance.builtin(case["model"], case["batch"], "port").build_tables(case["devices"])
    n = inst.n_layers
    assert [inst.config_count(l) for l in range(n)] == case["config_counts"]
    assert sha([inst.node(l) for l in range(n)]) == case["node_sha256"]
    assert sha([inst.compute(l) for l in range(n)]) == case["compute_sha256"]
    assert sha([inst.sync(l) for l in range(n)]) == case["sync_sha256"]
    assert [sha([inst.xfer(e)]) for e in range(inst.n_edges)] == case["xfer_sha256"]
    p = inst.plan()
    assert [int(x) for x in p.indices] == case["indices"] and float(p.cost).hex() == case["cost"]
    inst.reduce()
    assert [list(r) for r in inst.log()] == case["log"]


@pytest.mark.parametrize("case", [c for c in GOLD["synthetic"] if c["configs"] <= 64], ids=lambda c: f"C{c['configs']}")
def test_port_matches_reference_golden_synthetic(case):
    p = O.Instance.synthetic(case["seed"], case["nodes"], case["configs"], case["bp"], "port").plan()
    assert [int(x) for x in p.indices] == case["indices"] and float(p.cost).hex() == case["cost"]


def test_survey_reference_values():
    """SURVEY §8(c) reference values measured on the real reference."""
    want = {("alexnet", 4): "0.0060945131263999992", ("vgg16", 16): "0.021980223487999995",
            ("inception_chain", 16): "0.012209959391999975"}
    for (m, D), v in want.items():
        c = next(c for c in GOLD["builtins"] if c["model"] == m and c["devices"] == D)
        assert float.fromhex(c["cost"]) == float(v)
    i64 = next(c for c in GOLD["builtins"] if c["model"] == "inception_chain" and c["devices"] == 64)
    assert float.fromhex(i64["cost"]) == 0.0045765530799999976
    c256 = next(c for c in GOLD["synthetic"] if c["configs"] == 256)
    assert float.fromhex(c256["cost"]) == 727.421875 and c256["indices"][0] == 208
