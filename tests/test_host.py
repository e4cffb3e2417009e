"""Host logic of libparplan_cuda.so that runs without a GPU: graph creation and
validation, catalogs, the symbolic elimination scheduler (vs the reference log),
error mapping, and the exported C ABI (every symbol include/parplan_c.h declares)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def P():
    import paper_1802_04924_b200 as pkg

    return pkg


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "parplan_c.h")).read()
    declared = set(re.findall(r"\b(pp_[a-z_]+)\s*\(", header))
    lib = os.path.join(ROOT, "paper_1802_04924_b200", "libparplan_cuda.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert declared and declared <= exported, declared - exported
    P().lib()  # loads, ABI version check


def test_no_gpu_means_no_context():
    pkg = P()
    if pkg.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(pkg.CudaError):
        pkg.Context(0)


@pytest.mark.parametrize("model,D", [("lenet5", 4), ("alexnet", 4), ("vgg16", 16), ("inception_chain(3)", 4),
                                     ("inception_chain", 16), ("inception_chain", 64)])
def test_graph_catalogs_schedule_match_reference(model, D):
    g = P().builtin_model(model, 32)
    o = O.Instance.builtin(model, 32, "port")
    assert (g.shapes() == o.shapes()).all() and (g.topo_order() == o.topo()).all()
    s, d, p = g.edges()
    so, do, po = o.edges()
    assert (s == so).all() and (d == do).all() and (p == po).all()
    for l, c in enumerate(g.catalogs(D)):
        assert (c == O.enumerate_configs(o.layer(l)[0], o.shapes()[l], D)).all()
    o.build_tables(D if D <= 16 else 2)  # the schedule is topology-only
    o.reduce()
    sched, waves = g.schedule()
    assert [r[:7] for r in sched] == o.log()
    # waves respect the dependency DAG
    wave_of = {}
    for r in sched:
        for e in (r[2], r[3]):
            assert wave_of.get(e, 0) < r[7]
        wave_of[r[4]] = r[7]


def _graph_of(inst):
    pkg = P()
    names = {v: k for k, v in O.KINDS.items()}
    layers, inputs = [], [[] for _ in range(inst.n_layers)]
    for l in range(inst.n_layers):
        k, p, _ = inst.layer(l)
        layers.append(pkg.Layer(f"n{l}", names[k], list(p)))
    s, d, _ = inst.edges()
    for e in range(len(s)):
        inputs[d[e]].append(f"n{s[e]}")
    return pkg.ComputationGraph.create(layers, inputs, 8)


def test_scheduler_matches_reference_on_random_graphs():
    for seed in range(300):
        inst = O.Instance.random(seed, 1 + seed % 40, 2, 0.15 * (seed % 5), 4)
        inst.reduce()
        assert [r[:7] for r in _graph_of(inst).schedule()[0]] == inst.log()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_scheduler_matches_reference_on_1k_node_graphs(seed):
    inst = O.Instance.synthetic(seed, 1000, 2, 0.3)
    inst.reduce()
    g = P().series_parallel_graph(seed, 1000, 0.3)
    assert [r[:7] for r in g.schedule()[0]] == inst.log()


def test_graph_errors_match_reference_messages():
    pkg = P()
    L = pkg.Layer
    with pytest.raises(pkg.InputError, match="ghost"):
        pkg.ComputationGraph.create([L("in", "input", [1, 4, 4]), L("c", "softmax")], [[], ["ghost"]], 1)
    with pytest.raises(pkg.InputError, match="duplicate layer id 'x'"):
        pkg.ComputationGraph.create([L("x", "input", [1, 4, 4]), L("x", "softmax")], [[], ["x"]], 1)
    with pytest.raises(pkg.InputError, match="cycle"):
        pkg.ComputationGraph.create([L("in", "input", [2, 4, 4]), L("a", "softmax"), L("b", "softmax")],
                                    [[], ["b"], ["a"]], 1)
    with pytest.raises(pkg.InputError, match="non-positive inferred extent"):
        pkg.ComputationGraph.create([L("in", "input", [3, 4, 4]), L("c", "conv2d", [4, 7, 7, 1, 1, 0, 0])],
                                    [[], ["in"]], 1)
    with pytest.raises(pkg.InputError, match="unknown model 'resnet50'"):
        pkg.builtin_model("resnet50")
    with pytest.raises(pkg.InputError, match="module count must be >= 1"):
        pkg.builtin_model("inception_chain(0)")
    with pytest.raises(pkg.InputError, match="invalid module count"):
        pkg.builtin_model("inception_chain(x)")


def test_python_layer_api_round_trip():
    pkg = P()
    g = pkg.builtin_model("vgg16", 32)
    assert g.layer_count() == 21 and g.index_of("pool5") >= 0
    assert list(g.shapes()[g.index_of("pool5")]) == [32, 512, 7, 7]
    assert list(g.shapes()[g.index_of("fc1")]) == [32, 4096, 1, 1]
