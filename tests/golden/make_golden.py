"""Generates tests/golden/*.json from the REAL reference (oracle/_ref, compiled
from /root/reference by oracle/Makefile).  Run here (the CPU container); the
fixtures travel with the repo so GPU-box tests never need /root/reference.

  python tests/golden/make_golden.py [--big]

--big adds Inception-chain(12)@64 (~2 min of reference CPU time) and the
config-5 synthetic graph at C=256 (~45 s).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def sha(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def builtin_case(model, D, batch=32):
    t0 = time.time()
    inst = O.Instance.builtin(model, batch, "reference").build_tables(D)
    t_tables = time.time() - t0
    t0 = time.time()
    p = inst.plan()
    t_plan = time.time() - t0
    inst.reduce()
    log = inst.log()
    am = [sha([inst.log_argmin(r).astype(np.int32)]) for r, rec in enumerate(log) if rec[0] == 0]
    return {
        "model": model, "devices": D, "batch": batch,
        "config_counts": [inst.config_count(l) for l in range(inst.n_layers)],
        "node_sha256": sha([inst.node(l) for l in range(inst.n_layers)]),
        "compute_sha256": sha([inst.compute(l) for l in range(inst.n_layers)]),
        "sync_sha256": sha([inst.sync(l) for l in range(inst.n_layers)]),
        "xfer_sha256": [sha([inst.xfer(e)]) for e in range(inst.n_edges)],
        "xfer_sample": [[e, float(inst.xfer(e).reshape(-1)[k]).hex()] for e in range(0, inst.n_edges, 7)
                        for k in (0, inst.xfer(e).size // 2, inst.xfer(e).size - 1)],
        "indices": [int(x) for x in p.indices], "cost": float(p.cost).hex(), "cost_repr": repr(p.cost),
        "stats": [p.final_graph_nodes, p.node_eliminations, p.edge_eliminations],
        "log": [list(r) for r in log], "argmin_sha256": am,
        "reference_cpu_s": {"build_cost_tables": t_tables, "plan_with_tables": t_plan},
    }


def synthetic_case(seed, n, C):
    inst = O.Instance.synthetic(seed, n, C, 0.3, "reference")
    t0 = time.time()
    p = inst.plan()
    dt = time.time() - t0
    return {"seed": seed, "nodes": n, "configs": C, "bp": 0.3, "indices": [int(x) for x in p.indices],
            "cost": float(p.cost).hex(), "cost_repr": repr(p.cost),
            "stats": [p.final_graph_nodes, p.node_eliminations, p.edge_eliminations], "reference_cpu_s": dt}


def main():
    big = "--big" in sys.argv
    assert O.available("reference"), "build oracle/_ref first (make -C oracle)"
    cases = [("lenet5", 4), ("alexnet", 4), ("vgg16", 4), ("vgg16", 16), ("inception_chain(3)", 4),
             ("inception_chain", 16), ("inception_chain(13)", 16)]
    if big:
        cases.append(("inception_chain", 64))
    out = {"generator": "tests/golden/make_golden.py (real reference via oracle/_ref)", "builtins": []}
    for m, D in cases:
        print("builtin", m, D, flush=True)
        out["builtins"].append(builtin_case(m, D))
    out["synthetic"] = []
    for C in ([16, 64, 256] if big else [16, 64]):
        print("synthetic C", C, flush=True)
        out["synthetic"].append(synthetic_case(1, 1000, C))
    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main()
