"""Config-5 goldens at large C from the REAL reference (oracle/_ref):

  python tests/golden/make_golden_synth.py C [seed]

writes tests/golden/reference_synth_C{C}.json with the reference's
plan_with_tables result (indices, cost as hex-float, elimination counts) on
the config-5 synthetic graph: 1000 layers, bp 0.3, reference draw order
(oracle.hpp:121-185 with C-sized catalogs; SURVEY §9 probe7).

Reference CPU cost on this container: C=512 ~7 min / 9 GB, C=1024 ~2 h /
34 GB (single-threaded; run once, the fixture travels with the repo).
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def main():
    C = int(sys.argv[1])
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    assert O.available("reference"), "build oracle/_ref first (make -C oracle)"
    t0 = time.time()
    inst = O.Instance.synthetic(seed, 1000, C, 0.3, "reference")
    t_gen = time.time() - t0
    t0 = time.time()
    p = inst.plan()
    dt = time.time() - t0
    out = {"generator": "tests/golden/make_golden_synth.py (real reference via oracle/_ref)",
           "seed": seed, "nodes": 1000, "configs": C, "bp": 0.3,
           "indices": [int(x) for x in p.indices], "cost": float(p.cost).hex(), "cost_repr": repr(p.cost),
           "stats": [p.final_graph_nodes, p.node_eliminations, p.edge_eliminations],
           "reference_cpu_s": {"generate": t_gen, "plan_with_tables": dt}}
    path = os.path.join(HERE, f"reference_synth_C{C}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, out["cost_repr"], out["stats"], f"{dt:.0f} s")


if __name__ == "__main__":
    main()
