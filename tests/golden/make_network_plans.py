"""Pin the executor's BASELINE network plans against the REFERENCE planner.

TEST INFRASTRUCTURE (runs only where /root/reference exists).  For one
network (arch, batch, H) it exports the executor's tensor graph (vertex =
activation tensor, cost = arena bytes), runs the reference `solve_acg`
(/root/reference/proj/include/reforward/acg.hpp:579-600, compiled in place by
oracle/Makefile into oracle/_ref/libreforward_ref.so) on it single-threaded,
and writes tests/golden/net_plans/<arch>_b<batch>_<H>.json with the chosen set,
Eq. 1 totals, candidate max term and the reference's wall time.
tests/test_planner_networks.py checks the product planner against these files.

    python tests/golden/make_network_plans.py vgg16 32 224
    nohup nice -n 10 python tests/golden/make_network_plans.py densenet121 32 224 &

Every BASELINE network is listed in NETWORKS; the reference needs seconds
for the linear nets and ResNets and hours for DenseNet-121 / Inception-v3.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT_DIR = os.path.join(HERE, "net_plans")

# (arch, batch, H, classes): every network of BASELINE.json configs[1..4]
NETWORKS = [
    ("alexnet", 32, 224, 1000),
    ("vgg16", 32, 224, 1000),
    ("resnet50", 32, 224, 1000),
    ("resnet101", 32, 224, 1000),
    ("densenet121", 32, 224, 1000),
    ("densenet121", 64, 600, 1000),
    ("inception_v3", 32, 299, 1000),
    ("inception_v3", 64, 600, 1000),
]


def graph_of(arch: str, batch: int, hw: int, classes: int):
    from paper_1808_00079_b200.executor import ReforwardNet
    net = ReforwardNet.named(arch, batch, hw, hw, classes)
    verts, edges = net.graph()
    return verts, edges


def graph_key(verts, edges) -> str:
    h = hashlib.sha256()
    for n, c in verts:
        h.update(f"{n}:{c};".encode())
    for a, b in edges:
        h.update(f"{a}>{b};".encode())
    return h.hexdigest()


def out_path(arch: str, batch: int, hw: int) -> str:
    return os.path.join(OUT_DIR, f"{arch}_b{batch}_{hw}.json")


def run(arch: str, batch: int, hw: int, classes: int = 1000) -> dict:
    from paper_1808_00079_b200.planner import reference_planner
    verts, edges = graph_of(arch, batch, hw, classes)
    P = reference_planner()
    assert P.abi_name().startswith("reforward_ref"), P.abi_name()
    g = P.from_named_edges(verts, edges)
    t0 = time.time()
    s = g.solve_acg()
    dt = time.time() - t0
    sa = g.store_all()
    rec = {
        "generator": "tests/golden/make_network_plans.py",
        "command": f"python tests/golden/make_network_plans.py {arch} {batch} {hw}",
        "oracle": P.abi_name(),
        "arch": arch, "batch": batch, "H": hw, "W": hw, "classes": classes,
        "graph_key": graph_key(verts, edges),
        "n_vertices": len(verts), "n_edges": len(edges),
        "reference_seconds": round(dt, 1),
        "acg": {"stored": sorted(s.stored_names(g)), "stored_cost": s.stored_cost,
                "realized_max": s.realized_max, "total": s.total,
                "candidate_max_term": s.candidate_max_term},
        "store_all_total": sa.total,
    }
    os.makedirs(OUT_DIR, exist_ok=True)
    with open(out_path(arch, batch, hw), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    return rec


def main(argv):
    if len(argv) >= 3:
        arch, batch, hw = argv[0], int(argv[1]), int(argv[2])
        rec = run(arch, batch, hw)
        print(json.dumps({k: rec[k] for k in ("arch", "batch", "H", "reference_seconds")}), rec["acg"]["total"])
        return
    for arch, batch, hw, classes in NETWORKS:
        if not os.path.exists(out_path(arch, batch, hw)):
            print("missing", arch, batch, hw)


if __name__ == "__main__":
    main(sys.argv[1:])
