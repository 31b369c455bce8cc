"""TEST INFRASTRUCTURE — export oracle/fixtures/<arch>_b<batch>_<hw>.json.gz.

Run where /root/reference exists (this container):

    python oracle/make_fixture.py resnet50 32 224

The stored set comes from the reference planner (oracle/_ref: the reference
``solve_acg`` compiled in place), or, for graphs the reference needs hours on,
from the pinned golden plan tests/golden/net_plans/<arch>_b<batch>_<hw>.json
(written by the reference, see tests/golden/make_network_plans.py).  The
network description and the re-forward schedule for that set are read from
the executor's graph builder once; the fixture then lets the CPU oracle run
without the product library (bench.py --impl reference).
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.fixture import export, fixture_path  # noqa: E402


def main(arch: str, batch: int, hw: int, classes: int = 1000) -> None:
    from paper_1808_00079_b200.executor import ReforwardNet
    from paper_1808_00079_b200.planner import reference_planner
    net = ReforwardNet.named(arch, batch, hw, hw, classes)
    verts, edges = net.graph()
    golden = os.path.join(ROOT, "tests", "golden", "net_plans", f"{arch}_b{batch}_{hw}.json")
    t0 = time.time()
    if os.path.exists(golden):
        with open(golden) as f:
            names = json.load(f)["acg"]["stored"]
        source = f"reference solve_acg, pinned in {os.path.relpath(golden, ROOT)}"
    else:
        R = reference_planner()
        g = R.from_named_edges(verts, edges)
        names = g.solve_acg().stored_names(g)
        source = f"reference solve_acg ({R.abi_name()}), {time.time() - t0:.1f} s"
    ids = {t.name: t.id for t in net.tensors()}
    rep = net.plan_with_stored([ids[n] for n in names], "reference plan")
    meta = {"arch": arch, "batch": batch, "H": hw, "W": hw, "classes": classes, "plan_source": source,
            "planned_total": rep.planned_total, "store_all_total": rep.store_all_total,
            "generator": "oracle/make_fixture.py"}
    path = fixture_path(arch, batch, hw)
    export(net, path, meta)
    print(path, os.path.getsize(path), "bytes;", source)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1]), int(a[2]), int(a[3]) if len(a) > 3 else 1000)
