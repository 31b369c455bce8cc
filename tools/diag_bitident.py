"""Diagnostic: where do re-forward and store-all (or two identical runs) diverge?

    python tools/diag_bitident.py inception_v3 64 600 [graph]

Runs one forward+backward per configuration (eager, or through the captured
graph with lr 0) and prints, in op order, the parameters whose gradients
differ bitwise, and whether a re-run of the same policy is deterministic.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402
from _parity import plan  # noqa: E402

arch = sys.argv[1]
B, HW = int(sys.argv[2]), int(sys.argv[3])
use_graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
x, y = random_batch(ReforwardNet.named(arch, B, HW, HW, 1000), seed=3)


def run(policy):
    net = ReforwardNet.named(arch, B, HW, HW, 1000)
    plan(net, arch, B, HW, policy)
    net.setup(seed=0)
    net.load_batch(x, y)
    if use_graph:
        net.step(lr=0.0, momentum=0.0, weight_decay=0.0, use_graph=True)
    else:
        net.forward_backward()
    torch.cuda.synchronize()
    out = (net.read_loss(), [(p.name, net.read_param(p.index, 1)) for p in net.params()])
    bn = [o for o in net.ops() if o.kind in ("bn", "bn_add_relu")]
    run_stats = [(o.name, net.read_bn_running(o.id)) for o in bn]
    del net
    torch.cuda.synchronize()
    return out, run_stats


def diff(a, b, label):
    (la, ga), sa = a
    (lb, gb), sb = b
    nd = [n for (n, u), (_, v) in zip(ga, gb) if not np.array_equal(u, v)]
    ns = [n for (n, (m1, v1)), (_, (m2, v2)) in zip(sa, sb) if not (np.array_equal(m1, m2) and np.array_equal(v1, v2))]
    print(f"{label}: loss {la!r} vs {lb!r}; {len(nd)} params differ; {len(ns)} BN running stats differ")
    # the backward finishes parameters in reverse op order: the LAST differing
    # parameter in op order is where the divergence started
    for n in nd[-8:]:
        print("   grad differs:", n)
    for n in ns[:8]:
        print("   running stats differ:", n)


r1 = run("reforward")
r2 = run("reforward")
s1 = run("store_all")
diff(r1, r2, "reforward vs reforward")
diff(r1, s1, "reforward vs store_all")
if os.environ.get("TWICE_STORE_ALL"):
    diff(s1, run("store_all"), "store_all vs store_all")
