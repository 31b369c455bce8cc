"""In-stream time of every instruction of one re-forward step, grouped (run on the GPU).

    python tools/step_breakdown.py [arch] [policy] [batch] [hw]

Events between eager launches (launch overhead hidden behind the GPU queue);
groups by (pass, op kind) where pass is forward / re-forward / backward, and
lists the slowest instructions.  The sum is close to the CUDA-graph step time.
"""
import json
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
policy = sys.argv[2] if len(sys.argv) > 2 else "reforward"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 32
hw = int(sys.argv[4]) if len(sys.argv) > 4 else 224

net = ReforwardNet.named(arch, batch, hw, hw, 1000)
net.plan(policy)
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
net.step(lr=0.01, use_graph=True)
torch.cuda.synchronize()
ms = net.instr_profile(iters=3)
sched = net.schedule()
ops = net.ops()
agg = defaultdict(lambda: [0, 0.0])
rows = []
for (kind, o, seg, refwd, ph), t in zip(sched, ms):
    if kind == "release":
        continue
    p = "reforward" if refwd else kind
    k = (p, ops[o].kind)
    agg[k][0] += 1
    agg[k][1] += t
    rows.append((t, p, ops[o].name, ops[o].kind, ph))
agg[("update", "sgd")] = [1, ms[-1]]
tot = sum(ms)
print(f"{arch} b{batch} {policy}: {len(rows)} instructions, {tot:.3f} ms (eager, in-stream)")
for (p, k), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {p:10s} {k:10s} n={c:4d} {t:7.3f} ms {100 * t / tot:5.1f}%")
print("slowest instructions:")
for t, p, name, k, ph in sorted(rows, reverse=True)[:30]:
    print(f"  {t * 1e3:7.1f} us  {p:10s} {k:10s} {name} {'(phase %d)' % ph if ph else ''}")
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"total_ms": tot, "groups": {f"{p}/{k}": v for (p, k), v in agg.items()},
           "instrs": [{"us": t * 1e3, "pass": p, "op": n, "kind": k} for t, p, n, k, _ in rows]},
          open(f"gpurun_out/step_breakdown_{arch}_{policy}.json", "w"), indent=0)
