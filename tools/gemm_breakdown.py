"""Per-GEMM timing breakdown of one ResNet-50 re-forward step (run on the GPU)."""
import json
import sys
import torch
sys.path.insert(0, ".")
from oracle.train_oracle import random_batch
from paper_1808_00079_b200.executor import ReforwardNet

net = ReforwardNet.named("resnet50", 32, 224, 224, 1000)
net.plan(sys.argv[1] if len(sys.argv) > 1 else "reforward")
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
net.step(lr=0.01, use_graph=True)
torch.cuda.synchronize()
rows = net.gemm_profile_detail(iters=3)
kinds = {0: "K2D", 1: "MN2D", 2: "im2colK", 3: "im2colMN", 4: "Wtaps"}
tot = sum(r["ms"] for r in rows)
fl = sum(r["flops"] for r in rows)
print(f"GEMMs {len(rows)}: {tot:.3f} ms, {fl / tot / 1e9:.1f} TFLOP/s")
agg = {}
for r in rows:
    key = f"{kinds[int(r['a_kind'])]}x{kinds[int(r['b_kind'])]}"
    a = agg.setdefault(key, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += r["ms"]
    a[2] += r["flops"]
for k, (c, ms, f) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:18s} n={c:3d} {ms:7.3f} ms  {f / ms / 1e9:7.1f} TFLOP/s")
print("slowest launches:")
for r in sorted(rows, key=lambda r: -r["ms"])[:25]:
    print(f"  M={int(r['M']):7d} N={int(r['N']):5d} K={int(r['K']):7d} {kinds[int(r['a_kind'])]:8s} "
          f"{kinds[int(r['b_kind'])]:8s} splits={int(r['splits']):2d} {r['ms'] * 1e3:7.1f} us "
          f"{r['flops'] / r['ms'] / 1e9:7.1f} TFLOP/s")
json.dump(rows, open("gpurun_out/gemm_breakdown.json", "w"))
