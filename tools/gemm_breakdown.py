"""Per-GEMM timing breakdown of one re-forward step (run on the GPU).

    python tools/gemm_breakdown.py [policy] [arch] [batch] [hw]

For every GEMM launch of the step: measured time (CUDA events between eager
launches), algorithmic flops and bytes, and its roofline time
max(flops / tensor peak, bytes / HBM peak) with the measured peaks of
MEASURED_PEAKS.json.  The ratio roofline / measured is how far that launch is
from its own bound (1.0 = at the roofline).
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "reforward"
arch = sys.argv[2] if len(sys.argv) > 2 else "resnet50"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 32
hw = int(sys.argv[4]) if len(sys.argv) > 4 else 224
try:
    peaks = json.load(open("MEASURED_PEAKS.json"))
except Exception:
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
PT, PB = peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9

net = ReforwardNet.named(arch, batch, hw, hw, 1000)
net.plan(policy)
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
net.step(lr=0.01, use_graph=True)
torch.cuda.synchronize()
rows = net.gemm_profile_detail(iters=3)
kinds = {0: "K2D", 1: "MN2D", 2: "im2colK", 3: "im2colMN", 4: "Wtaps"}
for r in rows:
    r["t_roof_ms"] = max(r["flops"] / PT, r["bytes"] / PB) * 1e3
    r["bound"] = "tensor" if r["flops"] / PT >= r["bytes"] / PB else "hbm"
tot = sum(r["ms"] for r in rows)
fl = sum(r["flops"] for r in rows)
roof = sum(r["t_roof_ms"] for r in rows)
print(f"{arch} b{batch} {policy}: GEMMs {len(rows)}: {tot:.3f} ms, {fl / tot / 1e9:.1f} TFLOP/s, "
      f"roofline {roof:.3f} ms -> {roof / tot:.3f} of roofline")
agg = {}
for r in rows:
    key = f"{kinds[int(r['a_kind'])]}x{kinds[int(r['b_kind'])]}"
    a = agg.setdefault(key, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += r["ms"]
    a[2] += r["flops"]
    a[3] += r["t_roof_ms"]
for k, (c, ms, f, rf) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:18s} n={c:3d} {ms:7.3f} ms  {f / ms / 1e9:7.1f} TFLOP/s  roof {rf:6.3f} ms ({rf / ms:.2f})")
print("largest gaps to the roofline (measured - roofline):")
for r in sorted(rows, key=lambda r: -(r["ms"] - r["t_roof_ms"]))[:30]:
    print(f"  M={int(r['M']):7d} N={int(r['N']):5d} K={int(r['K']):6d} {kinds[int(r['a_kind'])]:8s} "
          f"{kinds[int(r['b_kind'])]:8s} bn={int(r['block_n']):3d} sp={int(r['splits']):2d} "
          f"{r['ms'] * 1e3:7.1f} us roof {r['t_roof_ms'] * 1e3:6.1f} us ({r['bound']}) "
          f"{r['flops'] / r['ms'] / 1e9:7.1f} TF/s {r['bytes'] / r['ms'] / 1e6:7.1f} GB/s")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open(f"gpurun_out/gemm_breakdown_{arch}_{policy}.json", "w"))
