"""Dump one re-forward step's loss and every parameter gradient (GPU) to a
.npz, for bitwise A/B comparison of two library builds (RF_LIB_PATH):

    RF_LIB_PATH=build/ab/lib_base.so python tools/dump_step.py resnet50 8 224 /tmp/a.npz
    RF_LIB_PATH=build/ab/lib_new.so  python tools/dump_step.py resnet50 8 224 /tmp/b.npz
    python tools/dump_step.py --compare /tmp/a.npz /tmp/b.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    diff = [k for k in a.files if not np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32))]
    print(f"{len(a.files)} arrays, {len(diff)} differ bitwise" + (f": {diff[:8]}" if diff else ""))
    sys.exit(1 if diff else 0)

import torch  # noqa: E402

from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch, B, HW, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
net = ReforwardNet.named(arch, B, HW, HW, 1000)
cache = os.path.join("plans", f"{arch}_b{B}_{HW}_reforward.json")
net.plan_cached("reforward", cache) if os.path.exists(cache) else net.plan("reforward")
net.setup(seed=0)
x, y = random_batch(net, seed=3)
net.load_batch(x.cuda(), y.cuda())
net.forward_backward()
torch.cuda.synchronize()
res = {"loss": np.array([net.read_loss()], dtype=np.float32)}
for p in net.params():
    res[f"g{p.index}_{p.name}"] = np.ascontiguousarray(net.read_param(p.index, 1), dtype=np.float32)
np.savez(out, **res)
print("saved", len(res), "arrays, loss", res["loss"][0])
