"""Step time with kernels ablated (RFK_ABLATE, timing experiments only).

    RFK_ABLATE=<mask> python tools/ablate_time.py [arch] [batch] [hw]

Prints the CUDA-graph step time of the re-forward plan; the loss is
meaningless when kernels are skipped -- this bounds what fusing them away
could save.
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
hw = int(sys.argv[3]) if len(sys.argv) > 3 else 224
net = ReforwardNet.named(arch, batch, hw, hw, 1000)
cache = os.path.join("plans", f"{arch}_b{batch}_{hw}_reforward.json")
if os.path.exists(cache):
    net.plan_cached("reforward", cache)  # the exact plan, computed once (minutes for Inception-v3)
else:
    net.plan("reforward")
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
s = torch.cuda.Stream()
for _ in range(5):
    net.step(lr=0.0, momentum=0.0, weight_decay=0.0, use_graph=True, stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 30
e0.record(s)
for _ in range(n):
    net.step(lr=0.0, momentum=0.0, weight_decay=0.0, use_graph=True, stream=s)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"RFK_ABLATE={os.environ.get('RFK_ABLATE', '0')}: {ms:.3f} ms/step  {batch / ms * 1e3:.0f} img/s")
