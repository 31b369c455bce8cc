"""Early SGD (each finished gradient bucket updated on the side stream during
the backward, runtime.cpp forward_backward) equals one update pass after the
backward, bit for bit: a parameter is never read again in a step after its
own backward, and the update is elementwise.  Two captured SGD steps with
momentum and weight decay per setting, in child processes (the knob is read
once per process), on networks with BN, residual adds, concatenations and a
plain chain; parameters, momentum-updated weights and losses compared bitwise.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from oracle.train_oracle import random_batch
from paper_1808_00079_b200.executor import ReforwardNet
arch, B, HW, out = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
net = ReforwardNet.named(arch, B, HW, HW, 10)
net.plan("reforward")
net.setup(seed=0)
x, y = random_batch(net, seed=4)
net.load_batch(x.cuda(), y.cuda())
losses = []
for _ in range(2):
    net.step(lr=0.05, momentum=0.9, weight_decay=1e-4, use_graph=True)
    torch.cuda.synchronize()
    losses.append(net.read_loss())
res = {"loss": np.array(losses, dtype=np.float32)}
for p in net.params():
    res[f"w{p.index}"] = np.ascontiguousarray(net.read_param(p.index, 0), dtype=np.float32)
np.savez(out, **res)
"""


@pytest.mark.parametrize("arch,B,HW", [("resnet18", 4, 64), ("densenet_tiny", 4, 32), ("chain8", 4, 32)])
def test_early_sgd_bit_identical(tmp_path, arch, B, HW):
    got = {}
    for mode in ("0", "1"):
        out = tmp_path / f"{arch}_{mode}.npz"
        env = dict(os.environ, RFK_EARLY_SGD=mode, RFK_SGD_BUCKET_MB="1")  # several buckets even on a small net
        subprocess.run([sys.executable, "-c", CHILD, ROOT, arch, str(B), str(HW), str(out)], env=env, check=True,
                       timeout=600)
        got[mode] = np.load(out)
    a, b = got["0"], got["1"]
    assert np.isfinite(a["loss"]).all()
    for k in a.files:
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
