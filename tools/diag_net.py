"""Per-parameter GPU vs CPU-oracle gradient errors for one small network (GPU)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.train_oracle import OracleNet, random_batch, rel_err  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch, batch, hw, classes = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
probe = ReforwardNet.named(arch, batch, hw, hw, classes)
probe.plan("reforward")
o = OracleNet(probe, emulate_bf16=True)
o.init_weights(seed=11, residual_gamma=0.1)
if arch in ("vgg11", "alexnet"):
    last = [op for op in probe.ops() if op.kind == "fc"][-1].name + ".weight"
    o.weights[last] = o.weights[last] * 0.1
x, y = random_batch(probe, seed=5)
stored, seg = probe.plan_sets()
ref_loss, ref_grads, _ = o.run_step(x, y, probe.schedule(), stored, seg)
net = ReforwardNet.named(arch, batch, hw, hw, classes)
net.plan("reforward")
net.setup(seed=0)
o.push_weights_to(net)
net.load_batch(x, y)
net.forward_backward()
torch.cuda.synchronize()
print("loss gpu", net.read_loss(), "cpu", ref_loss)
for p in net.params():
    g = net.read_param(p.index, 1)
    r = ref_grads[p.name].numpy()
    print(f"{p.name:28s} rel {rel_err(g, r):.3e} |g| {np.linalg.norm(r):.3e}")
