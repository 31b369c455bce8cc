"""Diagnostic: GPU forward tensors vs the CPU bf16-emulating forward, op by op
(free-running, not teacher-forced): where does the divergence grow?

    python tools/diag_forward_drift.py inception_v3 2 139 [classes]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.train_oracle import OracleNet, random_batch, rel_err  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch, B, HW = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
K = int(sys.argv[4]) if len(sys.argv) > 4 else 10
net = ReforwardNet.named(arch, B, HW, HW, K)
net.set_keep_grads(True)
net.plan("store_all")
net.setup(seed=0)
o = OracleNet(net, emulate_bf16=True)
o.init_weights(seed=11)
o.push_weights_to(net)
x, y = random_batch(net, seed=5)
net.load_batch(x, y)
net.forward_backward()
torch.cuda.synchronize()
vals = {o.ops[0].out: o.rb(x)}
prev = 0.0
for op in o.ops[1:]:
    if op.kind == "loss":
        ref = float(o.op_forward(op, [vals[op.inputs[0]]], y))
        print("loss gpu", net.read_loss(), "cpu", ref)
        break
    ins = [vals[i] for i in op.inputs]
    if op.kind == "fc":
        ins = [ins[0].reshape(B, -1)]
    out = o.op_forward(op, ins, y).detach()
    vals[op.out] = out
    g = net.read_tensor(op.out)
    g = torch.from_numpy(np.ascontiguousarray(g))
    if g.dim() == 4:
        g = g.permute(0, 3, 1, 2)
    e = rel_err(g.reshape(out.shape).numpy(), out.numpy())
    if e > 4e-3 and (e > 1.3 * prev or op.kind in ("fc", "avgpool", "concat")):
        print(f"{op.id:4d} {op.kind:10s} {op.name:40s} rel {e:.3e}")
    prev = max(prev, e)
