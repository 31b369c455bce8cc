"""Diagnostic: per-parameter GPU vs CPU-oracle gradient errors, against the
plain fp32 oracle and the bf16-storage-emulating oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle.train_oracle import OracleNet, random_batch, rel_err
from paper_1808_00079_b200.executor import ReforwardNet

arch = sys.argv[1] if len(sys.argv) > 1 else "chain8"
B, HW, K = [int(v) for v in sys.argv[2:5]] if len(sys.argv) > 4 else (4, 32, 10)
net = ReforwardNet.named(arch, B, HW, HW, K)
net.plan("reforward")
net.setup(0)
o = OracleNet(net); o.init_weights(11); o.push_weights_to(net)
e = OracleNet(net, emulate_bf16=True); e.weights = o.weights
x, y = random_batch(net, 5)
net.load_batch(x, y)
net.forward_backward(); torch.cuda.synchronize()
stored, seg = net.plan_sets()
sched = net.schedule()
l32, g32, _ = o.run_step(x, y, sched, stored, seg)
l16, g16, _ = e.run_step(x, y, sched, stored, seg)
print(f"{arch} B={B} HW={HW}: loss gpu {net.read_loss():.6f} fp32 {l32:.6f} bf16-emul {l16:.6f}")
w32 = w16 = 0
for p in net.params():
    gg = net.read_param(p.index, 1)
    a, b = rel_err(gg, g32[p.name].numpy()), rel_err(gg, g16[p.name].numpy())
    w32, w16 = max(w32, a), max(w16, b)
    print(f"  {p.name:28s} vs fp32 {a:.3e}  vs bf16-emul {b:.3e}  (emul vs fp32 {rel_err(g16[p.name].numpy(), g32[p.name].numpy()):.3e})")
print(f"WORST {arch}: vs fp32 {w32:.3e} vs bf16-emul {w16:.3e}")
