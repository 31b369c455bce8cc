import sys; sys.path.insert(0, ".")
import torch
from oracle.train_oracle import random_batch
from paper_1808_00079_b200.executor import ReforwardNet
for arch in ("resnet50", "densenet121"):
    net = ReforwardNet.named(arch, 32, 224, 224, 1000); net.plan("reforward"); net.setup(0)
    x, y = random_batch(net, 0); net.load_batch(x.cuda(), y.cuda())
    print(arch, "backward convs:", sum(1 for o in net.ops() if o.kind == "conv"), flush=True)
    net.forward_backward(); torch.cuda.synchronize()
