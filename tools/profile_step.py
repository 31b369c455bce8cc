"""One eager ResNet-50 re-forward train step (for ncu launch lists / captures)."""
import sys
import torch
sys.path.insert(0, ".")
from oracle.train_oracle import random_batch
from paper_1808_00079_b200.executor import ReforwardNet

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
policy = sys.argv[2] if len(sys.argv) > 2 else "reforward"
net = ReforwardNet.named(arch, 32, 224, 224, 1000)
net.plan(policy)
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
torch.cuda.synchronize()
net.step(lr=0.01, use_graph=False)
torch.cuda.synchronize()
print("loss", net.read_loss())
