"""The in-graph NCCL gradient all-reduce path on one GPU.

A one-rank communicator exercises everything the multi-GPU step does inside
its CUDA graph -- bucket events after the backward instructions that finalise
each range, the side-stream NCCL all-reduce (average over 1 rank = identity),
the join of the side-stream weight-gradient GEMMs before every bucket, the
final join -- so the step must reproduce the no-communication step exactly.
"""
import numpy as np
import pytest
import torch

from oracle.train_oracle import random_batch
from paper_1808_00079_b200.executor import ReforwardNet

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch,hw,bucket_mb,comm_sms", [("resnet18", 32, 1, None), ("resnet50", 64, 4, None),
                                                       ("densenet_tiny", 32, 1, None), ("resnet50", 64, 4, "40")])
def test_single_rank_nccl_step_matches_local_step(monkeypatch, arch, hw, bucket_mb, comm_sms):
    """comm_sms: persistent GEMMs issued while a bucket is in flight leave that
    many SMs to NCCL (RFK_COMM_SMS; default 16 when world > 1) -- a different
    tile -> CTA mapping with the same per-tile K order, so still bit-identical."""
    if comm_sms is not None:
        monkeypatch.setenv("RFK_COMM_SMS", comm_sms)
    nets = []
    for with_comm in (False, True):
        net = ReforwardNet.named(arch, 4, hw, hw, 10)
        net.plan("reforward")
        net.setup(seed=7)
        x, y = random_batch(net, seed=8)
        net.load_batch(x, y)
        if with_comm:
            assert net.set_comm(1, 0, ReforwardNet.comm_unique_id(), bucket_mb << 20) >= 1
        losses = []
        for _ in range(3):
            net.step(lr=0.05, momentum=0.9, weight_decay=1e-4, use_graph=True)
            losses.append(net.read_loss())
        torch.cuda.synchronize()
        nets.append((net, losses))
    (a, la), (b, lb) = nets
    assert la == lb
    for p in a.params():
        assert np.array_equal(a.read_param(p.index, 0), b.read_param(p.index, 0)), p.name


def test_lr_schedule_reuses_the_captured_step_graph():
    """SGD hyperparameters are read from device memory: a graph step under a
    changing learning rate equals the eager step, with one capture."""
    runs = []
    for use_graph in (False, True):
        net = ReforwardNet.named("resnet18", 4, 32, 32, 10)
        net.plan("reforward")
        net.setup(seed=2)
        x, y = random_batch(net, seed=3)
        net.load_batch(x, y)
        losses = []
        for k in range(4):
            net.step(lr=0.1 / (k + 1), momentum=0.9, weight_decay=1e-4 * k, use_graph=use_graph)
            losses.append(net.read_loss())
        runs.append((net, losses))
    (a, la), (b, lb) = runs
    assert la == lb
    for p in a.params():
        assert np.array_equal(a.read_param(p.index, 0), b.read_param(p.index, 0)), p.name
