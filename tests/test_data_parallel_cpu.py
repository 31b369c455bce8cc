"""Data-parallel host logic, checked on CPU (no GPU, gloo, world size 2).

* The all-reduce bucket plan covers the flat gradient buffer exactly once and
  only reduces a range after every op owning it has run its backward.
* Data-parallel semantics: each rank runs the CPU re-forward step (oracle) on
  its shard of the batch; averaging the per-rank gradients with a gloo
  all-reduce reproduces the full-batch gradient of the BN-free conv chain
  (BASELINE.json configs[0]) — the same averaging the GPU step performs with
  NCCL inside its CUDA graph.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.train_oracle import OracleNet, random_batch, rel_err
from paper_1808_00079_b200.executor import ReforwardNet


@pytest.mark.parametrize("arch", ["chain8", "resnet18", "resnet50"])
@pytest.mark.parametrize("bucket_mb", [1, 25, 1000])
def test_bucket_plan_covers_buffer_after_producers(arch, bucket_mb):
    net = ReforwardNet.named(arch, 4, 32 if arch == "chain8" else 64, 32 if arch == "chain8" else 64, 10)
    net.plan("reforward")
    buckets = net.bucket_plan(bucket_mb << 20)
    offs = net.param_offsets()
    total = offs[-1][0] + ((offs[-1][1] + 63) // 64 * 64)
    # exact, disjoint cover of [0, total)
    spans = sorted((lo, hi) for _, lo, hi in buckets)
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    # a range is reduced only after the backward of every op owning it
    sched = net.schedule()
    params = net.params()
    pos = {}
    for k, (kind, op, _, _, _) in enumerate(sched):
        if kind == "backward":
            pos[op] = k
    op_of_param = {}
    for o in net.ops():
        for p in params:
            if p.name.startswith(o.name + "."):
                op_of_param[p.index] = o.id
    for after, lo, hi in buckets:
        for p, (off, n) in zip(params, offs):
            if off < hi and off + n > lo:
                assert pos[op_of_param[p.index]] <= after, (p.name, after)
    if bucket_mb >= 1000:
        assert len(buckets) == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    full = ReforwardNet.named("chain8", 4, 32, 32, 10)
    full.plan("reforward")
    x, y = random_batch(full, seed=21)
    shard = ReforwardNet.named("chain8", 4 // world, 32, 32, 10)
    shard.plan("reforward")
    o = OracleNet(shard)
    o.init_weights(seed=5)
    lo, hi = rank * (4 // world), (rank + 1) * (4 // world)
    stored, seg = shard.plan_sets()
    loss, grads, _ = o.run_step(x[lo:hi].contiguous(), y[lo:hi].contiguous(), shard.schedule(), stored, seg)
    names = sorted(grads)
    flat = torch.cat([grads[n].flatten() for n in names])
    dist.all_reduce(flat)
    flat /= world
    if rank == 0:
        of = OracleNet(full)
        of.init_weights(seed=5)
        st, sg = full.plan_sets()
        _, ref, _ = of.run_step(x, y, full.schedule(), st, sg)
        ref_flat = torch.cat([ref[n].flatten() for n in names])
        q.put(rel_err(flat.numpy(), ref_flat.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_gradient_average_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-5, err


def _flat_grads(net, grads):
    """Oracle gradients (canonical layout) -> the product's flat fp32 gradient
    buffer, through the product's own host-side layout (rfx_net_pack_param)."""
    import numpy as np
    ps = net.params()
    slots = [net.param_slot(p.index) for p in ps]
    total = max(o + c for o, c in slots)
    flat = np.zeros(total, dtype=np.float32)
    for p, (o, c) in zip(ps, slots):
        flat[o:o + c] = net.pack_param(p.index, grads[p.name].float().numpy())
    return torch.from_numpy(flat)


def _worker_buckets(rank, world, port, arch, hw, q):
    """Each rank: CPU re-forward step on its shard -> product flat layout ->
    all-reduce bucket by bucket in rfx_net_bucket_plan order (the order and
    ranges the GPU step issues its NCCL calls in) -> averaged flat gradient."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    per = 2
    full = ReforwardNet.named(arch, per * world, hw, hw, 10)
    full.plan("reforward")
    x, y = random_batch(full, seed=31)
    shard = ReforwardNet.named(arch, per, hw, hw, 10)
    shard.plan("reforward")
    st, sg = shard.plan_sets()

    def shard_grads(r):
        o = OracleNet(shard)
        o.init_weights(seed=6)
        lo, hi = r * per, (r + 1) * per
        _, g, _ = o.run_step(x[lo:hi].contiguous(), y[lo:hi].contiguous(), shard.schedule(), st, sg)
        return g

    flat = _flat_grads(shard, shard_grads(rank))
    buckets = shard.bucket_plan(64 << 10)  # small buckets: many NCCL-sized ranges
    covered = torch.zeros(flat.numel(), dtype=torch.int32)
    for _, lo, hi in buckets:
        seg = flat[lo:hi].clone()
        dist.all_reduce(seg)
        flat[lo:hi] = seg / world
        covered[lo:hi] += 1
    if rank == 0:
        # expected: mean of every shard's gradient (per-replica BN statistics,
        # as in data-parallel training without synchronised BN)
        ref = sum(_flat_grads(shard, shard_grads(r)) for r in range(world)) / world
        res = {"buckets": len(buckets), "cover_ok": bool((covered == 1).all()),
               "err_mean": rel_err(flat.numpy(), ref.numpy())}
        if arch == "chain8":  # no BN: the average is the full-batch gradient
            of = OracleNet(full)
            of.init_weights(seed=6)
            fst, fsg = full.plan_sets()
            _, gref, _ = of.run_step(x, y, full.schedule(), fst, fsg)
            res["err_full"] = rel_err(flat.numpy(), _flat_grads(full, gref).numpy())
        # unpacking the averaged buffer gives every parameter back in canonical layout
        g0 = shard_grads(0)
        p0 = shard.params()[0]
        o0, c0 = shard.param_slot(p0.index)
        res["unpack_shape_ok"] = shard.unpack_param(p0.index, flat[o0:o0 + c0].numpy()).shape == tuple(g0[p0.name].shape)
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("arch,hw", [("chain8", 32), ("resnet18", 32)])
def test_gloo_two_rank_bucketed_allreduce_of_product_flat_layout(arch, hw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_buckets, args=(r, 2, port, arch, hw, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["cover_ok"] and res["buckets"] > 1, res
    assert res["err_mean"] < 1e-6, res
    assert res["unpack_shape_ok"]
    if arch == "chain8":
        assert res["err_full"] < 1e-5, res
