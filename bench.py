#!/usr/bin/env python
"""Headline benchmark: ResNet-50 re-forward training on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One "step" = one SGD iteration of ResNet-50 at batch 32 per GPU on synthetic
(32, 3, 224, 224) images with random-init weights: first forward storing only
the planner's V^R, backward re-forwarding each segment, SGD update (BASELINE.json
configs[3], the config the headline metric is quoted on).  Prints ONE JSON line
(rank 0).  `value` = whole-job images/s with inputs resident in HBM; `e2e` =
the same through the public API with a pinned-host H2D copy of the batch and a
D2H read of the loss inside every timed step.  The same run also times the
store-all plan to report the re-forward time overhead, and reports the
activation memory (planner Eq. 1 vs store-all) the overhead buys.

`--impl reference` times the CPU path instead: the CPU fp32 re-forward train
step (oracle/train_oracle.py) at the same batch, following the plan the
reference planner chose (committed fixture oracle/fixtures/, exported once
with oracle/_ref), on every host core; the product library is not loaded.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 train imgs/s at re-forward peak mem; overhead vs store-all"
ARCH, HW, CLASSES = "resnet50", 224, 1000


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) is polled every few milliseconds from a thread, so
    even a ~100 ms timed region gets tens of samples; nvidia-smi (one query
    per ~0.2 s) is the fallback when NVML is unavailable.
    """

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index: int = 0, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            self._stop.wait(self.period)

    def _run_smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                self.samples.append((float(f[0]), float(f[1]), int(f[2], 16)))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
        except Exception:
            return self._run_smi()
        try:
            self._run_nvml(nv)
        finally:
            nv.nvmlShutdown()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(s[0] for s in self.samples)
        mask = 0
        for s in self.samples:
            mask |= int(s[2])
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": [n for n, bit in self.REASONS if mask & bit], "samples": len(self.samples)}


def dist_setup(n):
    import torch
    import torch.distributed as dist
    if n > 1 or "WORLD_SIZE" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
        rank, world = dist.get_rank(), dist.get_world_size()
    else:
        rank, world = 0, 1
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    return rank, world, local


class GradView:
    """Zero-copy torch view of the executor's flat fp32 gradient buffer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def time_steps(net, steps, warmup, stream, world, allreduce=None, e2e=None):
    """Device time of `steps` steps (CUDA events on the launching stream)."""
    import torch
    import torch.distributed as dist

    def one():
        if e2e is not None:
            e2e()
        if allreduce is None:
            net.step(lr=0.01, momentum=0.9, weight_decay=1e-4, use_graph=True, stream=stream)
        else:
            net.run_phase(0, use_graph=True, stream=stream)
            allreduce()
            net.run_phase(1, lr=0.01, momentum=0.9, weight_decay=1e-4, use_graph=True, stream=stream)
        if e2e is not None:
            net.read_loss(stream=stream)  # D2H of the step's result

    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
    return ms / steps


def time_e2e(net, steps, warmup, stream, world, xh, yh):
    """Device time of `steps` end-to-end steps: H2D of each step's batch (staged
    one step ahead on a copy stream), pack, the step graph, D2H of the loss."""
    import torch
    import torch.distributed as dist
    copy = torch.cuda.Stream()

    losses = torch.zeros(max(steps, warmup) + 1, dtype=torch.float32).pin_memory()

    def run(n, start_event=None):
        if start_event is not None:
            copy.wait_event(start_event)
        net.stage_batch(xh, yh, 0, copy_stream=copy)
        for k in range(n):
            if k + 1 < n:
                net.stage_batch(xh, yh, (k + 1) % 2, copy_stream=copy)
            net.use_batch(k % 2, stream=stream)
            net.step(lr=0.01, momentum=0.9, weight_decay=1e-4, use_graph=True, stream=stream)
            # D2H of the step's result into pinned memory, in stream order (the
            # host reads the values after the run, as an async training loop
            # would log them)
            net.copy_loss(losses, k, stream=stream)

    run(warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(steps, start_event=e0)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if not all(math.isfinite(v) for v in losses[:steps].tolist()):
        raise RuntimeError("non-finite loss in the end-to-end run")
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
    return ms / steps


def build_net(batch, policy, seed=0):
    from paper_1808_00079_b200.executor import ReforwardNet
    net = ReforwardNet.named(ARCH, batch, HW, HW, CLASSES)
    t0 = time.time()
    cache = os.path.join(ROOT, "plans", f"{ARCH}_b{batch}_{HW}_{policy}.json")
    if policy == "reforward" and os.path.exists(cache):
        rep = net.plan_cached(policy, cache)  # exact plan computed once (minutes for Inception-v3)
    else:
        rep = net.plan(policy)
    plan_s = time.time() - t0
    net.setup(seed=seed)
    return net, rep, plan_s


def cpu_baseline_sample(threads=None, gpu_stored=None, batch=32):
    """Bounded CPU sample: one re-forward train step of the benched network.

    With a fixture (oracle/fixtures/<arch>_b<batch>_<hw>.json.gz: the graph,
    the REFERENCE planner's stored set and the re-forward schedule, exported
    once by oracle/make_fixture.py) the step runs at the benched batch without
    touching the product library.  Networks without a fixture fall back to
    batch 2 with the plan of the GPU run."""
    import torch
    from oracle.fixture import FixtureNet, fixture_path
    from oracle.train_oracle import OracleNet, random_batch
    if threads:
        torch.set_num_threads(threads)
    if os.path.exists(fixture_path(ARCH, batch, HW)):
        net = FixtureNet.named(ARCH, batch, HW)
        b = batch
        plan_kind = net.meta["plan_source"]
    else:
        from paper_1808_00079_b200.executor import ReforwardNet
        b = 2
        net = ReforwardNet.named(ARCH, b, HW, HW, CLASSES)
        # every Eq. 1 cost scales with the batch, so the GPU run's optimal
        # vertex set is also optimal at batch 2 (same tensor ids)
        net.plan_with_stored(gpu_stored, "gpu-plan") if gpu_stored is not None else net.plan("reforward")
        plan_kind = "the GPU run's plan" if gpu_stored is not None else "product planner"
    o = OracleNet(net)
    o.init_weights(0)
    x, y = random_batch(net, 0)
    st, seg = net.plan_sets()
    sched = net.schedule()
    t0 = time.time()
    loss, _, _ = o.run_step(x, y, sched, st, seg)
    dt = time.time() - t0
    if not math.isfinite(loss):
        raise RuntimeError("non-finite CPU loss")
    return {"value": b / dt, "unit": "imgs/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"1 re-forward train step of {ARCH} at batch {b}, 3x{HW}x{HW}, fp32 CPU "
                      f"(oracle/train_oracle.py following the re-forward schedule; plan: {plan_kind})",
            "batch": b, "seconds": dt}


def run_reference(args):
    """The reference arm: the CPU re-forward train step (oracle/train_oracle.py,
    a port -- the reference has no training code) on every host core, at the
    GPU arm's config (batch per step = --batch), plan from the reference
    planner via the committed fixture; no product code on this path."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count()
    torch.set_num_threads(threads)
    for _ in range(max(args.warmup, 0)):
        cpu_baseline_sample(threads, batch=args.batch)
    vals = []
    t0 = time.time()
    for _ in range(args.steps):
        vals.append(cpu_baseline_sample(threads, batch=args.batch))
    total = time.time() - t0
    b = vals[0]["batch"]
    v = b * len(vals) / sum(x["seconds"] for x in vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "imgs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic random images/labels, random-init weights",
            "config": {"workload": f"{ARCH} re-forward training, batch {b}/step, 3x{HW}x{HW}, SGD (CPU)",
                       "model": ARCH, "global_batch": b, "seq_len": None, "parallelism": "cpu",
                       "same_config_as_gpu_arm": b == args.batch},
            "cpu_baseline": {"value": v, "unit": "imgs/s", "cores": threads, "kind": "port",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": "imgs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-store-all", action="store_true")
    ap.add_argument("--arch", default="resnet50",
                    help="resnet50 (headline) | resnet18/34/101/152 | densenet121/169/201/161 | vgg11-19 | alexnet")
    ap.add_argument("--hw", type=int, default=224)
    args = ap.parse_args()
    global ARCH, HW
    ARCH, HW = args.arch, args.hw
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from oracle.train_oracle import random_batch

    rank, world, local = dist_setup(args.gpus)
    stream = torch.cuda.Stream()
    peaks, peak_kind = _peaks()

    net, rep, plan_s = build_net(args.batch, "reforward", seed=1234)
    dev_bytes = net.report().device_bytes  # after setup, before the e2e staging buffers
    gpu_stored = net.plan_sets()[0] if ARCH.startswith(("densenet", "inception")) else None
    x, y = random_batch(net, seed=rank)
    net.load_batch(x.cuda(), y.cuda(), stream=stream)
    allreduce = None
    buckets = 0
    uid = None
    if world > 1:
        # gradient averaging runs inside the step: NCCL all-reduce per bucket on
        # a side stream as the backward finishes each range (torch.distributed
        # only carries the NCCL unique id)
        from paper_1808_00079_b200.executor import ReforwardNet
        obj = [ReforwardNet.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
        buckets = net.set_comm(world, rank, uid)

    with ClockSampler(local) as clk:
        ms = time_steps(net, args.steps, args.warmup, stream, world, allreduce)
    value = args.batch * world / (ms / 1000.0)
    launches = net.report().launches_per_step

    # end to end through the public API: every step copies its batch from
    # pinned host memory (double-buffered staging: batch k+1's copy runs on a
    # copy stream while step k computes) and reads its loss back
    xh, yh = x.pin_memory(), y.pin_memory()
    ms_e2e = time_e2e(net, args.steps, max(args.warmup, 3), stream, world, xh, yh)
    e2e_value = args.batch * world / (ms_e2e / 1000.0)

    # live roofline probe of the dominant kernel family (tcgen05 GEMMs)
    g_ms, g_flops, g_launch = net.gemm_profile(iters=5, stream=stream)
    achieved = g_flops / (g_ms / 1000.0) / 1e12
    peak = peaks.get("bf16_tflops", 1590.0)
    # per-launch roofline: many ResNet-50 convs at batch 32 are HBM-bound, so
    # the honest bound of the family is sum_i max(flops_i / tensor peak,
    # bytes_i / HBM peak) over the step's GEMM launches
    rows = net.gemm_profile_detail(iters=1, stream=stream)
    roof_ms = sum(max(r["flops"] / (peak * 1e12), r["bytes"] / (peaks.get("hbm_gbs", 6650.0) * 1e9))
                  for r in rows) * 1e3
    alg_bytes = sum(r["bytes"] for r in rows)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_gemm_summary.json")) as f:
            summ = json.load(f)
        # the capture is of one workload (tools/profile_step.py); other
        # networks / sizes report no traffic rather than a foreign number
        if summ.get("workload", "resnet50_b32_224") == f"{ARCH}_b{args.batch}_{HW}":
            traffic = summ.get("dram_bytes_per_step")
    except Exception:
        pass

    # store-all comparison (same kernels, plan = every tensor stored)
    overhead = None
    sa_value = None
    sa_device = None
    if not args.no_store_all:
        del net
        torch.cuda.synchronize()
        net_sa, rep_sa, _ = build_net(args.batch, "store_all", seed=1234)
        net_sa.load_batch(x.cuda(), y.cuda(), stream=stream)
        if world > 1:
            # a NCCL unique id bootstraps exactly one communicator: fresh one
            obj = [ReforwardNet.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            net_sa.set_comm(world, rank, obj[0])
        ms_sa = time_steps(net_sa, args.steps, args.warmup, stream, world)
        sa_value = args.batch * world / (ms_sa / 1000.0)
        overhead = ms / ms_sa
        sa_device = net_sa.report().device_bytes
        del net_sa

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(os.cpu_count(), gpu_stored, batch=args.batch)
            cpu.pop("seconds", None)
            cpu.pop("batch", None)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "imgs/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC if ARCH == "resnet50" else METRIC.replace("ResNet-50", ARCH), "value": value,
            "unit": "imgs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (N,3,224,224) random images + random labels; random-init weights",
            "config": {"workload": f"{ARCH} re-forward training, batch {args.batch}/GPU, 3x{HW}x{HW}, SGD",
                       "model": ARCH, "global_batch": args.batch * world, "seq_len": None,
                       "parallelism": f"dp{world}", "policy": "reforward (Algorithm 5 plan)",
                       "l2": "working set (activations + weights) far exceeds the 126 MB L2; no flush"},
            "memory": {"activation_peak_bytes": rep.tracked_peak, "planned_eq1_bytes": rep.planned_total,
                       "store_all_bytes": rep.store_all_total,
                       "cut_percent": 100.0 * (1 - rep.planned_total / rep.store_all_total),
                       "arena_bytes": rep.arena_bytes, "grad_arena_bytes": rep.grad_arena_bytes,
                       "workspace_bytes": rep.workspace_bytes, "reforward_ops": rep.reforward_ops,
                       "plan_seconds": plan_s,
                       # every cudaMalloc of the net (arena + guard band, gradient arena,
                       # workspace, parameters / gradients / momentum / bf16 copies, BN state,
                       # input and staging buffers), re-forward vs store-all
                       "device_bytes": dev_bytes, "device_peak_bytes": dev_bytes,
                       "store_all_device_bytes": sa_device,
                       "device_cut_percent": (100.0 * (1 - dev_bytes / sa_device)) if sa_device else None},
            "store_all": {"value": sa_value, "unit": "imgs/s"},
            "overhead_vs_store_all": overhead,
            "e2e": {"value": e2e_value, "unit": "imgs/s",
                    "h2d_bytes_per_step": int(x.numel() * 4 + y.numel() * 4), "d2h_bytes_per_step": 4},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "gemm_kernel (tcgen05 implicit-GEMM conv fprop/dgrad/wgrad + fc)",
                         "gemm_ms_per_step": g_ms, "gemm_share_of_step": g_ms / ms, "gemm_launches": g_launch,
                         "algorithmic_bytes_per_step": alg_bytes,
                         "traffic_note": "ncu dram read+write bytes of the step's GEMM launches (profiles/ncu_gemm_summary.json)",
                         "roofline_ms_per_step": roof_ms, "frac_of_roofline_time": roof_ms / g_ms,
                         "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({peak_kind}, burst)"},
            "cpu_baseline": cpu,
            "gpu_launches": launches * args.steps,
            "allreduce_buckets": buckets,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
