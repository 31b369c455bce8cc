"""GPU parity at the BASELINE.json configurations (the shapes the bench runs).

The benchmarked sizes reach code paths small shapes never do: persistent GEMMs
with hundreds to thousands of tiles, bf16 split-K finishes on the 14^2 / 7^2
layers, sub-pixel dgrad classes on parallel streams, the whole-batch stem
im2col cache, lazy weight-gradient joins, CUDA-graph replay.  Three checks:

1. Per-op teacher-forced parity against the CPU fp32 oracle (tests/_parity.py)
   at batch 32 / 224^2 (ResNet-50, VGG-16, AlexNet) and batch 2 / 600^2
   (DenseNet-121, Inception-v3): rel L2 <= 5e-3 (under one bf16 ulp) for every
   forward output, activation gradient and parameter gradient.
2. Re-forward vs store-all bit identity of the captured train step (two SGD
   steps through the CUDA graph, exactly as bench.py runs it) at every
   BASELINE config, including batch 64 at 600^2.
3. Whole-step parity with a stated tolerance: the GPU
   step's loss and gradients against the CPU step
   (a) that stores bf16 at the same points: for the whole gradient and for
       every parameter, ||g_gpu - g_cpu|| / ||g_cpu|| <= max(2e-2, 3 x floor),
       floor = the distance of that CPU step from the same step with fp64
       instead of fp32 accumulation (how far bf16 rounding flips alone move
       this configuration; the GPU's fp32 accumulation order is a second,
       independent draw of that noise);
   (b) in plain fp32 (no bf16 anywhere): the GPU step is no further from it
       than the bf16-storing CPU step is (<= 1.5x + 1e-3), i.e. the kernels
       add nothing beyond the storage precision;
   and the loss to 1e-3 relative.  No initialisation crutches (residual BN
   gammas at 1).
"""
import numpy as np
import pytest
import torch

from oracle.train_oracle import OracleNet, random_batch, rel_err
from _parity import Timer, gpu_step, plan, report, teacher_forced, worst

pytestmark = pytest.mark.gpu
TOL = 5e-3

TEACHER = [("resnet50", 32, 224, 1000), ("vgg16", 32, 224, 1000), ("alexnet", 32, 224, 1000),
           ("densenet121", 2, 600, 1000), ("inception_v3", 2, 600, 1000), ("inception_v3", 4, 299, 1000)]


@pytest.mark.parametrize("arch,batch,hw,classes", TEACHER)
def test_teacher_forced_every_op_at_baseline_shape(arch, batch, hw, classes):
    with Timer() as t:
        res = teacher_forced(arch, batch, hw, classes)
    report(f"baseline_teacher_{arch}_b{batch}_{hw}", {"worst": worst(res), "seconds": t.s, **res})
    assert res["loss"] <= 1e-5, res["loss"]
    bad = [(k, n, e) for k in ("fwd", "dgrad", "pgrad") for n, e in res[k].items() if e > TOL]
    assert not bad, sorted(bad, key=lambda b: -b[2])[:20]


BIT = [("alexnet", 32, 224), ("vgg16", 32, 224), ("resnet50", 32, 224), ("resnet101", 32, 224),
       ("densenet121", 64, 600), ("inception_v3", 64, 600)]


@pytest.mark.parametrize("arch,batch,hw", BIT)
def test_reforward_bit_identical_to_store_all_at_baseline_shape(arch, batch, hw):
    from paper_1808_00079_b200.executor import ReforwardNet
    x, y = random_batch(ReforwardNet.named(arch, batch, hw, hw, 1000), seed=3)
    out = {}
    for policy in ("reforward", "store_all"):
        net, rep, losses, grads, values = gpu_step(arch, batch, hw, 1000, policy, x=x, y=y, steps=2, lr=0.01,
                                                   wd=1e-4, use_graph=True)
        assert np.all(np.isfinite(losses)), losses
        out[policy] = (rep, losses, grads, values)
        if policy == "reforward":
            assert rep.tracked_peak == rep.planned_total == rep.arena_bytes
            assert net.arena_guard_intact()
        del net
        torch.cuda.synchronize()
    (rr, lr_, gr, vr), (rs, ls, gs, vs) = out["reforward"], out["store_all"]
    report(f"bitident_{arch}_b{batch}_{hw}", {"losses": lr_, "planned": rr.planned_total,
                                              "store_all": rs.planned_total})
    assert rr.planned_total < rs.planned_total
    assert lr_ == ls
    for n in gr:
        assert np.array_equal(gr[n], gs[n]), n
        assert np.array_equal(vr[n], vs[n]), n


# (arch, batch, hw, classes, residual BN gamma init): 1.0 = plain init; 0.0 =
# the zero-init of each residual block's last BN gamma of the standard
# large-batch ResNet recipe (Goyal et al. 2017), under which a deep ResNet
# starts well conditioned -- its floor is ~1 % instead of ~100 %, so the bar
# is tight there
WHOLE = [("resnet50", 32, 224, 1000, 0.0), ("resnet50", 32, 224, 1000, 1.0), ("alexnet", 32, 224, 1000, 1.0),
         ("vgg16", 8, 224, 1000, 1.0), ("densenet121", 4, 224, 1000, 1.0), ("inception_v3", 4, 299, 1000, 1.0)]


def _cat(g, names):
    return np.concatenate([np.asarray(g[n], dtype=np.float64).ravel() for n in names])


@pytest.mark.parametrize("arch,batch,hw,classes,gamma", WHOLE)
def test_whole_step_within_stated_tolerance(arch, batch, hw, classes, gamma):
    from paper_1808_00079_b200.executor import ReforwardNet
    probe = ReforwardNet.named(arch, batch, hw, hw, classes)
    plan(probe, arch, batch, hw)
    stored, seg = probe.plan_sets()
    sched = probe.schedule()
    x, y = random_batch(probe, seed=5)
    o16 = OracleNet(probe, emulate_bf16=True)
    o16.init_weights(seed=11, residual_gamma=gamma)
    with Timer() as t:
        l16, g16, peak = o16.run_step(x, y, sched, stored, seg)
        o64 = OracleNet(probe, dtype=torch.float64, emulate_bf16=True)
        o64.weights = {k: v.double() for k, v in o16.weights.items()}
        l64, g64, _ = o64.run_step(x, y, sched, stored, seg)
        o32 = OracleNet(probe, emulate_bf16=False)
        o32.weights = dict(o16.weights)
        l32, g32, _ = o32.run_step(x, y, sched, stored, seg)
    net, rep, losses, g, _ = gpu_step(arch, batch, hw, classes, "reforward", o16.weights, x, y)
    assert rep.tracked_peak == rep.planned_total == peak
    names = sorted(g16)
    a, b16, b64, b32 = _cat(g, names), _cat(g16, names), _cat(g64, names), _cat(g32, names)
    err16 = rel_err(a, b16)
    floor = rel_err(b16, b64)
    err32 = rel_err(a, b32)
    bf16_cost = rel_err(b16, b32)
    per_param = {n: rel_err(g[n], g16[n].numpy()) for n in names}
    floor_p = {n: rel_err(g16[n].numpy(), g64[n].numpy()) for n in names}
    ratio = {n: per_param[n] / max(2e-2, 3 * floor_p[n]) for n in names}
    worst_p = max(ratio, key=ratio.get)
    loss_floor = abs(l16 - l64)
    rep_ = {"residual_gamma": gamma, "loss_gpu": losses[0], "loss_cpu_bf16": l16, "loss_cpu_fp64": l64,
            "loss_cpu_fp32": l32, "grad_err_vs_cpu_bf16": err16, "noise_floor_fp64": floor,
            "grad_err_vs_cpu_fp32": err32, "cpu_bf16_vs_fp32": bf16_cost,
            "worst_param": [worst_p, per_param[worst_p], floor_p[worst_p]], "cpu_seconds": t.s}
    report(f"wholestep_{arch}_b{batch}_{hw}_g{gamma:g}", rep_)
    assert abs(losses[0] - l16) <= max(1e-3 * abs(l16), 3 * loss_floor), rep_
    assert abs(losses[0] - l32) <= 1.5 * abs(l16 - l32) + max(1e-3 * abs(l32), 3 * loss_floor), rep_
    assert err16 <= max(2e-2, 3 * floor), rep_
    assert ratio[worst_p] <= 1.0, rep_
    assert err32 <= 1.5 * bf16_cost + 1e-3, rep_


def test_multi_step_loss_trajectory_resnet50():
    """Three momentum-SGD steps through the captured graph against the CPU
    step + the same SGD update on the host (fp32 masters, bf16 copies), with
    the trajectory's own floor (the same CPU run with fp64 accumulation)."""
    from paper_1808_00079_b200.executor import ReforwardNet
    arch, batch, hw, classes = "resnet50", 8, 224, 1000
    probe = ReforwardNet.named(arch, batch, hw, hw, classes)
    plan(probe, arch, batch, hw)
    stored, seg = probe.plan_sets()
    sched = probe.schedule()
    x, y = random_batch(probe, seed=9)
    o = OracleNet(probe, emulate_bf16=True)
    o.init_weights(seed=12, residual_gamma=0.0)
    w0 = {k: v.clone() for k, v in o.weights.items()}
    lr, mom, wd, steps = 0.05, 0.9, 1e-4, 3

    def cpu_run(dtype):
        oc = OracleNet(probe, dtype=dtype, emulate_bf16=True)
        oc.weights = {k: v.to(dtype) for k, v in w0.items()}
        buf = {k: torch.zeros_like(v) for k, v in oc.weights.items()}
        losses = []
        for _ in range(steps):
            loss, g, _ = oc.run_step(x, y, sched, stored, seg)
            losses.append(loss)
            for k in oc.weights:
                d = g[k] + wd * oc.weights[k]
                buf[k] = mom * buf[k] + d
                oc.weights[k] = oc.weights[k] - lr * buf[k]
        return losses, {k: v.double().numpy() for k, v in oc.weights.items()}

    cpu_losses, cpu_w = cpu_run(torch.float32)
    cpu64_losses, cpu64_w = cpu_run(torch.float64)
    _, _, gpu_losses, _, vals = gpu_step(arch, batch, hw, classes, "reforward", w0, x, y, steps=steps, lr=lr,
                                         momentum=mom, wd=wd, use_graph=True)
    names = sorted(vals)
    # distance travelled from w0, GPU vs CPU, relative to the CPU's own floor
    d_gpu = _cat(vals, names) - _cat({k: v.numpy() for k, v in w0.items()}, names)
    d_cpu = _cat(cpu_w, names) - _cat({k: v.numpy() for k, v in w0.items()}, names)
    d_64 = _cat(cpu64_w, names) - _cat({k: v.numpy() for k, v in w0.items()}, names)
    werr, wfloor = rel_err(d_gpu, d_cpu), rel_err(d_cpu, d_64)
    report("trajectory_resnet50_b8_224", {"gpu": gpu_losses, "cpu": cpu_losses, "cpu_fp64": cpu64_losses,
                                          "update_err": werr, "update_floor": wfloor})
    for a, b, c in zip(gpu_losses, cpu_losses, cpu64_losses):
        assert abs(a - b) <= max(2e-3 * abs(b), 3 * abs(b - c)), (gpu_losses, cpu_losses, cpu64_losses)
    assert gpu_losses[-1] < gpu_losses[0]
    assert werr <= max(2e-2, 3 * wfloor), (werr, wfloor)


@pytest.mark.parametrize("arch,batch,hw", [("resnet50", 32, 224), ("inception_v3", 4, 299), ("densenet121", 8, 224)])
def test_bn_batch_statistics_accuracy_at_baseline_shape(arch, batch, hw):
    """BN batch statistics are one-pass (sum and sum of squares of the stored
    bf16 values, fp32 per-CTA partial rows from the conv epilogue, fixed-order
    finalize).  Cancellation would show where |mean| >> sigma; measured at
    the benched shapes against fp64 statistics of the GPU's own conv outputs:
    mean within 1e-5 sigma, variance within 5e-5 relative, every channel."""
    from paper_1808_00079_b200.executor import ReforwardNet
    net = ReforwardNet.named(arch, batch, hw, hw, 1000)
    net.set_keep_grads(True)
    net.plan("store_all")
    net.setup(seed=0)
    x, y = random_batch(net, seed=8)
    net.load_batch(x, y)
    net.forward_backward()
    torch.cuda.synchronize()
    worst = {"mean_sigma": 0.0, "var_rel": 0.0, "max_abs_mean_over_sigma": 0.0}
    for o in net.ops():
        if o.kind not in ("bn", "bn_add_relu"):
            continue
        m, v = net.read_bn_running(o.id)  # one momentum-0.1 update from (0, 1)
        t = net.read_tensor(o.inputs[0]).astype(np.float64)
        t = t.reshape(-1, t.shape[-1])
        n = t.shape[0]
        tm, tv = t.mean(0), t.var(0) * n / (n - 1)
        ok = tv > 1e-12
        bm, bv = m.astype(np.float64) / 0.1, (v.astype(np.float64) - 0.9) / 0.1
        worst["mean_sigma"] = max(worst["mean_sigma"], float(np.max(np.abs(bm - tm)[ok] / np.sqrt(tv[ok]))))
        # the running variance stores 0.9 + 0.1 var in fp32: its rounding
        # (~6e-8 absolute) is part of what this reads back
        worst["var_rel"] = max(worst["var_rel"], float(np.max((np.abs(bv - tv)[ok] - 1e-6) / tv[ok])))
        worst["max_abs_mean_over_sigma"] = max(worst["max_abs_mean_over_sigma"],
                                               float(np.max(np.abs(tm[ok]) / np.sqrt(tv[ok]))))
    report(f"bnstats_{arch}_b{batch}_{hw}", worst)
    assert worst["mean_sigma"] <= 1e-5, worst
    assert worst["var_rel"] <= 5e-5, worst
