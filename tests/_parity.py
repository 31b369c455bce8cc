"""Shared GPU-vs-oracle parity helpers (test infrastructure).

teacher_forced(): per-op parity of every kernel of one real train step.  The
GPU's own stored inputs (and, backward, its own incoming gradient) are fed to
the CPU fp32 restatement of that op (oracle/train_oracle.py), so each op is
judged in isolation.  The oracle output is rounded to bf16 where the GPU
stores bf16, so a correct kernel differs only by accumulation order (an
occasional one-ulp rounding flip) -- rel L2 well under one bf16 ulp (2^-8).

report(): parity numbers are also written to $RF_PARITY_OUT/<name>.json when
that variable is set (the GPU runs set it to gpurun_out/parity).
"""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch

from oracle.train_oracle import OracleNet, random_batch, rel_err
from paper_1808_00079_b200.executor import ReforwardNet


def _nchw(a):
    a = torch.from_numpy(np.ascontiguousarray(a))
    return a.permute(0, 3, 1, 2).contiguous() if a.dim() == 4 else a


def report(name: str, data: dict) -> None:
    out = os.environ.get("RF_PARITY_OUT")
    if not out:
        return
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, name + ".json"), "w") as f:
        json.dump(data, f, indent=1, sort_keys=True, default=float)


def teacher_forced(arch: str, batch: int, hw: int, classes: int, seed: int = 7):
    """Returns {'fwd': {op: err}, 'dgrad': {tensor: err}, 'pgrad': {param: err}}."""
    net = ReforwardNet.named(arch, batch, hw, hw, classes)
    net.set_keep_grads(True)
    net.plan("store_all")
    net.setup(seed=0)
    o = OracleNet(net, emulate_bf16=True)
    o.init_weights(seed=seed)
    o.push_weights_to(net)
    x, y = random_batch(net, seed=seed + 1)
    net.load_batch(x, y)
    net.forward_backward()
    torch.cuda.synchronize()

    src = o.ops[0].out
    sink = o.ops[-1].out
    vals = {t.id: _nchw(net.read_tensor(t.id)) for t in o.tensors if t.id not in (sink,)}
    vals[src] = o.rb(x)
    grads = {t.id: _nchw(net.read_grad_tensor(t.id)) for t in o.tensors if t.id not in (src, sink)}
    logits_t = o.ops[-1].inputs[0]
    vals[logits_t] = vals[logits_t].reshape(batch, classes)
    grads[logits_t] = grads[logits_t].reshape(batch, classes)
    res = {"fwd": {}, "dgrad": {}, "pgrad": {}, "loss": None}
    for op in o.ops[1:]:
        if op.kind == "loss":
            ref = float(o.op_forward(op, [vals[op.inputs[0]]], y))
            res["loss"] = abs(net.read_loss() - ref) / abs(ref)
            continue
        ins = [vals[i] for i in op.inputs]
        if op.kind == "fc":
            ins = [ins[0].reshape(batch, -1)]
        ref = o.op_forward(op, ins, y).detach()
        res["fwd"][op.name] = rel_err(vals[op.out].reshape(ref.shape), ref)
    contrib = {}
    pgrad_ref = {}
    for op in reversed(o.ops[1:]):
        dout = None if op.out == sink else grads[op.out]
        if op.kind == "fc":
            vals_fc = dict(vals)
            vals_fc[op.inputs[0]] = vals[op.inputs[0]].reshape(batch, -1)
            ig, pg = o.op_vjp(op, vals_fc, dout, y, src)
            ig = [(i, g.reshape(vals[i].shape)) for i, g in ig]
        else:
            ig, pg = o.op_vjp(op, vals, dout, y, src)
        for i, g in ig:
            if i != src:
                contrib[i] = contrib[i] + g.detach() if i in contrib else g.detach()
        pgrad_ref.update(pg)
    for t, ref in contrib.items():
        res["dgrad"][o.tensors[t].name] = rel_err(grads[t].reshape(ref.shape), ref)
    for p in net.params():
        res["pgrad"][p.name] = rel_err(net.read_param(p.index, 1), pgrad_ref[p.name].numpy())
    return res


def worst(res: dict) -> dict:
    out = {}
    for k in ("fwd", "dgrad", "pgrad"):
        if res[k]:
            name = max(res[k], key=res[k].get)
            out[k] = (name, res[k][name])
    return out


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def plan(net, arch, batch, hw, policy="reforward"):
    """plan(policy); the exact re-forward plan is memoised in plans/ (keyed by
    the graph hash): Inception-v3's takes minutes."""
    if policy != "reforward":
        return net.plan(policy)
    return net.plan_cached(policy, os.path.join(ROOT, "plans", f"{arch}_b{batch}_{hw}_{policy}.json"))


def gpu_step(arch, batch, hw, classes, policy, weights=None, x=None, y=None, steps=0, lr=0.0, momentum=0.9,
             wd=0.0, use_graph=False):
    """One forward+backward (steps=0) or `steps` SGD steps; returns net, report,
    [losses], {param: grad of the last step}, {param: value after}."""
    net = ReforwardNet.named(arch, batch, hw, hw, classes)
    rep = plan(net, arch, batch, hw, policy)
    net.setup(seed=0)
    if weights is not None:
        for p in net.params():
            net.write_param(p.index, weights[p.name].float().numpy())
    net.load_batch(x, y)
    losses = []
    if steps == 0:
        net.forward_backward()
        torch.cuda.synchronize()
        losses.append(net.read_loss())
    else:
        for _ in range(steps):
            net.step(lr=lr, momentum=momentum, weight_decay=wd, use_graph=use_graph)
            losses.append(net.read_loss())
    grads = {p.name: net.read_param(p.index, 1) for p in net.params()}
    values = {p.name: net.read_param(p.index, 0) for p in net.params()}
    return net, rep, losses, grads, values


class Timer:
    def __enter__(self):
        self.t = time.time()
        return self

    def __exit__(self, *a):
        self.s = time.time() - self.t
