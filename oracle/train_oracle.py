"""TEST INFRASTRUCTURE — CPU (fp32) restatement of one re-forward training step.

Never imported by the product.  Used as the numerical checker by tests/ and as
the CPU baseline leg of bench.py (``cpu_baseline`` / ``--impl reference``).

The reference repository stops at the plan (proj/include/reforward/acg.hpp
``solve_acg`` -> stored set V^R); the training step it is meant to drive is
described in the paper (§3 Overview: "during the first forward, we only store
tensors at selected vertices ... During backward, the tensors and gradients at
missing vertices are recovered by local forward operations") and modelled by
the reference simulator (simulate.hpp:38-94: stored set resident, one segment
re-forwarded at a time, segments visited in reverse order).  This module
executes exactly that on the CPU:

* the network is read from a ``ReforwardNet`` (ops, tensors, parameters in
  PyTorch layout) and computed in fp32 with plain torch CPU ops — conv2d,
  training-mode batch norm (biased variance, eps 1e-5), ReLU, max/avg pooling,
  linear, mean softmax cross-entropy;
* ``run_step`` follows the executor's exported schedule (forward / backward /
  release instructions): only planned tensors survive the first forward, and
  each segment is recomputed before the backward ops that need it; every op's
  backward is its local vector-Jacobian product (torch.autograd.grad on the
  single re-executed op), so gradients accumulate per tensor exactly as in the
  schedule;
* ``live_peak`` reports the activation high-water mark (tensor bytes at the
  executor's cost granularity) observed while doing so.

Layout note: tensors are NCHW here.  The executor flattens a hidden linear
layer's input in NHWC order and stores its weight accordingly; read_param /
write_param convert to the canonical NCHW-flatten layout used here.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import numpy as np
import torch
import torch.nn.functional as F

EPS = 1e-5


class OracleNet:
    def __init__(self, net, dtype=torch.float32, emulate_bf16: bool = False):
        """emulate_bf16: round every tensor the GPU stores in bf16 (activations,
        activation gradients, conv/fc weight copies) at the same points, so a
        correct GPU step must agree to accumulation-order noise."""
        self.net = net
        self.dtype = dtype
        self.emulate_bf16 = emulate_bf16
        self.tensors = net.tensors()
        self.ops = net.ops()
        self.params = {p.name: p for p in net.params()}
        self.weights: Dict[str, torch.Tensor] = {}
        self.attrs = {op.id: net.op_attrs(op.id) for op in self.ops}

    def init_weights(self, seed: int = 0, residual_gamma: float = 1.0) -> None:
        """Deterministic fp32 init (Kaiming convs, unit BN, small classifier).

        residual_gamma scales the BN gamma that feeds each residual add (the
        usual small/zero init of a block's last BN); deep random ResNets are
        otherwise so ill-conditioned that bf16 storage alone decorrelates
        their gradients from an fp32 step."""
        g = torch.Generator().manual_seed(seed)
        joins = {op.name for op in self.ops if op.kind == "bn_add_relu"}
        for p in self.params.values():
            if p.kind == 0:
                fan = p.shape[1] * p.shape[2] * p.shape[3]
                w = torch.randn(p.shape, generator=g) * (2.0 / fan) ** 0.5
            elif p.kind == 1:
                w = 1.0 + 0.1 * torch.randn(p.shape, generator=g)
                if p.name[: -len(".weight")] in joins:
                    w = w * residual_gamma
            elif p.kind in (2, 4):
                w = 0.1 * torch.randn(p.shape, generator=g)
            elif p.kind == 5:  # hidden linear layer (Kaiming over the fan-in)
                w = torch.randn(p.shape, generator=g) * (2.0 / p.shape[1]) ** 0.5
            else:
                w = torch.randn(p.shape, generator=g) * 0.05
            self.weights[p.name] = w.to(self.dtype)

    def push_weights_to(self, net) -> None:
        for p in net.params():
            net.write_param(p.index, self.weights[p.name].float().numpy())

    def load_weights_from(self, net=None):
        net = net or self.net
        for p in net.params():
            self.weights[p.name] = torch.from_numpy(net.read_param(p.index, 0)).to(self.dtype)

    def rb(self, t: torch.Tensor) -> torch.Tensor:
        """bf16 rounding (straight-through for autograd) when emulating."""
        if not self.emulate_bf16:
            return t
        return t + (t.detach().to(torch.bfloat16).to(t.dtype) - t.detach())

    # ------------------------------------------------------------ ops (fp32)
    def op_forward(self, op, ins: List[torch.Tensor], labels: torch.Tensor) -> torch.Tensor:
        out = self._op_forward(op, ins, labels)
        if op.kind in ("fc", "loss"):
            return out
        return self.rb(out)

    def _op_forward(self, op, ins: List[torch.Tensor], labels: torch.Tensor) -> torch.Tensor:
        k = op.kind
        a = self.attrs[op.id]
        if k == "conv":
            w = self.rb(self.weights[op.name + ".weight"])
            return F.conv2d(ins[0], w, stride=a["stride"], padding=(a["pad"], a["pad_w"]))
        if k in ("bn", "bn_add_relu"):
            y = ins[0]
            mean = y.mean(dim=(0, 2, 3), keepdim=True)
            var = ((y - mean) ** 2).mean(dim=(0, 2, 3), keepdim=True)
            g = self.weights[op.name + ".weight"].view(1, -1, 1, 1)
            b = self.weights[op.name + ".bias"].view(1, -1, 1, 1)
            out = (y - mean) / torch.sqrt(var + EPS) * g + b
            if k == "bn_add_relu":
                return torch.relu(out + ins[1])
            return torch.relu(out) if a["k"] == 1 else out
        if k == "relu":
            return torch.relu(ins[0])
        if k == "maxpool":
            return F.max_pool2d(ins[0], a["k"], a["stride"], a["pad"])
        if k == "avgpool":
            return ins[0].mean(dim=(2, 3), keepdim=True)
        if k == "avgpool2d":
            return F.avg_pool2d(ins[0], a["k"], a["stride"], a["pad"], count_include_pad=True)
        if k == "fc":
            x = ins[0].flatten(1)
            return F.linear(x, self.rb(self.weights[op.name + ".weight"]), self.weights[op.name + ".bias"])
        if k == "linear":  # hidden layer: NCHW flatten (the canonical weight layout), [N, out, 1, 1]
            x = ins[0].flatten(1)
            y = F.linear(x, self.rb(self.weights[op.name + ".weight"]), self.weights[op.name + ".bias"])
            return y.view(y.shape[0], -1, 1, 1)
        if k == "concat":
            return torch.cat(ins, dim=1)
        if k == "loss":
            return F.cross_entropy(ins[0], labels.long())
        raise ValueError(k)

    def _bn_only(self, op, y):
        mean = y.mean(dim=(0, 2, 3), keepdim=True)
        var = ((y - mean) ** 2).mean(dim=(0, 2, 3), keepdim=True)
        g = self.weights[op.name + ".weight"].view(1, -1, 1, 1)
        b = self.weights[op.name + ".bias"].view(1, -1, 1, 1)
        return (y - mean) / torch.sqrt(var + EPS) * g + b

    # ------------------------------------------------------------ store-all reference
    def reference_step(self, images: torch.Tensor, labels: torch.Tensor):
        """Plain autograd over the whole graph: loss, {param: grad}."""
        ws = {n: w.clone().requires_grad_(True) for n, w in self.weights.items()}
        saved = self.weights
        self.weights = ws
        vals: Dict[int, torch.Tensor] = {}
        for op in self.ops:
            if op.kind == "input":
                vals[op.out] = images.to(self.dtype)
                continue
            vals[op.out] = self.op_forward(op, [vals[i] for i in op.inputs], labels)
        loss = vals[self.ops[-1].out]
        loss.backward()
        grads = {n: w.grad.detach().clone() if w.grad is not None else torch.zeros_like(w) for n, w in ws.items()}
        self.weights = saved
        return loss.item(), grads

    def op_vjp(self, op, vals, dout, labels, src):
        """Local vector-Jacobian product of one op from the tensors the executor
        keeps for its backward.  Returns ([(input tensor, grad)], {param: grad})."""
        wnames = [n for n in (op.name + ".weight", op.name + ".bias") if n in self.weights]
        ws = [self.weights[n].clone().requires_grad_(True) for n in wnames]
        saved = {n: self.weights[n] for n in wnames}
        for n, w in zip(wnames, ws):
            self.weights[n] = w
        try:
            if op.kind == "bn_add_relu":
                y = vals[op.inputs[0]].detach().clone().requires_grad_(True)
                z = self._bn_only(op, y)
                g = dout * (vals[op.out] > 0).to(dout.dtype)
                gs = torch.autograd.grad(z, [y] + ws, grad_outputs=g)
                in_grads = [(op.inputs[0], gs[0]), (op.inputs[1], g)]
                wgr = gs[1:]
            elif op.kind == "bn" and self.attrs[op.id]["k"] == 1:
                # BN + ReLU: the ReLU mask from the op's own output (as for
                # the residual add above); recomputing it would let a value
                # sitting exactly at 0 flip with the last bit of the stats
                y = vals[op.inputs[0]].detach().clone().requires_grad_(True)
                z = self._bn_only(op, y)
                out = vals[op.out] if op.out in vals else self.rb(torch.relu(z.detach()))
                g = dout * (out > 0).to(dout.dtype)
                gs = torch.autograd.grad(z, [y] + ws, grad_outputs=g)
                in_grads = [(op.inputs[0], gs[0])]
                wgr = gs[1:]
            elif op.kind == "relu":  # mask from the output (the input may be released)
                in_grads = [(op.inputs[0], dout * (vals[op.out] > 0).to(dout.dtype))]
                wgr = []
            elif op.kind == "avgpool":  # shape only
                _, h, w, _c = self.tensors[op.inputs[0]].shape
                in_grads = [(op.inputs[0], (dout / (h * w)).expand(-1, -1, h, w).contiguous())]
                wgr = []
            elif op.kind == "avgpool2d":  # linear and shape only: the input itself is not kept
                n, h, w, c = self.tensors[op.inputs[0]].shape
                x = torch.zeros(n, c, h, w, dtype=dout.dtype, requires_grad=True)
                a = self.attrs[op.id]
                z = F.avg_pool2d(x, a["k"], a["stride"], a["pad"], count_include_pad=True)
                in_grads = [(op.inputs[0], torch.autograd.grad(z, x, grad_outputs=dout)[0])]
                wgr = []
            elif op.kind == "concat":
                ca = self.tensors[op.inputs[0]].shape[3]
                in_grads = [(op.inputs[0], dout[:, :ca].contiguous()), (op.inputs[1], dout[:, ca:].contiguous())]
                wgr = []
            elif op.kind == "fc" and self.emulate_bf16:
                # the GPU feeds bf16 dlogits to the dgrad / wgrad GEMMs, fp32 to the bias sum
                x = vals[op.inputs[0]].flatten(1)
                db16 = self.rb(dout)
                wb = self.rb(saved[op.name + ".weight"])
                dx = (db16 @ wb).view_as(vals[op.inputs[0]])
                in_grads = [(op.inputs[0], dx)]
                wgr = [db16.t() @ x, dout.sum(0)]
            else:
                ins = [vals[i].detach().clone().requires_grad_(i != src) for i in op.inputs]
                out = self.op_forward(op, ins, labels)
                targets = [x for x, i in zip(ins, op.inputs) if i != src] + ws
                gs = torch.autograd.grad(out, targets, grad_outputs=dout, allow_unused=True)
                in_grads = []
                gi = 0
                for x, i in zip(ins, op.inputs):
                    if i == src:
                        continue
                    in_grads.append((i, gs[gi] if gs[gi] is not None else torch.zeros_like(x)))
                    gi += 1
                wgr = gs[gi:]
        finally:
            for n in wnames:
                self.weights[n] = saved[n]
        return in_grads, {n: (g if g is not None else torch.zeros_like(saved[n])) for n, g in zip(wnames, wgr)}

    # ------------------------------------------------------------ schedule-following re-forward step
    def run_step(self, images: torch.Tensor, labels: torch.Tensor, schedule, stored: List[int],
                 seg_of: List[int]):
        """Execute the executor's schedule on the CPU; returns (loss, grads, live_peak)."""
        cost = {t.id: t.cost for t in self.tensors}
        src = self.ops[0].out
        sink = self.ops[-1].out
        vals: Dict[int, torch.Tensor] = {src: self.rb(images.to(self.dtype))}
        grads_t: Dict[int, torch.Tensor] = {}
        pgrads: Dict[str, torch.Tensor] = {}
        f32_tensors = {t.id for t in self.tensors if t.dtype == "f32"}
        live = 0
        peak = 0

        def materialize(t, v):
            nonlocal live, peak
            if t not in vals and t not in (src, sink):
                live += cost[t]
                peak = max(peak, live)
            vals[t] = v

        partial: Dict[int, Dict[int, torch.Tensor]] = {}
        for kind, o, seg, _re, phase in schedule:
            if kind == "release":
                for t in [t for t in list(vals) if seg_of[t] == seg]:
                    del vals[t]
                    live -= cost[t]
                continue
            op = self.ops[o]
            if kind == "forward":
                if phase == 0:
                    out = self.op_forward(op, [vals[i] for i in op.inputs], labels).detach()
                elif op.kind == "bn_add_relu" and phase == 1:  # out <- skip
                    out = vals[op.inputs[1]].clone()
                elif op.kind == "bn_add_relu":  # out <- relu(bn(y) + out)
                    out = self._bn_only(op, vals[op.inputs[0]]).detach()
                    out = self.rb(torch.relu(out + vals[op.out]))
                else:  # concat slice
                    partial.setdefault(op.out, {})[phase] = vals[op.inputs[phase - 1]]
                    if len(partial[op.out]) < 2:
                        if op.out not in vals:
                            materialize(op.out, torch.empty(0))
                        continue
                    out = torch.cat([partial[op.out][1], partial[op.out][2]], dim=1)
                materialize(op.out, out)
                continue
            # backward: local VJP of this op, re-executed on the tensors the
            # executor keeps for it (the residual add uses its output's mask
            # instead of the skip input)
            dout = None if op.out == sink else grads_t.pop(op.out)
            in_grads, wgr_named = self.op_vjp(op, vals, dout, labels, src)
            wnames = list(wgr_named)
            wgr = [wgr_named[n] for n in wnames]
            for i, g in in_grads:
                if i == src:
                    continue
                g = g.detach()
                acc = grads_t[i] + g if i in grads_t else g
                grads_t[i] = acc if i in f32_tensors else self.rb(acc)
            for n, g in zip(wnames, wgr):
                pgrads[n] = g if g is not None else torch.zeros_like(self.weights[n])
        loss = float(vals[sink]) if sink in vals else float("nan")
        return loss, pgrads, peak


def random_batch(net, seed: int = 0, classes: Optional[int] = None):
    ts = net.tensors()
    n, h, w, _ = ts[0].shape
    g = torch.Generator().manual_seed(seed)
    images = torch.randn(n, 3, h, w, generator=g)
    k = classes or ts[net.ops()[-1].inputs[0]].shape[3]
    labels = torch.randint(0, k, (n,), generator=g, dtype=torch.int32)
    return images.contiguous(), labels.contiguous()


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
