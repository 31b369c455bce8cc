"""Per-op parity of every sm_100a kernel in a real train step, teacher-forced.

End-to-end gradients of a random-init ResNet under bf16 storage differ from
an fp32 CPU step by tens of percent in small configs (the CPU oracle in its
bf16-emulating mode shows the same spread against its own fp32 mode, see
DESIGN.md "Parity"), which would hide kernel bugs.  So each op is checked in
isolation: the GPU's own stored inputs (and, backward, its own incoming
gradient) are fed to the CPU fp32 restatement of that op
(oracle/train_oracle.py), and the op's GPU output / input gradients / parameter
gradients must match it up to one bf16 rounding:

    forward outputs, activation gradients:  rel L2 err <= 1.5e-2
    parameter gradients (fp32 on the GPU):   rel L2 err <= 1.5e-2
"""
import numpy as np
import pytest
import torch

from oracle.train_oracle import OracleNet, random_batch, rel_err
from paper_1808_00079_b200.executor import ReforwardNet

pytestmark = pytest.mark.gpu
TOL = 1.5e-2

CASES = [("chain8", 4, 32, 10), ("resnet18", 4, 64, 16), ("resnet50", 2, 64, 16)]


def _nchw(a):
    a = torch.from_numpy(np.ascontiguousarray(a))
    return a.permute(0, 3, 1, 2).contiguous() if a.dim() == 4 else a


@pytest.mark.parametrize("arch,batch,hw,classes", CASES)
def test_every_op_forward_and_backward(arch, batch, hw, classes):
    net = ReforwardNet.named(arch, batch, hw, hw, classes)
    net.set_keep_grads(True)
    net.plan("store_all")
    net.setup(seed=0)
    o = OracleNet(net, emulate_bf16=True)
    o.init_weights(seed=7)
    o.push_weights_to(net)
    x, y = random_batch(net, seed=8)
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

    bad = []
    # ---- forward, op by op from the GPU's own inputs
    for op in o.ops[1:]:
        if op.kind == "loss":
            ref = float(o.op_forward(op, [vals[op.inputs[0]]], y))
            assert abs(net.read_loss() - ref) <= 1e-4 * abs(ref) + 1e-5
            continue
        ins = [vals[i] for i in op.inputs]
        if op.kind == "fc":
            ins = [ins[0].reshape(batch, -1)]
        ref = o.op_forward(op, ins, y).detach()
        e = rel_err(vals[op.out].reshape(ref.shape), ref)
        if e > TOL:
            bad.append(("fwd", op.name, e))

    # ---- backward: CPU VJP from the GPU's incoming gradient, summed over consumers
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
        e = rel_err(grads[t].reshape(ref.shape), ref)
        if e > TOL:
            bad.append(("dgrad", o.tensors[t].name, e))
    for p in net.params():
        e = rel_err(net.read_param(p.index, 1), pgrad_ref[p.name].numpy())
        if e > TOL:
            bad.append(("pgrad", p.name, e))
    assert not bad, bad[:20]
