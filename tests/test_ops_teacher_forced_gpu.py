"""Per-op parity of every sm_100a kernel in a real train step, teacher-forced.

Each op is checked in isolation (tests/_parity.py:teacher_forced): the GPU's
own stored inputs (and, backward, its own incoming gradient) are fed to the CPU
fp32 restatement of that op (oracle/train_oracle.py), rounded to bf16 where the
GPU stores bf16.  A correct kernel then differs only by fp32 accumulation order
(an occasional one-ulp bf16 rounding flip), so the bar is well under one bf16
ulp (2^-8 = 3.9e-3 relative) in relative L2:

    forward outputs, activation gradients, parameter gradients: rel L2 <= 5e-3

Small configurations here; the BASELINE.json shapes (batch 32 at 224^2, batch 2
at 600^2) run the same check in tests/test_baseline_shapes_gpu.py.
"""
import pytest

from _parity import report, teacher_forced, worst

pytestmark = pytest.mark.gpu
TOL = 5e-3

CASES = [("chain8", 4, 32, 10), ("resnet18", 4, 64, 16), ("resnet50", 2, 64, 16), ("densenet_tiny", 4, 32, 10),
         ("inception_v3", 2, 139, 10), ("vgg11", 4, 32, 10), ("alexnet", 4, 64, 10)]


@pytest.mark.parametrize("arch,batch,hw,classes", CASES)
def test_every_op_forward_and_backward(arch, batch, hw, classes):
    res = teacher_forced(arch, batch, hw, classes)
    report(f"teacher_{arch}_b{batch}_{hw}", {"worst": worst(res), **res})
    assert res["loss"] <= 1e-5, res["loss"]
    bad = [(k, n, e) for k in ("fwd", "dgrad", "pgrad") for n, e in res[k].items() if e > TOL]
    assert not bad, sorted(bad, key=lambda b: -b[2])[:20]
