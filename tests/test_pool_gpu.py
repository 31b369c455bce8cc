"""Max-pool backward (rfx_maxpool_bwd): the fused tiled kernel is bit-identical
to the two-pass argmax + gather form and matches torch's max_pool2d gradient."""
import pytest
import torch
import torch.nn.functional as F

from paper_1808_00079_b200 import kernels as K

pytestmark = pytest.mark.gpu

CASES = [(2, 112, 112, 64, 3, 2, 1),   # ResNet / DenseNet stem pool
         (2, 55, 55, 64, 3, 2, 0),     # AlexNet
         (2, 32, 32, 128, 2, 2, 0),    # VGG
         (1, 147, 147, 64, 3, 2, 0),   # Inception-v3
         (3, 21, 17, 520, 3, 2, 1)]    # ragged tiles, wide channels (smaller window tile)


@pytest.mark.parametrize("N,H,W,C,k,s,pad", CASES)
@pytest.mark.parametrize("acc", [False, True])
def test_maxpool_bwd_fused_matches_two_pass_and_torch(monkeypatch, N, H, W, C, k, s, pad, acc):
    torch.manual_seed(1)
    x = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
    P, Q = (H + 2 * pad - k) // s + 1, (W + 2 * pad - k) // s + 1
    dy = torch.randn(N, P, Q, C, device="cuda").to(torch.bfloat16)
    base = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16) if acc else torch.zeros(N, H, W, C, device="cuda",
                                                                                                dtype=torch.bfloat16)
    fused = K.maxpool_bwd(x, dy, k, s, pad, dx=base.clone(), accumulate=acc)
    monkeypatch.setenv("RFK_POOL_TWO_PASS", "1")
    two = K.maxpool_bwd(x, dy, k, s, pad, dx=base.clone(), accumulate=acc)
    torch.cuda.synchronize()
    assert torch.equal(fused, two)
    xf = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    y = F.max_pool2d(xf, k, s, pad)
    y.backward(dy.float().permute(0, 3, 1, 2))
    ref = xf.grad.permute(0, 2, 3, 1) + (base.float() if acc else 0)
    assert torch.equal(fused, ref.to(torch.bfloat16)) or (fused.float() - ref).abs().max().item() <= 1e-2
