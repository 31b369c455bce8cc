"""Explicit im2col (the few-channel stem path, rfx_im2col) vs torch unfold: bit-exact."""
import pytest
import torch
import torch.nn.functional as F

from paper_1808_00079_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _ref(x, C, R, S, stride, pad, kpad):
    N, H, W, Cs = x.shape
    u = F.unfold(x[..., :C].permute(0, 3, 1, 2).float(), (R, S), padding=pad, stride=stride)
    L = u.shape[-1]
    u = u.view(N, C, R, S, L).permute(0, 4, 2, 3, 1).reshape(N * L, R * S * C)
    o = torch.zeros(N * L, kpad, device=x.device)
    o[:, :R * S * C] = u
    return o.to(torch.bfloat16)


@pytest.mark.parametrize("N,H,W,C,Cs,R,stride,pad,kpad", [
    (2, 224, 224, 3, 8, 7, 2, 3, 192),   # ResNet / DenseNet stem
    (3, 299, 299, 3, 8, 3, 2, 0, 64),    # Inception-v3 stem
    (2, 37, 29, 3, 8, 7, 2, 3, 192),     # ragged: P not a multiple of the run length, W != H
    (1, 20, 20, 5, 8, 3, 1, 1, 64),      # stride 1
    (2, 16, 16, 12, 16, 3, 1, 1, 128),   # two 16-byte vectors per pixel
])
def test_im2col_matches_unfold(N, H, W, C, Cs, R, stride, pad, kpad):
    torch.manual_seed(0)
    x = torch.randn(N, H, W, Cs, device="cuda").to(torch.bfloat16)
    out = K.im2col(x, C, R, R, stride, pad, kpad)
    torch.cuda.synchronize()
    assert torch.equal(out, _ref(x, C, R, R, stride, pad, kpad))
