"""The GEMM engine's pipeline shape never changes results.

The K blocks per ring stage (RFK_GEMM_KPS: 1 = one 64-wide K block per
full/empty hand-off, 2 = two for BN <= 128 -- the default -- 3 = two for every
tile width) only regroups the TMA loads and the barrier hand-offs; the MMAs
accumulate the same K blocks in the same order, so every output must be
bit-identical.  The knob is read once per process, so each setting runs in a
child process over the same seeded operands: im2col convs with an odd number
of K blocks per tile (a half-empty last stage), the B-resident A-only ring,
multi-wave 2-D GEMMs at every tile width, and a split-K weight gradient.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_1808_00079_b200 import kernels as K
dev = "cuda"

def bf(*shape, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * 0.5).to(torch.bfloat16).to(dev)

outs = []
# 3x3 im2col fprop, 56x56x64 -> 64 (9 K blocks per tile, B resident, statistics)
x = bf(4, 56, 56, 64, seed=1); w = bf(64, 9 * 64, seed=2)
o = torch.zeros(4 * 56 * 56, 64, device=dev, dtype=torch.bfloat16); st = torch.zeros(160, 2, 64, device=dev)
g = K.ConvGeom(4, 56, 56, 64, 56, 56, 3, 3, 1, 1, 1, 1)
K.gemm(K.GemmArgs(M=4 * 56 * 56, N=64, K=576, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                  b=w.data_ptr(), b_ld=576, out=o.data_ptr(), ldc=64, stats=st.data_ptr(), splits=1))
outs += [o, st]
# 3x3 im2col fprop 28x28x192 -> 256 (27 K blocks, two n tiles, bn 128)
x2 = bf(4, 28, 28, 192, seed=3); w2 = bf(256, 9 * 192, seed=4)
o2 = torch.zeros(4 * 28 * 28, 256, device=dev, dtype=torch.bfloat16)
g2 = K.ConvGeom(4, 28, 28, 192, 28, 28, 3, 3, 1, 1, 1, 1)
K.gemm(K.GemmArgs(M=4 * 28 * 28, N=256, K=9 * 192, a_kind=K.IM2COL_K, a=x2.data_ptr(), a_geom=g2,
                  b_kind=K.KMAJOR, b=w2.data_ptr(), b_ld=9 * 192, out=o2.data_ptr(), ldc=256, splits=1, block_n=128))
outs.append(o2)
# multi-wave 2-D GEMMs, K = 320 (5 K blocks), every tile width, bf16 and fp32
a = bf(40000, 320, seed=5); b = bf(256, 320, seed=6)
for bn, f32 in ((64, False), (128, True), (256, False)):
    oc = torch.zeros(40000, 256, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    K.gemm(K.GemmArgs(M=40000, N=256, K=320, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=320, b_kind=K.KMAJOR,
                      b=b.data_ptr(), b_ld=320, out=oc.data_ptr(), ldc=256, out_f32=int(f32), splits=1, block_n=bn))
    outs.append(oc)
# weight gradient: dY (MN-major) x im2col(X) (MN-major), split-K fp32 partials
dy = bf(4 * 28 * 28, 128, seed=7); xw = bf(4, 28, 28, 64, seed=8)
gw = K.ConvGeom(4, 28, 28, 64, 28, 28, 3, 3, 1, 1, 1, 1)
ws = torch.zeros(6, 128, 576, device=dev)
K.gemm(K.GemmArgs(M=128, N=576, K=4 * 28 * 28, a_kind=K.MNMAJOR, a=dy.data_ptr(), a_ld=128, b_kind=K.IM2COL_MN,
                  b=xw.data_ptr(), b_geom=gw, out=ws.data_ptr(), ldc=576, out_f32=1, splits=6,
                  split_stride=128 * 576, block_n=128))
outs.append(ws)
torch.cuda.synchronize()
torch.save([t.cpu() for t in outs], sys.argv[2])
"""


def _run(tmp_path, kps):
    out = tmp_path / f"kps{kps}.pt"
    env = dict(os.environ)
    env.pop("RFK_GEMM_KPS", None)
    if kps:
        env["RFK_GEMM_KPS"] = str(kps)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(out)], env=env, check=True, timeout=300)
    return torch.load(out)


def test_k_blocks_per_stage_bit_identical(tmp_path):
    ref = _run(tmp_path, 1)
    for kps in (0, 3):
        got = _run(tmp_path, kps)
        assert len(got) == len(ref)
        for i, (r, g) in enumerate(zip(ref, got)):
            assert torch.equal(r.view(torch.int16) if r.dtype == torch.bfloat16 else r.view(torch.int32),
                               g.view(torch.int16) if g.dtype == torch.bfloat16 else g.view(torch.int32)), \
                f"output {i} differs with RFK_GEMM_KPS={kps}"
        assert any(t.abs().sum() > 0 for t in got)


@pytest.mark.parametrize("C,Co", [(64, 64), (32, 128), (64, 32)])
def test_band_kernel_bit_identical_to_im2col_with_one_channel_block(C, Co):
    """With one 64-channel block of A the shifted-band kernel sums the K blocks
    (filter taps) in the TMA im2col kernel's order, so the two produce the same
    bits (the executor relies on it: a conv may run either way in different
    plans, e.g. band in the first forward and im2col with a fused BN in the
    re-forward).  Forward (K-major weights) and data gradient (flipped taps)."""
    from paper_1808_00079_b200 import kernels as K
    torch.manual_seed(0)
    n, h = 8, 56
    x = (torch.randn(n, h, h, C, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(Co, 9 * 64, device="cuda") * 0.1).to(torch.bfloat16)
    w[:, :].view(Co, 9, 64)[:, :, C:] = 0
    wt = (torch.randn(C, 3, 3, Co, device="cuda") * 0.1).to(torch.bfloat16)  # dgrad: [cout=C of dy][tap][cin=Co]
    g = K.ConvGeom(n, h, h, C, h, h, 3, 3, 1, 1, 1, 1)
    outs = {}
    for band in (0, 1):
        o = torch.zeros(n * h * h, Co, device="cuda", dtype=torch.bfloat16)
        K.gemm(K.GemmArgs(M=n * h * h, N=Co, K=9 * 64, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                          b=w.data_ptr(), b_ld=9 * 64, out=o.data_ptr(), ldc=Co, splits=1, band=band))
        d = torch.zeros(n * h * h, Co, device="cuda", dtype=torch.bfloat16)
        ga = K.GemmArgs(M=n * h * h, N=Co, K=9 * 64, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=4,
                        b=wt.data_ptr(), out=d.data_ptr(), ldc=Co, splits=1, band=band)
        for k, v in {"b_extent": Co, "b_taps": 9, "b_cpad": Co, "b_rows": C}.items():
            setattr(ga, k, v)
        K.gemm(ga)
        torch.cuda.synchronize()
        outs[band] = (o, d)
    for a, b in zip(outs[0], outs[1]):
        assert a.abs().sum() > 0
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
