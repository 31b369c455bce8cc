"""tcgen05 GEMM engine vs a plain PyTorch fp32 reference of the same contraction.

Operands are bf16 (exactly representable in fp32), so the reference is the
fp32 product of the same values (TF32 disabled in torch; convolution references
in fp64 -- cuDNN's fp32 conv may pick FFT / Winograd algorithms whose error
exceeds a bf16 ulp).  Tolerances:

* fp32 outputs:  max |out - ref| <= 1e-4 * max |ref|  (accumulation order only)
* bf16 outputs:  |out - ref| <= 2^-7 |ref| + 1e-4 max |ref| elementwise, i.e. at
  most one bf16 ulp (round-to-nearest plus an order-dependent flip); when the
  output is accumulated in bf16 (out = prev + bf16(D), two roundings) the ulps
  are of the operands: <= 2^-7 (|prev| + |D|) + 2^-7 |ref|.
"""
import pytest
import torch
import torch.nn.functional as F

from paper_1808_00079_b200 import kernels as K

pytestmark = pytest.mark.gpu
dev = "cuda"
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False


@pytest.fixture(params=[0, 1, -1], ids=["auto", "pair", "single"], autouse=True)
def cta_pair_mode(request, monkeypatch):
    """Every case runs with the automatic choice, with CTA pairs (2-CTA
    clusters, cta_group::2 M = 256 tiles) wherever the shape allows them --
    including odd M-tile counts, whose second CTA drains an all-out-of-bounds
    tile -- and with single CTAs only."""
    orig = K.gemm

    def gemm(args, *a, **kw):
        if args.pair == 0:
            args.pair = request.param
        return orig(args, *a, **kw)

    monkeypatch.setattr(K, "gemm", gemm)


def _bf(*shape, scale=1.0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).to(torch.bfloat16).to(dev)


def _check(out, ref, rtol=None, ulps=1, mag=None):
    f32 = out.dtype == torch.float32
    out = out.float()
    ref = ref.float()
    scale = ref.abs().max().item() + 1e-6
    if f32 or rtol is not None:
        err = (out - ref).abs().max().item()
        tol = (rtol if rtol is not None else 1e-4) * scale
        assert err <= tol, f"max err {err} vs tol {tol} (scale {scale})"
        return
    bound = ulps * 2.0 ** -7 * (ref.abs() if mag is None else mag.float()) + 1e-4 * scale
    bad = ((out - ref).abs() > bound)
    assert not bad.any(), f"{int(bad.sum())} elements beyond {ulps} bf16 ulp, worst {(out - ref).abs().max().item()}"


@pytest.mark.parametrize("M,N,Kd,bn,f32", [(256, 128, 128, 128, False), (200, 96, 96, 0, False),
                                           (128, 256, 320, 256, False), (384, 64, 64, 64, False),
                                           (130, 1000, 2048, 0, True), (33, 48, 40, 64, True)])
def test_gemm_kmajor(M, N, Kd, bn, f32):
    a = _bf(M, Kd, seed=1)
    b = _bf(N, Kd, seed=2)
    ref = a.float() @ b.float().t()
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.randn(N, device=dev) if f32 else None
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                      b_ld=Kd, out=out.data_ptr(), ldc=N, out_f32=int(f32), splits=1, block_n=bn,
                      bias=None if bias is None else bias.data_ptr())
    K.gemm(args)
    torch.cuda.synchronize()
    if bias is not None:
        ref = ref + bias
    _check(out, ref)


@pytest.mark.parametrize("M,N,Kd,a_mn,b_mn", [(128, 128, 128, True, True), (1000, 2048, 32, True, True),
                                              (64, 2048, 1000, False, True), (256, 192, 192, True, False)])
def test_gemm_mn_major(M, N, Kd, a_mn, b_mn):
    a = _bf(M, Kd, seed=3)
    b = _bf(N, Kd, seed=4)
    ref = a.float() @ b.float().t()
    at = a.t().contiguous() if a_mn else a
    bt = b.t().contiguous() if b_mn else b
    out = torch.zeros(M, N, device=dev, dtype=torch.float32)
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.MNMAJOR if a_mn else K.KMAJOR, a=at.data_ptr(),
                      a_ld=M if a_mn else Kd, b_kind=K.MNMAJOR if b_mn else K.KMAJOR, b=bt.data_ptr(),
                      b_ld=N if b_mn else Kd, out=out.data_ptr(), ldc=N, out_f32=1, splits=1)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


def _pad_w(w_nchw, cpad):
    # [Cout, Cin, R, S] -> [Cout, R, S, Cpad] bf16
    co, ci, r, s = w_nchw.shape
    out = torch.zeros(co, r, s, cpad, device=dev, dtype=torch.bfloat16)
    out[..., :ci] = w_nchw.permute(0, 2, 3, 1).to(torch.bfloat16)
    return out.contiguous()


CONV_CASES = [(2, 8, 8, 64, 128, 3, 1, 1), (2, 9, 9, 64, 64, 3, 1, 2), (2, 16, 16, 128, 256, 1, 0, 1),
              (2, 15, 15, 64, 64, 7, 3, 2), (1, 7, 7, 512, 512, 3, 1, 1), (2, 10, 10, 96, 64, 3, 1, 1),
              (4, 14, 14, 256, 256, 3, 1, 1), (2, 16, 16, 64, 128, 1, 0, 2)]


@pytest.mark.parametrize("N,H,W,Ci,Co,R,pad,st", CONV_CASES)
def test_conv_fprop_im2col(N, H, W, Ci, Co, R, pad, st):
    x = _bf(N, Ci, H, W, seed=5)
    w = _bf(Co, Ci, R, R, scale=0.1, seed=6)
    ref = F.conv2d(x.double(), w.double(), stride=st, padding=pad).permute(0, 2, 3, 1).contiguous().float()
    g = K.conv_geom(N, H, W, Ci, R, R, pad, st)
    cpad = (Ci + 63) // 64 * 64
    xn = x.permute(0, 2, 3, 1).contiguous()
    wp = _pad_w(w, cpad)
    M = N * g.P * g.Q
    out = torch.zeros(N, g.P, g.Q, Co, device=dev, dtype=torch.bfloat16)
    mt = (M + 127) // 128
    stats = torch.zeros(160, 2, Co, device=dev)  # one row per persistent CTA (<= SM count)
    del mt
    args = K.GemmArgs(M=M, N=Co, K=R * R * cpad, a_kind=K.IM2COL_K, a=xn.data_ptr(), a_geom=g,
                      b_kind=K.KMAJOR, b=wp.data_ptr(), b_ld=R * R * cpad, out=out.data_ptr(), ldc=Co,
                      stats=stats.data_ptr(), splits=1)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)
    r2 = out.float().reshape(M, Co)  # statistics are of the stored bf16 values
    _check(stats[:, 0].sum(0), r2.sum(0), rtol=1e-5)
    _check(stats[:, 1].sum(0), (r2 * r2).sum(0), rtol=1e-5)


@pytest.mark.parametrize("N,H,W,Ci,Co,R,pad,st", CONV_CASES)
@pytest.mark.parametrize("splits", [1, 3])
def test_conv_wgrad_im2col(N, H, W, Ci, Co, R, pad, st, splits):
    x = _bf(N, Ci, H, W, seed=7)
    g = K.conv_geom(N, H, W, Ci, R, R, pad, st)
    dy = _bf(N, Co, g.P, g.Q, seed=8)
    ref = torch.nn.grad.conv2d_weight(x.double(), (Co, Ci, R, R), dy.double(), stride=st, padding=pad).float()
    cpad = (Ci + 63) // 64 * 64
    xn = x.permute(0, 2, 3, 1).contiguous()
    dyn = dy.permute(0, 2, 3, 1).contiguous()
    M = N * g.P * g.Q
    ktot = R * R * cpad
    out = torch.zeros(splits, Co, ktot, device=dev)
    args = K.GemmArgs(M=Co, N=ktot, K=M, a_kind=K.MNMAJOR, a=dyn.data_ptr(), a_ld=Co, b_kind=K.IM2COL_MN,
                      b=xn.data_ptr(), b_geom=g, out=out.data_ptr(), ldc=ktot, out_f32=1, splits=splits,
                      split_stride=Co * ktot)
    K.gemm(args)
    torch.cuda.synchronize()
    got = out.sum(0).reshape(Co, R, R, cpad)[..., :Ci].permute(0, 3, 1, 2)
    _check(got, ref)


def test_scatter_remap():
    # 1x1 stride-2 dgrad: rows of dY (N,P,Q) land at (n, 2p, 2q) of dX
    N, H, W, Co, Ci = 2, 8, 8, 64, 128
    P, Q = 4, 4
    dy = _bf(N * P * Q, Co, seed=9)
    wt = _bf(Ci, Co, seed=10)  # [Cin, Cout], K-major over Cout
    ref = torch.zeros(N, H, W, Ci, device=dev)
    ref[:, ::2, ::2, :] = (dy.float() @ wt.float().t()).reshape(N, P, Q, Ci)
    out = torch.zeros(N, H, W, Ci, device=dev, dtype=torch.bfloat16)
    args = K.GemmArgs(M=N * P * Q, N=Ci, K=Co, a_kind=K.KMAJOR, a=dy.data_ptr(), a_ld=Co, b_kind=K.KMAJOR,
                      b=wt.data_ptr(), b_ld=Co, out=out.data_ptr(), ldc=Ci, splits=1, remap=1, rP=P, rQ=Q, rH=H,
                      rW=W, rsh=2, rsw=2)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


DGRAD_CASES = [(2, 8, 8, 64, 128, 3, 1), (2, 10, 10, 96, 64, 3, 1), (1, 7, 7, 512, 512, 3, 1),
               (2, 15, 15, 64, 64, 5, 2)]


@pytest.mark.parametrize("N,H,W,Ci,Co,R,pad", DGRAD_CASES)
def test_conv_dgrad_weight_taps(N, H, W, Ci, Co, R, pad):
    # stride-1 dgrad: im2col over dY (pad' = R-1-pad) x flipped weights read
    # in place through a 3-D transposing TMA map
    g = K.conv_geom(N, H, W, Ci, R, R, pad, 1)
    dy = _bf(N, Co, g.P, g.Q, seed=11)
    w = _bf(Co, Ci, R, R, scale=0.1, seed=12)
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), w.double(), dy.double(), stride=1, padding=pad).float()
    ref = ref.permute(0, 2, 3, 1).contiguous()
    cpad = (Ci + 63) // 64 * 64
    wp = _pad_w(w, cpad)  # [Co][R][S][Cpad]
    dyn = dy.permute(0, 2, 3, 1).contiguous()
    pd = R - 1 - pad
    ga = K.ConvGeom(N, g.P, g.Q, Co, H, W, R, R, pd, pd, 1, 1)
    copad = (Co + 63) // 64 * 64
    out = torch.zeros(N, H, W, Ci, device=dev, dtype=torch.bfloat16)
    args = K.GemmArgs(M=N * H * W, N=Ci, K=R * R * copad, a_kind=K.IM2COL_K, a=dyn.data_ptr(), a_geom=ga,
                      b_kind=4, b=wp.data_ptr(), out=out.data_ptr(), ldc=Ci, splits=1)
    args.b_extent = Ci
    args.b_taps = R * R
    args.b_cpad = cpad
    args.b_rows = Co
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


def _subpixel_dim(a, s, R, pad, H):
    r0 = (a + pad) % s
    J = (R - r0 + s - 1) // s if r0 < R else 0
    c = (a + pad) // s
    return r0, J, c, J - 1 - c, (H - a + s - 1) // s


@pytest.mark.parametrize("N,H,W,Ci,Co,R,pad,s", [(2, 16, 16, 64, 64, 3, 1, 2), (1, 15, 13, 72, 40, 3, 0, 2),
                                                 (2, 14, 14, 128, 96, 3, 1, 2)])
def test_conv_dgrad_subpixel_classes(N, H, W, Ci, Co, R, pad, s):
    """Strided dgrad as s*s stride-1 class GEMMs: im2col over dY with the
    class's taps (asymmetric box), weight taps through the general tap map,
    rows scattered to the class's pixels (remap)."""
    P, Q = (H + 2 * pad - R) // s + 1, (W + 2 * pad - R) // s + 1
    dy = _bf(N, Co, P, Q, seed=21)
    w = _bf(Co, Ci, R, R, scale=0.1, seed=22)
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), w.double(), dy.double(), stride=s, padding=pad).float()
    ref = ref.permute(0, 2, 3, 1).contiguous()
    cpad = (Ci + 63) // 64 * 64
    wp = _pad_w(w, cpad)
    dyn = dy.permute(0, 2, 3, 1).contiguous()
    copad = (Co + 63) // 64 * 64
    out = torch.zeros(N, H, W, Ci, device=dev, dtype=torch.bfloat16)
    for a in range(s):
        for b in range(s):
            r0a, Ja, ca, pla, Pa = _subpixel_dim(a, s, R, pad, H)
            r0b, Jb, cb, plb, Qb = _subpixel_dim(b, s, R, pad, W)
            if Ja == 0 or Jb == 0 or Pa == 0 or Qb == 0:
                continue
            ga = K.ConvGeom(N, P, Q, Co, Pa, Qb, Ja, Jb, pla, plb, 1, 1)
            args = K.GemmArgs(M=N * Pa * Qb, N=Ci, K=Ja * Jb * copad, a_kind=K.IM2COL_K, a=dyn.data_ptr(), a_geom=ga,
                              b_kind=4, b=wp.data_ptr(), out=out.data_ptr() + (a * W + b) * Ci * 2, ldc=Ci,
                              splits=1, remap=1, rP=Pa, rQ=Qb, rH=H, rW=W, rsh=s, rsw=s)
            args.b_extent = Ci
            args.b_taps = R * R
            args.b_cpad = cpad
            args.b_rows = Co
            args.b_tap_map = 1
            args.b_tap_base = (r0a + (Ja - 1) * s) * R + r0b + (Jb - 1) * s
            args.b_tap_dr = s * R
            args.b_tap_ds = s
            K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


@pytest.mark.parametrize("M,N,Kd,f32", [(256, 256, 64, False), (200, 72, 96, False), (130, 40, 128, True)])
def test_gemm_accumulate_out(M, N, Kd, f32):
    # out += A B^T (TMA reduce-add epilogue)
    a = _bf(M, Kd, seed=15)
    b = _bf(N, Kd, seed=16)
    prev = _bf(M, N, seed=17)
    out = prev.float().clone() if f32 else prev.clone()
    d = a.float() @ b.float().t()
    ref = prev.float() + d
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                      b_ld=Kd, out=out.data_ptr(), ldc=N, out_f32=int(f32), accumulate_out=1, splits=1)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref, mag=prev.float().abs() + d.abs() + ref.abs())


def test_gemm_split_partials_isolated():
    # split-K partials: rows past M of one split must not spill into the next
    M, N, Kd, S = 64, 192, 512, 4
    a = _bf(M, Kd, seed=18)
    b = _bf(N, Kd, seed=19)
    out = torch.full((S, M, N), 7.0, device=dev)
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                      b_ld=Kd, out=out.data_ptr(), ldc=N, out_f32=1, splits=S, split_stride=M * N)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out.sum(0), a.float() @ b.float().t())


# Shifted-band implicit GEMM (gemm_band.cu): stride-1 convs with Q >= 24, the
# ResNet / DenseNet / Inception 3x3 (and 1x7 / 7x1) shapes.
BAND_CASES = [(2, 28, 28, 64, 64, 3, 3, 1, 1), (1, 56, 56, 64, 64, 3, 3, 1, 1), (2, 28, 28, 128, 128, 3, 3, 1, 1),
              (2, 30, 30, 96, 64, 3, 3, 0, 0), (2, 35, 35, 64, 96, 5, 5, 2, 2), (2, 28, 28, 64, 192, 1, 7, 0, 3),
              (2, 28, 28, 64, 72, 7, 1, 3, 0), (1, 32, 40, 160, 200, 3, 3, 1, 1),
              (2, 56, 56, 128, 32, 3, 3, 1, 1), (3, 28, 28, 256, 32, 3, 3, 1, 1)]  # DenseNet growth convs (row-aligned bands)


@pytest.mark.parametrize("N,H,W,Ci,Co,R,S,ph,pw", BAND_CASES)
@pytest.mark.parametrize("accumulate", [False, True])
def test_conv_fprop_band(N, H, W, Ci, Co, R, S, ph, pw, accumulate):
    x = _bf(N, Ci, H, W, seed=21)
    w = _bf(Co, Ci, R, S, scale=0.1, seed=22)
    ref = F.conv2d(x.double(), w.double(), padding=(ph, pw)).permute(0, 2, 3, 1).contiguous().float()
    P, Q = H + 2 * ph - R + 1, W + 2 * pw - S + 1
    cpad = (Ci + 63) // 64 * 64
    xn = x.permute(0, 2, 3, 1).contiguous()
    wp = torch.zeros(Co, R, S, cpad, device=dev, dtype=torch.bfloat16)
    wp[..., :Ci] = w.permute(0, 2, 3, 1)
    g = K.ConvGeom(N, H, W, Ci, P, Q, R, S, ph, pw, 1, 1)
    M = N * P * Q
    base = _bf(N, P, Q, Co, seed=23) if accumulate else torch.zeros(N, P, Q, Co, device=dev, dtype=torch.bfloat16)
    out = base.clone()
    stats = torch.zeros(160, 2, Co, device=dev)
    args = K.GemmArgs(M=M, N=Co, K=R * S * cpad, a_kind=K.IM2COL_K, a=xn.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                      b=wp.data_ptr(), b_ld=R * S * cpad, out=out.data_ptr(), ldc=Co, splits=1,
                      stats=None if accumulate else stats.data_ptr(), accumulate_out=int(accumulate), band=1)
    K.gemm(args)
    torch.cuda.synchronize()
    want = ref + base.float() if accumulate else ref
    _check(out, want, mag=(base.float().abs() + ref.abs() + want.abs()) if accumulate else None)
    if not accumulate:
        r2 = out.float().reshape(M, Co)  # statistics are of the stored bf16 values
        _check(stats[:, 0].sum(0), r2.sum(0), rtol=1e-5)
        _check(stats[:, 1].sum(0), (r2 * r2).sum(0), rtol=1e-5)


@pytest.mark.parametrize("N,H,W,Ci,Co,R,pad", [(2, 28, 28, 64, 64, 3, 1), (1, 56, 56, 64, 128, 3, 1),
                                               (2, 28, 28, 128, 64, 3, 1)])
def test_conv_dgrad_band(N, H, W, Ci, Co, R, pad):
    dy = _bf(N, Co, H, W, seed=24)
    w = _bf(Co, Ci, R, R, scale=0.1, seed=25)
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), w.double(), dy.double(), stride=1, padding=pad).float()
    ref = ref.permute(0, 2, 3, 1).contiguous()
    cpad = (Ci + 63) // 64 * 64
    wp = _pad_w(w, cpad)
    dyn = dy.permute(0, 2, 3, 1).contiguous()
    pd = R - 1 - pad
    ga = K.ConvGeom(N, H, W, Co, H, W, R, R, pd, pd, 1, 1)
    copad = (Co + 63) // 64 * 64
    out = torch.zeros(N, H, W, Ci, device=dev, dtype=torch.bfloat16)
    args = K.GemmArgs(M=N * H * W, N=Ci, K=R * R * copad, a_kind=K.IM2COL_K, a=dyn.data_ptr(), a_geom=ga,
                      b_kind=4, b=wp.data_ptr(), out=out.data_ptr(), ldc=Ci, splits=1, band=1)
    args.b_extent = Ci
    args.b_taps = R * R
    args.b_cpad = cpad
    args.b_rows = Co
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


# ---- persistent multi-wave launches (> 2 x 148 tiles): the TMEM double-buffer
# phase flips, the smem ring wraps across tiles, and a CTA's fused statistics
# are flushed every time its column block changes
@pytest.mark.parametrize("bn", [64, 0])
def test_conv_fprop_multiwave_with_stats(bn):
    N, H, W, Ci, Co, R, pad, st = 8, 56, 56, 64, 256, 3, 1, 1
    x = _bf(N, Ci, H, W, seed=31)
    w = _bf(Co, Ci, R, R, scale=0.05, seed=32)
    ref = F.conv2d(x.double(), w.double(), stride=st, padding=pad).permute(0, 2, 3, 1).contiguous().float()
    g = K.conv_geom(N, H, W, Ci, R, R, pad, st)
    cpad = 64
    xn = x.permute(0, 2, 3, 1).contiguous()
    wp = _pad_w(w, cpad)
    M = N * g.P * g.Q
    tiles = (M + 127) // 128 * ((Co + (bn or 256) - 1) // (bn or 256))
    if bn:
        assert tiles > 2 * 148
    out = torch.zeros(N, g.P, g.Q, Co, device=dev, dtype=torch.bfloat16)
    stats = torch.zeros(160, 2, Co, device=dev)
    args = K.GemmArgs(M=M, N=Co, K=R * R * cpad, a_kind=K.IM2COL_K, a=xn.data_ptr(), a_geom=g,
                      b_kind=K.KMAJOR, b=wp.data_ptr(), b_ld=R * R * cpad, out=out.data_ptr(), ldc=Co,
                      stats=stats.data_ptr(), splits=1, block_n=bn)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)
    r2 = out.float().reshape(M, Co).double()
    _check(stats[:, 0].sum(0).double(), r2.sum(0), rtol=1e-5)
    _check(stats[:, 1].sum(0).double(), (r2 * r2).sum(0), rtol=1e-5)
    # rows of CTAs beyond the grid stay untouched
    assert stats[148:].abs().sum().item() == 0


@pytest.mark.parametrize("bn,f32", [(64, True), (128, False), (256, True)])
def test_gemm_kmajor_multiwave(bn, f32):
    M, N, Kd = 100352, 256, 64  # ResNet-50 layer1 1x1 conv shape at batch 32
    a = _bf(M, Kd, seed=33)
    b = _bf(N, Kd, seed=34)
    ref = a.float() @ b.float().t()
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                      b_ld=Kd, out=out.data_ptr(), ldc=N, out_f32=int(f32), splits=1, block_n=bn)
    K.gemm(args)
    torch.cuda.synchronize()
    _check(out, ref)


@pytest.mark.parametrize("splits", [1, 37])
def test_conv_wgrad_multiwave(splits):
    N, H, W, Ci, Co, R, pad, st = 8, 56, 56, 64, 64, 3, 1, 1
    x = _bf(N, Ci, H, W, seed=35)
    g = K.conv_geom(N, H, W, Ci, R, R, pad, st)
    dy = _bf(N, Co, g.P, g.Q, seed=36)
    ref = torch.nn.grad.conv2d_weight(x.double(), (Co, Ci, R, R), dy.double(), stride=st, padding=pad).float()
    xn = x.permute(0, 2, 3, 1).contiguous()
    dyn = dy.permute(0, 2, 3, 1).contiguous()
    M = N * g.P * g.Q
    ktot = R * R * 64
    out = torch.zeros(splits, Co, ktot, device=dev)
    args = K.GemmArgs(M=Co, N=ktot, K=M, a_kind=K.MNMAJOR, a=dyn.data_ptr(), a_ld=Co, b_kind=K.IM2COL_MN,
                      b=xn.data_ptr(), b_geom=g, out=out.data_ptr(), ldc=ktot, out_f32=1, splits=splits,
                      split_stride=Co * ktot, block_n=64)
    K.gemm(args)
    torch.cuda.synchronize()
    got = out.sum(0).reshape(Co, R, R, 64)[..., :Ci].permute(0, 3, 1, 2)
    _check(got, ref)


def _bwd_stats_case(kind, M, N, Kd, bn, seed):
    """A data-gradient GEMM whose output is dout of a BN+ReLU output."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    y = (torch.randn(M, N, generator=g) * 2 + 0.3).to(torch.bfloat16).to(dev)   # the BN input
    mean = (torch.randn(N, generator=g) * 0.1).to(dev)
    scale = (torch.rand(N, generator=g) + 0.5).to(dev)
    shift = (torch.randn(N, generator=g) * 0.5).to(dev)
    a = _bf(M, Kd, seed=seed + 1)
    if kind == "kmajor":
        b = _bf(N, Kd, seed=seed + 2)
        ref = a.float() @ b.float().t()
        kw = dict(b_kind=K.KMAJOR, b=b.data_ptr(), b_ld=Kd)
        keep = (a, b)
    else:  # 1x1 dgrad: W [Cout=K][Cin=N] MN-major
        wt = _bf(Kd, N, seed=seed + 2)
        ref = a.float() @ wt.float()
        kw = dict(b_kind=K.MNMAJOR, b=wt.data_ptr(), b_ld=N)
        keep = (a, wt)
    return y, mean, scale, shift, a, ref, kw, keep


@pytest.mark.parametrize("kind,M,N,Kd,bn", [("kmajor", 6272, 256, 512, 128), ("mnmajor", 25088, 128, 512, 64),
                                            ("mnmajor", 1000, 72, 256, 64), ("kmajor", 100352, 64, 256, 64)])
def test_bn_backward_statistics_epilogue_and_replay(kind, M, N, Kd, bn):
    """The dgrad GEMM epilogue stores dout and emits per-CTA rows of (sum g,
    sum g*(y - mean)), g = dout * [y*scale + shift > 0]; a replay launch (no GEMM,
    the epilogue re-reads the stored output) writes bit-identical rows -- so a
    BN backward gets the same statistics whether or not its input was resident
    when the dgrad ran."""
    y, mean, scale, shift, a, ref, kw, keep = _bwd_stats_case(kind, M, N, Kd, bn, seed=40)
    out = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    rows = torch.full((160, 2, N), 0.0, device=dev)
    args = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, out=out.data_ptr(), ldc=N,
                      stats=rows.data_ptr(), splits=1, block_n=bn, stats_bwd=1, bs_y=y.data_ptr(), bs_ldy=N,
                      bs_mean=mean.data_ptr(), bs_scale=scale.data_ptr(), bs_shift=shift.data_ptr(),
                      b_extent=N if kind == "mnmajor" else 0, **kw)
    K.gemm(args)
    torch.cuda.synchronize()
    mask = (y.float() * scale + shift) > 0
    # stored output: dout itself (one bf16 rounding of the GEMM)
    _check(out, ref)
    gm = torch.where(mask, out.float(), torch.zeros_like(ref)).double()  # exactly what the statistics sum
    s_ref = gm.sum(0)
    q_ref = (gm * (y.double() - mean.double())).sum(0)
    s, q = rows[:, 0].double().sum(0), rows[:, 1].double().sum(0)
    assert torch.allclose(s, s_ref, rtol=1e-5, atol=1e-3 * gm.abs().sum(0).max().item() / M), (s - s_ref).abs().max()
    assert torch.allclose(q, q_ref, rtol=1e-4, atol=1e-5 * (gm * (y.double() - mean.double())).abs().sum(0).max().item())
    # replay over the stored output: bit-identical rows
    rows2 = torch.full((160, 2, N), 0.0, device=dev)
    args2 = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=0, a_ld=Kd, out=out.data_ptr(), ldc=N,
                       stats=rows2.data_ptr(), splits=1, block_n=bn, stats_bwd=1, replay=1, bs_y=y.data_ptr(),
                       bs_ldy=N, bs_mean=mean.data_ptr(), bs_scale=scale.data_ptr(), bs_shift=shift.data_ptr())
    before = out.clone()
    K.gemm(args2)
    torch.cuda.synchronize()
    assert torch.equal(rows2, rows)
    assert torch.equal(out, before)  # the replay writes nothing
    # replay over the dout of a plain launch (a dgrad without the fused
    # epilogue): the same output bits, the same rows
    out_unmasked = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    plain = K.GemmArgs(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, out=out_unmasked.data_ptr(), ldc=N,
                       splits=1, block_n=bn, b_extent=N if kind == "mnmajor" else 0, **kw)
    K.gemm(plain)
    torch.cuda.synchronize()
    assert torch.equal(out_unmasked, out)
    rows3 = torch.full((160, 2, N), 0.0, device=dev)
    args2.out = out_unmasked.data_ptr()
    args2.stats = rows3.data_ptr()
    K.gemm(args2)
    torch.cuda.synchronize()
    assert torch.equal(rows3, rows)
