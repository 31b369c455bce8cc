"""Isolated timing of representative ResNet-50 GEMM launches (run on the GPU).

python tools/gemm_probe.py            # time every case
python tools/gemm_probe.py --only 3   # one case, a few launches (for ncu)
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K  # noqa: E402

dev = "cuda"


def bf(*shape):
    return (torch.randn(*shape, device=dev) * 0.5).to(torch.bfloat16)


def cases():
    out = []
    # 1x1 fprop, K=64 -> N=256 at 56x56 (stage-1 expand), with fused BN stats
    M, Kd, N = 32 * 56 * 56, 64, 256
    a, b, o = bf(M, Kd), bf(N, Kd), bf(M, N)
    st = torch.zeros(160, 2, N, device=dev)
    out.append(("1x1 fprop K64 N256 +stats", M, N, Kd,
                dict(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                     b_ld=Kd, out=o.data_ptr(), ldc=N, stats=st.data_ptr(), splits=1), (a, b, o, st), {}))
    out.append(("1x1 fprop K64 N256", M, N, Kd,
                dict(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.KMAJOR, b=b.data_ptr(),
                     b_ld=Kd, out=o.data_ptr(), ldc=N, splits=1), (a, b, o), {}))
    # 1x1 dgrad 64 -> 256 accumulating into the skip gradient
    wt = bf(Kd, N)  # [Cout=64][Cin=256]: MN-major B
    out.append(("1x1 dgrad K64 N256 accumulate", M, N, Kd,
                dict(M=M, N=N, K=Kd, a_kind=K.KMAJOR, a=a.data_ptr(), a_ld=Kd, b_kind=K.MNMAJOR, b=wt.data_ptr(),
                     b_ld=N, out=o.data_ptr(), ldc=N, accumulate_out=1, splits=1), (a, wt, o), {"b_extent": N}))
    # 3x3 dgrad (stage 4 stride-2 via zero insert): M=6272 N=512 K=4608, weights in place
    n, h, ci, co = 32, 14, 512, 512
    dy = bf(n, h, h, co)
    w = bf(co, 3, 3, ci)
    o2 = bf(n, h, h, ci)
    g = K.ConvGeom(n, h, h, co, h, h, 3, 3, 1, 1, 1, 1)
    out.append(("3x3 dgrad Wtaps 14x14x512", n * h * h, ci, 9 * co,
                dict(M=n * h * h, N=ci, K=9 * co, a_kind=K.IM2COL_K, a=dy.data_ptr(), a_geom=g, b_kind=4,
                     b=w.data_ptr(), out=o2.data_ptr(), ldc=ci, splits=1), (dy, w, o2),
                {"b_extent": ci, "b_taps": 9, "b_cpad": ci, "b_rows": co}))
    # same contraction as a 3x3 fprop (K-major weights)
    wk = bf(co, 9 * ci)
    out.append(("3x3 fprop im2col 14x14x512", n * h * h, co, 9 * ci,
                dict(M=n * h * h, N=co, K=9 * ci, a_kind=K.IM2COL_K, a=dy.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                     b=wk.data_ptr(), b_ld=9 * ci, out=o2.data_ptr(), ldc=co, splits=1), (dy, wk, o2), {}))
    # plain 2-D GEMM of the same size
    a3 = bf(n * h * h, 9 * ci)
    out.append(("2D K-major 6272x512x4608", n * h * h, co, 9 * ci,
                dict(M=n * h * h, N=co, K=9 * ci, a_kind=K.KMAJOR, a=a3.data_ptr(), a_ld=9 * ci, b_kind=K.KMAJOR,
                     b=wk.data_ptr(), b_ld=9 * ci, out=o2.data_ptr(), ldc=co, splits=1), (a3, wk, o2), {}))
    # layer-1 3x3 conv (56x56x64 -> 64) on the im2col and the shifted-band paths
    n1, h1 = 32, 56
    x1 = bf(n1, h1, h1, 64)
    w1 = bf(64, 9 * 64)
    o1 = bf(n1, h1, h1, 64)
    s1 = torch.zeros(160, 2, 64, device=dev)
    g1 = K.ConvGeom(n1, h1, h1, 64, h1, h1, 3, 3, 1, 1, 1, 1)
    for band in (0, 1):
        out.append((f"3x3 56x56x64 fprop +stats band={band}", n1 * h1 * h1, 64, 576,
                    dict(M=n1 * h1 * h1, N=64, K=576, a_kind=K.IM2COL_K, a=x1.data_ptr(), a_geom=g1,
                         b_kind=K.KMAJOR, b=w1.data_ptr(), b_ld=576, out=o1.data_ptr(), ldc=64,
                         stats=s1.data_ptr(), splits=1, band=band), (x1, w1, o1, s1), {}))
    # same work without any out-of-bounds columns: 58x58 input, pad 0 -> 56x56
    x2 = bf(n1, 58, 58, 64)
    g2 = K.ConvGeom(n1, 58, 58, 64, h1, h1, 3, 3, 0, 0, 1, 1)
    out.append(("3x3 58x58 pad0 fprop +stats band=1", n1 * h1 * h1, 64, 576,
                dict(M=n1 * h1 * h1, N=64, K=576, a_kind=K.IM2COL_K, a=x2.data_ptr(), a_geom=g2,
                     b_kind=K.KMAJOR, b=w1.data_ptr(), b_ld=576, out=o1.data_ptr(), ldc=64,
                     stats=s1.data_ptr(), splits=1, band=1), (x2, w1, o1, s1), {}))
    # stem (7x7/2, 3 -> 64 at 112x112): explicit im2col K = 192, whole batch
    # and one 4-image chunk (the chunk's A stays in L2 across replays)
    Ms, Ks = 32 * 112 * 112, 192
    As, Bs, Os = bf(Ms, Ks), bf(64, Ks), bf(Ms, 64)
    Ss = torch.zeros(160, 2, 64, device=dev)
    for m in (Ms, Ms // 8):
        out.append((f"stem fprop M={m} K192 N64 +stats", m, 64, Ks,
                    dict(M=m, N=64, K=Ks, a_kind=K.KMAJOR, a=As.data_ptr(), a_ld=Ks, b_kind=K.KMAJOR,
                         b=Bs.data_ptr(), b_ld=Ks, out=Os.data_ptr(), ldc=64, stats=Ss.data_ptr(), splits=1),
                    (As, Bs, Os, Ss), {}))
    Ws = torch.zeros(32, 64, Ks, device=dev)
    out.append(("stem wgrad 64x192 K=401408 s32", 64, Ks, Ms,
                dict(M=64, N=Ks, K=Ms, a_kind=K.MNMAJOR, a=Os.data_ptr(), a_ld=64, b_kind=K.MNMAJOR,
                     b=As.data_ptr(), b_ld=Ks, out=Ws.data_ptr(), ldc=Ks, out_f32=1, splits=32,
                     split_stride=64 * Ks), (As, Os, Ws), {"block_n": 256}))
    # the 56x56x64 3x3 conv as a plain 2-D GEMM (A materialised): is the
    # im2col-mode TMA or the N=64 tile shape the limit?
    a56 = bf(n1 * h1 * h1, 576)
    for bn_ in (64, 128):
        out.append((f"2D 100352x64x576 (3x3 56x56 shape) bn={bn_}", n1 * h1 * h1, 64, 576,
                    dict(M=n1 * h1 * h1, N=64, K=576, a_kind=K.KMAJOR, a=a56.data_ptr(), a_ld=576, b_kind=K.KMAJOR,
                         b=w1.data_ptr(), b_ld=576, out=o1.data_ptr(), ldc=64, splits=1), (a56, w1, o1),
                    {"block_n": bn_}))
    out.append(("3x3 56x56x64 fprop im2col no stats", n1 * h1 * h1, 64, 576,
                dict(M=n1 * h1 * h1, N=64, K=576, a_kind=K.IM2COL_K, a=x1.data_ptr(), a_geom=g1,
                     b_kind=K.KMAJOR, b=w1.data_ptr(), b_ld=576, out=o1.data_ptr(), ldc=64, splits=1),
                (x1, w1, o1), {}))
    # sub-pixel dgrad class (layer2.0 3x3/2): dy 28x28x128 -> odd/odd class
    # of dx 56x56x128, 2x2 taps, with and without the output row remap
    dyc = bf(32, 28, 28, 128)
    wc = bf(128, 3, 3, 128)
    dxc = bf(32, 56, 56, 128)
    gc = K.ConvGeom(32, 28, 28, 128, 28, 28, 2, 2, 0, 0, 1, 1)
    for remap in (1, 0):
        out.append((f"subpixel class 2x2 K512 remap={remap}", 25088, 128, 512,
                    dict(M=25088, N=128, K=512, a_kind=K.IM2COL_K, a=dyc.data_ptr(), a_geom=gc, b_kind=4,
                         b=wc.data_ptr(), out=dxc.data_ptr(), ldc=128, splits=1, remap=remap, rP=28, rQ=28, rH=56,
                         rW=56, rsh=2, rsw=2), (dyc, wc, dxc),
                    {"b_extent": 128, "b_taps": 9, "b_cpad": 128, "b_rows": 128}))
    gc1 = K.ConvGeom(32, 28, 28, 128, 28, 28, 1, 1, 0, 0, 1, 1)
    out.append(("subpixel class 1x1 K128 remap=1", 25088, 128, 128,
                dict(M=25088, N=128, K=128, a_kind=K.IM2COL_K, a=dyc.data_ptr(), a_geom=gc1, b_kind=4,
                     b=wc.data_ptr(), out=dxc.data_ptr(), ldc=128, splits=1, remap=1, rP=28, rQ=28, rH=56,
                     rW=56, rsh=2, rsw=2), (dyc, wc, dxc),
                {"b_extent": 128, "b_taps": 9, "b_cpad": 128, "b_rows": 128}))
    a2 = bf(25088, 128)
    out.append(("plain 2D 25088x128x128", 25088, 128, 128,
                dict(M=25088, N=128, K=128, a_kind=K.KMAJOR, a=a2.data_ptr(), a_ld=128, b_kind=K.KMAJOR,
                     b=wc.data_ptr(), b_ld=128, out=dxc.data_ptr(), ldc=128, splits=1), (a2, wc, dxc), {}))
    # launch + prologue + epilogue floor: one 128x128 tile per SM, one K block
    Mt = 128 * 148
    at, bt, ot = bf(Mt, 64), bf(128, 64), bf(Mt, 128)
    out.append(("floor: 148 tiles, K=64", Mt, 128, 64,
                dict(M=Mt, N=128, K=64, a_kind=K.KMAJOR, a=at.data_ptr(), a_ld=64, b_kind=K.KMAJOR, b=bt.data_ptr(),
                     b_ld=64, out=ot.data_ptr(), ldc=128, splits=1), (at, bt, ot), {}))
    # 1x1 dgrad shape of layer2 (dY 25088x512 K-major, W MN-major): the
    # largest gap to its roofline in the step breakdown; same with K-major B
    a5 = bf(25088, 512)
    w5 = bf(512, 256)   # [Cout=K][Cin=N]: MN-major B
    w5k = bf(256, 512)  # K-major B
    o5 = bf(25088, 256)
    for bn_ in (128, 256):
        out.append((f"1x1 dgrad 25088x256x512 MN-major B bn={bn_}", 25088, 256, 512,
                    dict(M=25088, N=256, K=512, a_kind=K.KMAJOR, a=a5.data_ptr(), a_ld=512, b_kind=K.MNMAJOR,
                         b=w5.data_ptr(), b_ld=256, out=o5.data_ptr(), ldc=256, splits=1), (a5, w5, o5),
                    {"b_extent": 256, "block_n": bn_}))
        out.append((f"1x1 25088x256x512 K-major B bn={bn_}", 25088, 256, 512,
                    dict(M=25088, N=256, K=512, a_kind=K.KMAJOR, a=a5.data_ptr(), a_ld=512, b_kind=K.KMAJOR,
                         b=w5k.data_ptr(), b_ld=512, out=o5.data_ptr(), ldc=256, splits=1), (a5, w5k, o5),
                    {"block_n": bn_}))
    # 1x1 stride-2 dgrad (layer2.0 downsample): rows scattered to the even
    # pixels of 56x56 and accumulated into the block-input gradient
    o6 = bf(32 * 56 * 56, 256)
    for acc in (0, 1):
        out.append((f"1x1/2 dgrad remap 25088x256x512 acc={acc}", 25088, 256, 512,
                    dict(M=25088, N=256, K=512, a_kind=K.KMAJOR, a=a5.data_ptr(), a_ld=512, b_kind=K.MNMAJOR,
                         b=w5.data_ptr(), b_ld=256, out=o6.data_ptr(), ldc=256, splits=1, remap=1, rP=28, rQ=28,
                         rH=56, rW=56, rsh=2, rsw=2, accumulate_out=acc), (a5, w5, o6), {"b_extent": 256}))
    # large square 2-D GEMM: the engine's best case
    S = 8192
    a4, b4, o4 = bf(S, S), bf(S, S), bf(S, S)
    out.append(("2D K-major 8192^3", S, S, S,
                dict(M=S, N=S, K=S, a_kind=K.KMAJOR, a=a4.data_ptr(), a_ld=S, b_kind=K.KMAJOR, b=b4.data_ptr(),
                     b_ld=S, out=o4.data_ptr(), ldc=S, splits=1), (a4, b4, o4), {}))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", type=int, default=-1)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    torch.manual_seed(0)
    for i, (name, M, N, Kd, kw, keep, extra) in enumerate(cases()):
        if args.only >= 0 and i != args.only:
            continue
        ga = K.GemmArgs(**kw)
        for k, v in extra.items():
            setattr(ga, k, v)
        iters = 3 if args.only >= 0 else args.iters
        for _ in range(2):
            K.gemm(ga)
        torch.cuda.synchronize()
        if args.only >= 0:  # a few eager launches for ncu
            for _ in range(iters):
                K.gemm(ga)
            torch.cuda.synchronize()
            continue
        # device time without host overhead: the launches captured in a graph
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                K.gemm(ga)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        fl = 2.0 * M * N * Kd
        print(f"[{i}] {name:32s} {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
