"""im2col-TMA vs shifted-band implicit GEMM on the ResNet-50 stride-1 3x3 shapes (GPU)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K  # noqa: E402

dev = "cuda"


def bf(*shape):
    return (torch.randn(*shape, device=dev) * 0.5).to(torch.bfloat16)


def timeit(ga, iters=20):
    for _ in range(2):
        K.gemm(ga)
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
    return e0.elapsed_time(e1) * 1e3 / iters


# ResNet-50 3x3 convs (c -> c) and DenseNet-121 growth convs (128 -> 32)
for (n, h, c, co) in [(32, 56, 64, 64), (32, 28, 128, 128), (32, 14, 256, 256), (32, 56, 128, 32), (32, 28, 128, 32),
                      (32, 14, 128, 32), (32, 35, 96, 96), (32, 17, 192, 192)]:
    x = bf(n, h, h, c)
    w = bf(co, 9 * ((c + 63) // 64 * 64))
    wt = bf(c, 3, 3, c)
    o = bf(n, h, h, max(c, co))
    st = torch.zeros(160, 2, co, device=dev)
    g = K.ConvGeom(n, h, h, c, h, h, 3, 3, 1, 1, 1, 1)
    M = n * h * h
    fl = 2.0 * M * co * 9 * c
    for band in (0, 1):
        cp = (c + 63) // 64 * 64
        fp = K.GemmArgs(M=M, N=co, K=9 * cp, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                        b=w.data_ptr(), b_ld=9 * cp, out=o.data_ptr(), ldc=co, stats=st.data_ptr(), splits=1, band=band)
        dg = K.GemmArgs(M=M, N=c, K=9 * cp, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=4, b=wt.data_ptr(),
                        out=o.data_ptr(), ldc=c, splits=1, band=band)
        for k, v in {"b_extent": c, "b_taps": 9, "b_cpad": c, "b_rows": c}.items():
            setattr(dg, k, v)
        for name, ga in (("fprop+stats", fp), ("dgrad", dg)):
            if name == "dgrad" and co != c:
                continue
            us = timeit(ga)
            print(f"3x3 {h}x{h}x{c}->{co} {name:12s} band={band}: {us:7.1f} us  {fl / us / 1e6:7.1f} TFLOP/s")
