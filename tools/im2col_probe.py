"""Stem im2col: exactness against torch unfold and graph-timed throughput (run on the GPU).

    python tools/im2col_probe.py
"""
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K  # noqa: E402


def ref(x, C, R, S, stride, pad, kpad):
    N, H, W, Cs = x.shape
    xc = x[..., :C].permute(0, 3, 1, 2).float()
    u = F.unfold(xc, (R, S), padding=pad, stride=stride)  # [N][C*R*S][L], (c, r, s) order
    L = u.shape[-1]
    u = u.view(N, C, R, S, L).permute(0, 4, 2, 3, 1).reshape(N * L, R * S * C)
    o = torch.zeros(N * L, kpad, device=x.device)
    o[:, :R * S * C] = u
    return o.to(torch.bfloat16)


def main():
    torch.manual_seed(0)
    for (N, H, C, Cs, R, st, pad, kpad) in [(2, 224, 3, 8, 7, 2, 3, 192), (32, 224, 3, 8, 7, 2, 3, 192),
                                            (32, 299, 3, 8, 3, 2, 0, 64)]:
        x = torch.randn(N, H, H, Cs, device="cuda").to(torch.bfloat16)
        out = K.im2col(x, C, R, R, st, pad, kpad)
        ok = torch.equal(out, ref(x, C, R, R, st, pad, kpad))
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        iters = 10
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                K.im2col(x, C, R, R, st, pad, kpad, out=out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        gb = (out.numel() * 2 + x.numel() * 2) / 1e9
        print(f"N={N} H={H} R={R} kpad={kpad}: exact={ok} {us:8.1f} us  {gb / us * 1e6:7.1f} GB/s")


if __name__ == "__main__":
    main()
