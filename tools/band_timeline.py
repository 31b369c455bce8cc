"""Per-tile timeline of CTA 0 of the band kernel (RFK_BAND_DEBUG=1; GPU)."""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K
dev = "cuda"
n1, h1 = 32, 56
x1 = (torch.randn(n1, h1, h1, 64, device=dev)).to(torch.bfloat16)
w1 = (torch.randn(64, 576, device=dev) * 0.1).to(torch.bfloat16)
o1 = torch.zeros(n1, h1, h1, 64, device=dev, dtype=torch.bfloat16)
g1 = K.ConvGeom(n1, h1, h1, 64, h1, h1, 3, 3, 1, 1, 1, 1)
args = K.GemmArgs(M=n1 * h1 * h1, N=64, K=576, a_kind=K.IM2COL_K, a=x1.data_ptr(), a_geom=g1, b_kind=K.KMAJOR,
                  b=w1.data_ptr(), b_ld=576, out=o1.data_ptr(), ldc=64, splits=1, band=1)
for _ in range(3):
    K.gemm(args)
torch.cuda.synchronize()
