import sys, torch
sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K
torch.manual_seed(0)
for (n, h, C, Co) in [(8, 56, 128, 256), (8, 56, 256, 256), (8, 56, 128, 32), (8, 56, 128, 128), (4, 28, 128, 32), (8, 56, 64, 128)]:
    x = (torch.randn(n, h, h, C, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(Co, 9 * C, device="cuda") * 0.05).to(torch.bfloat16)
    g = K.ConvGeom(n, h, h, C, h, h, 3, 3, 1, 1, 1, 1)
    res = {}
    for band in (0, 1):
        o = torch.zeros(n * h * h, Co, device="cuda", dtype=torch.bfloat16)
        st = torch.zeros(160, 2, Co, device="cuda")
        K.gemm(K.GemmArgs(M=n * h * h, N=Co, K=9 * C, a_kind=K.IM2COL_K, a=x.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                          b=w.data_ptr(), b_ld=9 * C, out=o.data_ptr(), ldc=Co, stats=st.data_ptr(), splits=1, band=band))
        torch.cuda.synchronize()
        res[band] = (o.float(), st.sum(0))
    d = (res[0][0] - res[1][0]).abs().max().item() / res[0][0].abs().max().item()
    ds = ((res[0][1] - res[1][1]).abs().max() / res[0][1].abs().max()).item()
    print(n, h, C, Co, "out rel", d, "stats rel", ds, flush=True)
