"""Band-kernel diagnostics: per-row-phase / per-column error of a 3x3 conv (GPU)."""
import sys
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
from paper_1808_00079_b200 import kernels as K  # noqa: E402

dev = "cuda"
N, H, W, Ci, Co, R, S, ph, pw = 1, 28, 28, 64, 64, 3, 3, 1, 1
torch.manual_seed(0)
x = torch.randn(N, Ci, H, W, device=dev).to(torch.bfloat16)
w = (torch.randn(Co, Ci, R, S, device=dev) * 0.1).to(torch.bfloat16)
mode = sys.argv[1] if len(sys.argv) > 1 else "full"
if mode == "center":  # only the centre tap
    w2 = torch.zeros_like(w); w2[:, :, 1, 1] = w[:, :, 1, 1]; w = w2
if mode == "tap00":
    w2 = torch.zeros_like(w); w2[:, :, 0, 0] = w[:, :, 0, 0]; w = w2
ref = F.conv2d(x.float(), w.float(), padding=(ph, pw)).permute(0, 2, 3, 1).contiguous()
P, Q = H, W
xn = x.permute(0, 2, 3, 1).contiguous()
wp = w.permute(0, 2, 3, 1).contiguous()
g = K.ConvGeom(N, H, W, Ci, P, Q, R, S, ph, pw, 1, 1)
out = torch.zeros(N, P, Q, Co, device=dev, dtype=torch.bfloat16)
args = K.GemmArgs(M=N * P * Q, N=Co, K=R * S * 64, a_kind=K.IM2COL_K, a=xn.data_ptr(), a_geom=g, b_kind=K.KMAJOR,
                  b=wp.data_ptr(), b_ld=R * S * 64, out=out.data_ptr(), ldc=Co, splits=1, band=1)
K.gemm(args)
torch.cuda.synchronize()
err = (out.float() - ref).abs().amax(-1)[0]  # [P, Q]
print(mode, "max err", err.max().item(), "ref scale", ref.abs().max().item())
Wp = W + 2 * pw
for h in range(0, 6):
    print("h", h, " ".join(f"{err[h, q].item():.2f}" for q in range(Q)))
# group by plane position phase
import collections
by = collections.defaultdict(list)
for h in range(P):
    for q in range(Q):
        j = h * Wp + q
        by[(j % 128) % 8].append(err[h, q].item())
print("by (j%128)%8:", {k: round(max(v), 2) for k, v in sorted(by.items())})
