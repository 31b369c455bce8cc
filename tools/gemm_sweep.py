"""Tile-width x split-K sweep over the distinct GEMM shapes of one step (run on the GPU).

    python tools/gemm_sweep.py [arch] [policy]

Writes gpurun_out/gemm_sweep_<arch>.json: per distinct (M, N, K, a_kind,
b_kind) the time of every (block_n, splits) pair, fp32 partial output.  Used
to calibrate the tile / split chooser in csrc/kernels/gemm.cu.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from oracle.train_oracle import random_batch  # noqa: E402
from paper_1808_00079_b200.executor import ReforwardNet  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
policy = sys.argv[2] if len(sys.argv) > 2 else "reforward"
net = ReforwardNet.named(arch, 32, 224, 224, 1000)
net.plan(policy)
net.setup(0)
x, y = random_batch(net, 0)
net.load_batch(x.cuda(), y.cuda())
net.step(lr=0.01, use_graph=True)
torch.cuda.synchronize()
rows = net.gemm_profile_detail(iters=1)
seen = {}
for i, r in enumerate(rows):
    key = (int(r["M"]), int(r["N"]), int(r["K"]), int(r["a_kind"]), int(r["b_kind"]))
    if key not in seen:
        seen[key] = (i, r)
out = []
for key, (i, r) in seen.items():
    M, N, K, ak, bk = key
    res = {}
    for bn in (64, 128, 256):
        if bn > 64 and N <= bn // 2:
            continue
        for sp in (1, 2, 3, 4, 6, 8):
            if sp > 1 and K < 64 * sp * 2:
                continue
            try:
                res[f"{bn}x{sp}"] = net.gemm_try(i, bn, sp, iters=5) * 1e3
            except Exception as e:  # noqa: BLE001
                res[f"{bn}x{sp}"] = None
    best = min((v, k) for k, v in res.items() if v)
    cur = r["ms"] * 1e3
    print(f"M={M:7d} N={N:5d} K={K:6d} a{ak} b{bk} cur bn={int(r['block_n'])} sp={int(r['splits'])} {cur:7.1f} us"
          f" | best {best[1]} {best[0]:7.1f} us | " + " ".join(f"{k}:{v:.0f}" for k, v in res.items() if v))
    out.append({"M": M, "N": N, "K": K, "a_kind": ak, "b_kind": bk, "cur_us": cur, "cur_bn": r["block_n"],
                "cur_splits": r["splits"], "flops": r["flops"], "bytes": r["bytes"], "times_us": res})
json.dump(out, open(f"gpurun_out/gemm_sweep_{arch}.json", "w"), indent=0)
