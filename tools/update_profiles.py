"""Copy one round refresh's outputs (tools/round_refresh.sh <tag>, merged back
into gpurun_out/) into profiles/ and regenerate DESIGN.md's measured table.

    python tools/update_profiles.py r2e
"""
import glob
import json
import os
import re
import shutil
import subprocess
import sys

tag = sys.argv[1]
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")
for f in glob.glob(os.path.join(G, f"bench_{tag}", "*.json")):
    shutil.copy(f, os.path.join(P, f"bench_{os.path.basename(f)[:-5]}_r2.json"))
prof = os.path.join(G, f"prof_{tag}")
run = lambda *a, out: open(os.path.join(P, out), "w").write(
    subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=R).stdout)
run("tools/ncu_traffic.py", os.path.join(prof, "traffic.csv"), "--gemm-json", "profiles/ncu_gemm_summary.json",
    out="ncu_traffic_r2.txt")
run("tools/summarize_launches.py", os.path.join(prof, "traffic.csv"), out="launches_r2.txt")
for rep, name in (("gemm_full", "ncu_gemm_r2"), ("bn_full", "ncu_bn_r2"), ("band_pool_full", "ncu_band_pool_r2")):
    if os.path.exists(os.path.join(prof, rep + ".ncu-rep")):
        subprocess.run([sys.executable, "tools/ncu_summary.py", os.path.join(prof, rep + ".ncu-rep"), f"profiles/{name}"],
                       cwd=R, capture_output=True)
for src, dst in (("gemm_breakdown.txt", "gemm_breakdown_r2.txt"), ("step_breakdown.txt", "step_breakdown_r2.txt"),
                 ("ablation.txt", "ablation_r2.txt")):
    shutil.copy(os.path.join(prof, src), os.path.join(P, dst))
shutil.copy(os.path.join(G, f"gpu_tests_{tag}.log"), os.path.join(P, "gpu_tests_r2.log"))

names = [("resnet50_b32_224", "ResNet-50 (headline)", "32, 224²"), ("resnet101_b32_224", "ResNet-101", "32, 224²"),
         ("densenet121_b32_224", "DenseNet-121", "32, 224²"),
         ("densenet121_b64_600", "DenseNet-121 (high-res stress, configs[4])", "64, 600²"),
         ("inception_v3_b32_299", "Inception-v3", "32, 299²"),
         ("inception_v3_b64_600", "Inception-v3 (high-res stress, configs[4])", "64, 600²"),
         ("vgg16_b32_224", "VGG-16", "32, 224²"), ("alexnet_b32_224", "AlexNet", "32, 224²")]
rows = []
for f, n, c in names:
    d = json.load(open(os.path.join(P, f"bench_{f}_r2.json")))
    m, r = d["memory"], d["roofline"]
    rows.append(f"| {n} | {c} | {d['value']:.0f} | {d['e2e']['value']:.0f} | {d['store_all']['value']:.0f} | "
                f"{d['overhead_vs_store_all']:.2f}x | {m['activation_peak_bytes'] / 1e6:.0f} MB / "
                f"{m['store_all_bytes'] / 1e6:.0f} MB ({m['cut_percent']:.1f} %) | {m['device_bytes'] / 1e6:.0f} MB / "
                f"{m['store_all_device_bytes'] / 1e6:.0f} MB ({m['device_cut_percent']:.1f} %) | "
                f"{r['achieved']:.0f} ({r['frac']:.3f}) | {r['frac_of_roofline_time']:.2f} |")
p = os.path.join(R, "DESIGN.md")
s = open(p).read()
i0 = s.index("| ResNet-50 (headline) | 32, 224² |")
i1 = s.index("\n\n(Mid-round-2 lines")
open(p, "w").write(s[:i0] + "\n".join(rows) + s[i1:])
print("\n".join(rows))
