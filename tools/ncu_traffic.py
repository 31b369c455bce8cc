"""Per-kernel-family DRAM traffic and time from one ncu pass over a whole step.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/profile_step.py
    python tools/ncu_traffic.py gpurun_out/traffic.csv [--gemm-json profiles/ncu_gemm_summary.json]

ncu times are cold-cache and serialised: compare shares, not absolutes.  The
GEMM summary (dram bytes of every GEMM launch of one step) is what bench.py
reports as roofline.traffic next to the algorithmic bytes.
"""
import argparse
import csv
import json
from collections import defaultdict

from summarize_launches import family


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--gemm-json")
    ap.add_argument("--label", default="")
    ap.add_argument("--workload", default="resnet50_b32_224", help="arch_bBATCH_HW of the profiled step")
    a = ap.parse_args()
    with open(a.csv) as f:
        lines = [l for l in f if not l.startswith("==")]
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
             "second": 1e9}
    for r in csv.DictReader(lines):
        i = int(r["ID"])
        names[i] = family(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r.get("Metric Unit", ""), 1)
        per[i][r["Metric Name"]] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        k = names[i]
        agg[k][0] += 1
        agg[k][1] += m.get("gpu__time_duration.sum", 0.0)
        agg[k][2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot_t = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'count':>5s} {'total_us':>9s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>7s}")
    for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:5d} {t / 1e3:9.1f} {100 * t / tot_t:5.1f}% {b / 1e6:9.1f} {b / max(t, 1):7.0f}")
    print(f"{'TOTAL':40s} {len(per):5d} {tot_t / 1e3:9.1f}")
    if a.gemm_json:
        g = [v for k, v in agg.items() if k.startswith("gemm_kernel")]
        launches = sum(v[0] for v in g)
        dram = sum(v[2] for v in g)
        out = {"source": a.csv, "label": a.label, "workload": a.workload, "gemm_launches": launches, "dram_bytes_per_step": dram,
               "dram_bytes_per_launch": dram / max(launches, 1),
               "gemm_ncu_us_per_step": sum(v[1] for v in g) / 1e3,
               "families": {k: {"count": c, "us": t / 1e3, "dram_bytes": b} for k, (c, t, b) in agg.items()}}
        json.dump(out, open(a.gemm_json, "w"), indent=1)


if __name__ == "__main__":
    main()
