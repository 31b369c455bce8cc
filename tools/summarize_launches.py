"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/summarize_launches.py gpurun_out/launches.csv [--json out.json]

Prints per-kernel-family count, total and mean duration and share of the
total; used to produce profiles/*launches*.md.
"""
import argparse
import csv
import json
import re
from collections import defaultdict


def family(name: str) -> str:
    m = re.search(r"(gemm_kernel<\d+>|gemm_kernelILi(\d+)E)", name)
    if m:
        return f"gemm_kernel<BN={m.group(2) or m.group(1)}>"
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^.*::", "", name)
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        rows.append((family(r["Kernel Name"]), ns))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    total = sum(v[1] for v in agg.values())
    out = []
    print(f"{'kernel':40s} {'count':>6s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:6d} {ns / 1e3:10.1f} {ns / c / 1e3:9.2f} {100 * ns / total:5.1f}%")
        out.append({"kernel": k, "count": c, "total_us": ns / 1e3, "mean_us": ns / c / 1e3, "share": ns / total})
    print(f"{'TOTAL':40s} {len(rows):6d} {total / 1e3:10.1f}")
    if a.json:
        json.dump({"total_us": total / 1e3, "launches": len(rows), "kernels": out}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
