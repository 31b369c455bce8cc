"""Summarise an `ncu --set full` report into profiles/ (markdown + JSON).

    python tools/ncu_summary.py gpurun_out/gemm_full_rX.ncu-rep profiles/ncu_gemm_rX [--flops F]

Per captured launch: duration, DRAM bytes read/write, tensor-pipe and DRAM
utilisation, occupancy, registers.  The JSON's `dram_bytes_per_launch`
(mean over launches) is what bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "Grid Size",
    "block": "Block Size",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = r[i]
            try:
                d[k] = float(v.replace(",", "")) * SCALE.get(units[i], 1)
            except ValueError:
                d[k] = v
        launches.append(d)
    n = max(1, len(launches))
    dram = sum(l.get("dram_read", 0) + l.get("dram_write", 0) for l in launches) / n
    summ = {"report": a.rep, "launches": launches, "dram_bytes_per_launch": dram}
    json.dump(summ, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu --set full summary: `{a.rep}`\n\n")
        f.write("| kernel | grid | dur us | DRAM MB (r+w) | tensor % | DRAM % | SM % | warps % | regs |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for l in launches:
            f.write(f"| {l['kernel'][:60]} | {l.get('grid', '')} | {l.get('dur_us', 0):.1f} | "
                    f"{(l.get('dram_read', 0) + l.get('dram_write', 0)) / 1e6:.2f} | {l.get('tensor_pct', 0):.1f} | "
                    f"{l.get('dram_pct', 0):.1f} | {l.get('sm_pct', 0):.1f} | {l.get('warps_active_pct', 0):.1f} | "
                    f"{l.get('regs', '')} |\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
