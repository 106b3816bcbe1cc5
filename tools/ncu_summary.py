"""Summarises ncu reports / launch lists into profiles/*.md (run here, no GPU needed).

    python tools/ncu_summary.py report  gpurun_out/x.ncu-rep  > profiles/x.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/launches.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed_pipe_uniform.sum",
    "lts__t_bytes.sum",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: `{path.split('/')[-1]}`\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"## {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
        extra = [i for i, h in enumerate(hdr) if ("tensor" in h.lower() or "utc" in h.lower()) and h not in KEYS]
        for i in extra[:12]:
            print(f"| {hdr[i]} | {r[i]} | {units[i]} |")
        print()


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v_us = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
        name = r["Kernel Name"].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += v_us
        total += v_us
    print(f"# launch list `{path.split('/')[-1]}` (ncu gpu__time_duration, cold-cache, serialised)\n")
    print(f"total {total/1000:.3f} ms over {sum(a[0] for a in agg.values())} launches\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {t:.1f} | {100*t/total:.1f}% |")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
