"""Summarise an ncu report (--set full) or a launch-list CSV into markdown for profiles/.

    python tools/ncu_summary.py rep  gpurun_out/spmv_sym.ncu-rep   > profiles/...md
    python tools/ncu_summary.py launches gpurun_out/launches.csv    > profiles/...md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"ncu --set full report `{path}`\n")
    print("| kernel | " + " | ".join(n for _, n in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:40]
        cells = []
        for k, _ in KEYS:
            if k in h:
                i = h.index(k)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        print(f"| {name} | " + " | ".join(cells) + " |")


def launches(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        name = r[ki].split("(")[0][:60]
        tot[name] += us
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"ncu launch list `{path}` (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    print(f"total {allt:.1f} us over {sum(cnt.values())} launches\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} | {100 * tot[k] / allt:.1f}% |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
