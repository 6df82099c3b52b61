"""Summarise ncu reports into markdown for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py full   gpurun_out/prof_gemm.ncu-rep   > profiles/...md   (or a raw .csv)
  python tools/ncu_summary.py launches gpurun_out/launches.csv       > profiles/...md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name):
    name = name.replace("memfine::", "").replace("sm100::", "")
    return name.split("(")[0]


def full(path):
    if path.endswith(".csv"):   # `ncu -i rep --page raw --csv` exported on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [(hdr.index(m), lab, units[hdr.index(m)]) for m, lab in METRICS if m in hdr]
    print(f"ncu --set full: `{path}`\n")
    print("| kernel | " + " | ".join(f"{lab} ({u})" if u else lab for _, lab, u in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in data:
        print("| " + short(r[hdr.index("Kernel Name")]) + " | " + " | ".join(r[i] for i, _, _ in cols) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[i + 1:]:
        if len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}.get(unit, 1.0)
        k = short(r[hdr.index("Kernel Name")])
        tot[k] += v * scale
        cnt[k] += 1
    s = sum(tot.values())
    print(f"ncu launch list (gpu__time_duration.sum, --clock-control none, serialised cold-cache): `{path}`\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k]} | {tot[k]:.3f} | {100 * tot[k] / s:.1f}% |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
