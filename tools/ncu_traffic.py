"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) per kernel class from
an `ncu --set full` capture, as JSON for bench.py's roofline.traffic field.

  python tools/ncu_traffic.py gpurun_out/prof.ncu-rep > profiles/r01_ncu_traffic.json
  python tools/ncu_traffic.py gpurun_out/prof_raw.csv  (ncu -i prof.ncu-rep --page raw --csv, exported on the box)
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

SLOT = {0: "gemm_gateup_swiglu", 1: "gemm_down", 2: "gemm_dact_epilogue", 3: "gemm_dx", 4: "gemm_wgrad_down",
        5: "gemm_wgrad_gateup"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    it = hdr.index("gpu__time_duration.sum")
    acc = defaultdict(list)
    for r in data:
        name = r[hdr.index("Kernel Name")]
        m = re.search(r"gemm_kernel<(\d+)", name)
        key = SLOT[int(m.group(1))] if m else re.sub(r"[<(].*", "", name.replace("void ", ""))
        b = float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]]
        acc[key].append((b, float(r[it])))
    out = {k: {"bytes_per_launch": sum(b for b, _ in v) / len(v), "launches_captured": len(v),
               "ncu_ms_per_launch": sum(t for _, t in v) / len(v)} for k, v in acc.items()}
    out["_source"] = path
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
