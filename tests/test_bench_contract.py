"""bench.py keeps the driver's contract: one JSON line with the required keys.

The reference arm (the oracle on the host cores) runs without a GPU; the GPU arm runs on the tiny
config (BASELINE.json configs[0]) under -m gpu.  Both as subprocesses, exactly as the driver
launches them.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    line = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1", "--ref-tokens", "8"],
                timeout=600)
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["steps"] == 2 and line["warmup"] == 1 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "workload" in line["config"]


@pytest.mark.gpu
def test_gpu_arm_line_tiny():
    line = _run(["--config", "tiny", "--steps", "3", "--warmup", "3", "--cpu-tokens", "4"], timeout=900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "per_C", "peak_act_gb", "kernel_ms_per_step"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["dtype"] == "bf16" and line["higher_is_better"] is True
    roof = line["roofline"]
    # the tiny layer is bound by its permute kernels, not the GEMMs
    assert (roof["bound"], roof["unit"]) in (("tensor", "TFLOP/s"), ("hbm", "GB/s"))
    assert 0 < roof["frac"] == roof["achieved"] / roof["peak"]
    assert roof["traffic"] is None   # the committed ncu capture is of the Mixtral workload, not this one
    sr = line["step_roofline"]   # the north star's 3-term roofline of the whole step
    assert sr["bound"] in ("tensor", "hbm", "nvlink") and 0 < sr["frac"] <= 1.0 and sr["t_roof4_ms"] >= sr["t_roof_ms"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle"
    # chunking: the peak activation falls with C (Table 2 rows 11-13 live for one chunk only)
    peaks = [line["per_C"][c]["peak_act_gb"] for c in sorted(line["per_C"], key=int)]
    assert all(a >= b for a, b in zip(peaks, peaks[1:]))
