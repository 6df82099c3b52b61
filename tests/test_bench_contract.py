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


def test_multi_rank_launcher_reference_arm():
    """`bench.py --gpus 2` without torchrun re-launches itself under torch.distributed.run (2 ranks on
    this node, rendezvous on 127.0.0.1); the ranks meet in a gloo group, rank 0 alone works and prints
    the one line, the other exits 0 - the driver's plain multi-GPU command, exercised on CPU."""
    line = _run(["--impl", "reference", "--gpus", "2", "--config", "tiny", "--steps", "1", "--warmup", "0",
                 "--ref-tokens", "4"], timeout=600)
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["ep"] == 2


@pytest.mark.gpu
def test_gpu_arm_line_tiny():
    line = _run(["--config", "tiny", "--steps", "3", "--warmup", "3", "--cpu-tokens", "4"], timeout=900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "per_C", "peak_act_gb", "kernel_ms_per_step"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["dtype"] == "bf16" and line["higher_is_better"] is True
    tuner = line["config"]["tuner"]
    assert tuner["in_timed_step"] and tuner["rule"].startswith("EXACT")
    assert tuner["fwd"]["C"] >= 1 and tuner["bwd"]["C"] >= 1
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
    pc = line["paper_context"]   # the paper's numbers with its hardware, beside this run's analogues
    assert pc["paper"]["activation_reduction_pct"] == 48.03 and pc["paper"]["throughput_vs_method1_pct"] == 4.42
    assert "activation_reduction_pct_c2" in pc["this_run"]
    # chunking: the peak activation falls with C (Table 2 rows 11-13 live for one chunk only)
    peaks = [line["per_C"][c]["peak_act_gb"] for c in sorted(line["per_C"], key=int)]
    assert all(a >= b for a, b in zip(peaks, peaks[1:]))


def test_step_roofline_terms():
    """The north star's 3-term step roofline on hand-made counts (EP = 2, E = 4, E_l = 2): rank 0 keeps
    10 copies for expert 0 and sends 30 to expert 2; rank 1 sends 5 to expert 1 and keeps 20 for
    expert 3.  s''_0 = 15, s''_1 = 50; off-rank traffic: rank 0 sends 30 / receives 5, rank 1 the
    reverse - so rank 1 is hot on FLOPs and both move 30 rows."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    counts = torch.zeros((2, 8, 4), dtype=torch.int32)
    counts[0, 0, 0], counts[0, 3, 2] = 10, 30
    counts[1, 5, 1], counts[1, 7, 3] = 5, 20
    h, g, k, T, El, C = 64, 128, 2, 40, 2, 2
    peaks = {"bf16_tflops_sustained": 1e-9, "hbm_gbs": 1e-3}       # FLOP/s 1e3, B/s 1e6
    r = bench.step_roofline(counts, h, g, k, T, El, C, ms=1000.0, peaks=peaks, nvlink_gbs=1e-3)
    F1 = 22 * h * g * 50 / 1e3                                       # seconds on the hot rank
    P = 10 * (k + 1) * h * T / 1e6
    N = 10 * h * 30 / 1e6
    W = 3 * El * h * g * 2
    P4 = (10 * (k + 1) * h * T + C * 8 / 3 * W + (4 * C - 2) * W) / 1e6
    assert r["hot_rank"] == 1 and r["bound"] == "tensor"
    assert abs(r["t_roof_ms"] - 1e3 * max(F1, P, N)) < 1e-6 * r["t_roof_ms"]
    assert abs(r["t_roof4_ms"] - 1e3 * max(F1, P4, N)) < 1e-6 * r["t_roof4_ms"]
    t = r["terms_ms_hot_rank"]
    assert abs(t["a2a_bytes"] - 1e3 * N) < 1e-9 and abs(t["permute_bytes"] - 1e3 * P) < 1e-9
    assert abs(r["frac"] - max(F1, P, N) / 1.0) < 1e-9
    # t_serial: the same terms not overlapped, on the rank where their sum is largest
    F0 = 22 * h * g * 15 / 1e3
    N0 = N
    assert abs(r["t_serial_ms"] - 1e3 * max(F0 + P4 + N0, F1 + P4 + N)) < 1e-6 * r["t_serial_ms"]
    pc = bench.per_c_roofline(counts, h, g, k, T, El, C, 1000.0, peaks)     # NVLink at its default 900 GB/s
    r9 = bench.step_roofline(counts, h, g, k, T, El, C, ms=1000.0, peaks=peaks)
    assert pc["t_roof4_ms"] == r9["t_roof4_ms"] and pc["t_serial_ms"] == r9["t_serial_ms"]
    assert pc["t_serial_ms"] >= pc["t_roof4_ms"]


def test_ep_emulation_shapes():
    """--ep-emulate R runs one rank's expert load at EP = R on one GPU: the config's T k copies over E/R
    local experts.  With fewer local experts than top-k (Mixtral at EP = 8: one expert per rank) the copies
    run as T k / E_l tokens of top-E_l routing - the same expert GEMM shapes - while tokens/s and the
    workload still count the real layer's T tokens per GPU."""
    import argparse
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    import synth
    for name, R in (("mixtral", 8), ("dsv3", 8), ("qwen3", 8), ("mixtral", 1)):
        a = argparse.Namespace(config=name, ep_emulate=R, tokens=0, placement=None)
        cfg, cfg0 = b.emulated_config(a), synth.CONFIGS[name]
        assert cfg.E == cfg0.E // R and cfg.k <= cfg.E
        assert cfg.T * cfg.k == cfg0.T * cfg0.k                    # the same copies
        wl = b.workload_config(cfg, a, 1)
        assert wl["tokens_per_gpu"] == cfg0.T and f"top-{cfg0.k}" in wl["workload"]
    a = argparse.Namespace(config="mixtral", ep_emulate=8, tokens=0, placement=None)
    assert (b.emulated_config(a).E, b.emulated_config(a).k, b.emulated_config(a).T) == (1, 1, 32768)
