"""Same-run comparison: our grouped expert GEMMs (inside the Mixtral-size step) vs cuBLAS
(torch.matmul, bf16) dense GEMMs with the same total M x N x K, back to back, with the SM clock
sampled during each.  Separates kernel efficiency from the power-capped clock.

  python tools/gemm_vs_cublas.py
"""
import json
import os
import statistics
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402


def sample_clock(stop, out):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append([float(x) for x in line.split(",")])
    p.terminate()


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=sample_clock, args=(stop, samples))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / iters
    mhz = statistics.median(s[0] for s in samples) if samples else None
    w = statistics.median(s[1] for s in samples) if samples else None
    return ms, mhz, w


def main():
    dev = "cuda:0"
    res = {}
    # the Mixtral-size expert GEMM shapes at EP=1 (32768 routed rows)
    shapes = {"gate_up (M=32768, N=2*14336, K=4096)": (32768, 28672, 4096),
              "down (M=32768, N=4096, K=14336)": (32768, 4096, 14336),
              "dX (M=32768, N=4096, K=28672)": (32768, 4096, 28672),
              "cuBLAS reference 8192^3": (8192, 8192, 8192)}
    for name, (M, N, K) in shapes.items():
        a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        b = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
        ms, mhz, w = timed(lambda: torch.matmul(a, b.t()))
        res[f"cublas {name}"] = {"ms": ms, "tflops": 2 * M * N * K / ms / 1e9, "sm_mhz": mhz, "power_w": w}
        del a, b
        torch.cuda.empty_cache()
    # ours: the bench step, per-kernel event times
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3",
                          "--sweep", "0", "--no-cpu-baseline"], capture_output=True, text=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    hg, rows = 4096 * 14336, 32768
    coef = {"gemm_gateup_swiglu": 8, "gemm_down": 2, "gemm_dact_epilogue": 2, "gemm_dx": 4, "gemm_wgrad_down": 2,
            "gemm_wgrad_gateup": 4}
    for k, c in coef.items():
        ms = d["kernel_ms_per_step"][k]
        res[f"memfine {k}"] = {"ms_per_step": ms, "tflops": c * hg * rows / ms / 1e9}
    res["memfine step"] = {"ms": d["ms_per_step"], "clocks": d["clocks"]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
