"""Sustained-power comparison on one box: ~4 s of back-to-back work each, SM clock and power sampled
by nvidia-smi during it.  (1) cuBLAS bf16 GEMMs of the gate/up shape (M = 32768 copies, N = 2 x 14336,
K = 4096) and the 8192^3 peak shape; (2) the library's forward (gate/up + down + permute) and full
fwd+bwd step on the Mixtral-size layer.  Whether the grouped kernels cost more energy per FLOP than
cuBLAS shows up as a lower sustained clock at the same work.  Prints one JSON object.

  python tools/sustained_clock.py
"""
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import capi, layer  # noqa: E402


def run_for(fn, seconds, flops_per_call):
    samples, stop = [], threading.Event()

    def sampler():
        p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                              "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        while not stop.is_set():
            ln = p.stdout.readline()
            if ln:
                try:
                    samples.append([float(v) for v in ln.split(",")])
                except ValueError:
                    pass
        p.terminate()

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=sampler)
    th.start()
    time.sleep(0.3)
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(5):
            fn()
        n += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    tail = samples[len(samples) // 4:] or samples   # skip the ramp
    return {"ms_per_call": ms, "tflops": flops_per_call / (ms / 1e3) / 1e12,
            "sm_mhz_median": statistics.median(s[0] for s in tail),
            "power_w_median": statistics.median(s[1] for s in tail), "samples": len(tail)}


def main():
    dev = torch.device("cuda", 0)
    out = {}
    a = torch.randn(32768, 4096, device=dev, dtype=torch.bfloat16)
    b = torch.randn(4096, 2 * 14336, device=dev, dtype=torch.bfloat16)
    if not os.environ.get("SKIP_CUBLAS"):
        out["cublas_gateup_shape"] = run_for(lambda: a @ b, 4.0, 2.0 * 32768 * 4096 * 2 * 14336)
        c = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        out["cublas_8192"] = run_for(lambda: c @ c, 4.0, 2.0 * 8192 ** 3)
        del c
    del a, b
    cfg = synth.CONFIGS["mixtral"]
    T, h, g, E, k = cfg.T, cfg.h, cfg.g, cfg.E, cfg.k
    x, dy = synth.make_x(T, h).to(dev), synth.make_dy(T, h).to(dev)
    ids_np, w_np = synth.make_routing(T, E, k, zipf_s=cfg.zipf_s, placement=cfg.placement)
    ids, w = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
    ws_ = []
    for e in range(E):
        gen = torch.Generator(device=dev).manual_seed(7000 + e)
        ws_.append(((torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).bfloat16(),
                    (torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).bfloat16(),
                    (torch.randn(h, g, generator=gen, device=dev) / math.sqrt(g)).bfloat16()))
    wg, wu, wd = (torch.stack([t[i] for t in ws_]).contiguous() for i in range(3))
    del ws_
    f32 = dict(dtype=torch.float32, device=dev)
    dwg, dwu, dwd = torch.empty(wg.shape, **f32), torch.empty(wu.shape, **f32), torch.empty(wd.shape, **f32)
    y, dx, ds = torch.empty_like(x), torch.empty_like(x), torch.empty(w.shape, **f32)
    mf = layer.MemFine(T, h, g, E, k)
    counts = mf.route_counts(ids).cpu()
    wsb = max(layer.workspace_bytes(counts, mf.dims, 1, p_) for p_ in (capi.FWD, capi.BWD))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    copies = T * k
    out["memfine_fwd"] = run_for(lambda: mf.moe_fwd(x, ids, w, wg, wu, wd, 1, ws, y=y), 4.0, 6.0 * h * g * copies)

    def step():
        mf.moe_fwd(x, ids, w, wg, wu, wd, 1, ws, y=y)
        mf.moe_bwd(dy, x, ids, w, wg, wu, wd, 1, ws, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd, dscore=ds)
    out["memfine_step"] = run_for(step, 4.0, 22.0 * h * g * copies)
    assert mf.sync() == 0
    for v in out.values():
        v["tflops_per_ghz"] = v["tflops"] / (v["sm_mhz_median"] / 1000.0)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
