"""Config 5: memory-budget sweep of the DeepSeek-V3-style layer (one rank's load at EP=8:
32 local experts, 8K tokens x top-8, Zipf(1.2) routing) from 180 GB down to where C steps.

For every activation budget: the tuner's C (paper model, Eqs. 8-9 + bins, on the device) and
the exact-workspace C (MEMFINE_MODEL_IMPL), then fwd+bwd timed at the IMPL C with a ballast
allocation leaving only the budget free.  Prints one JSON object (the throughput vs memory
curve); commit it under profiles/.

  python tools/budget_sweep.py [--steps 5] [--warmup 2]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import capi, layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    T, h, g, E, k = 8192, 7168, 2048, 32, 8
    dev = torch.device("cuda", 0)
    ids_np, w_np = synth.make_routing(T, E, k, rank=0, zipf_s=1.2)
    x = synth.make_x(T, h).to(dev)
    dy = synth.make_dy(T, h).to(dev)
    ids = torch.from_numpy(ids_np).to(dev)
    w = torch.from_numpy(w_np).to(dev)
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
    counts = mf.route_counts(ids, 8)
    counts_h = counts.cpu()
    wsb = {C: max(layer.workspace_bytes(counts_h, mf.dims, C, capi.FWD),
                  layer.workspace_bytes(counts_h, mf.dims, C, capi.BWD)) for C in (1, 2, 4, 8)}

    def step(C, wst):
        mf.moe_fwd(x, ids, w, wg, wu, wd, C, wst, y=y)
        mf.moe_bwd(dy, x, ids, w, wg, wu, wd, C, wst, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd, dscore=ds)

    for C in (1, 8):  # load every kernel before measuring what is static
        wst = torch.empty(wsb[C], dtype=torch.uint8, device=dev)
        step(C, wst)
        del wst
    layer.plan(counts, mf.dims, capi.make_budget(int(180e9)))
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0, total = torch.cuda.mem_get_info()
    static = total - free0
    budgets = [int(b * 1e9) for b in (180, 140, 100, 60, 40)] + [static + wsb[C] + (16 << 20) for C in (1, 2, 4, 8)]
    points = []
    for B in budgets:
        pp = layer.plan(counts, mf.dims, capi.make_budget(B, 1.0, static, 0))
        pi = layer.plan(counts, mf.dims, capi.make_budget(B, 1.0, static, 0, model=capi.MODEL_IMPL))
        C = pi["C"]
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        size = max(0, torch.cuda.mem_get_info()[0] - (B - static))
        ballast = None
        for _ in range(5):
            ballast = None
            torch.cuda.empty_cache()
            if size:
                ballast = torch.empty(size - size % (2 << 20), dtype=torch.uint8, device=dev)
            torch.cuda.synchronize()
            err = (B - static) - torch.cuda.mem_get_info()[0]
            if abs(err) < (8 << 20):
                break
            size = max(0, size - err)
        wst = torch.empty(wsb[C], dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            step(C, wst)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(C, wst)
        e1.record()
        torch.cuda.synchronize()
        assert mf.sync() == 0
        ms = e0.elapsed_time(e1) / args.steps
        points.append({"budget_gb": B / 1e9, "activation_budget_gb": (B - static) / 1e9,
                       "C_paper": pp["C"], "C_impl": C, "c_theory": pp["c_theory"],
                       "s_dd_max": pp["s_dd_max"], "s_prime_max": pp["s_prime_max"],
                       "peak_act_gb_measured": wsb[C] / 1e9,
                       "peak_act_gb_paper_model": pp["predicted_peak_bytes"] / 1e9 if pp["status"] == 0 else None,
                       "ms_per_step": ms, "tokens_per_s": T / (ms / 1000.0)})
        del wst, ballast
        torch.cuda.empty_cache()
    print(json.dumps({"config": "dsv3-style layer, one rank's load at EP=8: 32 local experts, 8192 tokens x top-8, "
                                "h=7168, ffn=2048, Zipf(1.2)", "static_gb": static / 1e9,
                      "peak_act_gb_by_C": {C: v / 1e9 for C, v in wsb.items()}, "points": points}))


if __name__ == "__main__":
    main()
