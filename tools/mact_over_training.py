"""MACT over training (Fig. 5 / Table 4 / Methods 1-3).

A stack of MoE layers runs forward+backward for several iterations at EP = 4 (four ranks as host
threads on one GPU, memfine in-process group: real dispatch / expert / combine exchanges).  Routing
skew grows with depth and peaks in early iterations ("larger chunks are concentrated in layers
7-15 during iterations 5-15 ... stabilizes after ~10 iterations") — a synthetic
Zipf stand-in, hot experts contiguous on rank 0 (the Fig. 2 extreme).  For every (iteration,
layer) cell the device tuner picks C from the all-gathered counts under a per-GPU activation
budget (MEMFINE_MODEL_IMPL: the exact workspace), and the three methods of PAPER.md:225-230 are
compared: Method 1 = no chunking (C=1; "OOM" when its workspace exceeds the budget),
Method 2 = fixed c_k = 8, Method 3 = MACT with bins [1,2,4,8].

  python tools/mact_over_training.py [--layers 8] [--iters 12]   -> one JSON object
"""
import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import capi, layer  # noqa: E402


def skew(i, l, L):
    """Zipf exponent of layer l at iteration i: deeper layers more skewed, peak early in training."""
    return 0.15 + 1.7 * ((l + 1) / L) * math.exp(-((i - 6) / 4.0) ** 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--ep", type=int, default=4)
    ap.add_argument("--budget-mb", type=float, default=1300.0, help="per-GPU activation budget")
    args = ap.parse_args()
    EP, L, I = args.ep, args.layers, args.iters
    T, h, g, E, k = 4096, 2048, 4096, 16, 4
    El = E // EP
    wg, wu, wd = synth.make_experts(range(E), h, g)
    group = layer.LocalGroup(EP)
    budget_act = int(args.budget_mb * 1e6)
    cells = {}          # (i, l) -> record
    lock = threading.Lock()
    errors = []
    barrier = threading.Barrier(EP)

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                dev = "cuda:0"
                mf = layer.MemFine(T, h, g, E, k, ep_size=EP, ep_rank=r, local_group=group)
                lwg, lwu, lwd = (t[r * El:(r + 1) * El].contiguous().to(dev) for t in (wg, wu, wd))
                x = synth.make_x(T, h, rank=r).to(dev)
                dy = synth.make_dy(T, h, rank=r).to(dev)
                f32 = dict(dtype=torch.float32, device=dev)
                grads = [torch.zeros(t.shape, **f32) for t in (lwg, lwu, lwd)]
                # warm-up (untimed): first launches of every kernel, tensor-map encodes, every C
                ids_np, w_np = synth.make_routing(T, E, k, rank=r, zipf_s=skew(0, 0, L), placement="contiguous", seed=7)
                ids, w = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
                ch = mf.route_counts(ids, nsub=8, stream=st).cpu()
                for C in (1, 2, 4, 8):
                    ws = torch.empty(layer.workspace_bytes(ch, mf.dims, C, capi.BWD), dtype=torch.uint8, device=dev)
                    barrier.wait()
                    mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws, stream=st)
                    mf.moe_bwd(dy, x, ids, w, lwg, lwu, lwd, C, ws, dw_gate=grads[0], dw_up=grads[1], dw_down=grads[2],
                               accumulate_dw=True, stream=st)
                    assert mf.sync(stream=st) == 0
                    del ws
                for i in range(I):
                    for l in range(L):
                        ids_np, w_np = synth.make_routing(T, E, k, rank=r, zipf_s=skew(i, l, L),
                                                          placement="contiguous", seed=100000 * i + 1000 * l)
                        ids = torch.from_numpy(ids_np).to(dev)
                        w = torch.from_numpy(w_np).to(dev)
                        counts = mf.route_counts(ids, nsub=8, stream=st)
                        st.synchronize()
                        ch = counts.cpu()
                        # the exact backward workspace of every rank for every C
                        ws_all = {C: max(layer.workspace_bytes(ch, layer.make_dims(T, h, g, E, k, EP, rr), C,
                                                               capi.BWD) for rr in range(EP)) for C in (1, 2, 4, 8)}
                        bi = capi.make_budget(budget_act, 1.0, 0, 0, model=capi.MODEL_IMPL)
                        plan = layer.plan(counts, mf.dims, bi)          # device counts -> C
                        paper = layer.plan(counts, mf.dims, capi.make_budget(budget_act, 1.0, 0, 0))
                        rec = {"C_mact": plan["C"], "C_paper_model": paper["C"], "s_dd_max": paper["s_dd_max"],
                               "hot_rank": paper["hot_rank"], "ws_gb": {C: ws_all[C] / 1e9 for C in ws_all},
                               "feasible_C1": ws_all[1] <= budget_act, "skew": skew(i, l, L)}
                        times = {}
                        for name, C in (("method3_mact", plan["C"]), ("method2_c8", 8), ("method1_c1", 1)):
                            wsb = layer.workspace_bytes(ch, mf.dims, C, capi.BWD)
                            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
                            barrier.wait()
                            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            e0.record(st)
                            y = mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws, stream=st)
                            mf.moe_bwd(dy, x, ids, w, lwg, lwu, lwd, C, ws, dw_gate=grads[0], dw_up=grads[1],
                                       dw_down=grads[2], accumulate_dw=True, stream=st)
                            e1.record(st)
                            assert mf.sync(stream=st) == 0
                            times[name] = e0.elapsed_time(e1)
                            del ws, y
                        with lock:
                            c = cells.setdefault((i, l), {})
                            if r == 0:
                                c.update(rec)
                            for n_, t_ in times.items():   # max over ranks
                                c[n_ + "_ms"] = max(c.get(n_ + "_ms", 0.0), t_)
                mf.close()
        except BaseException:  # noqa: BLE001
            import traceback
            errors.append(f"rank {r}: {traceback.format_exc()}")
            barrier.abort()

    t0 = time.time()
    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(EP)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    group.close()
    if errors:
        print("\n".join(errors), file=sys.stderr)
        sys.exit(1)
    heat = [[cells[(i, l)]["C_mact"] for l in range(L)] for i in range(I)]
    summ = {}
    for name in ("method1_c1", "method2_c8", "method3_mact"):
        summ[name] = {"total_ms_all_cells": sum(c[name + "_ms"] for c in cells.values()),
                      "cells_over_budget": sum(1 for c in cells.values() if name == "method1_c1"
                                               and not c["feasible_C1"]),
                      "tokens_per_s_per_gpu": EP * T * len(cells) / (sum(c[name + "_ms"] for c in cells.values())
                                                                     / 1e3) / EP}
    peak = {"method1_c1": max(c["ws_gb"][1] for c in cells.values()),
            "method2_c8": max(c["ws_gb"][8] for c in cells.values()),
            "method3_mact": max(c["ws_gb"][c["C_mact"]] for c in cells.values())}
    out = {"config": {"EP": EP, "tokens_per_gpu": T, "h": h, "ffn": g, "E": E, "k": k, "layers": L, "iters": I,
                      "activation_budget_gb": budget_act / 1e9, "routing": "Zipf(s(i,l)), hot experts on rank 0",
                      "note": "EP ranks are threads on one GPU (in-process group); times are per layer fwd+bwd, "
                              "max over ranks, ranks share the device"},
           "C_heatmap_iter_by_layer": heat, "methods": summ, "peak_activation_gb": peak,
           "cells": {f"{i},{l}": cells[(i, l)] for i in range(I) for l in range(L)},
           "wall_s": time.time() - t0}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
