"""Chunk pipelining of the EP exchange (MEMFINE_FLAG_OVERLAP), measured on ONE B200.

NCCL refuses two ranks on one device, so the EP data path runs over a 1-rank communicator
(MEMFINE_FLAG_EP_PATH): every chunk's dispatch and combine are real NCCL send/recv kernels (to
self) that move the same bytes per rank as an EP exchange's self segment would.  For each C the
fwd+bwd step is timed four ways:
  ep1        the EP = 1 path (no exchange at all) - the floor;
  serial     EP path, one stream: permute -> NCCL dispatch -> GEMMs -> NCCL combine per chunk;
  overlap    EP path, MEMFINE_FLAG_OVERLAP: chunk j+-1's exchange on the comm stream under chunk
             j's GEMMs (GEMMs on every SM);
  overlapR   the same with R SMs left to the comm stream (memfine_set_comm_sms).
exposed = (t - t_ep1); the pipeline hides exposed exchange time.  Prints one JSON object as the
last stdout line (NCCL may print its version line first).

  python tools/ep_overlap_bench.py [--config mixtral] [--steps 5] [--warmup 2]
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
    ap.add_argument("--config", default="mixtral", choices=sorted(synth.CONFIGS))
    ap.add_argument("--experts", type=int, default=0, help="local experts (default: all of the config's)")
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--chunks", default="2,4,8")
    ap.add_argument("--comm-sms", default="8,16")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    T = args.tokens or cfg.T
    h, g, k = cfg.h, cfg.g, cfg.k
    E = args.experts or cfg.E
    dev = torch.device("cuda", 0)
    ids_np, w_np = synth.make_routing(T, E, k, rank=0, zipf_s=cfg.zipf_s, placement=cfg.placement)
    x = synth.make_x(T, h).to(dev)
    dy = synth.make_dy(T, h).to(dev)
    ids = torch.from_numpy(ids_np).to(dev)
    w = torch.from_numpy(w_np).to(dev)
    parts = []
    for e in range(E):
        gen = torch.Generator(device=dev).manual_seed(7000 + e)
        parts.append(((torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).bfloat16(),
                      (torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).bfloat16(),
                      (torch.randn(h, g, generator=gen, device=dev) / math.sqrt(g)).bfloat16()))
    wg, wu, wd = (torch.stack([t[i] for t in parts]).contiguous() for i in range(3))
    del parts
    f32 = dict(dtype=torch.float32, device=dev)
    dwg, dwu, dwd = torch.empty(wg.shape, **f32), torch.empty(wu.shape, **f32), torch.empty(wd.shape, **f32)
    y, dx, ds = torch.empty_like(x), torch.empty_like(x), torch.empty(w.shape, **f32)

    def time_variant(mf, C):
        counts_h = mf.route_counts(ids, 8).cpu()
        wsb = max(layer.workspace_bytes(counts_h, mf.dims, C, capi.FWD),
                  layer.workspace_bytes(counts_h, mf.dims, C, capi.BWD))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)

        def step():
            mf.moe_fwd(x, ids, w, wg, wu, wd, C, ws, y=y)
            mf.moe_bwd(dy, x, ids, w, wg, wu, wd, C, ws, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd, dscore=ds)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        assert mf.sync() == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        assert mf.sync() == 0
        out = {"ms_per_step": e0.elapsed_time(e1) / args.steps, "workspace_gb": wsb / 1e9}
        del ws
        return out

    res = {"config": args.config, "tokens": T, "experts": E, "h": h, "g": g, "k": k, "per_C": {}}
    for C in [int(c) for c in args.chunks.split(",")]:
        row = {}
        mf = layer.MemFine(T, h, g, E, k)
        row["ep1"] = time_variant(mf, C)
        mf.close()
        mf = layer.MemFine(T, h, g, E, k, ep_path=True)
        row["serial"] = time_variant(mf, C)
        mf.close()
        mf = layer.MemFine(T, h, g, E, k, ep_path=True, overlap=True)
        row["overlap"] = time_variant(mf, C)
        for r in [int(v) for v in args.comm_sms.split(",") if v]:
            mf.set_comm_sms(r)
            row[f"overlap{r}"] = time_variant(mf, C)
        mf.close()
        base = row["ep1"]["ms_per_step"]
        for v in row.values():
            v["exposed_ms"] = v["ms_per_step"] - base
        res["per_C"][C] = row
        print(json.dumps({C: row}), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
