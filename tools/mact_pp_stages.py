"""MACT per pipeline stage: Eq. 2's m_g = v p + p - 2 r_pp - 1
micro-batches of activations live on stage r_pp, so s'_max (Eq. 8) - and with it C (Eq. 9 + bins) -
differs by stage.  Host planner only (memfine_plan on host counts; no GPU needed).

Workload: the DeepSeek-V3-style layer at EP = 8 (256 experts, top-8, 8K tokens per rank, Zipf(1.2)
routing with the hot experts on rank 0), p = 4 stages, v = 1 and 2, a 180 GB GPU whose static memory
leaves `--act-gb` for activations.  Prints one JSON object (commit it under profiles/).

  python tools/mact_pp_stages.py [--act-gb 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import capi, layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--act-gb", type=float, default=20.0)
    ap.add_argument("--placement", default="contiguous")
    args = ap.parse_args()
    T, h, g, E, k, EP = 8192, 7168, 2048, 256, 8, 8
    # counts [EP][8][E]: copies of each rank's sub-chunk j (tokens [jT/8, (j+1)T/8)) per expert
    counts = np.zeros((EP, 8, E), np.int32)
    for r in range(EP):
        ids = synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement=args.placement)[0]
        for j in range(8):
            counts[r, j] = np.bincount(ids[j * T // 8:(j + 1) * T // 8].ravel(), minlength=E)
    ct = torch.from_numpy(counts)
    cap = 180 * 10**9
    static = cap - int(args.act_gb * 1e9)
    out = {"workload": f"dsv3-style layer, EP=8, 8K tokens/rank, Zipf(1.2) {args.placement}", "gpu_gb": 180,
           "activation_budget_gb": args.act_gb, "stages": {}}
    for v in (1, 2):
        p = 4
        rows = []
        for r in range(p):
            mg = layer.m_g(v, p, r)
            dims = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=0)
            info = layer.plan(ct, dims, capi.make_budget(cap, 1.0, static, 0, m_g=mg))
            rows.append({"r_pp": r, "m_g": mg, "C": info["C"], "c_theory": info["c_theory"],
                         "s_prime_max": info["s_prime_max"], "s_dd_max": info["s_dd_max"],
                         "clamped": info["clamped"], "feasible": info["feasible"], "status": info["status"]})
        out["stages"][f"p{p}_v{v}"] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()
