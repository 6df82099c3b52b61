"""One fwd+bwd step of the Mixtral-size layer in BF16 and in the MXFP8 variant (C=1), for ncu:
per-kernel SM cycles / tensor-pipe activity of the two GEMM families on the same box.

  ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,... python tools/mx_profile.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import capi, layer  # noqa: E402


def main():
    cfg = synth.CONFIGS["mixtral"]
    T, h, g, E, k = cfg.T, cfg.h, cfg.g, cfg.E, cfg.k
    dev = torch.device("cuda", 0)
    x, dy = synth.make_x(T, h).to(dev), synth.make_dy(T, h).to(dev)
    ids_np, w_np = synth.make_routing(T, E, k, zipf_s=cfg.zipf_s, placement=cfg.placement)
    ids, w = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
    wg, wu, wd = (t.to(dev) for t in synth.make_experts(range(E), h, g))
    for mx in (False, True):
        mf = layer.MemFine(T, h, g, E, k, mx=mx)
        counts = mf.route_counts(ids).cpu()
        wsb = max(layer.workspace_bytes(counts, mf.dims, 1, p) for p in (capi.FWD, capi.BWD))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        if mx:
            mf.mx_quantize_weights(wg, wu, wd)
        mf.moe_fwd(x, ids, w, wg, wu, wd, 1, ws)
        mf.moe_bwd(dy, x, ids, w, wg, wu, wd, 1, ws)
        assert mf.sync() == 0
        mf.close()
        del ws


if __name__ == "__main__":
    main()
