"""Router step timing at the BASELINE configs' sizes: logits + top-k + softmax forward and
the backward (d_logits, dx, dW_r), CUDA events, one B200.  Prints one JSON object.

  python tools/router_bench.py
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_21431_b200 import layer  # noqa: E402


def timed(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = torch.device("cuda", 0)
    out = {}
    for name in ("mixtral", "dsv3", "qwen3"):
        cfg = synth.CONFIGS[name]
        T, h, E, k = cfg.T, cfg.h, cfg.E, cfg.k
        x = synth.make_x(T, h).to(dev)
        wr = (torch.randn(E, h, device=dev) / math.sqrt(h)).to(torch.bfloat16)
        mf = layer.MemFine(T, h, cfg.g, E, k)
        ids, scores = mf.router_fwd(x, wr)
        ds = torch.randn(T, k, device=dev)
        fwd = timed(lambda: mf.router_fwd(x, wr))
        bwd = timed(lambda: mf.router_bwd(x, wr, ids, scores, ds))
        assert mf.sync() == 0
        flops = 2.0 * T * h * E
        out[name] = {"T": T, "h": h, "E": E, "k": k, "fwd_ms": fwd, "bwd_ms": bwd,
                     "logits_tflops_if_fwd_were_all_gemm": flops / (fwd / 1e3) / 1e12}
        mf.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
