"""Programmatic dependent launch (launch boundaries) changes when kernels start, never
what they compute: the layer's outputs with PDL on (the default) and off (MEMFINE_PDL=0, read once
per process, hence the subprocesses) are bit-identical - Y, dX and every dW - at C = 1 and C = 3 (BF16)
and C = 2 (MXFP8 with MX weight gradients) (run with -m gpu)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from tests.harness import make_problem, GpuRun
out = {}
from paper_2511_21431_b200 import layer
for mode, C in (("bf16", 1), ("bf16", 3), ("mx", 2)):
    p = make_problem(1500, 256, 384, 8, 2, zipf_s=1.2, seed=21)
    run = GpuRun(p)
    if mode == "mx":
        run.mf = layer.MemFine(p.T, p.h, p.g, p.E, p.k, mx=True, mx_wgrad=True)
        run.mf.mx_quantize_weights(run.wg, run.wu, run.wd)
    y, st, _, _ = run.fwd(C)
    assert st == 0
    (dx, dwg, dwu, dwd, ds), st, _, _ = run.bwd(C)
    assert st == 0
    for n, t in zip(("y", "dx", "dwg", "dwu", "dwd"), (y, dx, dwg, dwu, dwd)):
        out[f"{mode}_{n}{C}"] = t.float().cpu().numpy()
np.savez(sys.argv[2], **out)
'''


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_pdl_on_off_bit_identical(tmp_path):
    res = {}
    for v in ("1", "0"):
        f = tmp_path / f"out_{v}.npz"
        env = dict(os.environ, MEMFINE_PDL=v)
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(f)], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[v] = np.load(f)
    for k in res["1"].files:
        assert np.array_equal(res["1"][k], res["0"][k]), k
