"""Shared helpers for the GPU parity tests: seeded problems (synth), the CUDA path through the
C ABI, and the oracle on the same inputs.  Test infrastructure only."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import oracle
import synth
from paper_2511_21431_b200 import capi, layer


@dataclass
class Problem:
    T: int
    h: int
    g: int
    E: int
    k: int
    dtype: torch.dtype
    x: torch.Tensor
    dy: torch.Tensor
    ids: torch.Tensor   # int32 [T,k]
    w: torch.Tensor     # fp32 [T,k]
    wg: torch.Tensor
    wu: torch.Tensor
    wd: torch.Tensor


def make_problem(T, h, g, E, k, dtype=torch.bfloat16, zipf_s=0.0, placement="random", seed=0,
                 ids=None) -> Problem:
    x = synth.make_x(T, h, rank=seed, dtype=dtype)
    dy = synth.make_dy(T, h, rank=seed, dtype=dtype)
    r_ids, w = synth.make_routing(T, E, k, rank=seed, zipf_s=zipf_s, placement=placement)
    if ids is not None:
        r_ids = ids
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    return Problem(T, h, g, E, k, dtype, x, dy, torch.from_numpy(np.ascontiguousarray(r_ids, dtype=np.int32)),
                   torch.from_numpy(w), wg, wu, wd)


def _np_in(t: torch.Tensor, dtype):
    if dtype == torch.bfloat16:
        return t.contiguous().view(torch.int16).numpy().view(np.uint16)
    return t.contiguous().numpy().astype(np.float32)


def oracle_dims(p: Problem):
    return oracle.Dims(T=p.T, h=p.h, g=p.g, E=p.E, k=p.k, in_dtype="bf16" if p.dtype == torch.bfloat16 else "f32")


def oracle_fwd_bwd(p: Problem, C: int = 1):
    d = oracle_dims(p)
    a = [_np_in(t, p.dtype) for t in (p.x, p.dy, p.wg, p.wu, p.wd)]
    ids = p.ids.numpy()
    w = p.w.numpy().astype(np.float64)
    y, cb, pk = oracle.fcda_forward(d, C, a[0], ids, w, a[2], a[3], a[4], D_t=2 if p.dtype == torch.bfloat16 else 4)
    dx, ds, dwg, dwu, dwd, _, _ = oracle.fcda_backward(d, C, a[1], a[0], ids, w, a[2], a[3], a[4])
    return dict(y=y, dx=dx, dscore=ds, dwg=dwg, dwu=dwu, dwd=dwd, meter_peak=int(pk[0]), meter_chunks=cb[0])


def oracle_tokens(p: Problem, toks):
    d = oracle_dims(p)
    a = [_np_in(t, p.dtype) for t in (p.x, p.dy, p.wg, p.wu, p.wd)]
    return oracle.moe_tokens(d, np.asarray(toks, np.int64), a[1], a[0], p.ids.numpy(),
                             p.w.numpy().astype(np.float64), a[2], a[3], a[4])


class GpuRun:
    """Runs route_counts -> plan -> fwd -> bwd on cuda:0 through the C ABI."""

    def __init__(self, p: Problem, dev="cuda:0", **mf_kw):
        self.p = p
        self.dev = dev
        self.mf = layer.MemFine(p.T, p.h, p.g, p.E, p.k, dtype=p.dtype, **mf_kw)
        g = lambda t: t.to(dev).contiguous()
        self.x, self.dy, self.ids, self.w = g(p.x), g(p.dy), g(p.ids), g(p.w)
        self.wg, self.wu, self.wd = g(p.wg), g(p.wu), g(p.wd)

    def counts(self, nsub):
        c = self.mf.route_counts(self.ids, nsub)
        torch.cuda.synchronize()
        return c

    def fwd(self, C, ws_bytes=None, counts_host=None):
        if ws_bytes is None:
            ch = counts_host if counts_host is not None else self.counts(C).cpu()
            ws_bytes = layer.workspace_bytes(ch, self.mf.dims, C, capi.FWD)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.dev)
        y = self.mf.moe_fwd(self.x, self.ids, self.w, self.wg, self.wu, self.wd, C, ws)
        st = self.mf.sync()
        return y, st, self.mf.last_stats(), ws_bytes

    def bwd(self, C, ws_bytes=None, accumulate=False, grads=None):
        if ws_bytes is None:
            ws_bytes = layer.workspace_bytes(self.counts(C).cpu(), self.mf.dims, C, capi.BWD)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.dev)
        kw = {}
        if grads is not None:
            kw = dict(dw_gate=grads[0], dw_up=grads[1], dw_down=grads[2])
        out = self.mf.moe_bwd(self.dy, self.x, self.ids, self.w, self.wg, self.wu, self.wd, C, ws,
                              accumulate_dw=accumulate, **kw)
        st = self.mf.sync()
        return out, st, self.mf.last_stats(), ws_bytes


def rel_err(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    if den == 0.0:
        return float(np.abs(got).max()) if got.size else 0.0
    return float(np.abs(got - ref).max() / den)


def tol(dtype) -> float:
    """BASELINE.json north star: max relative error <= 2e-2 (bf16) / 1e-5 (fp32 mode), read as
    max|got-ref| / max|ref| per tensor (reading R21)."""
    return 2e-2 if dtype == torch.bfloat16 else 1e-5


def tile_covering_tokens(src_of, k, rng, stride=1):
    """Sampled tokens whose copies hit every 128-row m-tile of the expert-major padded layout (src_of:
    each row's copy index i*k + slot, -1 for padding - memfine_debug_rows), chosen greedily: a tile
    already hit by an earlier token's other copy takes no new token.  stride > 1: every stride-th tile
    plus every tile holding an expert segment's last rows (the ragged tails)."""
    src_of = np.asarray(src_of)
    tile_of = {}
    for r in np.nonzero(src_of >= 0)[0]:
        tile_of[int(src_of[r])] = r // 128
    ntiles = (len(src_of) + 127) // 128
    want = set(range(0, ntiles, stride))
    for t in range(ntiles):       # a tile followed by padding ends a segment
        blk = src_of[t * 128:(t + 1) * 128]
        if len(blk) and blk[-1] < 0 and (blk >= 0).any():
            want.add(t)
    covered, toks = set(), []
    for t0 in rng.permutation(np.arange(0, len(src_of), 128)):
        if t0 // 128 in covered or t0 // 128 not in want:
            continue
        live = src_of[t0:t0 + 128]
        live = live[live >= 0]
        if not len(live):
            continue
        tok = int(rng.choice(live)) // k
        toks.append(tok)
        for s in range(k):
            if tok * k + s in tile_of:
                covered.add(tile_of[tok * k + s])
    return np.array(sorted(set(toks)), np.int64)
