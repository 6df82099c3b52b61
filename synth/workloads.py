"""Seeded synthetic workloads shared by the tests, the bench and the oracle.

This module holds NO arithmetic of the method (no dispatch, no expert, no
combine, no memory model): only random inputs with the shapes and structure of
the paper's workloads (recipe: DESIGN.md "Input recipe").

* X ~ N(0, 1), one torch CPU generator per rank (seed 1000 + rank), rounded to bf16.
* dY ~ N(0, 1), seed 3000 + rank, rounded to bf16.
* Expert weights per GLOBAL expert id e (seed 7000 + e), so any rank (and the
  oracle) can rebuild any expert:  W_gate, W_up ~ N(0, 1/h) [g, h];
  W_down ~ N(0, 1/g) [h, g]  (nn.Linear [out, in] layout).
* Routing: per token, top-k DISTINCT experts by Gumbel-top-k over log p_e with
  p_e ∝ pi(e)^(-s); s = 0 uniform, s = 1.2 Zipf.  pi is a seeded permutation of
  1..E shared by all ranks ("zipf-random") or the identity ("zipf-contiguous":
  the hottest experts sit on rank 0 — the Fig. 2 extreme).
  Scores: softmax of the k selected perturbed logits (fp32, sums to 1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class LayerConfig:
    name: str
    E: int          # experts
    k: int          # top-k
    h: int          # hidden
    g: int          # expert FFN size
    T: int          # tokens per GPU
    EP: int         # expert-parallel size the config is quoted at
    zipf_s: float = 0.0
    placement: str = "random"


# BASELINE.json "configs" (Qwen3's tokens/GPU is unstated there; 16K assumed).
CONFIGS = {
    "tiny": LayerConfig("tiny", E=4, k=2, h=64, g=128, T=256, EP=1),
    "mixtral": LayerConfig("mixtral", E=8, k=2, h=4096, g=14336, T=16384, EP=8, zipf_s=1.2),
    "dsv3": LayerConfig("dsv3", E=256, k=8, h=7168, g=2048, T=8192, EP=8, zipf_s=1.2),
    "qwen3": LayerConfig("qwen3", E=64, k=6, h=4096, g=1536, T=16384, EP=8, zipf_s=1.2),
}


def to_bf16_bits(a: torch.Tensor) -> np.ndarray:
    """float tensor -> raw bf16 bits (round-to-nearest-even), as uint16 numpy."""
    return a.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def make_x(T: int, h: int, rank: int = 0, seed: int = 1000, dtype=torch.bfloat16) -> torch.Tensor:
    """[T, h] activations for one rank (CPU tensor; bf16-rounded unless dtype=float32)."""
    gen = torch.Generator().manual_seed(seed + rank)
    return torch.randn(T, h, generator=gen, dtype=torch.float32).to(dtype)


def make_dy(T: int, h: int, rank: int = 0, seed: int = 3000, dtype=torch.bfloat16) -> torch.Tensor:
    gen = torch.Generator().manual_seed(seed + rank)
    return torch.randn(T, h, generator=gen, dtype=torch.float32).to(dtype)


def make_expert(e: int, h: int, g: int, seed: int = 7000, dtype=torch.bfloat16):
    """(W_gate [g,h], W_up [g,h], W_down [h,g]) for global expert e (CPU tensors)."""
    gen = torch.Generator().manual_seed(seed + e)
    wg = torch.randn(g, h, generator=gen) * (1.0 / math.sqrt(h))
    wu = torch.randn(g, h, generator=gen) * (1.0 / math.sqrt(h))
    wd = torch.randn(h, g, generator=gen) * (1.0 / math.sqrt(g))
    return wg.to(dtype), wu.to(dtype), wd.to(dtype)


def make_experts(experts, h: int, g: int, seed: int = 7000, dtype=torch.bfloat16):
    """Stacked weights for the listed global experts: [n,g,h], [n,g,h], [n,h,g].
    Experts are drawn in parallel threads (each from its own seeded generator, so the
    values do not depend on the thread count)."""
    from concurrent.futures import ThreadPoolExecutor
    experts = [int(e) for e in experts]
    n = len(experts)
    wg = torch.empty((n, g, h), dtype=dtype)
    wu = torch.empty((n, g, h), dtype=dtype)
    wd = torch.empty((n, h, g), dtype=dtype)

    def one(i):
        a, b, c = make_expert(experts[i], h, g, seed, dtype)
        wg[i].copy_(a)
        wu[i].copy_(b)
        wd[i].copy_(c)

    with ThreadPoolExecutor(max_workers=min(16, max(1, n))) as ex:
        list(ex.map(one, range(n)))
    return wg, wu, wd


def popularity_rank(E: int, placement: str, seed: int = 4242) -> np.ndarray:
    """pi(e) in 1..E: the popularity rank of each expert (1 = hottest)."""
    if placement == "contiguous":
        return np.arange(1, E + 1, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.permutation(E) + 1).astype(np.float64)


def make_routing(T: int, E: int, k: int, rank: int = 0, zipf_s: float = 0.0,
                 placement: str = "random", seed: int = 2000):
    """(ids int32 [T,k], scores fp32 [T,k]) by Gumbel-top-k over log p_e."""
    assert 1 <= k <= E
    pi = popularity_rank(E, placement)
    logp = -zipf_s * np.log(pi)
    logp = logp - np.log(np.exp(logp).sum())
    rng = np.random.Generator(np.random.PCG64(seed + rank))
    ids = np.empty((T, k), dtype=np.int32)
    scores = np.empty((T, k), dtype=np.float32)
    step = 4096
    for t0 in range(0, T, step):
        t1 = min(T, t0 + step)
        z = logp[None, :] + rng.gumbel(size=(t1 - t0, E))
        top = np.argsort(-z, axis=1, kind="stable")[:, :k]
        zt = np.take_along_axis(z, top, axis=1)
        zt = zt - zt.max(axis=1, keepdims=True)
        p = np.exp(zt)
        p = p / p.sum(axis=1, keepdims=True)
        ids[t0:t1] = top.astype(np.int32)
        scores[t0:t1] = p.astype(np.float32)
    return ids, scores


def local_experts(E: int, EP: int, rank: int):
    """Contiguous expert blocks: rank r hosts [r*E/EP, (r+1)*E/EP) (reading R4)."""
    El = E // EP
    return list(range(rank * El, (rank + 1) * El))
