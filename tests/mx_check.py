"""MXFP8 parity helpers (readings R28, R28b, R28c).  Test infrastructure only.

A quantised code is an integer decided by floating point.  The oracle decides every code on the
EXACT value of its operand; the kernels decide on the value they hold (an fp32 accumulator, or a
bf16-stored intermediate), so near a rounding boundary the two may pick neighbouring codes.  Parity
is therefore checked in two parts:
  1. every GPU decision is VALID: its scale and code are what the format's rule gives for SOME value
     within the kernel's precision window around the exact value (tight for values decided from fp32,
     wider for values decided from bf16 storage);
  2. everything downstream of the decisions matches the oracle FED with the GPU's own decisions
     (oracle.moe_mx(fed=...)), at a tolerance set by the remaining arithmetic (fp32 accumulation,
     bf16 output rounding).
The E4M3 decode table and round-to-nearest-even encode below are torch's float8_e4m3fn conversions,
pinned to the oracle's codec in tests/test_oracle_mx_pins.py."""
from __future__ import annotations

import numpy as np
import torch

E4M3 = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()


def sf_rows(scales_chunked: np.ndarray, rows: int, K: int) -> np.ndarray:
    """Scale bytes from the tcgen05 chunk layout back to [rows][K/32] (memfine.h's formula)."""
    r = np.arange(rows)[:, None]
    b = np.arange(K // 32)[None, :]
    off = ((r // 128) * (K // 128) + b // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + b % 4
    return scales_chunked[off]


def scale_exp(amax: np.ndarray) -> np.ndarray:
    """The scale rule (reading R28): smallest E with amax <= 448 * 2^E, 0 for amax = 0, clamped."""
    amax = np.asarray(amax, np.float64)
    m, ex = np.frexp(amax)                       # amax = m 2^ex, m in [0.5, 1)
    E = np.where(amax > 0, ex - 9 + (2 * m > 1.75), 0)
    return np.clip(E, -127, 127)


def rne_e4m3(s: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even onto the E4M3 grid, saturating at +-448 (values, not codes)."""
    s = np.clip(np.asarray(s, np.float64), -448.0, 448.0)
    return torch.from_numpy(s).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def deq(codes: np.ndarray, E: np.ndarray) -> np.ndarray:
    """codes [n][32k] with block exponents E [n][k] -> values."""
    return E4M3[codes] * np.ldexp(1.0, np.repeat(E, 32, axis=-1))


def windows(gu, da, w_copy, eps_rel, eps_abs=2.0 ** -19):
    """Per-element precision windows of the values the kernels quantise, propagated to first order from the
    exact G, U, dA (oracle return_exact) and the precision the kernel holds them in:
      |delta G| = eps_rel |G| + eps_abs max_row |G|  (likewise U, dA): eps_rel = the storage rounding (bf16:
      2^-8 covers its 2^-9 plus fp32; fp32 registers: ~2^-20), eps_abs = the fp32 GEMM accumulation's
      absolute error, relative to the row's largest value (K-term sums cancel: a small G can carry a large
      relative error).  With f(G) = sig(G)(1 + G(1 - sig(G))) = silu'(G):
      a   = silu(G) U      ->  |U| |f| dG + |silu| dU
      dG  = dA U f(G)      ->  |dA| (|U| |f'| dG + |f| dU) + |U f| ddA
      dU  = dA silu(G)     ->  |dA| |f| dG + |silu| ddA
      a_w = w a            ->  w (|U| |f| dG + |silu| dU)
    plus eps_rel of the value itself (its own rounding before the quantiser).  Near the zero of f
    (G = -1.278) dG cancels - where a fixed relative window fails.  Returns (tol_a, tol_dgu, tol_aw)."""
    g = gu.shape[1] // 2
    G, U = gu[:, :g], gu[:, g:]
    rmax = lambda v: np.abs(v).max(axis=1, keepdims=True)
    dGe = eps_rel * np.abs(G) + eps_abs * rmax(G)
    dUe = eps_rel * np.abs(U) + eps_abs * rmax(U)
    dAe = eps_rel * np.abs(da) + eps_abs * rmax(da)
    sg = 1.0 / (1.0 + np.exp(-G))
    f = sg * (1 + G * (1 - sg))
    fp = sg * (1 - sg) * (2 + G * (1 - 2 * sg))
    silu = G * sg
    a = silu * U
    dG = da * U * f
    dU = da * silu
    ta = np.abs(U) * np.abs(f) * dGe + np.abs(silu) * dUe + eps_rel * np.abs(a)
    tg = np.abs(da) * (np.abs(U) * np.abs(fp) * dGe + np.abs(f) * dUe) + np.abs(U * f) * dAe + eps_rel * np.abs(dG)
    tu = np.abs(da) * np.abs(f) * dGe + np.abs(silu) * dAe + eps_rel * np.abs(dU)
    taw = np.abs(w_copy)[:, None] * ta
    return ta, np.concatenate([tg, tu], axis=1), taw


def check_decisions(v_exact, codes, E_gpu, rel, absb, what=""):
    """v_exact, codes: [nblk, 32] blocks (padding rows 0); E_gpu [nblk].  Each GPU decision must be the
    rule's result for some value within |v' - v| <= rel |v| + absb * amax(block).  Returns the fraction
    of codes that differ from the oracle's own decision on the exact value (reported, not gated)."""
    v = np.asarray(v_exact, np.float64)
    amax = np.abs(v).max(axis=1)
    return check_decisions_tol(v, codes, E_gpu, rel * np.abs(v) + absb * amax[:, None], what)


def check_decisions_tol(v_exact, codes, E_gpu, tol, what=""):
    """As check_decisions with an explicit per-element window tol [nblk, 32]."""
    v = np.asarray(v_exact, np.float64)
    amax = np.abs(v).max(axis=1)
    tol = np.asarray(tol, np.float64) + 2.0 ** -20 * amax[:, None]
    lo_amax = np.maximum(np.abs(v) - tol, 0).max(axis=1)
    # a window reaching 0 admits any smaller scale (the rule's E = 0 for an all-zero block is a convention,
    # not the limit of small amax)
    E_lo = np.where(lo_amax > 0, scale_exp(lo_amax), -127)
    E_hi = scale_exp((np.abs(v) + tol).max(axis=1))
    E_hi = np.where((np.abs(v) + tol).max(axis=1) > 0, E_hi, 0)
    bad_E = (E_gpu < E_lo) | (E_gpu > E_hi)
    assert not bad_E.any(), f"{what}: {int(bad_E.sum())} block scales outside the window"
    sc = np.ldexp(1.0, E_gpu)[:, None]
    lo, hi = rne_e4m3((v - tol) / sc), rne_e4m3((v + tol) / sc)
    got = E4M3[codes]
    bad = ~((got >= lo) & (got <= hi))
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} codes are no rounding of a value in the window; "
                           f"first at {np.argwhere(bad)[0]}: got {got[bad][0]} window [{lo[bad][0]}, {hi[bad][0]}]")
    own = rne_e4m3(v / np.ldexp(1.0, scale_exp(amax))[:, None])
    return float(np.mean(got * sc != own * np.ldexp(1.0, scale_exp(amax))[:, None]))


def rowwise_per_copy(codes, sf, src_of, nq, width):
    """Row-major decisions [rows][width] (blocks along the row) of the expert-major rows -> per copy:
    (dequantised [nq][width], codes [nq][width], E [nq][width/32]); copies without a row stay 0."""
    rows = codes.shape[0]
    E = sf_rows(sf, rows, width).astype(np.int64) - 127
    live = src_of >= 0
    q = src_of[live]
    out_v = np.zeros((nq, width)); out_c = np.zeros((nq, width), np.uint8); out_e = np.zeros((nq, width // 32), np.int64)
    out_c[q] = codes[live]
    out_e[q] = E[live]
    out_v[q] = deq(codes[live], E[live])
    return out_v, out_c, out_e


def colwise_rows(codes_t, sf_t, rows_pad):
    """Columnwise decisions [ncols][Rcap] (blocks of 32 rows along Rcap) -> per ROW [rows_pad][ncols]
    dequantised values, codes and per-row-block exponents E [rows_pad/32][ncols]."""
    ncols, rcap = codes_t.shape
    E = (sf_rows(sf_t, ncols, rcap).astype(np.int64) - 127)[:, :rows_pad // 32]      # [ncols][blocks]
    c = codes_t[:, :rows_pad]
    v = E4M3[c] * np.ldexp(1.0, np.repeat(E, 32, axis=1))
    return v.T.copy(), c.T.copy(), E.T.copy()


def col_blocks(a_rows, rows_pad):
    """[rows_pad][ncols] -> [rows_pad/32 * ncols][32] blocks of 32 rows of one column."""
    nb = rows_pad // 32
    return a_rows.reshape(nb, 32, -1).transpose(0, 2, 1).reshape(-1, 32)
