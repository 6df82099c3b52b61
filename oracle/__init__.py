"""CPU oracle for the MemFine chunked MoE layer (arXiv 2511.21431).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2511_21431_b200``, ``libmemfine.so``) never
imports, links or calls it; the two share no code.  Inputs come from
``synth.workloads`` (seeded generators, no method arithmetic).

The arithmetic lives in ``memfine_oracle.c`` (plain C, fp64, fixed loop order);
this module compiles it with gcc and marshals numpy arrays through ctypes.
Every entry point cites the passage of PAPER.md it follows (see the C file).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "memfine_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-Wall", "-Wno-unused-function", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Dims(C.Structure):
    _fields_ = [("T", C.c_int64), ("h", C.c_int32), ("g", C.c_int32), ("E", C.c_int32),
                ("k", C.c_int32), ("EP", C.c_int32), ("in_dtype", C.c_int32)]


class _ActCfg(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("m_g", "t", "c", "D_t", "b", "s", "h", "a", "h_d", "k_a", "e_n", "g_e")]


class _Budget(C.Structure):
    _fields_ = [("budget_bytes", C.c_uint64), ("static_bytes", C.c_uint64),
                ("other_act_bytes", C.c_uint64), ("m_g", C.c_int64), ("tp", C.c_int64),
                ("cp", C.c_int64), ("micro_batch", C.c_int64), ("D_t", C.c_int64),
                ("bins", C.POINTER(C.c_int32)), ("nbins", C.c_int32), ("rule", C.c_int32)]


class _PlanOut(C.Structure):
    _fields_ = [("C", C.c_int32), ("c_theory", C.c_int32), ("clamped", C.c_int32),
                ("feasible", C.c_int32), ("hot_rank", C.c_int32), ("exact_peak", C.c_int32),
                ("s_dd_max", C.c_int64), ("s_prime_max", C.c_int64), ("s_chunk_max", C.c_int64),
                ("predicted_peak_bytes", C.c_uint64)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_chunk_begin.restype = C.c_int64
        _lib.oracle_chunk_begin.argtypes = [C.c_int64, C.c_int32, C.c_int32]
        _lib.oracle_route_counts.restype = C.c_int64
        _lib.oracle_act_bytes_eq2.restype = C.c_uint64
        _lib.oracle_s_prime_max_eq8.restype = C.c_int64
        _lib.oracle_s_prime_max_eq8.argtypes = [C.POINTER(_ActCfg), C.c_uint64, C.c_uint64]
        _lib.oracle_act_bytes_eq2.argtypes = [C.POINTER(_ActCfg), C.c_int64]
        _lib.oracle_plan.restype = C.c_int32
        _lib.oracle_dispatch_order.restype = C.c_int64
        _lib.oracle_moe_backward.restype = C.c_int32
        _lib.oracle_moe_fcda_forward.restype = C.c_int32
        _lib.oracle_moe_fcda_backward.restype = C.c_int32
        _lib.oracle_e4m3_decode.restype = C.c_double
        _lib.oracle_e4m3_decode.argtypes = [C.c_uint8]
        _lib.oracle_e4m3_encode.restype = C.c_uint8
        _lib.oracle_e4m3_encode.argtypes = [C.c_double]
        _lib.oracle_mx_scale_exp.restype = C.c_int32
        _lib.oracle_mx_scale_exp.argtypes = [C.c_double]
        _lib.oracle_moe_mx.restype = C.c_int32
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Dims:
    T: int      # tokens per rank
    h: int
    g: int
    E: int
    k: int
    EP: int = 1
    in_dtype: str = "f32"   # "f32" | "bf16" (raw uint16 bits) | "f64"

    def c(self):
        code = {"f32": 0, "bf16": 1, "f64": 2}[self.in_dtype]
        return _Dims(self.T, self.h, self.g, self.E, self.k, self.EP, code)


_NP = {"f32": np.float32, "bf16": np.uint16, "f64": np.float64}


def _wt(a, dt):
    """Activations / weights as the C side expects (float32, raw bf16 bits, or float64)."""
    a = np.ascontiguousarray(a)
    assert a.dtype == _NP[dt], f"expected {_NP[dt]} for in_dtype={dt}, got {a.dtype}"
    return a


def chunk_begin(T: int, C_: int, j: int) -> int:
    return int(lib().oracle_chunk_begin(T, C_, j))


def route_counts(d: Dims, ids: np.ndarray, nsub: int):
    """counts[nsub][E] for one rank's ids [T][k]; returns (counts, n_bad)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    counts = np.zeros((nsub, d.E), dtype=np.int64)
    bad = lib().oracle_route_counts(C.byref(d.c()), C.c_int32(nsub), _p(ids), _p(counts))
    return counts, int(bad)


def act_bytes_eq2(cfg: dict, s_prime: int) -> int:
    q = _ActCfg(**cfg)
    return int(lib().oracle_act_bytes_eq2(C.byref(q), s_prime))


def act_table2_rows(cfg: dict, s_prime: int) -> np.ndarray:
    q = _ActCfg(**cfg)
    rows = np.zeros(14, dtype=np.int64)
    lib().oracle_act_table2_rows(C.byref(q), C.c_int64(s_prime), _p(rows))
    return rows


def s_prime_max_eq8(cfg: dict, budget: int, static: int) -> int:
    q = _ActCfg(**cfg)
    return int(lib().oracle_s_prime_max_eq8(C.byref(q), budget, static))


def plan(counts: np.ndarray, d: Dims, *, budget_bytes: int, static_bytes: int = 0,
         other_act_bytes: int = 0, m_g: int = 1, tp: int = 1, cp: int = 1, micro_batch: int = 1,
         D_t: int = 2, bins=(1, 2, 4, 8), rule: int = 0):
    """MACT plan; counts [EP][nsub][E].  Returns (status, dict)."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    assert counts.ndim == 3
    b = np.ascontiguousarray(bins, dtype=np.int32)
    bud = _Budget(budget_bytes, static_bytes, other_act_bytes, m_g, tp, cp, micro_batch, D_t,
                  b.ctypes.data_as(C.POINTER(C.c_int32)), len(b), rule)
    out = _PlanOut()
    st = lib().oracle_plan(_p(counts), C.c_int32(counts.shape[1]), C.byref(d.c()), C.byref(bud),
                           C.byref(out))
    return int(st), {f: getattr(out, f) for f, _ in _PlanOut._fields_}


def dispatch_order(d: Dims, ids_all: np.ndarray, rank: int, C_: int, j: int) -> np.ndarray:
    """Canonical (expert, src, token, slot) order; entries src*T*k + i*k + slot."""
    ids_all = np.ascontiguousarray(ids_all, dtype=np.int32)
    cap = max(1, ids_all.size)
    perm = np.zeros(cap, dtype=np.int64)
    n = lib().oracle_dispatch_order(C.byref(d.c()), _p(ids_all), C.c_int32(rank), C.c_int32(C_),
                                    C.c_int32(j), _p(perm), C.c_int64(cap))
    assert n >= 0
    return perm[:n].copy()


def moe_forward(d: Dims, x, ids, w, wg, wu, wd) -> np.ndarray:
    """Eq. 4 per-token definition.  x [EP*T, h]; ids/w [EP*T, k]; weights all E experts."""
    bf = d.in_dtype
    x, wg, wu, wd = (_wt(a, bf) for a in (x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    y = np.zeros((d.EP * d.T, d.h), dtype=np.float64)
    lib().oracle_moe_forward(C.byref(d.c()), _p(x), _p(ids), _p(w), _p(wg), _p(wu), _p(wd), _p(y))
    return y


def moe_backward(d: Dims, dy, x, ids, w, wg, wu, wd):
    """Eq. 5, unchunked.  Returns dx, dscore, dwg, dwu, dwd (fp64)."""
    bf = d.in_dtype
    dy, x, wg, wu, wd = (_wt(a, bf) for a in (dy, x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = d.EP * d.T
    dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    dwg = np.zeros((d.E, d.g, d.h)); dwu = np.zeros((d.E, d.g, d.h)); dwd = np.zeros((d.E, d.h, d.g))
    st = lib().oracle_moe_backward(C.byref(d.c()), _p(dy), _p(x), _p(ids), _p(w), _p(wg), _p(wu),
                                   _p(wd), _p(dx), _p(ds), _p(dwg), _p(dwu), _p(dwd))
    assert st == 0
    return dx, ds, dwg, dwu, dwd


def moe_backward_experts(d: Dims, dy, x, ids, w, wg, wu, wd, sel):
    """Eq. 5 with the weight gradients of the experts `sel` only: dx, dscore, dwg, dwu, dwd
    ([len(sel)][g][h] / [len(sel)][h][g]) - the rows / expert slices of moe_backward."""
    bf = d.in_dtype
    dy, x, wg, wu, wd = (_wt(a, bf) for a in (dy, x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    n, m = d.EP * d.T, len(sel)
    dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    dwg = np.zeros((m, d.g, d.h)); dwu = np.zeros((m, d.g, d.h)); dwd = np.zeros((m, d.h, d.g))
    st = lib().oracle_moe_backward_experts(C.byref(d.c()), _p(dy), _p(x), _p(ids), _p(w), _p(wg), _p(wu), _p(wd),
                                           C.c_int32(m), _p(sel), _p(dx), _p(ds), _p(dwg), _p(dwu), _p(dwd))
    assert st == 0
    return dx, ds, dwg, dwu, dwd


def fcda_forward(d: Dims, C_: int, x, ids, w, wg, wu, wd, D_t: int = 2):
    """Eq. 6 chunk loop.  Returns y, chunk_bytes [EP][C], peak [EP] (paper meter)."""
    bf = d.in_dtype
    x, wg, wu, wd = (_wt(a, bf) for a in (x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    y = np.zeros((d.EP * d.T, d.h))
    cb = np.zeros((d.EP, C_), dtype=np.uint64); pk = np.zeros(d.EP, dtype=np.uint64)
    st = lib().oracle_moe_fcda_forward(C.byref(d.c()), C.c_int32(C_), _p(x), _p(ids), _p(w), _p(wg),
                                       _p(wu), _p(wd), _p(y), C.c_int64(D_t), _p(cb), _p(pk))
    assert st == 0
    return y, cb, pk


def fcda_backward(d: Dims, C_: int, dy, x, ids, w, wg, wu, wd, D_t: int = 2):
    """Eq. 7 chunked recompute backward.  Returns dx, dscore, dwg, dwu, dwd, chunk_bytes, peak."""
    bf = d.in_dtype
    dy, x, wg, wu, wd = (_wt(a, bf) for a in (dy, x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = d.EP * d.T
    dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    dwg = np.zeros((d.E, d.g, d.h)); dwu = np.zeros((d.E, d.g, d.h)); dwd = np.zeros((d.E, d.h, d.g))
    cb = np.zeros((d.EP, C_), dtype=np.uint64); pk = np.zeros(d.EP, dtype=np.uint64)
    st = lib().oracle_moe_fcda_backward(C.byref(d.c()), C.c_int32(C_), _p(dy), _p(x), _p(ids), _p(w),
                                        _p(wg), _p(wu), _p(wd), _p(dx), _p(ds), _p(dwg), _p(dwu),
                                        _p(dwd), C.c_int64(D_t), _p(cb), _p(pk))
    assert st == 0
    return dx, ds, dwg, dwu, dwd, cb, pk


def moe_tokens(d: Dims, toks, dy, x, ids, w, wg, wu, wd):
    """y, dx, dscore for the listed global token indices only (sampled full-size checks)."""
    bf = d.in_dtype
    dy, x, wg, wu, wd = (_wt(a, bf) for a in (dy, x, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    toks = np.ascontiguousarray(toks, dtype=np.int64)
    n = len(toks)
    y = np.zeros((n, d.h)); dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    lib().oracle_moe_tokens(C.byref(d.c()), C.c_int64(n), _p(toks), _p(dy), _p(x), _p(ids), _p(w),
                            _p(wg), _p(wu), _p(wd), _p(y), _p(dx), _p(ds))
    return y, dx, ds


def router_forward(d: Dims, x, wr):
    """Router: logits = x W_r^T, top-k (ties -> lower id), softmax over the k selected."""
    x, wr = _wt(x, d.in_dtype), _wt(wr, d.in_dtype)
    n = x.shape[0]
    logits = np.zeros((n, d.E))
    ids = np.zeros((n, d.k), np.int32)
    scores = np.zeros((n, d.k))
    lib().oracle_router_forward(C.byref(d.c()), C.c_int64(n), _p(x), _p(wr), _p(logits), _p(ids), _p(scores))
    return logits, ids, scores


def router_backward(d: Dims, x, wr, ids, scores, dscore):
    """d_logits (softmax Jacobian on the selected slots), dx = d_logits W_r, dW_r = d_logits^T x."""
    x, wr = _wt(x, d.in_dtype), _wt(wr, d.in_dtype)
    n = x.shape[0]
    ids = np.ascontiguousarray(ids, np.int32)
    scores = np.ascontiguousarray(scores, np.float64)
    dscore = np.ascontiguousarray(dscore, np.float64)
    dx = np.zeros((n, d.h))
    dwr = np.zeros((d.E, d.h))
    lib().oracle_router_backward(C.byref(d.c()), C.c_int64(n), _p(x), _p(wr), _p(ids), _p(scores), _p(dscore),
                                 _p(dx), _p(dwr))
    return dx, dwr


# ---------------------------------------------------------------- MXFP8 variant (reading R28)
def e4m3_decode(code: int) -> float:
    return float(lib().oracle_e4m3_decode(code))


def e4m3_encode(v: float) -> int:
    """Round-to-nearest-even onto the FP8 E4M3 grid, saturating at +-448."""
    return int(lib().oracle_e4m3_encode(float(v)))


def mx_scale_exp(amax: float) -> int:
    """Smallest E with amax <= 448 * 2^E (E = 0 for amax = 0), clamped to [-127, 127]."""
    return int(lib().oracle_mx_scale_exp(float(amax)))


def mx_quantize(v, in_dtype: str = "f32"):
    """Blocks of 32 consecutive values of v (flattened): (E4M3 codes uint8 [n], scale codes E+127 uint8 [n/32])."""
    v = _wt(v, in_dtype)
    n = v.size
    assert n % 32 == 0
    codes = np.zeros(n, np.uint8)
    scales = np.zeros(n // 32, np.uint8)
    lib().oracle_mx_quantize(_p(v), C.c_int32({"f32": 0, "bf16": 1, "f64": 2}[in_dtype]), C.c_int64(n),
                             _p(codes), _p(scales))
    return codes.reshape(v.shape), scales


def mx_weights(d: Dims, wg, wu, wd, mode: int = 1):
    """Dequantised weights (fp64): gate/up rows along h, down rows along g, gate/up columns along g
    (the five weight operand layouts of the MX variant)."""
    wg, wu, wd = (_wt(a, d.in_dtype) for a in (wg, wu, wd))
    out = [np.zeros((d.E, d.g, d.h)), np.zeros((d.E, d.g, d.h)), np.zeros((d.E, d.h, d.g)),
           np.zeros((d.E, d.g, d.h)), np.zeros((d.E, d.g, d.h))]
    arr = (C.POINTER(C.c_double) * 5)(*[a.ctypes.data_as(C.POINTER(C.c_double)) for a in out])
    lib().oracle_mx_weights(C.byref(d.c()), C.c_int32(mode), _p(wg), _p(wu), _p(wd), arr)
    return out


class _MxFed(C.Structure):
    _fields_ = [("a_q", C.c_void_p), ("dgu_q", C.c_void_p), ("dgu_col_q", C.c_void_p), ("aw_col_q", C.c_void_p)]


class _MxExact(C.Structure):
    _fields_ = [("a", C.c_void_p), ("dgu", C.c_void_p), ("gu", C.c_void_p), ("da", C.c_void_p)]


def _mx_exact(n, g, with_dy):
    arr = {"a": np.zeros((n, g)), "gu": np.zeros((n, 2 * g)),
           "dgu": np.zeros((n, 2 * g)) if with_dy else None, "da": np.zeros((n, g)) if with_dy else None}
    ptr = lambda v: v.ctypes.data if v is not None else None
    return arr, _MxExact(ptr(arr["a"]), ptr(arr["dgu"]), ptr(arr["gu"]), ptr(arr["da"]))


def _mx_fed(fed, nq, g):
    """fed: None or a dict with any of a_q [nq][g], dgu_q [nq][2g], dgu_col_q [nq][2g], aw_col_q [nq][g]
    (another implementation's decisions, dequantised per copy).  Returns (struct or None, keep-alive)."""
    if not fed:
        return None, []
    widths = {"a_q": g, "dgu_q": 2 * g, "dgu_col_q": 2 * g, "aw_col_q": g}
    keep, ptrs = [], {}
    for key, wdt in widths.items():
        v = fed.get(key)
        if v is None:
            ptrs[key] = None
            continue
        v = np.ascontiguousarray(v, dtype=np.float64).reshape(nq, wdt)
        keep.append(v)
        ptrs[key] = v.ctypes.data
    return _MxFed(**ptrs), keep


def moe_mx(d: Dims, x, ids, w, wq, dy=None, mode: int = 1, wd=None, wgrad_C: int = 0, fed=None,
           return_exact: bool = False):
    """MX variant of the layer (mode 0: quantisers off).  wq from mx_weights(mode); wd the unquantised
    W_down (needed with dy: the dA step keeps BF16 operands).  wgrad_C = 0: weight gradients from
    unquantised operands; wgrad_C = C >= 1: MXFP8 weight gradients (operand columns quantised along
    each expert's copies in each of the C chunks; reading R28c).  Every code is decided on
    the exact value; fed (see _mx_fed) replaces those decisions by another implementation's.
    Returns y, or (y, dx, dscore, dwg, dwu, dwd) when dy is given; with return_exact a further dict
    {"a": [nq][g], "dgu": [nq][2g], "gu": [nq][2g], "da": [nq][g]} of the exact values per copy
    (a, dG || dU: what the quantisers act on; G || U, dA: what those are functions of)."""
    x = _wt(x, d.in_dtype)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = d.EP * d.T
    nq = n * d.k
    y = np.zeros((n, d.h))
    arr = (C.POINTER(C.c_double) * 5)(*[np.ascontiguousarray(a).ctypes.data_as(C.POINTER(C.c_double)) for a in wq])
    fs, keep = _mx_fed(fed, nq, d.g)
    exact, ex = _mx_exact(nq, d.g, dy is not None) if return_exact else (None, None)
    fp = C.byref(fs) if fs is not None else None
    ep = C.byref(ex) if ex is not None else None
    if dy is None:
        st = lib().oracle_moe_mx(C.byref(d.c()), C.c_int32(mode), None, _p(x), _p(ids), _p(w), arr, None, _p(y),
                                 None, None, None, None, None, C.c_int32(0), fp, ep)
        assert st == 0
        del keep
        return (y, exact) if return_exact else y
    dy = _wt(dy, d.in_dtype)
    wd = _wt(wd, d.in_dtype)
    dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    dwg = np.zeros((d.E, d.g, d.h)); dwu = np.zeros((d.E, d.g, d.h)); dwd = np.zeros((d.E, d.h, d.g))
    st = lib().oracle_moe_mx(C.byref(d.c()), C.c_int32(mode), _p(dy), _p(x), _p(ids), _p(w), arr, _p(wd), _p(y), _p(dx),
                             _p(ds), _p(dwg), _p(dwu), _p(dwd), C.c_int32(wgrad_C), fp, ep)
    assert st == 0
    del keep
    out = (y, dx, ds, dwg, dwu, dwd)
    return out + (exact,) if return_exact else out


def moe_mx_tokens(d: Dims, toks, x, dy, ids, w, wg, wu, wd, mode: int = 1, fed=None, return_exact: bool = False):
    """MX layer on a token subset (full-size sampled parity): (y, dx, dscore) rows of toks, as
    moe_mx would give them; weights are quantised one expert at a time.  fed / return_exact as in
    moe_mx, indexed by the sampled copy p*k + slot (a_q and dgu_q only)."""
    toks = np.ascontiguousarray(toks, dtype=np.int64)
    x, dy, wg, wu, wd = (_wt(a, d.in_dtype) for a in (x, dy, wg, wu, wd))
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = len(toks)
    y = np.zeros((n, d.h)); dx = np.zeros((n, d.h)); ds = np.zeros((n, d.k))
    fs, keep = _mx_fed(fed, n * d.k, d.g)
    exact, ex = _mx_exact(n * d.k, d.g, True) if return_exact else (None, None)
    st = lib().oracle_moe_mx_tokens(C.byref(d.c()), C.c_int32(mode), C.c_int64(n), _p(toks), _p(dy), _p(x), _p(ids),
                                    _p(w), _p(wg), _p(wu), _p(wd), _p(y), _p(dx), _p(ds),
                                    C.byref(fs) if fs is not None else None, C.byref(ex) if ex is not None else None)
    assert st == 0
    del keep
    return (y, dx, ds, exact) if return_exact else (y, dx, ds)


def m_g(v: int, p: int, r_pp: int, full_recompute: bool = False) -> int:
    """Eq. 2's m_g: v p + p - 2 r_pp - 1, or 1 under full recomputation."""
    return int(lib().oracle_m_g(C.c_int32(v), C.c_int32(p), C.c_int32(r_pp), C.c_int32(int(bool(full_recompute)))))
