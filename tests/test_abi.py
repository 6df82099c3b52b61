"""The C-ABI library on CPU (no GPU calls): it loads, exports every symbol include/memfine.h
declares, validates arguments, and its host MACT planner equals the oracle bit for bit."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

import oracle
from paper_2511_21431_b200 import capi, layer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    return capi.lib()


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "memfine.h")).read()
    declared = set(re.findall(r"\b(memfine_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(capi.SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.memfine_abi_version() == 2
    for s in range(8):
        assert capi.status_str(s)


def test_create_fails_loudly_without_gpu(L):
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = layer.make_dims(16, 64, 64, 4, 2)
    h = C.c_void_p()
    assert L.memfine_create(C.byref(d), None, C.byref(h)) == capi.ERR_CUDA


def test_argument_validation(L):
    d = layer.make_dims(16, 64, 64, 4, 2)
    counts = torch.zeros((1, 8, 4), dtype=torch.int32)
    b = capi.make_budget(10**9)
    assert layer.plan(counts, d, b)["status"] == 0
    # the default rule EXACT needs every bin to divide the sub-chunk count; EQ9 does not
    c1 = torch.zeros((1, 1, 4), dtype=torch.int32)
    assert layer.plan(c1, d, b)["status"] == capi.ERR_INVALID_ARG
    assert layer.plan(c1, d, capi.make_budget(10**9, rule=capi.RULE_EQ9))["status"] == 0
    bad = layer.make_dims(16, 60, 64, 4, 2)       # hidden % 64
    assert layer.plan(counts, bad, b)["status"] == capi.ERR_INVALID_ARG
    assert layer.plan(counts, d, capi.make_budget(10**9, bins=(2, 2)))["status"] == capi.ERR_INVALID_ARG
    assert layer.plan(counts, d, capi.make_budget(10**9, bins=(0, 2)))["status"] == capi.ERR_INVALID_ARG
    assert layer.plan(counts, d, capi.make_budget(10**9, alpha=0.0))["status"] == capi.ERR_INVALID_ARG
    assert layer.plan(counts, d, capi.make_budget(10**9, static_bytes=2 * 10**9))["status"] == capi.ERR_INFEASIBLE
    ep = layer.make_dims(16, 64, 64, 6, 2, ep_size=4)  # E % EP
    assert layer.plan(torch.zeros((4, 1, 6), dtype=torch.int32), ep, b)["status"] == capi.ERR_INVALID_ARG
    out = C.c_uint64()
    assert L.memfine_workspace_bytes(None, 0, C.byref(d), 0, 0, C.byref(out)) == capi.ERR_INVALID_ARG
    assert L.memfine_workspace_bytes(None, 0, C.byref(d), 1, 7, C.byref(out)) == capi.ERR_INVALID_ARG


def _both(counts_np, h, g, E, EP, budget, static, other, bins, rule, D_t=2, m_g=1):
    """rule: the oracle's numbering (0 EQ9, 1 EXACT)."""
    d = layer.make_dims(1, h, g, E, 1, ep_size=EP, dtype=torch.bfloat16 if D_t == 2 else torch.float32)
    lib_rule = capi.RULE_EQ9 if rule == 0 else capi.RULE_EXACT
    got = layer.plan(torch.from_numpy(counts_np.astype(np.int32)), d,
                     capi.make_budget(budget, 1.0, static, other, m_g=m_g, bins=bins, rule=lib_rule))
    od = oracle.Dims(T=1, h=h, g=g, E=E, k=1, EP=EP)
    st, ref = oracle.plan(counts_np.astype(np.int64), od, budget_bytes=budget, static_bytes=static,
                          other_act_bytes=other, m_g=m_g, D_t=D_t, bins=bins, rule=rule)
    return got, st, ref


def test_host_plan_matches_oracle_spec_vectors():
    """SPEC.md:316-336 vectors through the library's host planner (h=4, g=8 -> beta=48 B)."""
    for sdd, c_th, C_, clamped in ((156, 1, 1, 0), (157, 2, 2, 0), (400, 3, 4, 0), (9 * 156, 9, 8, 1), (0, 1, 1, 0)):
        counts = np.zeros((1, 1, 2), np.int64)
        counts[0, 0, 0] = sdd
        # h and g must be multiples of 64 for the library; scale the toy by 16 and the budget by 16
        got, st, ref = _both(counts, 64, 128, 2, 1, 16 * 10000, 16 * 2000, 16 * 512, (1, 2, 4, 8), 0)
        assert got["status"] == st == 0
        assert got["s_prime_max"] == ref["s_prime_max"] == 156
        assert (got["c_theory"], got["C"], got["clamped"]) == (c_th, C_, clamped)


def test_host_plan_matches_oracle_random():
    """10^4 random count tensors (EP, bins, rule, budgets): identical outputs, bit for bit."""
    rng = np.random.default_rng(123)
    fields = ("C", "c_theory", "clamped", "feasible", "hot_rank", "exact_peak", "s_dd_max", "s_prime_max",
              "s_chunk_max", "predicted_peak_bytes")
    for it in range(10000):
        EP = int(rng.choice([1, 2, 4, 8]))
        E = EP * int(rng.integers(1, 5))
        nsub = int(rng.choice([1, 2, 4, 8]))
        h, g = 64 * int(rng.integers(1, 4)), 64 * int(rng.integers(1, 4))
        counts = rng.integers(0, 3000, size=(EP, nsub, E))
        beta = 2 * (2 * h + 2 * g)
        budget = int(rng.integers(1, 40)) * beta * 1000 + int(rng.integers(0, beta))
        static = int(rng.integers(0, budget // 2 + 1))
        other = int(rng.integers(0, budget // 4 + 1))
        bins = [(1, 2, 4, 8), (1, 2, 4), (2, 8), (1, 3, 5)][it % 4]
        rule = int(rng.integers(0, 2))
        if rule == 1 and any(nsub % b for b in bins):
            rule = 0
        got, st, ref = _both(counts, h, g, E, EP, budget, static, other, bins, rule)
        assert got["status"] == st, (it, got, st)
        if st == 0:
            for f in fields:
                assert got[f] == ref[f], (it, f, got[f], ref[f])


def test_workspace_bytes_formula_and_scaling():
    """Workspace grows with the hottest chunk's padded rows; chunking shrinks it ~1/C."""
    T, h, g, E, k = 4096, 256, 512, 8, 2
    d = layer.make_dims(T, h, g, E, k)
    rng = np.random.default_rng(0)
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    od = oracle.Dims(T=T, h=h, g=g, E=E, k=k)
    counts, _ = oracle.route_counts(od, ids, 8)
    ct = torch.from_numpy(counts.astype(np.int32))[None]
    ws = {C_: layer.workspace_bytes(ct, d, C_, capi.FWD) for C_ in (1, 2, 4, 8)}
    assert ws[1] > ws[2] > ws[4] > ws[8]
    row_bytes = 4 + 4 + 2 * (h + g + h)
    for C_ in (1, 2, 4, 8):
        per = 8 // C_
        pad = max(int(sum(-(-int(counts[j * per:(j + 1) * per, e].sum()) // 128) * 128 for e in range(E)))
                  for j in range(C_))
        meta = ws[C_] - pad * row_bytes
        assert 0 < meta < 2 * 1024 * 1024
    wsb = {C_: layer.workspace_bytes(ct, d, C_, capi.BWD) for C_ in (1, 8)}
    assert wsb[1] > ws[1] and wsb[8] < wsb[1] / 4


def test_workspace_bytes_overlap_slots():
    """MEMFINE_FLAG_OVERLAP: identical bytes where it does not apply (EP = 1, C = 1); with EP > 1
    and C > 1 exactly two slots of the exchanged rows - forward per-row bytes 2(16+8+2h) + 2g
    (o over X_disp), backward 2(16+12+4h) + 6g - on top of the hottest chunk's padded rows."""
    rng = np.random.default_rng(11)
    T, h, g, E, k, EP = 1024, 256, 512, 8, 2, 2
    ids = [np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32) for _ in range(EP)]
    od = oracle.Dims(T=T, h=h, g=g, E=E, k=k)
    counts = np.stack([oracle.route_counts(od, i, 8)[0] for i in ids]).astype(np.int32)
    ct = torch.from_numpy(counts)
    ct1 = ct[:1].contiguous()
    for C_ in (1, 2, 4):
        for pass_ in (capi.FWD, capi.BWD):
            # EP = 1: the flag is ignored
            a = layer.workspace_bytes(ct1, layer.make_dims(T, h, g, E, k), C_, pass_)
            b = layer.workspace_bytes(ct1, layer.make_dims(T, h, g, E, k, overlap=True), C_, pass_)
            assert a == b
            for r in range(EP):
                d0 = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=r)
                d1 = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=r, overlap=True)
                w0 = layer.workspace_bytes(ct, d0, C_, pass_)
                w1 = layer.workspace_bytes(ct, d1, C_, pass_)
                if C_ == 1:
                    assert w0 == w1
                    continue
                El, per = E // EP, 8 // C_
                pad = max(sum(-(-int(counts[:, j * per:(j + 1) * per, e].sum()) // 128) * 128
                              for e in range(r * El, (r + 1) * El)) for j in range(C_))
                rb0 = 16 + 8 + 2 * (2 * h + g) if pass_ == capi.FWD else 16 + 12 + 2 * (2 * h + 3 * g)
                rb1 = 2 * (16 + 8 + 2 * h) + 2 * g if pass_ == capi.FWD else 2 * (16 + 12 + 4 * h) + 6 * g
                meta0, meta1 = w0 - pad * rb0, w1 - pad * rb1
                # two copies of the metadata + send staging (256-byte aligned pieces)
                assert 0 < meta0 < meta1 <= 2 * meta0 + 256, (C_, pass_, r, meta0, meta1)
    out = C.c_uint64()
    bad = layer.make_dims(T, h, g, E, k)
    bad.flags = 1 << 10   # unknown flag
    assert capi.lib().memfine_workspace_bytes(None, 0, C.byref(bad), 1, 0, C.byref(out)) == capi.ERR_INVALID_ARG
    bad = layer.make_dims(T, h, g, E, k, mx_wgrad=True)             # MX_WGRAD needs the MXFP8 dtype
    assert capi.lib().memfine_workspace_bytes(None, 0, C.byref(bad), 1, 0, C.byref(out)) == capi.ERR_INVALID_ARG
    bad = layer.make_dims(T, h, g, E, k, ep_size=2, ep_path=True)   # EP_PATH is for ep_size == 1
    assert capi.lib().memfine_workspace_bytes(None, 0, C.byref(bad), 1, 0, C.byref(out)) == capi.ERR_INVALID_ARG
    # EP_PATH at ep_size == 1: the EP layout (send staging, row addresses), overlap slots apply
    for pass_ in (capi.FWD, capi.BWD):
        e1 = layer.workspace_bytes(ct1, layer.make_dims(T, h, g, E, k), 2, pass_)
        ep = layer.workspace_bytes(ct1, layer.make_dims(T, h, g, E, k, ep_path=True), 2, pass_)
        epo = layer.workspace_bytes(ct1, layer.make_dims(T, h, g, E, k, ep_path=True, overlap=True), 2, pass_)
        assert e1 < ep < epo


def test_impl_model_picks_smallest_fitting_bin():
    """MEMFINE_MODEL_IMPL: C = smallest bin whose exact backward workspace (max over EP ranks)
    fits B - static - other; checked against memfine_workspace_bytes directly."""
    rng = np.random.default_rng(5)
    T, h, g, E, k, EP = 2048, 256, 512, 16, 4, 4
    ids = [np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32) for _ in range(EP)]
    od = oracle.Dims(T=T, h=h, g=g, E=E, k=k)
    counts = torch.from_numpy(np.stack([oracle.route_counts(od, i, 8)[0] for i in ids]).astype(np.int32))
    dims0 = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=0)
    ws = {}
    for C_ in (1, 2, 4, 8):
        ws[C_] = max(layer.workspace_bytes(counts, layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=r), C_,
                                           capi.BWD) for r in range(EP))
    assert ws[1] > ws[2] > ws[4] > ws[8]
    static = 10**6
    for C_ in (1, 2, 4, 8):
        b = capi.make_budget(static + ws[C_], 1.0, static, 0, model=capi.MODEL_IMPL)
        p = layer.plan(counts, dims0, b)
        assert p["status"] == 0 and p["C"] == C_ and p["feasible"] and p["predicted_peak_bytes"] == ws[C_]
        b = capi.make_budget(static + ws[C_] - 1, 1.0, static, 0, model=capi.MODEL_IMPL)
        p = layer.plan(counts, dims0, b)
        assert p["C"] == (C_ * 2 if C_ < 8 else 8) and (p["clamped"] == (C_ == 8))


def test_m_g_matches_oracle_and_validates():
    import oracle
    oracle.build()
    for v in range(1, 4):
        for p in range(1, 9):
            for r in range(p):
                for fr in (False, True):
                    assert layer.m_g(v, p, r, fr) == oracle.m_g(v, p, r, fr)
    out = C.c_int32()
    for bad in ((0, 4, 0), (1, 0, 0), (1, 4, 4), (1, 4, -1)):
        assert capi.lib().memfine_m_g(*bad, 0, C.byref(out)) == capi.ERR_INVALID_ARG
