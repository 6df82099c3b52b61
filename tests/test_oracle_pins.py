"""Pins for the CPU oracle (run with -m "not gpu").

Each test checks the oracle against something other than itself: values the
paper prints (tests/golden/*.json, cited), hand-derived closed forms, finite
differences, a textbook/library reduction (torch autograd on a dense SwiGLU
MLP, numpy's stable argsort / lexsort), SPEC.md's printed vectors, or an
invariant the method guarantees (Eq. 6 = Eq. 4, conservation, linearity).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import Dims

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rand_problem(rng, T, h, g, E, k, EP=1, distinct=True, dtype="f64"):
    n = EP * T
    x = rng.standard_normal((n, h))
    dy = rng.standard_normal((n, h))
    if distinct:
        ids = np.stack([rng.permutation(E)[:k] for _ in range(n)]).astype(np.int32)
    else:
        ids = rng.integers(0, E, size=(n, k)).astype(np.int32)
    w = rng.random((n, k))
    wg = rng.standard_normal((E, g, h)) / math.sqrt(h)
    wu = rng.standard_normal((E, g, h)) / math.sqrt(h)
    wd = rng.standard_normal((E, h, g)) / math.sqrt(g)
    if dtype == "f32":
        x, dy, wg, wu, wd = (a.astype(np.float32) for a in (x, dy, wg, wu, wd))
    return x, dy, ids, w, wg, wu, wd


# ----------------------------------------------------------------------------- golden / closed form
def test_hand_2x2_golden(oracle_lib):
    """Hand-worked one-token example (tests/golden/hand_2x2.json)."""
    gold = json.load(open(os.path.join(GOLD, "hand_2x2.json")))
    inp = {k: np.array(v, dtype=np.float64) for k, v in gold["inputs"].items()}
    sig = 1.0 / (1.0 + math.e)
    ev = lambda tree: np.vectorize(lambda s: eval(s, {"sig": sig}))(np.array(tree, dtype=object)).astype(float)
    d = Dims(T=1, h=2, g=2, E=1, k=1, in_dtype="f64")
    ids = inp["ids"].astype(np.int32)
    y = oracle.moe_forward(d, inp["x"], ids, inp["scores"], inp["w_gate"], inp["w_up"], inp["w_down"])
    np.testing.assert_allclose(y, ev(gold["expected_expr"]["y"]), rtol=1e-14, atol=1e-15)
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, inp["dy"], inp["x"], ids, inp["scores"],
                                                inp["w_gate"], inp["w_up"], inp["w_down"])
    ex = gold["expected_expr"]
    for got, key in ((dx, "dx"), (ds, "dscore"), (dwg, "dw_gate"), (dwu, "dw_up"), (dwd, "dw_down")):
        np.testing.assert_allclose(got, ev(ex[key]), rtol=1e-13, atol=1e-15, err_msg=key)


def test_single_expert_reduces_to_dense_swiglu_mlp(oracle_lib):
    """E=1, k=1, w=1: the MoE layer is a dense bias-free SwiGLU MLP.  Forward via torch's
    F.silu/matmul, gradients via torch.autograd (library routines), fp64."""
    rng = np.random.default_rng(7)
    T, h, g = 9, 12, 20
    x, dy, _, _, wg, wu, wd = rand_problem(rng, T, h, g, 1, 1)
    ids = np.zeros((T, 1), np.int32)
    w = np.ones((T, 1))
    d = Dims(T=T, h=h, g=g, E=1, k=1, in_dtype="f64")
    y = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    X = torch.tensor(x, requires_grad=True)
    Wg = torch.tensor(wg[0], requires_grad=True)
    Wu = torch.tensor(wu[0], requires_grad=True)
    Wd = torch.tensor(wd[0], requires_grad=True)
    Y = torch.nn.functional.linear(
        torch.nn.functional.silu(torch.nn.functional.linear(X, Wg)) * torch.nn.functional.linear(X, Wu), Wd)
    np.testing.assert_allclose(y, Y.detach().numpy(), rtol=1e-12, atol=1e-13)
    Y.backward(torch.tensor(dy))
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    np.testing.assert_allclose(dx, X.grad.numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dwg[0], Wg.grad.numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dwu[0], Wu.grad.numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dwd[0], Wd.grad.numpy(), rtol=1e-11, atol=1e-12)
    # d_score = <dY, o> with o = Y at w = 1
    np.testing.assert_allclose(ds[:, 0], (dy * Y.detach().numpy()).sum(1), rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------- finite differences
@pytest.mark.parametrize("EP", [1, 2])
def test_backward_matches_central_finite_differences(oracle_lib, EP):
    """Central differences in fp64, step 1e-5, max relative error <= 1e-6."""
    rng = np.random.default_rng(11 + EP)
    T, h, g, E, k = 5, 6, 8, 4, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k, EP=EP)
    d = Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="f64")
    loss = lambda x_, w_, wg_, wu_, wd_: float((oracle.moe_forward(d, x_, ids, w_, wg_, wu_, wd_) * dy).sum())
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    eps = 1e-5

    def fd(arr, idx, which):
        a_p, a_m = arr.copy(), arr.copy()
        a_p[idx] += eps
        a_m[idx] -= eps
        args_p = {"x": x, "w": w, "wg": wg, "wu": wu, "wd": wd}
        args_m = dict(args_p)
        args_p[which], args_m[which] = a_p, a_m
        lp = loss(args_p["x"], args_p["w"], args_p["wg"], args_p["wu"], args_p["wd"])
        lm = loss(args_m["x"], args_m["w"], args_m["wg"], args_m["wu"], args_m["wd"])
        return (lp - lm) / (2 * eps)

    for name, arr, an in (("x", x, dx), ("w", w, ds), ("wg", wg, dwg), ("wu", wu, dwu), ("wd", wd, dwd)):
        idxs = list(np.ndindex(arr.shape))
        if len(idxs) > 40:
            sel = rng.choice(len(idxs), 40, replace=False)
            idxs = [idxs[i] for i in sel]
        num = np.array([fd(arr, i, name) for i in idxs])
        ana = np.array([an[i] for i in idxs])
        rel = np.abs(num - ana).max() / max(np.abs(ana).max(), 1e-30)
        assert rel <= 1e-6, (name, rel)


# ----------------------------------------------------------------------------- special cases
def test_zero_scores_and_zero_dy(oracle_lib):
    """Scores all 0 -> Y = 0 and dX = dW = 0; dY = 0 -> all grads 0."""
    rng = np.random.default_rng(3)
    T, h, g, E, k = 7, 8, 16, 4, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k)
    d = Dims(T=T, h=h, g=g, E=E, k=k, in_dtype="f64")
    z = np.zeros_like(w)
    assert np.all(oracle.moe_forward(d, x, ids, z, wg, wu, wd) == 0.0)
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, dy, x, ids, z, wg, wu, wd)
    assert np.all(dx == 0) and np.all(dwg == 0) and np.all(dwu == 0) and np.all(dwd == 0)
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, np.zeros_like(dy), x, ids, w, wg, wu, wd)
    for a in (dx, ds, dwg, dwu, dwd):
        assert np.all(a == 0)


def test_linearity_in_scores_and_duplicate_slots(oracle_lib):
    """Combine is linear in the scores (Eq. 4 / Table 2 row 13): Y(w1+w2) = Y(w1)+Y(w2);
    two slots on the same expert equal one slot carrying the summed score (reading R20)."""
    rng = np.random.default_rng(5)
    T, h, g, E, k = 6, 8, 12, 3, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k)
    d = Dims(T=T, h=h, g=g, E=E, k=k, in_dtype="f64")
    w2 = rng.random(w.shape)
    y12 = oracle.moe_forward(d, x, ids, w + w2, wg, wu, wd)
    y1 = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    y2 = oracle.moe_forward(d, x, ids, w2, wg, wu, wd)
    np.testing.assert_allclose(y12, y1 + y2, rtol=1e-12, atol=1e-13)
    dup = np.repeat(ids[:, :1], 2, axis=1)
    y_dup = oracle.moe_forward(d, x, dup, w, wg, wu, wd)
    d1 = Dims(T=T, h=h, g=g, E=E, k=1, in_dtype="f64")
    y_one = oracle.moe_forward(d1, x, ids[:, :1].copy(), w.sum(1, keepdims=True), wg, wu, wd)
    np.testing.assert_allclose(y_dup, y_one, rtol=1e-12, atol=1e-13)


def test_token_permutation_equivariance_and_bad_ids(oracle_lib):
    rng = np.random.default_rng(9)
    T, h, g, E, k = 8, 8, 8, 4, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k)
    d = Dims(T=T, h=h, g=g, E=E, k=k, in_dtype="f64")
    p = rng.permutation(T)
    y = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    yp = oracle.moe_forward(d, x[p], ids[p], w[p], wg, wu, wd)
    np.testing.assert_array_equal(yp, y[p])
    bad = ids.copy()
    bad[0, 1] = E + 3
    bad[3, 0] = -1
    yb = oracle.moe_forward(d, x, bad, w, wg, wu, wd)
    keep = np.ones_like(w)
    keep[0, 1] = 0
    keep[3, 0] = 0
    np.testing.assert_allclose(yb, oracle.moe_forward(d, x, ids, w * keep, wg, wu, wd), rtol=0, atol=1e-15)
    counts, nbad = oracle.route_counts(d, bad, 1)
    assert nbad == 2 and counts.sum() == T * k - 2


# ----------------------------------------------------------------------------- FCDA invariants
@pytest.mark.parametrize("EP", [1, 2, 4])
def test_fcda_chunked_equals_unchunked(oracle_lib, EP):
    """Eq. 6 == Eq. 4 and Eq. 7 == Eq. 5: forward
    and dX / d_score bit-exact for every C; dW bit-exact at EP=1 (same visiting order),
    <= 1e-12 relative at EP>1 (chunk-major order differs, reading R18)."""
    rng = np.random.default_rng(21 + EP)
    T, h, g, E, k = 13, 8, 16, 8, 3
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k, EP=EP, distinct=False)
    d = Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="f64")
    y = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    dx, ds, dwg, dwu, dwd = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    for C_ in range(1, 9):
        yc, cb, pk = oracle.fcda_forward(d, C_, x, ids, w, wg, wu, wd)
        np.testing.assert_array_equal(yc, y)
        dxc, dsc, dwgc, dwuc, dwdc, _, _ = oracle.fcda_backward(d, C_, dy, x, ids, w, wg, wu, wd)
        np.testing.assert_array_equal(dxc, dx)
        np.testing.assert_array_equal(dsc, ds)
        for a, b in ((dwgc, dwg), (dwuc, dwu), (dwdc, dwd)):
            if EP == 1:
                np.testing.assert_array_equal(a, b)
            else:
                assert np.abs(a - b).max() <= 1e-12 * max(np.abs(b).max(), 1e-300)
    # T < C: empty chunks are legal (reading R20)
    d2 = Dims(T=3, h=h, g=g, E=E, k=k, EP=1, in_dtype="f64")
    y2 = oracle.moe_forward(d2, x[:3], ids[:3], w[:3], wg, wu, wd)
    y2c, _, _ = oracle.fcda_forward(d2, 8, x[:3], ids[:3], w[:3], wg, wu, wd)
    np.testing.assert_array_equal(y2c, y2)


def test_chunk_partition(oracle_lib):
    """Reading R1: chunk j = [floor(jT/C), floor((j+1)T/C)): exhaustive, disjoint, sizes
    differ by <= 1, and the boundaries of every C | 8 nest in those of 8."""
    for T in (0, 1, 3, 7, 8, 13, 256, 16384, 10**9 + 7):
        for C_ in range(1, 9):
            b = [oracle.chunk_begin(T, C_, j) for j in range(C_ + 1)]
            assert b[0] == 0 and b[-1] == T
            sizes = np.diff(b)
            assert sizes.min() >= 0 and sizes.max() - sizes.min() <= 1
        b8 = {oracle.chunk_begin(T, 8, j) for j in range(9)}
        for C_ in (1, 2, 4):
            assert {oracle.chunk_begin(T, C_, j) for j in range(C_ + 1)} <= b8


# ----------------------------------------------------------------------------- counts / permutation
def test_counts_conservation_and_histogram(oracle_lib):
    rng = np.random.default_rng(4)
    T, E, k = 1000, 16, 4
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    d = Dims(T=T, h=1, g=1, E=E, k=k)
    for nsub in (1, 3, 8):
        counts, bad = oracle.route_counts(d, ids, nsub)
        assert bad == 0 and counts.sum() == T * k          # conservation
        for j in range(nsub):
            t0, t1 = oracle.chunk_begin(T, nsub, j), oracle.chunk_begin(T, nsub, j + 1)
            np.testing.assert_array_equal(counts[j], np.bincount(ids[t0:t1].ravel(), minlength=E))


def test_dispatch_order_is_stable_sort(oracle_lib):
    """EP=1: canonical order == numpy's stable argsort of the chunk's expert ids;
    EP>1: == numpy lexsort on (slot, token, src, expert) (reading R3)."""
    rng = np.random.default_rng(8)
    T, E, k = 37, 8, 3
    ids1 = rng.integers(0, E, size=(T, k)).astype(np.int32)
    d = Dims(T=T, h=1, g=1, E=E, k=k)
    for C_ in (1, 2, 4, 8):
        for j in range(C_):
            t0, t1 = oracle.chunk_begin(T, C_, j), oracle.chunk_begin(T, C_, j + 1)
            ref = np.argsort(ids1[t0:t1].ravel(), kind="stable") + t0 * k
            np.testing.assert_array_equal(oracle.dispatch_order(d, ids1, 0, C_, j), ref)
    EP = 4
    idsA = rng.integers(0, E, size=(EP * T, k)).astype(np.int32)
    dA = Dims(T=T, h=1, g=1, E=E, k=k, EP=EP)
    El = E // EP
    for C_ in (1, 3):
        for j in range(C_):
            t0, t1 = oracle.chunk_begin(T, C_, j), oracle.chunk_begin(T, C_, j + 1)
            src, tok, slot = np.meshgrid(np.arange(EP), np.arange(t0, t1), np.arange(k), indexing="ij")
            src, tok, slot = src.ravel(), tok.ravel(), slot.ravel()
            q = (src * T + tok) * k + slot
            e = idsA.ravel()[q]
            for r in range(EP):
                m = (e >= r * El) & (e < (r + 1) * El)
                o = np.lexsort((slot[m], tok[m], src[m], e[m]))
                np.testing.assert_array_equal(oracle.dispatch_order(dA, idsA, r, C_, j), q[m][o])


# ----------------------------------------------------------------------------- memory model
TOY = dict(m_g=1, t=1, c=1, D_t=2, b=1, s=8, h=4, a=2, h_d=2, k_a=1, e_n=4, g_e=8)


def test_memory_model_spec_vectors(oracle_lib):
    """SPEC.md:121-122 toy Eq. 2 values (512 B at s'=0, 1280 B at s'=16) and SPEC.md:316
    toy s'_max = 156 (alpha*M=10000, M_sta=2000)."""
    assert oracle.act_bytes_eq2(TOY, 0) == 512
    assert oracle.act_bytes_eq2(TOY, 16) == 1280
    assert oracle.s_prime_max_eq8(TOY, 10000, 2000) == 156
    # boundary: budget exactly static + s-term -> 0
    assert oracle.s_prime_max_eq8(TOY, 2512, 2000) == 0
    # affine in s' with slope D_t*b*(2h+2g_e)
    v = [oracle.act_bytes_eq2(TOY, s) for s in (0, 5, 10)]
    assert v[1] - v[0] == v[2] - v[1] == 5 * 2 * (8 + 16)


def test_memory_model_closed_form_equals_table2_rows(oracle_lib):
    """Eq. 2's closed form == the sum of Table 2's rows, 200 random configs."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        cfg = {k: int(rng.integers(1, 50)) for k in TOY}
        cfg["t"] = cfg["c"] = 1
        cfg["m_g"] = int(rng.integers(1, 8))
        sp = int(rng.integers(0, 10000))
        rows = oracle.act_table2_rows(cfg, sp)
        assert rows[6] == 0 and rows[13] == 0
        assert oracle.act_bytes_eq2(cfg, sp) == cfg["m_g"] * int(rows.sum())
        cfg["t"], cfg["c"] = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        assert oracle.act_bytes_eq2(cfg, sp) == (cfg["m_g"] * int(rows.sum())) // (cfg["t"] * cfg["c"])


def _plan_toy(sdd, bins=(1, 2, 4, 8), rule=0, nsub=1):
    d = Dims(T=1, h=4, g=8, E=2, k=1)
    counts = np.zeros((1, nsub, 2), np.int64)
    counts[0, 0, 0] = sdd
    return oracle.plan(counts, d, budget_bytes=10000, static_bytes=2000, other_act_bytes=512,
                       D_t=2, bins=bins, rule=rule)


def test_plan_spec_vectors(oracle_lib):
    """s'_max = 156; ceil(157/156) = 2; ceil(400/156) = 3 -> bin 4;
    c = 9 clamps to 8 (clamped, infeasible); s''=0 -> c = 1."""
    st, p = _plan_toy(156)
    assert st == 0 and p["s_prime_max"] == 156 and p["c_theory"] == 1 and p["C"] == 1 and p["feasible"]
    st, p = _plan_toy(157)
    assert p["c_theory"] == 2 and p["C"] == 2
    st, p = _plan_toy(400)
    assert p["c_theory"] == 3 and p["C"] == 4 and not p["clamped"]
    st, p = _plan_toy(9 * 156)
    assert p["c_theory"] == 9 and p["C"] == 8 and p["clamped"] and not p["feasible"]
    st, p = _plan_toy(0)
    assert p["c_theory"] == 1 and p["C"] == 1
    # static alone exceeds the budget -> infeasible
    d = Dims(T=1, h=4, g=8, E=2, k=1)
    st, _ = oracle.plan(np.zeros((1, 1, 2), np.int64), d, budget_bytes=1000, static_bytes=2000)
    assert st == 2
    # invalid bins
    st, _ = _plan_toy(10, bins=(2, 2))
    assert st == 1


def test_plan_paper_model_I_and_II_derive_c2(oracle_lib):
    """with bins [1,2,4,8] MACT derives c_k = 2 for Model I, and Table 4
    shows Model II at the same 11.9 GB.  With Table 4's fit (s-term 0.9 GB, s'-term 22.0 GB at
    c = 1) and the paper's beta = D_t(2h + 2g_e) (Table 3: h=7168, g_e=2048), any alpha in
    [0.858, 0.975) gives C = 2 for both models; alpha = 0.9 pins it.  Fixed c_k = 8 -> 8."""
    gold = json.load(open(os.path.join(GOLD, "paper_table4.json")))
    t3 = gold["table3"]
    beta = t3["D_t"] * (2 * t3["h"] + 2 * t3["g_e"])
    assert beta == 36864
    sdd = int(22.0e9 // beta)
    d = Dims(T=1, h=t3["h"], g=t3["g_e"], E=1, k=1)
    counts = np.array([[[sdd]]], np.int64)
    for model in ("model_I", "model_II"):
        st, p = oracle.plan(counts, d, budget_bytes=int(0.9 * 64e9),
                            static_bytes=int(gold[model]["static_gb"] * 1e9),
                            other_act_bytes=int(0.9e9), D_t=2, bins=gold["mact_bins"])
        assert st == 0 and p["C"] == gold["mact_derived_c"] and p["feasible"], (model, p)
        st, p = oracle.plan(counts, d, budget_bytes=int(0.9 * 64e9),
                            static_bytes=int(gold[model]["static_gb"] * 1e9),
                            other_act_bytes=int(0.9e9), D_t=2, bins=[8])
        assert p["C"] == 8
    # Table 4 arithmetic: totals = static + active; the printed reductions
    for model in ("model_I", "model_II"):
        m = gold[model]
        for c in ("1", "2", "8"):
            assert abs(m["static_gb"] + m["active_gb"][c] - m["all_gb"][c]) < 1e-9
            assert (m["all_gb"][c] <= gold["gpu_capacity_gb"]) == m["trainable"][c]
    a = gold["model_I"]["active_gb"]
    assert round(100 * (a["1"] - a["2"]) / a["1"], 2) == gold["reduction_pct"]["mact_vs_m1"]
    assert round(100 * (a["1"] - a["8"]) / a["1"], 2) == gold["reduction_pct"]["c8_vs_m1"]


def test_plan_properties(oracle_lib):
    """Safety, monotonicity and bin soundness on random cases."""
    rng = np.random.default_rng(17)
    for _ in range(300):
        EP = int(rng.choice([1, 2, 4, 8]))
        E = EP * int(rng.integers(1, 5))
        h, g = int(rng.integers(1, 64)), int(rng.integers(1, 64))
        nsub = 8
        counts = rng.integers(0, 50, size=(EP, nsub, E)).astype(np.int64)
        d = Dims(T=1, h=h, g=g, E=E, k=1, EP=EP)
        budget = int(rng.integers(1000, 200000))
        static = int(rng.integers(0, 1000))
        other = int(rng.integers(0, 1000))
        rule = int(rng.integers(0, 2))
        st, p = oracle.plan(counts, d, budget_bytes=budget, static_bytes=static, other_act_bytes=other,
                            bins=(1, 2, 4, 8), rule=rule)
        if st == 2:
            continue
        assert st == 0
        beta = 2 * (2 * h + 2 * g)
        if p["feasible"]:
            assert static + other + beta * p["s_chunk_max"] <= budget       # Eq. 3 holds
        if not p["clamped"] and rule == 0:
            assert p["C"] >= p["c_theory"]
        st2, p2 = oracle.plan(counts * 2, d, budget_bytes=budget, static_bytes=static,
                              other_act_bytes=other, bins=(1, 2, 4, 8), rule=0)
        st1, p1 = oracle.plan(counts, d, budget_bytes=budget, static_bytes=static,
                              other_act_bytes=other, bins=(1, 2, 4, 8), rule=0)
        if st2 == 0:
            assert p2["c_theory"] >= p1["c_theory"]


# ----------------------------------------------------------------------------- meter
def test_meter_peak_scales_as_one_over_c(oracle_lib):
    """Meter peak non-increasing in c for uniformly split routing; c=4 peak = 1/4
    (SPEC.md:265, 275, 474); per-chunk bytes sum to the unchunked bytes."""
    rng = np.random.default_rng(1)
    T, h, g, E, k = 64, 4, 8, 4, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k)
    d = Dims(T=T, h=h, g=g, E=E, k=k, in_dtype="f64")
    peaks = []
    for C_ in range(1, 9):
        _, cb, pk = oracle.fcda_forward(d, C_, x, ids, w, wg, wu, wd, D_t=2)
        assert int(cb.sum()) == 2 * T * k * (2 * h + 2 * g)
        peaks.append(int(pk[0]))
        _, _, _, _, _, cbb, pkb = oracle.fcda_backward(d, C_, dy, x, ids, w, wg, wu, wd, D_t=2)
        assert int(pkb[0]) == int(pk[0])
    assert all(peaks[i + 1] <= peaks[i] for i in range(7))
    assert peaks[3] * 4 == peaks[0]


# ----------------------------------------------------------------------------- router (N3)
def test_router_matches_torch_topk_softmax_and_autograd(oracle_lib):
    """Router forward == torch.topk + softmax over the selected logits; backward == torch.autograd
    of that composition (library routines), fp64, with an upstream d_score."""
    rng = np.random.default_rng(31)
    n, h, E, k = 23, 16, 12, 3
    x = rng.standard_normal((n, h))
    wr = rng.standard_normal((E, h))
    d = Dims(T=n, h=h, g=1, E=E, k=k, in_dtype="f64")
    logits, ids, scores = oracle.router_forward(d, x, wr)
    X = torch.tensor(x, requires_grad=True)
    W = torch.tensor(wr, requires_grad=True)
    L = X @ W.T
    top = torch.topk(L, k, dim=1)
    np.testing.assert_allclose(logits, L.detach().numpy(), rtol=1e-13, atol=1e-13)
    np.testing.assert_array_equal(ids, top.indices.numpy())
    S = torch.softmax(top.values, dim=1)
    np.testing.assert_allclose(scores, S.detach().numpy(), rtol=1e-13, atol=1e-14)
    ds = rng.standard_normal((n, k))
    S.backward(torch.tensor(ds))
    dx, dwr = oracle.router_backward(d, x, wr, ids, scores, ds)
    np.testing.assert_allclose(dx, X.grad.numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dwr, W.grad.numpy(), rtol=1e-11, atol=1e-12)


def test_router_ties_and_finite_differences(oracle_lib):
    """Ties resolve to the lower expert id; the backward matches central differences of
    sum(ds * scores) away from ties (fp64, step 1e-6)."""
    d = Dims(T=1, h=2, g=1, E=4, k=2, in_dtype="f64")
    x = np.array([[1.0, 0.0]])
    wr = np.array([[1.0, 0.0], [2.0, 0.0], [2.0, 0.0], [0.5, 0.0]])   # logits 1, 2, 2, 0.5
    _, ids, sc = oracle.router_forward(d, x, wr)
    assert ids.tolist() == [[1, 2]] and np.allclose(sc, 0.5)
    rng = np.random.default_rng(5)
    n, h, E, k = 6, 5, 7, 3
    x = rng.standard_normal((n, h))
    wr = rng.standard_normal((E, h))
    ds = rng.standard_normal((n, k))
    d = Dims(T=n, h=h, g=1, E=E, k=k, in_dtype="f64")
    _, ids, sc = oracle.router_forward(d, x, wr)
    dx, dwr = oracle.router_backward(d, x, wr, ids, sc, ds)

    def f(x_, w_):
        _, i2, s2 = oracle.router_forward(d, x_, w_)
        assert np.array_equal(i2, ids)
        return float((s2 * ds).sum())
    eps = 1e-6
    for arr, an in ((x, dx), (wr, dwr)):
        for idx in list(np.ndindex(arr.shape))[:15]:
            ap, am = arr.copy(), arr.copy()
            ap[idx] += eps
            am[idx] -= eps
            num = (f(ap, wr) - f(am, wr)) / (2 * eps) if arr is x else (f(x, ap) - f(x, am)) / (2 * eps)
            assert abs(num - an[idx]) <= 1e-6 * max(1.0, abs(an[idx]))


def test_m_g_pipeline_stage_pins():
    """Eq. 2's m_g (reading R29): full recomputation holds one micro-batch; without
    pipelining (p = 1, v = 1) one micro-batch is live; the last stage of a plain 1F1B pipeline
    (v = 1, r_pp = p - 1) runs each forward straight into its backward, so it holds one; every
    stage earlier holds two more; every extra virtual stage adds p."""
    import oracle
    oracle.build()
    assert oracle.m_g(3, 8, 5, full_recompute=True) == 1
    assert oracle.m_g(1, 1, 0) == 1
    for p in range(1, 9):
        assert oracle.m_g(1, p, p - 1) == 1
        for r in range(p - 1):
            assert oracle.m_g(1, p, r) == oracle.m_g(1, p, r + 1) + 2
        for v in range(1, 4):
            for r in range(p):
                assert oracle.m_g(v + 1, p, r) == oracle.m_g(v, p, r) + p


# ----------------------------------------------------------------------------- pins of the checkers themselves
@pytest.mark.parametrize("EP,dtype", [(1, "f64"), (2, "f32")])
def test_moe_tokens_equals_whole_layer_rows(oracle_lib, EP, dtype):
    """oracle_moe_tokens (the full-size sampled checker) returns exactly the rows of the whole-layer
    definitions: y of Eq. 4 (oracle_moe_forward), dx and d_score of Eq. 5 (oracle_moe_backward), for
    any token subset in any order - including duplicate slots and out-of-range ids."""
    rng = np.random.default_rng(23)
    T, h, g, E, k = 24, 16, 24, 6, 3
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k, EP=EP, distinct=False, dtype=dtype)
    ids[3, 1] = E + 2          # an id outside [0, E): contributes nothing
    ids[5, 2] = -1
    d = Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype=dtype)
    y = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    dx, ds, *_ = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    toks = np.array([0, 5, 3, EP * T - 1, 7, 5, 11])
    ys, dxs, dss = oracle.moe_tokens(d, toks, dy, x, ids, w, wg, wu, wd)
    for got, ref in ((ys, y[toks]), (dxs, dx[toks]), (dss, ds[toks])):
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert dss[2, 1] == 0.0 and np.all(dss[1, 2] == 0.0)


def test_plan_exact_rule_is_minimal(oracle_lib):
    """Rule EXACT (reading R11) picks the SMALLEST bin whose true per-chunk maximum fits s'_max: every
    smaller bin overflows, the chosen one fits, and a clamp means no bin fits.  Per-chunk loads are
    recomputed here with numpy from the counts (chunk jc of C = sub-chunks [jc*8/C, (jc+1)*8/C)) and
    s'_max from Eq. 8 directly."""
    rng = np.random.default_rng(29)
    bins = (1, 2, 4, 8)
    seen = {b: 0 for b in bins}
    clamped = 0
    for _ in range(400):
        EP = int(rng.choice([1, 2, 4]))
        E = EP * int(rng.integers(1, 4))
        h, g = int(rng.integers(1, 32)), int(rng.integers(1, 32))
        counts = rng.integers(0, 40, size=(EP, 8, E)).astype(np.int64)
        if rng.random() < 0.5:                         # skew: one hot rank and sub-chunk
            counts[0, int(rng.integers(0, 8)), 0] += int(rng.integers(0, 400))
        d = Dims(T=1, h=h, g=g, E=E, k=1, EP=EP)
        beta = 2 * (2 * h + 2 * g)
        budget = int(rng.integers(beta, 400 * beta))
        st, p = oracle.plan(counts, d, budget_bytes=budget, bins=bins, rule=1)
        assert st == 0
        spm = budget // beta
        assert p["s_prime_max"] == spm
        El = E // EP
        recv = counts.sum(axis=0).reshape(8, EP, El).sum(axis=2)        # [sub-chunk][receiving rank]
        def chunk_max(C_):
            return int(recv.reshape(C_, 8 // C_, EP).sum(axis=1).max())
        fits = [chunk_max(b) <= spm for b in bins]
        if p["clamped"]:
            clamped += 1
            assert not any(fits) and p["C"] == bins[-1] and not p["feasible"]
        else:
            i = bins.index(p["C"])
            seen[p["C"]] += 1
            assert fits[i] and not any(fits[:i]) and p["feasible"]
            assert p["s_chunk_max"] == chunk_max(p["C"])
    assert all(v > 0 for v in seen.values()) and clamped > 0


def test_moe_backward_experts_equals_whole_layer_slices(oracle_lib):
    """oracle_moe_backward_experts (the full-size dW checker) returns exactly moe_backward's expert
    slices (same copies, same canonical order: bit-identical) and its dx / d_score."""
    rng = np.random.default_rng(31)
    T, h, g, E, k = 30, 16, 24, 6, 2
    x, dy, ids, w, wg, wu, wd = rand_problem(rng, T, h, g, E, k, EP=2, dtype="f32")
    d = Dims(T=T, h=h, g=g, E=E, k=k, EP=2, in_dtype="f32")
    ref = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    sel = [4, 0, 5]
    got = oracle.moe_backward_experts(d, dy, x, ids, w, wg, wu, wd, sel)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    for a, b in zip(got[2:], ref[2:]):
        assert np.array_equal(a, b[sel])
