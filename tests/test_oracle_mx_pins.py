"""Pins for the oracle's MXFP8 variant (reading R28), CPU only.

The oracle's E4M3 codec is pinned to torch's float8_e4m3fn conversion (an independent library
routine) and to brute force over all 256 codes; the scale rule to its closed-form property; the
MX layer to the exact oracle with quantisers off, and — for the operand layouts (which tensors are
quantised along which axis) — to an independent numpy/torch re-derivation of one token."""
import numpy as np
import pytest
import torch

import oracle
import synth


def _dec_all():
    return np.array([oracle.e4m3_decode(c) for c in range(256)])


def test_e4m3_decode_matches_torch_all_codes():
    ref = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    got = _dec_all()
    nan = np.isnan(ref)
    assert (np.isnan(got) == nan).all() and nan.sum() == 2          # 0x7F and 0xFF
    assert (got[~nan] == ref[~nan]).all()
    assert np.nanmax(got) == 448.0 and got[1] == 2.0 ** -9               # max normal, min subnormal


def test_e4m3_encode_matches_torch_and_brute_force():
    rng = np.random.default_rng(5)
    mag = 2.0 ** rng.uniform(-12, np.log2(448), 4000)
    v = (mag * rng.choice([-1, 1], 4000)).astype(np.float32)
    # torch: float32 -> float8_e4m3fn, round to nearest even
    ref = torch.from_numpy(v).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = np.array([oracle.e4m3_encode(float(x)) for x in v], np.uint8)
    assert (got == ref).all()
    # exact midpoints between neighbouring codes tie to the even code (brute force over the grid)
    vals = _dec_all()
    pos = np.array(sorted({(float(vals[c]), c) for c in range(0x7F)}))
    for (a, ca), (b, cb) in zip(pos[:-1], pos[1:]):
        mid = (a + b) / 2
        want = int(ca) if int(ca) % 2 == 0 else int(cb)
        assert oracle.e4m3_encode(mid) == want
        assert oracle.e4m3_encode(-mid) == want | 0x80
    assert oracle.e4m3_encode(1e6) == 0x7E and oracle.e4m3_encode(-1e6) == 0xFE   # saturating
    assert oracle.e4m3_encode(0.0) == 0


def test_mx_scale_rule_closed_form():
    rng = np.random.default_rng(6)
    for amax in np.concatenate([2.0 ** rng.uniform(-100, 100, 2000), [448.0, 449.0, 1.75, 1.0, 896.0, 897.0]]):
        E = oracle.mx_scale_exp(amax)
        assert amax <= 448.0 * 2.0 ** E                 # nothing clips
        assert amax > 448.0 * 2.0 ** (E - 1)            # and E is the smallest such
    assert oracle.mx_scale_exp(0.0) == 0
    assert oracle.mx_scale_exp(1e-300) == -127 and oracle.mx_scale_exp(1e300) == 127


def test_mx_quantize_block_error_bound():
    rng = np.random.default_rng(7)
    v = (rng.standard_normal(32 * 64) * 2.0 ** rng.integers(-20, 20, 32 * 64)).astype(np.float32)
    v[:32] = 0.0                                                          # an all-zero block
    codes, sc = oracle.mx_quantize(v)
    vals = _dec_all()
    E = sc.astype(np.int64) - 127
    deq = vals[codes] * 2.0 ** np.repeat(E, 32)
    assert (deq[:32] == 0).all() and E[0] == 0
    for b in range(64):
        blk = v[b * 32:(b + 1) * 32].astype(np.float64)
        if not blk.any():
            continue
        assert E[b] == oracle.mx_scale_exp(np.abs(blk).max())
        # half an E4M3 spacing of each element (3 mantissa bits; subnormal spacing 2^-9 * 2^E)
        sp = np.maximum(2.0 ** (np.floor(np.log2(np.maximum(np.abs(blk) / 2.0 ** E[b], 2.0 ** -6))) - 3),
                        2.0 ** -9) * 2.0 ** E[b]
        assert (np.abs(deq[b * 32:(b + 1) * 32] - blk) <= sp / 2 + 1e-300).all()


def _problem(T=6, h=64, g=96, E=4, k=2, seed=3):
    d = oracle.Dims(T=T, h=h, g=g, E=E, k=k, in_dtype="f32")
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, h)).astype(np.float32)
    dy = rng.standard_normal((T, h)).astype(np.float32)
    wg = (rng.standard_normal((E, g, h)) / np.sqrt(h)).astype(np.float32)
    wu = (rng.standard_normal((E, g, h)) / np.sqrt(h)).astype(np.float32)
    wd = (rng.standard_normal((E, h, g)) / np.sqrt(g)).astype(np.float32)
    wd[1, 5, :] *= 300.0                         # an outlier row: row vs column blocking differ
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
    w = rng.dirichlet(np.ones(k), T)
    return d, x, dy, wg, wu, wd, ids, w


def test_mx_layer_mode0_equals_exact_oracle():
    d, x, dy, wg, wu, wd, ids, w = _problem()
    wq = oracle.mx_weights(d, wg, wu, wd, mode=0)
    y0 = oracle.moe_mx(d, x, ids, w, wq, mode=0)
    assert np.array_equal(y0, oracle.moe_forward(d, x, ids, w, wg, wu, wd))
    y, dx, ds, dwg, dwu, dwd = oracle.moe_mx(d, x, ids, w, wq, dy=dy, mode=0, wd=wd)
    ref = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    for a, b in zip((dx, ds, dwg, dwu, dwd), ref):
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())


def _mxq(v, axis):
    """Independent MX quantise-dequantise along `axis` (numpy frexp + torch float8 conversion)."""
    v = np.moveaxis(np.asarray(v, np.float64), axis, -1)
    sh = v.shape
    b = v.reshape(-1, 32)
    amax = np.abs(b).max(1)
    m, ex = np.frexp(amax)                       # amax = m 2^ex, m in [0.5, 1)
    E = np.where(amax > 0, ex - 1 - 8 + (2 * m > 1.75), 0)
    s = b / 2.0 ** E[:, None]
    q = torch.from_numpy(s.astype(np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    return np.moveaxis((q * 2.0 ** E[:, None]).reshape(sh), -1, axis)


def test_mx_layer_one_token_brute_force():
    """Every code decided on the exact value (reading R28): numpy/torch re-derivation of one token."""
    d, x, dy, wg, wu, wd, ids, w = _problem()
    wq = oracle.mx_weights(d, wg, wu, wd)
    y, dx, ds, *_, ex = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, return_exact=True)
    t = 2
    sig = lambda z: 1 / (1 + np.exp(-z))
    xq = _mxq(x[t], 0)
    y_ref = np.zeros(d.h); dx_ref = np.zeros(d.h); ds_ref = np.zeros(d.k)
    for s in range(d.k):
        e = ids[t, s]
        G = _mxq(wg[e], 1) @ xq                  # W_gate rows blocked along h
        U = _mxq(wu[e], 1) @ xq
        a = G * sig(G) * U
        o = _mxq(wd[e], 1) @ _mxq(a, 0)          # W_down rows and a along g
        y_ref += w[t, s] * o
        u = wd[e].astype(np.float64).T @ dy[t].astype(np.float64)   # dA: BF16 operands, not quantised
        ds_ref[s] = u @ a
        dA = w[t, s] * u
        dG = dA * U * sig(G) * (1 + G * (1 - sig(G)))
        dU = dA * G * sig(G)
        dx_ref += _mxq(wg[e], 0).T @ _mxq(dG, 0) + _mxq(wu[e], 0).T @ _mxq(dU, 0)   # columns along g
        q = t * d.k + s                          # the exact values the oracle reports per copy
        assert np.abs(ex["a"][q] - a).max() <= 1e-12 * np.abs(a).max()
        assert np.abs(ex["gu"][q] - np.concatenate([G, U])).max() <= 1e-12 * np.abs(np.concatenate([G, U])).max()
        assert np.abs(ex["da"][q] - dA).max() <= 1e-12 * np.abs(dA).max()
        assert np.abs(ex["dgu"][q] - np.concatenate([dG, dU])).max() <= 1e-12 * np.abs(np.concatenate([dG, dU])).max()
    for got, ref in ((y[t], y_ref), (dx[t], dx_ref), (ds[t], ds_ref)):
        assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()


def test_mx_fed_own_decisions_change_nothing():
    """Feeding the oracle's own decisions (its exact values quantised by an independent routine) back
    in reproduces its outputs: the fed path replaces the quantiser and nothing else."""
    d, x, dy, wg, wu, wd, ids, w = _problem()
    wq = oracle.mx_weights(d, wg, wu, wd)
    ref = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, return_exact=True)
    ex = ref[-1]
    g = d.g
    fed = {"a_q": _mxq(ex["a"], 1),
           "dgu_q": np.concatenate([_mxq(ex["dgu"][:, :g], 1), _mxq(ex["dgu"][:, g:], 1)], axis=1)}
    got = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, fed=fed)
    for a, b in zip(got, ref[:-1]):
        assert np.abs(a - b).max() <= 1e-12 * max(1e-300, np.abs(b).max())


def test_mx_fed_codes_enter_linearly():
    """A fed decision moves the output by exactly its own term: perturbing copy q's a by da moves
    y[token] by w_q W_down^q(e) da; perturbing its dG || dU moves dx[token] by W_gate^q(e)^T ddG +
    W_up^q(e)^T ddU (the column-quantised weights) - which pins the copy indexing of the fed arrays."""
    d, x, dy, wg, wu, wd, ids, w = _problem(T=6)
    wq = oracle.mx_weights(d, wg, wu, wd)
    ex = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, return_exact=True)[-1]
    g, k = d.g, d.k
    base = {"a_q": _mxq(ex["a"], 1),
            "dgu_q": np.concatenate([_mxq(ex["dgu"][:, :g], 1), _mxq(ex["dgu"][:, g:], 1)], axis=1)}
    y0, dx0, *_ = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, fed=base)
    rng = np.random.default_rng(11)
    for q in (1, 7, 10):
        t, e = q // k, ids[q // k, q % k]
        da, dgu = rng.standard_normal(g), rng.standard_normal(2 * g)
        fed = {key: v.copy() for key, v in base.items()}
        fed["a_q"][q] += da
        fed["dgu_q"][q] += dgu
        y1, dx1, *_ = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, fed=fed)
        want_y = w[t, q % k] * (wq[2][e] @ da)
        want_dx = wq[3][e].T @ dgu[:g] + wq[4][e].T @ dgu[g:]
        assert np.abs((y1 - y0)[t] - want_y).max() <= 1e-10 * np.abs(want_y).max()
        assert np.abs((dx1 - dx0)[t] - want_dx).max() <= 1e-10 * np.abs(want_dx).max()
        others = np.arange(d.T) != t
        assert np.array_equal(y1[others], y0[others]) and np.array_equal(dx1[others], dx0[others])


def test_mx_layer_quantisation_error_is_small_but_present():
    d = oracle.Dims(T=64, h=128, g=192, E=4, k=2, in_dtype="bf16")
    x = synth.make_x(64, 128, rank=0).view(torch.int16).numpy().view(np.uint16)
    wg, wu, wd = (t.view(torch.int16).numpy().view(np.uint16) for t in synth.make_experts(range(4), 128, 192))
    ids, w = synth.make_routing(64, 4, 2, rank=0, zipf_s=1.2)
    y_mx = oracle.moe_mx(d, x, ids, w, oracle.mx_weights(d, wg, wu, wd))
    y = oracle.moe_forward(d, x, ids, w, wg, wu, wd)
    err = np.abs(y_mx - y).max() / np.abs(y).max()
    assert 1e-4 < err < 0.1          # E4M3 keeps 3 mantissa bits: a few % at most, never zero


# ---------------------------------------------------------------- MXFP8 weight gradients (R28c)
def test_mx_wgrad_mode0_equals_exact_dw():
    """Quantisers and roundings off: the chunked columnwise path is the definition W_grad = sum over
    chunks of the copies' outer products (reading R18), whatever C."""
    d, x, dy, wg, wu, wd, ids, w = _problem(T=40)
    wq = oracle.mx_weights(d, wg, wu, wd, mode=0)
    ref = oracle.moe_backward(d, dy, x, ids, w, wg, wu, wd)
    for C in (1, 3):
        *_, dwg, dwu, dwd = oracle.moe_mx(d, x, ids, w, wq, dy=dy, mode=0, wd=wd, wgrad_C=C)
        for a, b in zip((dwg, dwu, dwd), ref[2:]):
            assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


def test_mx_wgrad_brute_force():
    """Independent re-derivation: per copy the exact G, U, dG, dU, a_w (numpy, torch float8
    conversion), then per chunk and expert the copies stacked in (token, slot)
    order (reading R3, EP = 1), zero-padded to a multiple of 32 rows, every column quantised per
    32-row block (_mxq along the copies), and dW_gate = dG^T x, dW_up = dU^T x, dW_down = dY^T a_w."""
    T = 80
    d, x, dy, wg, wu, wd, ids, w = _problem(T=T, seed=9)
    wq = oracle.mx_weights(d, wg, wu, wd)
    sig = lambda z: 1 / (1 + np.exp(-z))
    per = {}
    for t in range(T):
        xq = _mxq(x[t], 0)
        for s in range(d.k):
            e = ids[t, s]
            G, U = _mxq(wg[e], 1) @ xq, _mxq(wu[e], 1) @ xq     # exact values (reading R28)
            a = G * sig(G) * U
            u = wd[e].astype(np.float64).T @ dy[t].astype(np.float64)
            dA = w[t, s] * u
            per[t, s] = (dA * U * sig(G) * (1 + G * (1 - sig(G))), dA * G * sig(G), w[t, s] * a)
    for C in (1, 2):
        ref = [np.zeros((d.E, d.g, d.h)), np.zeros((d.E, d.g, d.h)), np.zeros((d.E, d.h, d.g))]
        for j in range(C):
            t0, t1 = j * T // C, (j + 1) * T // C
            for e in range(d.E):
                cp = [(t, s) for t in range(t0, t1) for s in range(d.k) if ids[t, s] == e]
                n = -(-len(cp) // 32) * 32
                if not cp:
                    continue
                pad = lambda rows, width: np.vstack([np.array(rows, np.float64), np.zeros((n - len(rows), width))])
                colq = lambda m: np.vstack([_mxq(m[i:i + 32], 0) for i in range(0, n, 32)])
                X = colq(pad([x[t] for t, _ in cp], d.h))
                Y = colq(pad([dy[t] for t, _ in cp], d.h))
                dG = colq(pad([per[c][0] for c in cp], d.g))
                dU = colq(pad([per[c][1] for c in cp], d.g))
                Aw = colq(pad([per[c][2] for c in cp], d.g))
                ref[0][e] += dG.T @ X
                ref[1][e] += dU.T @ X
                ref[2][e] += Y.T @ Aw
        *_, dwg, dwu, dwd = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=C)
        for got, r in zip((dwg, dwu, dwd), ref):
            assert np.abs(got - r).max() <= 1e-10 * np.abs(r).max()


def test_mx_wgrad_error_small_present_and_chunk_dependent():
    """Against unquantised operands the MX weight gradients differ by a few % at most (3 mantissa
    bits per operand) and never by zero; the blocks follow the chunk partition, so C matters."""
    d, x, dy, wg, wu, wd, ids, w = _problem(T=64, seed=4)
    wq = oracle.mx_weights(d, wg, wu, wd)
    *_, e0, e1, e2 = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=0)
    outs = {C: oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=C)[3:] for C in (1, 2)}
    for C, (g1, u1, d1) in outs.items():
        for got, ref in ((g1, e0), (u1, e1), (d1, e2)):
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert 1e-4 < err < 0.1, (C, err)
    assert not np.array_equal(outs[1][0], outs[2][0])


def test_mx_token_subset_equals_whole_layer():
    """The full-size sampled evaluator (weights quantised one expert at a time) reproduces the whole
    layer's rows bit for bit - it is the same per-copy arithmetic on a token subset."""
    d, x, dy, wg, wu, wd, ids, w = _problem(T=40, seed=21)
    wq = oracle.mx_weights(d, wg, wu, wd)
    y, dx, ds, *_ = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd)
    toks = np.array([3, 17, 0, 39, 22])
    ys, dxs, dss = oracle.moe_mx_tokens(d, toks, x, dy, ids, w, wg, wu, wd)
    assert np.array_equal(ys, y[toks]) and np.array_equal(dxs, dx[toks]) and np.array_equal(dss, ds[toks])


def test_mx_wgrad_fed_columnwise_codes_enter_linearly():
    """A fed columnwise dG || dU (a_w) value of copy q moves dW_gate / dW_up (dW_down) of its expert by
    the outer product with that copy's columnwise-quantised x (dY) row - nothing else moves."""
    T = 40
    d, x, dy, wg, wu, wd, ids, w = _problem(T=T, seed=12)
    wq = oracle.mx_weights(d, wg, wu, wd)
    g, k = d.g, d.k
    *_, ex = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, return_exact=True)
    # columnwise decisions of the exact values, blocked as reading R28c says (C = 1, EP = 1)
    gu_col, aw_col = np.zeros((T * k, 2 * g)), np.zeros((T * k, g))
    xq_col, yq_col = np.zeros((T * k, d.h)), np.zeros((T * k, d.h))
    aw = ex["a"] * w.reshape(-1)[:, None]
    for e in range(d.E):
        cp = [t * k + s for t in range(T) for s in range(k) if ids[t, s] == e]
        for b in range(0, len(cp), 32):
            rows = cp[b:b + 32]
            pad = lambda m: np.vstack([m, np.zeros((32 - len(rows), m.shape[1]))])
            gu_col[rows] = _mxq(pad(ex["dgu"][rows]), 0)[:len(rows)]
            aw_col[rows] = _mxq(pad(aw[rows]), 0)[:len(rows)]
            xq_col[rows] = _mxq(pad(x[[q // k for q in rows]].astype(np.float64)), 0)[:len(rows)]
            yq_col[rows] = _mxq(pad(dy[[q // k for q in rows]].astype(np.float64)), 0)[:len(rows)]
    base = {"dgu_col_q": gu_col, "aw_col_q": aw_col}
    r0 = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=1, fed=base)
    own = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=1)
    for a, b in zip(r0[3:], own[3:]):            # feeding its own decisions back changes nothing
        assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
    rng = np.random.default_rng(13)
    q = 9
    e = ids[q // k, q % k]
    dgu, daw = rng.standard_normal(2 * g), rng.standard_normal(g)
    fed = {key: v.copy() for key, v in base.items()}
    fed["dgu_col_q"][q] += dgu
    fed["aw_col_q"][q] += daw
    r1 = oracle.moe_mx(d, x, ids, w, wq, dy=dy, wd=wd, wgrad_C=1, fed=fed)
    want = (np.outer(dgu[:g], xq_col[q]), np.outer(dgu[g:], xq_col[q]), np.outer(yq_col[q], daw))
    for got1, got0, wnt in zip(r1[3:], r0[3:], want):
        diff = got1 - got0
        assert np.abs(diff[e] - wnt).max() <= 1e-10 * np.abs(wnt).max()
        assert np.array_equal(np.delete(got1, e, 0), np.delete(got0, e, 0))
