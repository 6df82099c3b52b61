"""MXFP8 variant (readings R28, R28b, R28c) on the GPU vs the oracle
(run with -m gpu).

The oracle decides every E4M3 code on the EXACT value of its operand.  Quantising the layer's bf16
inputs (x, dY) is exact in any precision, so those codes and scales must equal the oracle's bit
for bit.  Codes of intermediates (a, dG || dU, a_w) are decided by the kernels on the values they
hold, so each one is checked for VALIDITY against the exact value (tests/mx_check.py: a rounding
of some value inside the kernel's precision window), and everything downstream of the decisions is
compared with the oracle FED with the GPU's own decisions (oracle.moe_mx(fed=...)):
  - y and dx against the fed oracle: FED_TOL = 5e-3 (max-norm; bf16 output rounding 2^-9 plus fp32
    accumulation);
  - d_score and BF16-operand dW involve no decision: against the oracle with MX_TOL = 1e-2 (the
    bf16 storage of G, U, dG, dU between fp32-accumulated GEMMs, as in the BF16 path);
  - MX weight gradients (R28c) against the fed oracle with FED_TOL.
The gap between the MX result and the exact (unquantised) oracle - the quantisation error itself,
a few % - is asserted present, not gated."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21431_b200 import capi, layer
from tests import mx_check as mc
from tests.harness import GpuRun, _np_in, make_problem, oracle_dims, rel_err, tile_covering_tokens

pytestmark = pytest.mark.gpu
MX_TOL = 1e-2
FED_TOL = 5e-3
# precision windows of the kernels' decisions (tests/mx_check.windows, propagated from the exact G, U, dA):
# a from the fp32 accumulators of the gate/up GEMM (EPS_FP32); dG || dU and a_w from the dA epilogue, which
# reads the recomputed G || U as stored (bf16, reading R19) and rounds dG, dU, a_w to bf16 before
# quantising (EPS_BF16)
EPS_FP32 = 2.0 ** -20
EPS_BF16 = 2.0 ** -8


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_mx_quantize_bit_exact():
    gen = torch.Generator().manual_seed(3)
    rows, K = 256, 384
    x = torch.randn(rows, K, generator=gen) * torch.pow(2.0, torch.randint(-30, 30, (rows, 1), generator=gen).float())
    x[5, :32] = 0.0                        # an all-zero block
    x[7, 40] = 1e30                        # a block with a huge outlier
    xb = x.to(torch.bfloat16)
    codes, scales = layer.mx_quantize(xb.cuda())
    torch.cuda.synchronize()
    ref_codes, ref_scales = oracle.mx_quantize(xb.view(torch.int16).numpy().view(np.uint16), "bf16")
    assert np.array_equal(codes.cpu().numpy(), ref_codes)
    assert np.array_equal(mc.sf_rows(scales.cpu().numpy(), rows, K), ref_scales.reshape(rows, K // 32))


def _mx_run(p, C, debug=False, **mf_kw):
    """fwd + bwd of the MX variant; with debug, the decisions of every chunk (memfine_debug_mx)."""
    run = GpuRun(p)
    run.mf.close()
    run.mf = layer.MemFine(p.T, p.h, p.g, p.E, p.k, mx=True, **mf_kw)
    run.mf.mx_quantize_weights(run.wg, run.wu, run.wd)
    if debug:
        run.mf.set_debug(True)
    y, st, _, _ = run.fwd(C)
    assert st == 0
    cap = {"fwd": [], "bwd": []}
    if debug:
        cap["fwd"] = [(run.mf.debug_rows(j), run.mf.debug_mx(j, 0)) for j in range(C)]
    (dx, dwg, dwu, dwd, ds), st, _, _ = run.bwd(C)
    assert st == 0
    if debug:
        wg = bool(mf_kw.get("mx_wgrad"))
        cap["bwd"] = [(run.mf.debug_rows(j), run.mf.debug_mx(j, 1),
                       [run.mf.debug_mx(j, w) for w in (2, 3, 4, 5)] if wg else None) for j in range(C)]
    out = dict(y=y.float().cpu().numpy(), dx=dx.float().cpu().numpy(), dscore=ds.cpu().numpy(),
               dwg=dwg.cpu().numpy(), dwu=dwu.cpu().numpy(), dwd=dwd.cpu().numpy())
    run.mf.close()
    return out, cap


def _inputs(p):
    d = oracle_dims(p)
    a = [_np_in(t, p.dtype) for t in (p.x, p.dy, p.wg, p.wu, p.wd)]
    return d, a, p.ids.numpy(), p.w.numpy().astype(np.float64)


def _check_and_feed(p, cap, mx_wgrad=False, wgrad_C=0):
    """Validity of every GPU decision against the oracle's exact values, and the fed dict."""
    d, a, ids, w = _inputs(p)
    nq, g, h, k = p.T * p.k, p.g, p.h, p.k
    wq = oracle.mx_weights(d, a[2], a[3], a[4])
    *_, ex = oracle.moe_mx(d, a[0], ids, w, wq, dy=a[1], wd=a[4], return_exact=True)
    tol_a = mc.windows(ex["gu"], ex["da"], w.reshape(-1), EPS_FP32)[0]
    _, tol_dgu, tol_aw = mc.windows(ex["gu"], ex["da"], w.reshape(-1), EPS_BF16)
    fed = {"a_q": np.zeros((nq, g)), "dgu_q": np.zeros((nq, 2 * g))}
    if mx_wgrad:
        fed.update(dgu_col_q=np.zeros((nq, 2 * g)), aw_col_q=np.zeros((nq, g)))
    flips = {}
    x_bits = a[0].view(np.uint16)
    dy_bits = a[1].view(np.uint16)
    for j, (src, (codes, sf)) in enumerate(cap["fwd"]):
        if not len(src):
            continue
        v, c, E = mc.rowwise_per_copy(codes, sf, src, nq, g)
        q = src[src >= 0]
        fed["a_q"][q] = v[q]
        flips[f"a/{j}"] = mc.check_decisions_tol(ex["a"][q].reshape(-1, 32), c[q].reshape(-1, 32), E[q].reshape(-1),
                                                 tol_a[q].reshape(-1, 32), what=f"a chunk {j}")
    for j, (src, (codes, sf), cols) in enumerate(cap["bwd"]):
        if not len(src):
            continue
        v, c, E = mc.rowwise_per_copy(codes, sf, src, nq, 2 * g)
        q = src[src >= 0]
        fed["dgu_q"][q] = v[q]
        flips[f"dgu/{j}"] = mc.check_decisions_tol(ex["dgu"][q].reshape(-1, 32), c[q].reshape(-1, 32),
                                                   E[q].reshape(-1), tol_dgu[q].reshape(-1, 32),
                                                   what=f"dG||dU chunk {j}")
        if not mx_wgrad:
            continue
        rp = len(src)
        live = src >= 0
        tok = np.where(live, src // k, 0)
        # exact operand rows of the expert-major layout (padding rows are zero)
        xr = np.where(live[:, None], x_bits[tok], 0).astype(np.uint16)
        yr = np.where(live[:, None], dy_bits[tok], 0).astype(np.uint16)
        qs = np.where(live, src, 0)
        gur = np.where(live[:, None], ex["dgu"][qs], 0.0)
        awr = np.where(live[:, None], ex["a"][qs] * w.reshape(-1)[qs][:, None], 0.0)
        tgr = np.where(live[:, None], tol_dgu[qs], 0.0)
        tar = np.where(live[:, None], tol_aw[qs], 0.0)
        (xq, xs), (yq, ys), (gq, gs), (aq, as_) = cols
        for name, (cq, cs), rows_bits in (("x", (xq, xs), xr), ("dY", (yq, ys), yr)):
            # the layer's bf16 inputs: decisions bit-exact with the oracle's quantiser, columnwise blocks
            vt, ct, Et = mc.colwise_rows(cq, cs, rp)
            ref_c, ref_s = oracle.mx_quantize(np.ascontiguousarray(mc.col_blocks(rows_bits, rp)), "bf16")
            assert np.array_equal(mc.col_blocks(ct, rp).reshape(-1), ref_c.reshape(-1)), f"{name} codes chunk {j}"
            assert np.array_equal(Et.reshape(-1) + 127, ref_s.astype(np.int64)), f"{name} scales chunk {j}"
        for name, (cq, cs), exact, tl, key in (("dG||dU col", (gq, gs), gur, tgr, "dgu_col_q"),
                                               ("a_w col", (aq, as_), awr, tar, "aw_col_q")):
            vt, ct, Et = mc.colwise_rows(cq, cs, rp)
            flips[f"{name}/{j}"] = mc.check_decisions_tol(mc.col_blocks(exact, rp), mc.col_blocks(ct, rp),
                                                          Et.reshape(-1), mc.col_blocks(tl, rp),
                                                          what=f"{name} chunk {j}")
            fed[key][src[live]] = vt[live]
    return fed, flips, ex


def _oracle(p, fed=None, wgrad_C=0):
    d, a, ids, w = _inputs(p)
    wq = oracle.mx_weights(d, a[2], a[3], a[4])
    y, dx, ds, dwg, dwu, dwd = oracle.moe_mx(d, a[0], ids, w, wq, dy=a[1], wd=a[4], wgrad_C=wgrad_C, fed=fed)
    return dict(y=y, dx=dx, dscore=ds, dwg=dwg, dwu=dwu, dwd=dwd)


def _gate(got, fed_ref, own_ref, wgrad):
    """y, dx (and MX dW) vs the fed oracle; d_score and BF16-operand dW vs the oracle."""
    errs = {}
    for key in ("y", "dx"):
        errs[key] = (rel_err(got[key], fed_ref[key]), FED_TOL)
    errs["dscore"] = (rel_err(got["dscore"], own_ref["dscore"]), MX_TOL)
    for key in ("dwg", "dwu", "dwd"):
        errs[key] = (rel_err(got[key], fed_ref[key]), FED_TOL) if wgrad else (rel_err(got[key], own_ref[key]), MX_TOL)
    bad = {k_: v for k_, v in errs.items() if not v[0] <= v[1]}
    assert not bad, bad
    return {k_: f"{v[0]:.2e}" for k_, v in errs.items()}


@pytest.mark.parametrize("T,h,g,E,k,C,zipf", [(300, 256, 384, 4, 2, 1, 0.0), (300, 256, 384, 4, 2, 2, 1.2),
                                              (700, 384, 640, 8, 2, 3, 1.2)])
def test_mx_layer_matches_mx_oracle(T, h, g, E, k, C, zipf):
    # (h=384, g=640: ragged last N tiles of the down / dA / dX GEMMs, incl. a half scale chunk)
    p = make_problem(T, h, g, E, k, zipf_s=zipf, seed=31)
    got, cap = _mx_run(p, C, debug=True)
    fed, flips, _ = _check_and_feed(p, cap)
    fed_ref, own_ref = _oracle(p, fed), _oracle(p)
    errs = _gate(got, fed_ref, own_ref, wgrad=False)
    d, a, ids, w = _inputs(p)
    exact_y = oracle.moe_forward(d, a[0], ids, w, a[2], a[3], a[4])
    print("mx vs fed oracle", errs, "| decisions differing from the exact-value ones",
          {k_: f"{v:.1e}" for k_, v in flips.items()}, "| vs exact y", f"{rel_err(got['y'], exact_y):.2e}")
    # the variant is really quantised: the GPU result sits at the MX oracle, not at the exact one
    assert rel_err(got["y"], fed_ref["y"]) < 0.2 * rel_err(got["y"], exact_y)
    assert all(v < 0.05 for v in flips.values()), flips


def test_mx_errors():
    import ctypes
    d = layer.make_dims(256, 64, 128, 4, 2, mx=True)        # hidden % 128 != 0
    out = ctypes.c_uint64()
    assert capi.lib().memfine_mx_weights_bytes(ctypes.byref(d), ctypes.byref(out)) == capi.ERR_INVALID_ARG
    p = make_problem(256, 128, 128, 4, 2, seed=2)
    mf = layer.MemFine(p.T, p.h, p.g, p.E, p.k, mx=True)
    ws = torch.empty(1 << 24, dtype=torch.uint8, device="cuda:0")
    g = lambda t: t.cuda()
    with pytest.raises(capi.MemfineError):                    # weights not quantised yet
        mf.moe_fwd(g(p.x), g(p.ids), g(p.w), g(p.wg), g(p.wu), g(p.wd), 1, ws)
    small = torch.empty(16, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(capi.MemfineError):
        mf.mx_quantize_weights(g(p.wg), g(p.wu), g(p.wd), wq=small)


@pytest.mark.parametrize("C,mx_wgrad", [(1, False), (3, False), (2, True)])
def test_mx_nccl_ep_path_bit_identical(C, mx_wgrad):
    """MXFP8 over the NCCL transport (MEMFINE_FLAG_EP_PATH, 1-rank communicator): the rows travel
    in bf16 and are quantised on arrival - the same codes the EP = 1 gather writes - so every
    output equals the EP = 1 MX path bit for bit - except d_score, whose per-row partials from
    the dA GEMM's N tiles (g = 384: two) meet in an fp32 atomicAdd of run-dependent order."""
    p = make_problem(700, 256, 384, 8, 2, zipf_s=1.2, seed=5)
    a, _ = _mx_run(p, C, mx_wgrad=mx_wgrad)
    b, _ = _mx_run(p, C, ep_path=True, mx_wgrad=mx_wgrad)
    for key in a:
        if key == "dscore":
            assert rel_err(b[key], a[key]) <= 1e-6
        else:
            np.testing.assert_array_equal(a[key], b[key], err_msg=key)


@pytest.mark.parametrize("T,h,g,E,k,C,zipf", [(300, 256, 384, 4, 2, 1, 0.0), (700, 384, 640, 8, 2, 3, 1.2),
                                              (2048, 256, 256, 4, 2, 2, 1.2)])
def test_mx_wgrad_matches_mx_oracle(T, h, g, E, k, C, zipf):
    """MEMFINE_FLAG_MX_WGRAD (reading R28c): the weight gradients from columnwise MXFP8 operands -
    blocks of 32 copies of an expert inside a chunk.  x's and dY's columnwise codes bit-exact with the
    oracle's quantiser, dG || dU's and a_w's valid, and dW against the oracle fed with them."""
    p = make_problem(T, h, g, E, k, zipf_s=zipf, seed=37)
    got, cap = _mx_run(p, C, debug=True, mx_wgrad=True)
    fed, flips, _ = _check_and_feed(p, cap, mx_wgrad=True, wgrad_C=C)
    fed_ref = _oracle(p, fed, wgrad_C=C)
    own_ref = _oracle(p, None, wgrad_C=C)
    errs = _gate(got, fed_ref, own_ref, wgrad=True)
    print("mx-wgrad vs fed oracle", errs, {k_: f"{v:.1e}" for k_, v in flips.items()})
    # the gradients really are quantised: at the MX-wgrad definition, away from BF16 operands
    bf16w = _oracle(p, fed, wgrad_C=0)
    for key in ("dwg", "dwu", "dwd"):
        assert rel_err(got[key], fed_ref[key]) < 0.5 * rel_err(got[key], bf16w[key]), key
    assert all(v < 0.05 for v in flips.values()), flips


@pytest.mark.parametrize("C", [1, 2])
def test_mx_wgrad_empty_expert_and_ragged_chunks(C):
    """MX weight gradients with an expert that receives no copies (its dW tiles written as zeros by the
    first chunk, skipped by the accumulating ones), an expert whose copies fall in one chunk only, and
    chunks with ragged 32-copy blocks."""
    T, E, k = 333, 6, 2
    rng = np.random.default_rng(41)
    ids = np.stack([rng.choice([0, 1, 2, 4], k, replace=False) for _ in range(T)]).astype(np.int32)  # 3, 5 empty
    ids[T // 2:][ids[T // 2:] == 4] = 1          # expert 4 only in the first half of the tokens
    p = make_problem(T, 256, 256, E, k, seed=43, ids=ids)
    got, cap = _mx_run(p, C, debug=True, mx_wgrad=True)
    fed, _, _ = _check_and_feed(p, cap, mx_wgrad=True, wgrad_C=C)
    ref = _oracle(p, fed, wgrad_C=C)
    for key in ("dwg", "dwu", "dwd"):
        assert np.all(got[key][3] == 0) and np.all(got[key][5] == 0), key
        assert rel_err(got[key], ref[key]) <= FED_TOL, key


@pytest.mark.parametrize("mx_wgrad", [False, True])
def test_mx_fewer_tokens_than_chunks(mx_wgrad):
    """T < C (empty chunks issue nothing) with every copy on one expert (the others empty)."""
    T, E, k, C = 5, 4, 2, 8
    ids = np.tile(np.array([[0, 2]], np.int32), (T, 1))
    p = make_problem(T, 128, 256, E, k, seed=47, ids=ids)
    got, cap = _mx_run(p, C, debug=True, mx_wgrad=mx_wgrad)
    fed, _, _ = _check_and_feed(p, cap, mx_wgrad=mx_wgrad, wgrad_C=C if mx_wgrad else 0)
    _gate(got, _oracle(p, fed, wgrad_C=C if mx_wgrad else 0), _oracle(p, None, wgrad_C=C if mx_wgrad else 0),
          wgrad=mx_wgrad)
    for key in ("dwg", "dwu", "dwd"):
        assert np.all(got[key][1] == 0) and np.all(got[key][3] == 0), key


@pytest.mark.parametrize("mx_wgrad", [False, True])
def test_mx_mixtral_full_size_sampled(mx_wgrad):
    """The MXFP8 variant at BASELINE configs[1]'s shape in bench.py's launch configuration (EP = 1,
    16K tokens, C = 1): tokens sampled across the expert segments' m-tiles (below); their a and
    dG || dU decisions valid against the exact values, and y, dx of those tokens against the oracle's
    MX layer fed with them (weights quantised one expert at a time); d_score against the oracle.  (The
    BF16 full-size tests sample every m-tile.)"""
    p = make_problem(16384, 4096, 14336, 8, 2, zipf_s=1.2, seed=5)
    got, cap = _mx_run(p, 1, debug=True, mx_wgrad=mx_wgrad)
    src_f, (ca, sa) = cap["fwd"][0]
    src_b, (cg, sg), _ = cap["bwd"][0]
    # every 6th m-tile and every segment's ragged last tile (the fp64 MX evaluator quantises each expert's
    # weights in five layouts and runs ~6 h x g matvecs per copy: ~40 tokens keep the test near a minute)
    toks = tile_covering_tokens(src_f, p.k, np.random.default_rng(1), stride=6)
    d, a, ids, w = _inputs(p)
    sel = (toks[:, None] * p.k + np.arange(p.k)[None, :]).reshape(-1)

    def pick(src, codes, sf, width):   # the sampled copies' rows only (the full arrays are GBs in fp64)
        row_of = np.full(p.T * p.k, -1, np.int64)
        row_of[src[src >= 0]] = np.nonzero(src >= 0)[0]
        r = row_of[sel]
        assert (r >= 0).all()
        E = mc.sf_rows(sf, codes.shape[0], width).astype(np.int64)[r] - 127
        return mc.deq(codes[r], E), codes[r], E

    va, ca_c, Ea = pick(src_f, ca, sa, p.g)
    vg, cg_c, Eg = pick(src_b, cg, sg, 2 * p.g)
    fed = {"a_q": va, "dgu_q": vg}
    ry, rdx, rds, ex = oracle.moe_mx_tokens(d, toks, a[0], a[1], ids, w, a[2], a[3], a[4], fed=fed, return_exact=True)
    tol_a = mc.windows(ex["gu"], ex["da"], w[toks].reshape(-1), EPS_FP32)[0]
    _, tol_dgu, _ = mc.windows(ex["gu"], ex["da"], w[toks].reshape(-1), EPS_BF16)
    fa = mc.check_decisions_tol(ex["a"].reshape(-1, 32), ca_c.reshape(-1, 32), Ea.reshape(-1),
                                tol_a.reshape(-1, 32), what="a")
    fg = mc.check_decisions_tol(ex["dgu"].reshape(-1, 32), cg_c.reshape(-1, 32), Eg.reshape(-1),
                                tol_dgu.reshape(-1, 32), what="dG||dU")
    errs = {"y": rel_err(got["y"][toks], ry), "dx": rel_err(got["dx"][toks], rdx)}
    assert all(v <= FED_TOL for v in errs.values()), errs
    assert rel_err(got["dscore"][toks], rds) <= MX_TOL
    print(f"{len(toks)} tokens", errs, f"differing decisions a {fa:.1e} dG||dU {fg:.1e}")
    for key in ("dwg", "dwu", "dwd"):
        assert np.isfinite(got[key]).all() and np.abs(got[key]).max() > 0, key
