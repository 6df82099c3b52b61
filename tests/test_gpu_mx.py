"""MXFP8 variant (reading R28) on the GPU vs the oracle (run with -m gpu).

Quantisation is an integer decision taken on bf16 inputs, exact in fp32 and fp64 alike, so the
GPU's codes and scales must equal the oracle's bit for bit.  The layer is compared with the
oracle's MX layer (oracle.moe_mx: the same quantised operands, fp64 arithmetic, codes of a and
dG||dU decided in the kernel's precision - reading R28b).  Tolerance MX_TOL = 1e-2 (max-norm):
the bf16 output rounding (2^-9) plus the fp32-vs-fp64 accumulation of G, U, u before a code is
decided, where a rare flip moves one element by one E4M3 step (2^-4); measured 1.5e-3..4.8e-3.
The gap between the MX oracle and the exact oracle (the quantisation error itself, ~6e-2) is
reported, not gated."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21431_b200 import capi, layer
from tests.harness import GpuRun, _np_in, make_problem, oracle_dims, rel_err

pytestmark = pytest.mark.gpu
MX_TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _sf_rows(scales_chunked: np.ndarray, rows: int, K: int) -> np.ndarray:
    """Scale codes from the tcgen05 chunk layout back to [rows][K/32] (the header's formula)."""
    r = np.arange(rows)[:, None]
    b = np.arange(K // 32)[None, :]
    off = ((r // 128) * (K // 128) + b // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + b % 4
    return scales_chunked[off]


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
    assert np.array_equal(_sf_rows(scales.cpu().numpy(), rows, K), ref_scales.reshape(rows, K // 32))


def _mx_run(p, C, **mf_kw):
    run = GpuRun(p)
    run.mf.close()
    run.mf = layer.MemFine(p.T, p.h, p.g, p.E, p.k, mx=True, **mf_kw)
    run.mf.mx_quantize_weights(run.wg, run.wu, run.wd)
    y, st, _, _ = run.fwd(C)
    assert st == 0
    (dx, dwg, dwu, dwd, ds), st, _, _ = run.bwd(C)
    assert st == 0
    return dict(y=y.float().cpu().numpy(), dx=dx.float().cpu().numpy(), dscore=ds.cpu().numpy(),
                dwg=dwg.cpu().numpy(), dwu=dwu.cpu().numpy(), dwd=dwd.cpu().numpy())


def _mx_oracle(p, wgrad_C=0):
    d = oracle_dims(p)
    a = [_np_in(t, p.dtype) for t in (p.x, p.dy, p.wg, p.wu, p.wd)]
    ids, w = p.ids.numpy(), p.w.numpy().astype(np.float64)
    wq = oracle.mx_weights(d, a[2], a[3], a[4])
    y, dx, ds, dwg, dwu, dwd = oracle.moe_mx(d, a[0], ids, w, wq, dy=a[1], wd=a[4], wgrad_C=wgrad_C)
    exact_y = oracle.moe_forward(d, a[0], ids, w, a[2], a[3], a[4])
    return dict(y=y, dx=dx, dscore=ds, dwg=dwg, dwu=dwu, dwd=dwd), exact_y


@pytest.mark.parametrize("T,h,g,E,k,C,zipf", [(300, 256, 384, 4, 2, 1, 0.0), (300, 256, 384, 4, 2, 2, 1.2),
                                              (700, 384, 640, 8, 2, 3, 1.2)])
def test_mx_layer_matches_mx_oracle(T, h, g, E, k, C, zipf):
    # (h=384, g=640: ragged last N tiles of the down / dA / dX GEMMs, incl. a half scale chunk)
    p = make_problem(T, h, g, E, k, zipf_s=zipf, seed=31)
    got = _mx_run(p, C)
    ref, exact_y = _mx_oracle(p)
    t_ = MX_TOL
    errs = {key: rel_err(got[key], ref[key]) for key in ("y", "dx", "dscore", "dwg", "dwu", "dwd")}
    print("mx vs mx-oracle", {k_: f"{v:.2e}" for k_, v in errs.items()},
          "| vs exact y", f"{rel_err(got['y'], exact_y):.2e}")
    for key, e in errs.items():
        assert e <= t_, f"{key}: {e}"
    # the variant is really quantised: the GPU result sits at the MX oracle, not at the exact one
    assert rel_err(got["y"], ref["y"]) < 0.5 * rel_err(got["y"], exact_y)


def test_mx_errors():
    d = layer.make_dims(256, 64, 128, 4, 2, mx=True)        # hidden % 128 != 0
    out = __import__("ctypes").c_uint64()
    assert capi.lib().memfine_mx_weights_bytes(__import__("ctypes").byref(d), __import__("ctypes").byref(out)) \
        == capi.ERR_INVALID_ARG
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
    a = _mx_run(p, C, mx_wgrad=mx_wgrad)
    b = _mx_run(p, C, ep_path=True, mx_wgrad=mx_wgrad)
    for key in a:
        if key == "dscore":
            assert rel_err(b[key], a[key]) <= 1e-6
        else:
            np.testing.assert_array_equal(a[key], b[key], err_msg=key)


@pytest.mark.parametrize("T,h,g,E,k,C,zipf", [(300, 256, 384, 4, 2, 1, 0.0), (700, 384, 640, 8, 2, 3, 1.2),
                                              (2048, 256, 256, 4, 2, 2, 1.2)])
def test_mx_wgrad_matches_mx_oracle(T, h, g, E, k, C, zipf):
    """MEMFINE_FLAG_MX_WGRAD (reading R28c): the weight gradients from columnwise MXFP8 operands -
    blocks of 32 copies of an expert inside a chunk - against the oracle's definition of exactly
    that (oracle.moe_mx(wgrad_C=C)); every other output is the MX variant's as before."""
    p = make_problem(T, h, g, E, k, zipf_s=zipf, seed=37)
    got = _mx_run(p, C, mx_wgrad=True)
    ref, _ = _mx_oracle(p, wgrad_C=C)
    ref_bf16w, _ = _mx_oracle(p, wgrad_C=0)
    errs = {key: rel_err(got[key], ref[key]) for key in ("y", "dx", "dscore", "dwg", "dwu", "dwd")}
    print("mx-wgrad vs oracle", {k_: f"{v:.2e}" for k_, v in errs.items()})
    for key, e in errs.items():
        assert e <= MX_TOL, f"{key}: {e}"
    # the gradients really are quantised: closer to the MX-wgrad definition than to BF16 operands
    for key in ("dwg", "dwu", "dwd"):
        assert rel_err(got[key], ref[key]) < 0.5 * rel_err(got[key], ref_bf16w[key]), key


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
    got = _mx_run(p, C, mx_wgrad=True)
    ref, _ = _mx_oracle(p, wgrad_C=C)
    for key in ("dwg", "dwu", "dwd"):
        assert np.all(got[key][3] == 0) and np.all(got[key][5] == 0), key
        assert rel_err(got[key], ref[key]) <= MX_TOL, key


@pytest.mark.parametrize("mx_wgrad", [False, True])
def test_mx_fewer_tokens_than_chunks(mx_wgrad):
    """T < C (empty chunks issue nothing) with every copy on one expert (the others empty)."""
    T, E, k, C = 5, 4, 2, 8
    ids = np.tile(np.array([[0, 2]], np.int32), (T, 1))
    p = make_problem(T, 128, 256, E, k, seed=47, ids=ids)
    got = _mx_run(p, C, mx_wgrad=mx_wgrad)
    ref, _ = _mx_oracle(p, wgrad_C=C if mx_wgrad else 0)
    for key in ("y", "dx", "dscore", "dwg", "dwu", "dwd"):
        assert rel_err(got[key], ref[key]) <= MX_TOL, key
    for key in ("dwg", "dwu", "dwd"):
        assert np.all(got[key][1] == 0) and np.all(got[key][3] == 0), key


@pytest.mark.parametrize("mx_wgrad", [False, True])
def test_mx_mixtral_full_size_sampled(mx_wgrad):
    """The MXFP8 variant at BASELINE configs[1]'s shape in bench.py's launch configuration (EP = 1,
    16K tokens, C = 1): Y, dX and d_score of sampled tokens against the oracle's MX layer (weights
    quantised one expert at a time); the weight gradients finite and non-zero."""
    p = make_problem(16384, 4096, 14336, 8, 2, zipf_s=1.2, seed=5)
    got = _mx_run(p, 1, mx_wgrad=mx_wgrad)
    toks = np.random.default_rng(1).choice(16384, 6, replace=False)
    d = oracle_dims(p)
    a = [_np_in(t, p.dtype) for t in (p.x, p.dy, p.wg, p.wu, p.wd)]
    ry, rdx, rds = oracle.moe_mx_tokens(d, toks, a[0], a[1], p.ids.numpy(), p.w.numpy().astype(np.float64),
                                        a[2], a[3], a[4])
    for key, ref in (("y", ry), ("dx", rdx), ("dscore", rds)):
        assert rel_err(got[key][toks], ref) <= MX_TOL, key
    for key in ("dwg", "dwu", "dwd"):
        assert np.isfinite(got[key]).all() and np.abs(got[key]).max() > 0, key
