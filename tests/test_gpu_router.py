"""Router step on the GPU vs the oracle (run with -m gpu).

Top-k is an integer decision taken on floating-point logits: the GPU's selected set must be a valid
top-k of the oracle's fp64 logits up to the fp32 accumulation error (the unique part), scores are
compared with the oracle's softmax over the GPU-selected experts, and the backward is compared on
the GPU's own ids / scores."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2511_21431_b200 import layer
from tests.harness import rel_err, tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _np(t, dtype):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16) if dtype == torch.bfloat16 else \
        t.contiguous().numpy().astype(np.float32)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("T,h,E,k", [(300, 64, 8, 2), (1000, 512, 256, 8), (77, 128, 64, 6)])
def test_router_fwd_bwd(dtype, T, h, E, k):
    dev = "cuda:0"
    x = synth.make_x(T, h, rank=3, dtype=dtype)
    gen = torch.Generator().manual_seed(11)
    wr = (torch.randn(E, h, generator=gen) / h ** 0.5).to(dtype)
    mf = layer.MemFine(T, h, 64, E, k, dtype=dtype)
    logits = torch.empty((T, E), dtype=torch.float32, device=dev)
    xd, wd = x.to(dev), wr.to(dev)
    ids, scores = mf.router_fwd(xd, wd, logits=logits)
    assert mf.sync() == 0
    d = oracle.Dims(T=T, h=h, g=1, E=E, k=k, in_dtype="bf16" if dtype == torch.bfloat16 else "f32")
    ref_logits, ref_ids, ref_scores = oracle.router_forward(d, _np(x, dtype), _np(wr, dtype))
    assert rel_err(logits.cpu().numpy(), ref_logits) <= 1e-5
    g_ids = ids.cpu().numpy()
    # the unique part: a valid top-k of the exact logits (up to the fp32 accumulation error)
    eps = 1e-5 * np.abs(ref_logits).max()
    for t in range(T):
        sel = g_ids[t]
        assert len(set(sel.tolist())) == k and sel.min() >= 0 and sel.max() < E
        rest = np.setdiff1d(np.arange(E), sel)
        if len(rest):
            assert ref_logits[t, sel].min() >= ref_logits[t, rest].max() - eps
    assert (g_ids == ref_ids).mean() > 0.99
    # scores: softmax over the GPU-selected experts of the exact logits
    sl = np.take_along_axis(ref_logits, g_ids.astype(np.int64), 1)
    sl = np.exp(sl - sl.max(1, keepdims=True))
    sref = sl / sl.sum(1, keepdims=True)
    assert rel_err(scores.cpu().numpy(), sref) <= 1e-5
    # backward on the GPU's ids / scores
    ds = torch.from_numpy(np.random.default_rng(2).standard_normal((T, k)).astype(np.float32))
    dx0 = synth.make_dy(T, h, rank=4, dtype=dtype).to(dev)
    dwr0 = torch.randn(E, h, generator=gen).to(dev)
    dx, dwr = mf.router_bwd(xd, wd, ids, scores, ds.to(dev), dx=dx0.clone(), accumulate_dx=True,
                            dw_router=dwr0.clone(), accumulate_dw=True)
    assert mf.sync() == 0
    rdx, rdw = oracle.router_backward(d, _np(x, dtype), _np(wr, dtype), g_ids, scores.cpu().numpy().astype(np.float64),
                                      ds.numpy().astype(np.float64))
    t_ = tol(dtype)
    # accumulate mode: the whole output (dx0 + router term, rounded once to dtype) and dW
    assert rel_err(dx.float().cpu().numpy(), dx0.float().cpu().numpy() + rdx) <= t_
    assert rel_err(dwr.cpu().numpy(), dwr0.cpu().numpy() + rdw) <= t_
    # overwrite mode
    dx2, dwr2 = mf.router_bwd(xd, wd, ids, scores, ds.to(dev))
    assert mf.sync() == 0
    assert rel_err(dwr2.cpu().numpy(), rdw) <= t_
    assert rel_err(dx2.float().cpu().numpy(), rdx) <= t_


@pytest.mark.parametrize("T,h,E,k,bwd", [(16384, 4096, 8, 2, True), (8192, 7168, 256, 8, False)])
def test_router_full_size(T, h, E, k, bwd):
    """BASELINE sizes (Mixtral, DSv3) in bf16, the launch configuration tools/router_bench.py times:
    logits / ids / scores on a sample of tokens (rows are independent); dx and dW_r over all tokens
    at the Mixtral size (the oracle's dW_r loop is O(E T h): ~40 s at the DSv3 size, so there the
    backward is covered by the small cases above)."""
    dev = "cuda:0"
    dtype = torch.bfloat16
    x = synth.make_x(T, h, rank=5, dtype=dtype)
    gen = torch.Generator().manual_seed(13)
    wr = (torch.randn(E, h, generator=gen) / h ** 0.5).to(dtype)
    mf = layer.MemFine(T, h, 64, E, k, dtype=dtype)
    logits = torch.empty((T, E), dtype=torch.float32, device=dev)
    xd, wd = x.to(dev), wr.to(dev)
    ids, scores = mf.router_fwd(xd, wd, logits=logits)
    assert mf.sync() == 0
    rng = np.random.default_rng(T)
    sample = np.unique(np.concatenate([[0, T - 1], rng.choice(T, 384, replace=False)]))
    d = oracle.Dims(T=len(sample), h=h, g=1, E=E, k=k, in_dtype="bf16")
    xs = _np(x, dtype)[sample]
    ref_logits, _, _ = oracle.router_forward(d, xs, _np(wr, dtype))
    assert rel_err(logits.cpu().numpy()[sample], ref_logits) <= 1e-5
    g_ids = ids.cpu().numpy()
    eps = 1e-5 * np.abs(ref_logits).max()
    for i, t in enumerate(sample):
        sel = g_ids[t]
        assert len(set(sel.tolist())) == k and sel.min() >= 0 and sel.max() < E
        rest = np.setdiff1d(np.arange(E), sel)
        assert ref_logits[i, sel].min() >= ref_logits[i, rest].max() - eps
    sl = np.take_along_axis(ref_logits, g_ids[sample].astype(np.int64), 1)
    sl = np.exp(sl - sl.max(1, keepdims=True))
    sref = sl / sl.sum(1, keepdims=True)
    # softmax is 2-Lipschitz per score in the max logit error: |ds_j| <= s_j (|dl_j| + sum_q s_q |dl_q|)
    # <= 2 s_j max|dl|, so the scores' bound follows from the logits' measured error (K = h long sums
    # on the tensor cores put max|dl| at a few 1e-5 at the DSv3 size)
    dl = np.abs(logits.cpu().numpy()[sample] - ref_logits).max()
    e_s = np.abs(scores.cpu().numpy()[sample] - sref).max()
    print(f"router full size T={T} E={E}: max|dlogit| {dl:.2e}, max|dscore| {e_s:.2e}")
    assert e_s <= 2 * dl * sref.max() + 1e-6
    if not bwd:
        return
    # backward over all tokens (dW_r needs every row)
    ds = torch.from_numpy(np.random.default_rng(3).standard_normal((T, k)).astype(np.float32))
    dx, dwr = mf.router_bwd(xd, wd, ids, scores, ds.to(dev))
    assert mf.sync() == 0
    dfull = oracle.Dims(T=T, h=h, g=1, E=E, k=k, in_dtype="bf16")
    rdx, rdw = oracle.router_backward(dfull, _np(x, dtype), _np(wr, dtype), g_ids,
                                      scores.cpu().numpy().astype(np.float64), ds.numpy().astype(np.float64))
    e_dx = rel_err(dx.float().cpu().numpy(), rdx)
    e_dw = rel_err(dwr.cpu().numpy(), rdw)
    print(f"router full size T={T} E={E}: dx rel {e_dx:.2e}, dW_r rel {e_dw:.2e}")
    assert e_dx <= tol(dtype)
    assert e_dw <= tol(dtype)


@pytest.mark.parametrize("T,h,E,k", [(0, 64, 8, 2), (1, 64, 1, 1), (5, 128, 33, 16), (130, 64, 1024, 3)])
def test_router_edges(T, h, E, k):
    """Degenerate router shapes in bf16 (the cuBLAS path): no tokens (dW_r overwritten with zeros or
    left as is), one expert, k = 16 (the largest the kernels take), E = 1024 (the top-k mask's limit)."""
    dev = "cuda:0"
    dtype = torch.bfloat16
    x = synth.make_x(max(T, 1), h, rank=6, dtype=dtype)[:T]
    gen = torch.Generator().manual_seed(17)
    wr = (torch.randn(E, h, generator=gen) / h ** 0.5).to(dtype)
    mf = layer.MemFine(T, h, 64, E, k, dtype=dtype)
    xd, wd = x.to(dev), wr.to(dev)
    ids, scores = mf.router_fwd(xd, wd)
    ds = torch.from_numpy(np.random.default_rng(4).standard_normal((T, k)).astype(np.float32)).to(dev)
    dw0 = torch.randn(E, h, generator=gen).to(dev)
    dx, dwr = mf.router_bwd(xd, wd, ids, scores, ds, dw_router=dw0.clone(), accumulate_dw=True)
    dx2, dwr2 = mf.router_bwd(xd, wd, ids, scores, ds, dw_router=torch.full((E, h), 7.0, device=dev))
    assert mf.sync() == 0
    if T == 0:
        assert torch.equal(dwr, dw0) and not dwr2.any()
        return
    d = oracle.Dims(T=T, h=h, g=1, E=E, k=k, in_dtype="bf16")
    ref_logits, ref_ids, _ = oracle.router_forward(d, _np(x, dtype), _np(wr, dtype))
    g_ids = ids.cpu().numpy()
    eps = 1e-5 * np.abs(ref_logits).max()
    for t in range(T):
        sel = g_ids[t]
        assert len(set(sel.tolist())) == k and sel.min() >= 0 and sel.max() < E
        rest = np.setdiff1d(np.arange(E), sel)
        if len(rest):
            assert ref_logits[t, sel].min() >= ref_logits[t, rest].max() - eps
    if E == 1:
        assert torch.equal(scores.cpu(), torch.ones(T, 1))
    rdx, rdw = oracle.router_backward(d, _np(x, dtype), _np(wr, dtype), g_ids,
                                      scores.cpu().numpy().astype(np.float64), ds.cpu().numpy().astype(np.float64))
    assert rel_err(dwr.cpu().numpy(), dw0.cpu().numpy() + rdw) <= tol(dtype)
    assert rel_err(dwr2.cpu().numpy(), rdw) <= tol(dtype) or (not rdw.any() and not dwr2.any())
    assert rel_err(dx2.float().cpu().numpy(), rdx) <= tol(dtype) or (not rdx.any() and not dx2.float().any())
