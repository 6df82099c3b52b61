"""The expert-parallel data path on ONE GPU (run with -m gpu): EP = 2 / 4 ranks as host threads
of one process (memfine_local_group_create), exchanging rows with device copies in exactly the
NCCL path's layouts.  Every rank's Y, dX, d_score and its local experts' dW are compared with
the oracle's EP emulation (all ranks, canonical chunk-major dW order)."""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2511_21431_b200 import capi, layer
from tests.harness import rel_err, tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _bits(t, dtype):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16) if dtype == torch.bfloat16 else \
        t.contiguous().numpy().astype(np.float32)


def _run_group(EP, C, dtype, transport, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=False, mx_wgrad=False,
               nan_dw=False):
    """Every rank of an in-process EP group: fwd + bwd; returns (per-rank outputs, counts seen)."""
    El = E // EP
    group = layer.LocalGroup(EP)
    results, errors = [None] * EP, []
    counts_seen = [None] * EP

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ov = transport == "overlap"
                mf = layer.MemFine(T, h, g, E, k, ep_size=EP, ep_rank=r, dtype=dtype, local_group=group, overlap=ov,
                                   mx=mx, mx_wgrad=mx_wgrad)
                mf.set_ep_transport(capi.EP_COPY if ov else transport)
                if ov:
                    mf.set_comm_sms(16)
                dev = "cuda:0"
                x, dy = xs[r].to(dev), dys[r].to(dev)
                ids = torch.from_numpy(routes[r][0]).to(dev)
                w = torch.from_numpy(routes[r][1]).to(dev)
                lwg, lwu, lwd = (t[r * El:(r + 1) * El].contiguous().to(dev) for t in (wg, wu, wd))
                if mx:
                    mf.mx_quantize_weights(lwg, lwu, lwd, stream=st)
                counts = mf.route_counts(ids, nsub=C, stream=st)
                st.synchronize()
                ch = counts.cpu()
                counts_seen[r] = ch.numpy().copy()
                wsb = max(layer.workspace_bytes(ch, mf.dims, C, capi.FWD), layer.workspace_bytes(ch, mf.dims, C, capi.BWD))
                ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
                y = mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws, stream=st)
                kw = {}
                if nan_dw:   # dW buffers holding garbage: the call must overwrite every element
                    kw = {n_: torch.full(t_.shape, float("nan"), dtype=torch.float32, device=dev)
                          for n_, t_ in (("dw_gate", lwg), ("dw_up", lwu), ("dw_down", lwd))}
                dx, dwg, dwu, dwd, ds = mf.moe_bwd(dy, x, ids, w, lwg, lwu, lwd, C, ws, stream=st, **kw)
                s_ = mf.sync(stream=st)
                assert s_ == 0, capi.status_str(s_)
                results[r] = [t.float().cpu().numpy() for t in (y, dx, ds, dwg, dwu, dwd)]
                mf.close()
        except BaseException:  # noqa: BLE001
            import traceback
            errors.append(f"rank {r}: {traceback.format_exc()}")

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(EP)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    group.close()
    assert not errors, "\n".join(errors)
    return results, counts_seen


@pytest.mark.parametrize("transport", [capi.EP_COPY, capi.EP_P2P, "overlap"])
@pytest.mark.parametrize("EP,C,dtype", [(2, 1, torch.bfloat16), (2, 3, torch.bfloat16), (4, 2, torch.bfloat16),
                                        (4, 1, torch.float32), (2, 2, torch.float32)])
def test_ep_local_group_matches_oracle(EP, C, dtype, transport):
    """transport EP_COPY: send buffers + stream-ordered copies (the NCCL path's layouts);
    EP_P2P: dispatch and combine fused into the permute kernel and the down/dX GEMM epilogues,
    storing rows straight into peer buffers; "overlap": EP_COPY with MEMFINE_FLAG_OVERLAP (chunk
    j+-1's exchange on the comm stream while chunk j's GEMMs run; GEMMs leave 16 SMs free)."""
    T, h, g, E, k = 300, 128, 256, 8, 2
    El = E // EP
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, counts_seen = _run_group(EP, C, dtype, transport, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    # every rank saw the same all-gathered counts, equal to the oracle's per-rank histograms
    od1 = oracle.Dims(T=T, h=h, g=g, E=E, k=k)
    ref_counts = np.stack([oracle.route_counts(od1, routes[r][0], C)[0] for r in range(EP)])
    for r in range(EP):
        np.testing.assert_array_equal(counts_seen[r], ref_counts)
    # oracle EP emulation
    d = oracle.Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="bf16" if dtype == torch.bfloat16 else "f32")
    xa = np.concatenate([_bits(x, dtype) for x in xs])
    dya = np.concatenate([_bits(x, dtype) for x in dys])
    ida = np.concatenate([r[0] for r in routes])
    wa = np.concatenate([r[1] for r in routes]).astype(np.float64)
    W = [_bits(t, dtype) for t in (wg, wu, wd)]
    y_ref, _, _ = oracle.fcda_forward(d, C, xa, ida, wa, *W)
    dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref, _, _ = oracle.fcda_backward(d, C, dya, xa, ida, wa, *W)
    t_ = tol(dtype)
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        sl = slice(r * T, (r + 1) * T)
        es = slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(y, y_ref[sl]), "dx": rel_err(dx, dx_ref[sl]), "dscore": rel_err(ds, ds_ref[sl]),
                "dw_gate": rel_err(dwg, dwg_ref[es]), "dw_up": rel_err(dwu, dwu_ref[es]),
                "dw_down": rel_err(dwd, dwd_ref[es])}
        assert all(v <= t_ for v in errs.values()), (r, errs)


@pytest.mark.parametrize("EP,C", [(2, 3), (4, 4)])
def test_ep_overlap_bit_identical(EP, C):
    """MEMFINE_FLAG_OVERLAP changes when the exchange runs, not what any kernel reads: every
    output is bit-identical to the one-stream order (the dW first-chunk overwrite included)."""
    T, h, g, E, k = 700, 128, 256, 8, 2
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="random") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    a, _ = _run_group(EP, C, dtype, capi.EP_COPY, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    b, _ = _run_group(EP, C, dtype, "overlap", xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    for r in range(EP):
        for name, u, v in zip(("y", "dx", "dscore", "dw_gate", "dw_up", "dw_down"), a[r], b[r]):
            np.testing.assert_array_equal(u, v, err_msg=f"rank {r} {name}")


@pytest.mark.parametrize("EP,C", [(2, 1), (2, 3), (4, 2)])
def test_ep_local_group_mx_matches_mx_oracle(EP, C):
    """MXFP8 with EP (reading R28): rows travel in bf16, each rank quantises what it received; every
    rank's Y, dX, d_score and local dW against the oracle's MX layer over all ranks' tokens."""
    from tests.test_gpu_mx import MX_TOL
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_COPY, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True)
    d = oracle.Dims(T=T * EP, h=h, g=g, E=E, k=k, in_dtype="bf16")
    xa = np.concatenate([_bits(x, dtype) for x in xs])
    dya = np.concatenate([_bits(x, dtype) for x in dys])
    ida = np.concatenate([r[0] for r in routes])
    wa = np.concatenate([r[1] for r in routes]).astype(np.float64)
    W = [_bits(t, dtype) for t in (wg, wu, wd)]
    wq = oracle.mx_weights(d, *W)
    y_ref, dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref = oracle.moe_mx(d, xa, ida, wa, wq, dy=dya, wd=W[2])
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        sl, es = slice(r * T, (r + 1) * T), slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(y, y_ref[sl]), "dx": rel_err(dx, dx_ref[sl]), "dscore": rel_err(ds, ds_ref[sl]),
                "dw_gate": rel_err(dwg, dwg_ref[es]), "dw_up": rel_err(dwu, dwu_ref[es]),
                "dw_down": rel_err(dwd, dwd_ref[es])}
        assert all(v <= MX_TOL for v in errs.values()), (r, errs)


@pytest.mark.parametrize("EP,C", [(2, 1), (2, 3), (4, 2)])
def test_ep_local_group_mx_wgrad_matches_oracle(EP, C):
    """MXFP8 weight gradients with EP (reading R28c): each rank's K for its local expert e is the
    chunk's copies in (src rank, token, slot) order - the received expert-major layout - quantised
    columnwise in 32-copy blocks; against the oracle's definition over the EP ranks' chunks."""
    from tests.test_gpu_mx import MX_TOL
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_COPY, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True,
                            mx_wgrad=True)
    d = oracle.Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="bf16")
    xa = np.concatenate([_bits(x, dtype) for x in xs])
    dya = np.concatenate([_bits(x, dtype) for x in dys])
    ida = np.concatenate([r[0] for r in routes])
    wa = np.concatenate([r[1] for r in routes]).astype(np.float64)
    W = [_bits(t, dtype) for t in (wg, wu, wd)]
    wq = oracle.mx_weights(d, *W)
    y_ref, dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref = oracle.moe_mx(d, xa, ida, wa, wq, dy=dya, wd=W[2], wgrad_C=C)
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        sl, es = slice(r * T, (r + 1) * T), slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(y, y_ref[sl]), "dx": rel_err(dx, dx_ref[sl]), "dscore": rel_err(ds, ds_ref[sl]),
                "dw_gate": rel_err(dwg, dwg_ref[es]), "dw_up": rel_err(dwu, dwu_ref[es]),
                "dw_down": rel_err(dwd, dwd_ref[es])}
        assert all(v <= MX_TOL for v in errs.values()), (r, errs)


@pytest.mark.parametrize("EP,C,mx_wgrad", [(2, 2, False), (4, 1, False), (2, 3, True)])
def test_ep_local_group_mx_p2p_matches_oracle(EP, C, mx_wgrad):
    """MXFP8 over the fused peer-memory exchange (EP_P2P): rows pushed in bf16 by the permute kernel
    and quantised on arrival, o / dX rows stored into the sources' buffers by the MX down / dX
    epilogues; every rank against the oracle's MX layer (and, with MX weight gradients, R28c)."""
    from tests.test_gpu_mx import MX_TOL
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_P2P, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True,
                            mx_wgrad=mx_wgrad)
    d = oracle.Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="bf16")
    xa = np.concatenate([_bits(x, dtype) for x in xs])
    dya = np.concatenate([_bits(x, dtype) for x in dys])
    ida = np.concatenate([r[0] for r in routes])
    wa = np.concatenate([r[1] for r in routes]).astype(np.float64)
    W = [_bits(t, dtype) for t in (wg, wu, wd)]
    wq = oracle.mx_weights(d, *W)
    y_ref, dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref = oracle.moe_mx(d, xa, ida, wa, wq, dy=dya, wd=W[2],
                                                                    wgrad_C=C if mx_wgrad else 0)
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        sl, es = slice(r * T, (r + 1) * T), slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(y, y_ref[sl]), "dx": rel_err(dx, dx_ref[sl]), "dscore": rel_err(ds, ds_ref[sl]),
                "dw_gate": rel_err(dwg, dwg_ref[es]), "dw_up": rel_err(dwu, dwu_ref[es]),
                "dw_down": rel_err(dwd, dwd_ref[es])}
        assert all(v <= MX_TOL for v in errs.values()), (r, errs)


def _oracle_ep(EP, C, dtype, xs, dys, routes, wg, wu, wd, T, h, g, E, k):
    d = oracle.Dims(T=T, h=h, g=g, E=E, k=k, EP=EP, in_dtype="bf16" if dtype == torch.bfloat16 else "f32")
    xa = np.concatenate([_bits(x, dtype) for x in xs])
    dya = np.concatenate([_bits(x, dtype) for x in dys])
    ida = np.concatenate([r[0] for r in routes])
    wa = np.concatenate([r[1] for r in routes]).astype(np.float64)
    W = [_bits(t, dtype) for t in (wg, wu, wd)]
    y_ref, _, _ = oracle.fcda_forward(d, C, xa, ida, wa, *W)
    dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref, _, _ = oracle.fcda_backward(d, C, dya, xa, ida, wa, *W)
    return y_ref, dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref


def _check_ranks(results, refs, EP, T, El, t_):
    y_ref, dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref = refs
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        sl, es = slice(r * T, (r + 1) * T), slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(y, y_ref[sl]), "dx": rel_err(dx, dx_ref[sl]), "dscore": rel_err(ds, ds_ref[sl]),
                "dw_gate": rel_err(dwg, dwg_ref[es]), "dw_up": rel_err(dwu, dwu_ref[es]),
                "dw_down": rel_err(dwd, dwd_ref[es])}
        assert all(v <= t_ for v in errs.values()), (r, errs)
        for name, a in (("dw_gate", dwg), ("dw_up", dwu), ("dw_down", dwd)):
            assert np.isfinite(a).all(), (r, name)


@pytest.mark.parametrize("transport", [capi.EP_COPY, capi.EP_P2P, "overlap"])
@pytest.mark.parametrize("EP,C", [(2, 1), (4, 3)])
def test_ep_rank_without_rows(EP, C, transport):
    """A rank whose experts receive no copy in any chunk (hot-expert routing, the case MACT exists for):
    its weight-gradient GEMMs have no rows, so the call itself must overwrite its dW with zeros (the dW
    buffers start as NaN here), and its (empty) exchanges must still move every other rank's rows."""
    T, h, g, E, k = 300, 128, 256, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    cold = set(range((EP - 1) * El, E))               # the last rank's experts: never routed to
    hot = [e for e in range(E) if e not in cold]
    routes = []
    for r in range(EP):
        rng = np.random.default_rng(100 + r)
        ids = np.stack([rng.choice(hot, k, replace=False) for _ in range(T)]).astype(np.int32)
        lg = rng.standard_normal((T, k))
        w = (np.exp(lg) / np.exp(lg).sum(1, keepdims=True)).astype(np.float32)
        routes.append((ids, w))
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, transport, xs, dys, routes, wg, wu, wd, T, h, g, E, k, nan_dw=True)
    refs = _oracle_ep(EP, C, dtype, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    _check_ranks(results, refs, EP, T, El, tol(dtype))
    for a in results[EP - 1][3:]:
        assert np.all(a == 0)


@pytest.mark.parametrize("transport", [capi.EP_COPY, capi.EP_P2P])
@pytest.mark.parametrize("E,C,dtype", [(16, 1, torch.bfloat16), (16, 3, torch.bfloat16), (32, 3, torch.bfloat16),
                                       (32, 1, torch.float32)])
def test_ep8_local_group_matches_oracle(E, C, dtype, transport):
    """EP = 8 (the north star's box): E = 16 (2 local experts) and E = 32 (4), top-2 with Zipf skew and
    the hot experts on rank 0; every rank's Y, dX, d_score and local dW against the oracle."""
    EP, T, h, g, k = 8, 256, 128, 256, 2
    El = E // EP
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, transport, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    refs = _oracle_ep(EP, C, dtype, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    _check_ranks(results, refs, EP, T, El, tol(dtype))
