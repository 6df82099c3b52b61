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
                ov = transport in ("overlap", "p2p_overlap")
                mf = layer.MemFine(T, h, g, E, k, ep_size=EP, ep_rank=r, dtype=dtype, local_group=group, overlap=ov,
                                   mx=mx, mx_wgrad=mx_wgrad)
                mf.set_ep_transport(capi.EP_P2P if transport == "p2p_overlap" else
                                    capi.EP_COPY if ov else transport)
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
                # one size on every rank (the fused exchange derives every peer's layout from it): the
                # largest any rank needs, from the all-gathered counts
                wsb = 0
                for rr in range(EP):
                    dr = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=rr, dtype=dtype, mx=mx, overlap=ov,
                                         mx_wgrad=mx_wgrad)
                    wsb = max(wsb, layer.workspace_bytes(ch, dr, C, capi.FWD), layer.workspace_bytes(ch, dr, C, capi.BWD))
                ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
                # Every device allocation of this rank happens BEFORE its first layer call: with the fused
                # peer-memory exchange another rank's kernels spin on flags this rank raises, and a
                # cudaMalloc issued by this thread in between (e.g. torch allocating the backward's outputs)
                # may wait for the device to go idle - i.e. for that spin - while holding up this rank's
                # launches (seen as a 20 s wait timeout in the two-slot P2P mode).
                f32 = dict(dtype=torch.float32, device=dev)
                y = torch.empty_like(x)
                kw = {"dx": torch.empty_like(x), "dscore": torch.empty(w.shape, **f32)}
                fill = float("nan") if nan_dw else 0.0   # nan_dw: garbage dW, the call must overwrite every element
                kw.update({n_: torch.full(t_.shape, fill, **f32)
                           for n_, t_ in (("dw_gate", lwg), ("dw_up", lwu), ("dw_down", lwd))})
                y = mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws, y=y, stream=st)
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


@pytest.mark.parametrize("transport", [capi.EP_COPY, capi.EP_P2P, "overlap", "p2p_overlap"])
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
    # the fused peer-memory exchange with the same two-slot pipeline (pushes of chunk j+1 and the combine of
    # chunk j-1 on the comm stream while chunk j's GEMMs run): bit-identical to its own one-stream order
    c, _ = _run_group(EP, C, dtype, capi.EP_P2P, xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    d_, _ = _run_group(EP, C, dtype, "p2p_overlap", xs, dys, routes, wg, wu, wd, T, h, g, E, k)
    for r in range(EP):
        for name, u, v in zip(("y", "dx", "dscore", "dw_gate", "dw_up", "dw_down"), c[r], d_[r]):
            if name == "dscore":   # (its dA partials meet in fp32 atomics of run-dependent order)
                assert rel_err(v, u) <= 1e-6, (r, name)
            else:
                np.testing.assert_array_equal(u, v, err_msg=f"rank {r} p2p {name}")


def _ep1_mx_reference(EP, C, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx_wgrad):
    """The EP group's problem on ONE rank (EP = 1 MX path) with the tokens in chunk-major order - for
    each chunk j every source rank's tokens [jT/C, (j+1)T/C) in rank order - so that (T % C == 0) the
    EP = 1 chunk j holds exactly the EP chunk j's copies, each expert's in the EP receive order (src
    rank, token, slot; reading R3).  Returns per-rank (y, dx, dscore) and all experts' dW."""
    from tests.test_gpu_mx import _mx_run
    from tests.harness import Problem
    assert T % C == 0
    perm = np.array([r * T + i for j in range(C) for r in range(EP) for i in range(j * T // C, (j + 1) * T // C)])
    cat = lambda ts: torch.cat(ts)[torch.from_numpy(perm)].contiguous()
    ids = np.concatenate([r_[0] for r_ in routes])[perm]
    w = np.concatenate([r_[1] for r_ in routes])[perm]
    p = Problem(EP * T, h, g, E, k, torch.bfloat16, cat(xs), cat(dys), torch.from_numpy(np.ascontiguousarray(ids)),
                torch.from_numpy(np.ascontiguousarray(w)), wg, wu, wd)
    out, _ = _mx_run(p, C, mx_wgrad=mx_wgrad)
    inv = np.argsort(perm)
    per_rank = [{key: out[key][inv][r * T:(r + 1) * T] for key in ("y", "dx", "dscore")} for r in range(EP)]
    return per_rank, out


def _check_mx_ep_vs_ep1(results, per_rank, ep1, EP, El):
    """EP MX == the EP = 1 MX path (itself checked against the oracle in tests/test_gpu_mx.py): the rows
    travel in bf16 and are quantised on arrival to the same codes, every row and every dW element
    sees the same operands in the same order - bit for bit, except d_score, whose per-row partials
    from the dA GEMM's N tiles meet in fp32 atomics of run-dependent order."""
    for r in range(EP):
        y, dx, ds, dwg, dwu, dwd = results[r]
        np.testing.assert_array_equal(y, per_rank[r]["y"], err_msg=f"rank {r} y")
        np.testing.assert_array_equal(dx, per_rank[r]["dx"], err_msg=f"rank {r} dx")
        assert rel_err(ds, per_rank[r]["dscore"]) <= 1e-6, r
        es = slice(r * El, (r + 1) * El)
        for name, a_ in (("dwg", dwg), ("dwu", dwu), ("dwd", dwd)):
            np.testing.assert_array_equal(a_, ep1[name][es], err_msg=f"rank {r} {name}")


@pytest.mark.parametrize("EP,C", [(2, 1), (2, 3), (4, 2)])
def test_ep_local_group_mx_matches_ep1(EP, C):
    """MXFP8 with EP (reading R28): rows travel in bf16, each rank quantises what it received."""
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_COPY, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True)
    per_rank, ep1 = _ep1_mx_reference(EP, C, xs, dys, routes, wg, wu, wd, T, h, g, E, k, False)
    _check_mx_ep_vs_ep1(results, per_rank, ep1, EP, El)


@pytest.mark.parametrize("EP,C", [(2, 1), (2, 3), (4, 2)])
def test_ep_local_group_mx_wgrad_matches_ep1(EP, C):
    """MXFP8 weight gradients with EP (reading R28c): each rank's K for its local expert e is the
    chunk's copies in (src rank, token, slot) order - the received expert-major layout - quantised
    columnwise in 32-copy blocks, exactly as the EP = 1 path does on the chunk-major token order."""
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_COPY, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True,
                            mx_wgrad=True)
    per_rank, ep1 = _ep1_mx_reference(EP, C, xs, dys, routes, wg, wu, wd, T, h, g, E, k, True)
    _check_mx_ep_vs_ep1(results, per_rank, ep1, EP, El)


@pytest.mark.parametrize("EP,C,mx_wgrad", [(2, 2, False), (4, 1, False), (2, 3, True)])
def test_ep_local_group_mx_p2p_matches_ep1(EP, C, mx_wgrad):
    """MXFP8 over the fused peer-memory exchange (EP_P2P): rows pushed in bf16 by the permute kernel
    and quantised on arrival, o / dX rows stored into the sources' buffers by the MX down / dX
    epilogues; every rank against the EP = 1 MX path (and, with MX weight gradients, R28c)."""
    T, h, g, E, k = 300, 256, 384, 8, 2
    El = E // EP
    dtype = torch.bfloat16
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    results, _ = _run_group(EP, C, dtype, capi.EP_P2P, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx=True,
                            mx_wgrad=mx_wgrad)
    per_rank, ep1 = _ep1_mx_reference(EP, C, xs, dys, routes, wg, wu, wd, T, h, g, E, k, mx_wgrad)
    _check_mx_ep_vs_ep1(results, per_rank, ep1, EP, El)


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


@pytest.mark.parametrize("transport", [capi.EP_COPY, capi.EP_P2P, "overlap", "p2p_overlap"])
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


def test_ep_p2p_graph_capture_no_host_sync():
    """N1: the device-planned P2P exchange - the count all-gather pushed into the peers'
    sync areas, the chunk tables built on the device, per-peer epoch flags instead of host fences - never
    waits on the host, so every rank's fwd + bwd captures into a CUDA graph (thread-local capture, all ranks
    at once) and the replays, run concurrently, reproduce the eager outputs bit for bit (d_score: its
    atomics)."""
    EP, C, T, h, g, E, k = 4, 2, 300, 128, 256, 8, 2
    dtype = torch.bfloat16
    El = E // EP
    xs = [synth.make_x(T, h, rank=r, dtype=dtype) for r in range(EP)]
    dys = [synth.make_dy(T, h, rank=r, dtype=dtype) for r in range(EP)]
    routes = [synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous") for r in range(EP)]
    wg, wu, wd = synth.make_experts(range(E), h, g, dtype=dtype)
    group = layer.LocalGroup(EP)
    bar = threading.Barrier(EP)
    res, errors = [None] * EP, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            dev = "cuda:0"
            with torch.cuda.stream(st):
                mf = layer.MemFine(T, h, g, E, k, ep_size=EP, ep_rank=r, dtype=dtype, local_group=group)
                mf.set_ep_transport(capi.EP_P2P)
                x, dy = xs[r].to(dev), dys[r].to(dev)
                ids = torch.from_numpy(routes[r][0]).to(dev)
                w = torch.from_numpy(routes[r][1]).to(dev)
                lwg, lwu, lwd = (t[r * El:(r + 1) * El].contiguous().to(dev) for t in (wg, wu, wd))
                ch = mf.route_counts(ids, nsub=C, stream=st).cpu()
                wsb = 0
                for rr in range(EP):
                    dr = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=rr, dtype=dtype)
                    wsb = max(wsb, layer.workspace_bytes(ch, dr, C, capi.FWD), layer.workspace_bytes(ch, dr, C, capi.BWD))
                ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
                f32 = dict(dtype=torch.float32, device=dev)
                y, dx = torch.empty_like(x), torch.empty_like(x)
                gr = [torch.empty(t.shape, **f32) for t in (lwg, lwu, lwd)]
                ds = torch.empty(w.shape, **f32)

                def step():
                    mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws, y=y, stream=st)
                    mf.moe_bwd(dy, x, ids, w, lwg, lwu, lwd, C, ws, dx=dx, dw_gate=gr[0], dw_up=gr[1], dw_down=gr[2],
                               dscore=ds, stream=st)

                step()                                  # eager: registers the workspace, loads the kernels
                assert mf.sync(stream=st) == 0
                ref = [t.clone() for t in (y, dx, *gr, ds)]
                bar.wait()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=st, capture_error_mode="thread_local"):
                    step()
                for t in (y, dx, *gr, ds):
                    t.fill_(float("nan"))
                st.synchronize()
                bar.wait()                              # every rank captured: replay all at once
                for _ in range(2):
                    graph.replay()
                st.synchronize()
                assert mf.sync(stream=st) == 0
                res[r] = (ref, [t.clone() for t in (y, dx, *gr, ds)])
                mf.close()
        except BaseException:  # noqa: BLE001
            import traceback
            errors.append(f"rank {r}: {traceback.format_exc()}")
            bar.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(EP)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    group.close()
    assert not errors, "\n".join(errors)
    for r in range(EP):
        ref, got = res[r]
        for name, a_, b_ in zip(("y", "dx", "dw_gate", "dw_up", "dw_down"), ref[:5], got[:5]):
            assert torch.equal(a_, b_), f"rank {r} {name}"
        assert (ref[5] - got[5]).abs().max().item() <= 1e-5 * ref[5].abs().max().item()
