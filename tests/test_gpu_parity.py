"""CUDA path vs the oracle, element by element, through the C ABI (run with -m gpu).

Integer outputs (routing counts, permutation, C) bit-exact; floating point within the
north star's tolerance: max|got-ref|/max|ref| <= 2e-2 (bf16), <= 1e-5 (fp32 mode)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21431_b200 import capi, layer
from tests.harness import (GpuRun, make_problem, oracle_dims, oracle_fwd_bwd, oracle_tokens, rel_err,
                           tile_covering_tokens, tol)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check_all(p, run, C, ref):
    y, st, stats, wsb = run.fwd(C)
    assert st == 0, capi.status_str(st)
    t = tol(p.dtype)
    assert rel_err(y.float().cpu().numpy(), ref["y"]) <= t
    (dx, dwg, dwu, dwd, ds), st, bstats, _ = run.bwd(C)
    assert st == 0, capi.status_str(st)
    errs = {
        "dx": rel_err(dx.float().cpu().numpy(), ref["dx"]),
        "dscore": rel_err(ds.cpu().numpy(), ref["dscore"]),
        "dw_gate": rel_err(dwg.cpu().numpy(), ref["dwg"]),
        "dw_up": rel_err(dwu.cpu().numpy(), ref["dwu"]),
        "dw_down": rel_err(dwd.cpu().numpy(), ref["dwd"]),
    }
    for k_, v in errs.items():
        assert v <= t, (k_, v, errs)
    return y, dx, stats, bstats, wsb


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("C", [1, 2, 4])
def test_tiny_config(dtype, C):
    """BASELINE configs[0]: 4 experts, top-2, h=64, FFN=128, 256 tokens, C = 1/2/4."""
    p = make_problem(256, 64, 128, 4, 2, dtype=dtype)
    run = GpuRun(p)
    ref = oracle_fwd_bwd(p, C)
    _check_all(p, run, C, ref)


@pytest.mark.parametrize("T,h,g,E", [(1000, 256, 384, 8), (2600, 512, 256, 5)])
def test_quad_tiles_match_pairs_and_oracle(T, h, g, E, monkeypatch):
    """The 512 x 256 quad tiles of the down and dX GEMMs (two 256-row pair halves sharing each staged B tile;
    an expert's odd last pair is a one-half tile), forced on with MEMFINE_QUAD=2 at sizes the automatic
    choice would leave to pairs: Y and dX bit-identical to the 256 x 256 pair tiles (the same MMAs in the
    same K order per row), everything within tolerance of the oracle, at C = 1 and 3."""
    p = make_problem(T, h, g, E, 2, dtype=torch.bfloat16, zipf_s=1.2, placement="contiguous", seed=5)
    run = GpuRun(p)
    for C in (1, 3):
        ref = oracle_fwd_bwd(p, C)
        monkeypatch.setenv("MEMFINE_QUAD", "0")
        y0, dx0, _, _, _ = _check_all(p, run, C, ref)
        y0, dx0 = y0.clone(), dx0.clone()
        monkeypatch.setenv("MEMFINE_QUAD", "2")
        y1, dx1, _, _, _ = _check_all(p, run, C, ref)
        assert torch.equal(y0.view(torch.int16), y1.view(torch.int16)), C
        assert torch.equal(dx0.view(torch.int16), dx1.view(torch.int16)), C


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_medium_ragged_skewed(dtype):
    """Several M/N/K tiles, ragged token count (1000), Zipf(1.2) skew, C = 1 and 3."""
    p = make_problem(1000, 256, 384, 8, 2, dtype=dtype, zipf_s=1.2, placement="contiguous", seed=1)
    run = GpuRun(p)
    for C in (1, 3):
        _check_all(p, run, C, oracle_fwd_bwd(p, C))


def test_counts_permutation_plan_bit_exact():
    p = make_problem(1000, 64, 128, 8, 3, zipf_s=1.2, seed=2)
    run = GpuRun(p)
    d = oracle_dims(p)
    for nsub in (1, 3, 8):
        c = run.counts(nsub).cpu().numpy()[0]
        ref, bad = oracle.route_counts(d, p.ids.numpy(), nsub)
        assert bad == 0
        np.testing.assert_array_equal(c, ref)
    # canonical dispatch order (reading R3) of every chunk
    run.mf.set_debug(True)
    for C in (1, 2, 4, 3):
        run.fwd(C)
        for j in range(C):
            np.testing.assert_array_equal(run.mf.debug_perm(j), oracle.dispatch_order(d, p.ids.numpy(), 0, C, j))
    run.mf.set_debug(False)
    # device tuner == host planner == oracle
    counts_d = run.counts(8)
    rng = np.random.default_rng(0)
    for _ in range(20):
        budget = int(rng.integers(10**5, 10**7))
        b = capi.make_budget(budget, 1.0, int(rng.integers(0, 1000)), int(rng.integers(0, 1000)),
                             rule=int(rng.integers(0, 2)))
        dd = layer.plan(counts_d, run.mf.dims, b)
        dh = layer.plan(counts_d.cpu(), run.mf.dims, b)
        assert dd == dh
        st, ro = oracle.plan(counts_d.cpu().numpy().astype(np.int64), d, budget_bytes=budget,
                             static_bytes=b.static_bytes, other_act_bytes=b.other_act_bytes,
                             rule=0 if b.rule == capi.RULE_EQ9 else 1)
        assert st == dh["status"]
        if st == 0:
            for f in ro:
                assert ro[f] == dh[f], f


def test_chunking_invariance_on_gpu():
    """Eq. 6/7 on the device: Y and dX bit-identical for every C (row-local arithmetic)."""
    p = make_problem(777, 128, 256, 6, 2, seed=3)
    run = GpuRun(p)
    y1, st, _, _ = run.fwd(1)
    (dx1, *_), st, _, _ = run.bwd(1)
    for C in (2, 4, 8, 5):
        yc, st, _, _ = run.fwd(C)
        assert st == 0
        assert torch.equal(yc, y1)
        (dxc, *_), st, _, _ = run.bwd(C)
        assert torch.equal(dxc, dx1)


def test_run_to_run_determinism():
    """Two runs on the same inputs: Y, dX and every dW bit-identical (each output element has one
    writer per launch and the chunks accumulate in order); d_score's per-row partials from the dA
    GEMM's N tiles meet in fp32 atomics, so it is reproducible to rounding only."""
    p = make_problem(1500, 256, 384, 8, 2, zipf_s=1.2, seed=12)
    run = GpuRun(p)
    outs = []
    for _ in range(2):
        y, st, _, _ = run.fwd(3)
        assert st == 0
        (dx, dwg, dwu, dwd, ds), st, _, _ = run.bwd(3)
        assert st == 0
        outs.append([t.clone() for t in (y, dx, dwg, dwu, dwd, ds)])
    for a, b in zip(outs[0][:5], outs[1][:5]):
        assert torch.equal(a, b)
    assert rel_err(outs[0][5].cpu().numpy(), outs[1][5].cpu().numpy()) <= 1e-6


def test_peak_workspace_scales_one_over_c():
    """Measured workspace high-water == the prediction (memfine_workspace_bytes) exactly, and
    peak(C)/peak(1) tracks max_j s''_j / s'' (Table 2 rows 11-13)."""
    p = make_problem(4096, 256, 512, 8, 2, seed=4)
    run = GpuRun(p)
    peaks, maxrows = {}, {}
    row_bytes = 4 + 4 + 2 * (256 + 512 + 256)
    for C in (1, 2, 4, 8):
        y, st, stats, wsb = run.fwd(C)
        assert st == 0
        assert stats["workspace_used_bytes"] == wsb
        peaks[C] = wsb
        rows = stats["rows"]
        assert sum(rows) == 4096 * 2
        maxrows[C] = max(rows)
        # padded rows of the hottest chunk: at most 127 padding rows per local expert
        assert max(stats["rows_padded"]) <= maxrows[C] + 8 * 127
    assert peaks[1] > peaks[2] > peaks[4] > peaks[8]
    for C in (2, 4, 8):
        assert peaks[C] / peaks[1] <= (maxrows[C] + 8 * 128) / maxrows[1] + 0.01


def test_edge_cases():
    # T < C: empty chunks; duplicated ids inside a token's top-k; an expert with no tokens
    ids = np.array([[0, 0], [2, 2], [0, 2]], np.int32)
    p = make_problem(3, 64, 128, 4, 2, ids=ids)
    run = GpuRun(p)
    ref = oracle_fwd_bwd(p, 8)
    _check_all(p, run, 8, ref)
    # every token on one expert
    p = make_problem(300, 64, 128, 4, 2, ids=np.tile(np.array([[3, 1]], np.int32), (300, 1)))
    _check_all(p, GpuRun(p), 2, oracle_fwd_bwd(p, 2))


def test_maximum_experts_and_topk():
    """The largest routing the ABI accepts: 1024 experts (the dispatch scan's limit) and top-16
    (the copy-ranking limit) - ~8 copies per expert, every segment padded to 128 rows, 1024 expert
    segments in the grouped GEMMs; C = 2."""
    p = make_problem(512, 128, 128, 1024, 16, zipf_s=1.2, seed=8)
    _check_all(p, GpuRun(p), 2, oracle_fwd_bwd(p, 2))


def test_errors_surface():
    p = make_problem(64, 64, 128, 4, 2)
    run = GpuRun(p)
    # workspace too small -> latched, reported by memfine_sync
    y, st, stats, _ = run.fwd(1, ws_bytes=4096)
    assert st == capi.ERR_WORKSPACE
    # bad expert id -> MEMFINE_ERR_ROUTING at the next sync
    bad = p.ids.clone()
    bad[5, 1] = 99
    run.ids = bad.to(run.dev)
    y, st, stats, _ = run.fwd(1, counts_host=torch.zeros((1, 1, 4), dtype=torch.int32) + 64)
    assert st == capi.ERR_ROUTING


@pytest.mark.slow
@pytest.mark.parametrize("C", [1, 2])
def test_mixtral_full_size_sampled(C, monkeypatch):
    """BASELINE configs[1] shape at EP=1 (8 experts, top-2, h=4096, FFN=14336, 16K tokens):
    integer outputs in full; Y / dX / d_score vs the oracle on tokens sampled so that every 128-row
    m-tile of every expert segment of every chunk holds at least one of their copies.  C = 1 is the
    bench's launch configuration, where the down and dX GEMMs run 512 x 256 quad tiles: there Y and dX
    must also equal the 256 x 256 pair tiles' bit for bit."""
    p = make_problem(16384, 4096, 14336, 8, 2, zipf_s=1.2, seed=5)
    run = GpuRun(p)
    d = oracle_dims(p)
    c = run.counts(8).cpu().numpy()[0]
    ref, _ = oracle.route_counts(d, p.ids.numpy(), 8)
    np.testing.assert_array_equal(c, ref)
    run.mf.set_debug(True)      # the expert-major row layout, to sample every m-tile
    y, st, _, _ = run.fwd(C)
    assert st == 0
    rows = [run.mf.debug_rows(j) for j in range(C)]
    run.mf.set_debug(False)
    (dx, dwg, dwu, dwd, ds), st, _, _ = run.bwd(C)
    assert st == 0
    if C == 1:
        y, dx = y.clone(), dx.clone()
        monkeypatch.setenv("MEMFINE_QUAD", "0")
        y0, st, _, _ = run.fwd(C)
        assert st == 0
        (dx0, _, _, _, _), st, _, _ = run.bwd(C)
        assert st == 0
        assert torch.equal(y.view(torch.int16), y0.view(torch.int16))
        assert torch.equal(dx.view(torch.int16), dx0.view(torch.int16))
    rng = np.random.default_rng(0)
    toks = np.unique(np.concatenate([tile_covering_tokens(r, p.k, rng) for r in rows]))
    ry, rdx, rds = oracle_tokens(p, toks)
    assert rel_err(y.float().cpu().numpy()[toks], ry) <= 2e-2
    assert rel_err(dx.float().cpu().numpy()[toks], rdx) <= 2e-2
    assert rel_err(ds.cpu().numpy()[toks], rds) <= 2e-2
    assert torch.isfinite(dwg).all() and torch.isfinite(dwu).all() and torch.isfinite(dwd).all()


@pytest.mark.parametrize("C", [1, 2])
def test_many_tiles_per_cta(C):
    """8192 tokens x top-2 over 4 experts: ~512 gate/up tiles and 4096-deep weight-gradient K
    loops, so every persistent CTA runs several tiles through both TMEM accumulator stages."""
    p = make_problem(8192, 256, 512, 4, 2, zipf_s=1.2, seed=6)
    run = GpuRun(p)
    _check_all(p, run, C, oracle_fwd_bwd(p, C))


def test_cuda_graph_capture_replays_identically():
    """At EP=1 memfine_moe_fwd / memfine_moe_bwd do no host synchronisation, so a whole fwd+bwd
    step can be captured into a CUDA graph and replayed; the replay is bit-identical to eager, except
    d_score, whose per-row partial dots over the N-tiles are added with atomics (order not fixed)."""
    p = make_problem(1000, 256, 384, 8, 2, zipf_s=1.2, seed=21)
    run = GpuRun(p)
    C = 2
    wsb = max(layer.workspace_bytes(run.counts(C).cpu(), run.mf.dims, C, capi.FWD),
              layer.workspace_bytes(run.counts(C).cpu(), run.mf.dims, C, capi.BWD))
    ws = torch.empty(wsb, dtype=torch.uint8, device=run.dev)
    f32 = dict(dtype=torch.float32, device=run.dev)
    y, dx = torch.empty_like(run.x), torch.empty_like(run.x)
    g3 = [torch.empty(t.shape, **f32) for t in (run.wg, run.wu, run.wd)]
    ds = torch.empty(run.w.shape, **f32)

    def step():
        run.mf.moe_fwd(run.x, run.ids, run.w, run.wg, run.wu, run.wd, C, ws, y=y)
        run.mf.moe_bwd(run.dy, run.x, run.ids, run.w, run.wg, run.wu, run.wd, C, ws, dx=dx, dw_gate=g3[0],
                       dw_up=g3[1], dw_down=g3[2], dscore=ds)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()                      # warm-up: kernel attributes / modules loaded outside capture
        torch.cuda.synchronize()
        ref = [t.clone() for t in (y, dx, *g3, ds)]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            step()
    for t in (y, dx, *g3, ds):
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert run.mf.sync() == 0
    for a, b in zip((y, dx, *g3), ref[:5]):
        assert torch.equal(a, b)
    assert (ds - ref[5]).abs().max().item() <= 1e-5 * ref[5].abs().max().item()
