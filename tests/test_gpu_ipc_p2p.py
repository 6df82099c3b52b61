"""N1 across PROCESSES (run with -m gpu): EP = 2 ranks as two processes sharing the one GPU, each with a
memfine_create_ipc handle (no NCCL - NCCL refuses two ranks on one device).  The ranks exchange their
workspace mapping records over torch.distributed (gloo), map each other's workspace and sync area through
CUDA IPC (memfine_ipc_export / memfine_ipc_import), and run the device-planned fused exchange: counts pushed
into the peers' sync areas, rows pushed into the peers' expert-major buffers, down / dX epilogues storing
into the sources' combine buffers, epoch-stamped flags waited on by device kernels (system scope).  Every
rank's Y, dX, d_score and local dW are compared with the oracle's EP emulation, as for the in-process
group (tests/test_gpu_ep_local.py)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.harness import rel_err, tol

pytestmark = pytest.mark.gpu

T, H, G, E, K = 300, 128, 256, 8, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, C, overlap, out_dir):
    import torch.distributed as dist
    from paper_2511_21431_b200 import capi, layer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = "cuda:0"
        dt = torch.bfloat16
        El = E // world
        x = synth.make_x(T, H, rank=rank, dtype=dt).to(dev)
        dy = synth.make_dy(T, H, rank=rank, dtype=dt).to(dev)
        ids_np, w_np = synth.make_routing(T, E, K, rank=rank, zipf_s=1.2, placement="contiguous")
        ids, w = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
        wg, wu, wd = synth.make_experts(range(E), H, G, dtype=dt)
        lwg, lwu, lwd = (t[rank * El:(rank + 1) * El].contiguous().to(dev) for t in (wg, wu, wd))
        mf = layer.MemFine(T, H, G, E, K, ep_size=world, ep_rank=rank, dtype=dt, ipc=True, overlap=overlap)
        # A1 on this rank; the all-gather (A2) through gloo here, only to size the workspace - inside the
        # layer calls the counts travel through the peers' sync areas
        counts = mf.route_counts(ids, nsub=C)
        torch.cuda.synchronize()
        rows = [torch.zeros((C, E), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(rows, counts[rank].cpu().contiguous())
        ch = torch.stack(rows).contiguous()
        wsb = 0
        for r in range(world):
            dr = layer.make_dims(T, H, G, E, K, ep_size=world, ep_rank=r, dtype=dt, overlap=overlap)
            wsb = max(wsb, layer.workspace_bytes(ch, dr, C, capi.FWD), layer.workspace_bytes(ch, dr, C, capi.BWD))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        rec = mf.ipc_export(ws)
        recs = [None] * world
        dist.all_gather_object(recs, rec)
        mf.ipc_import(recs)
        dist.barrier()   # every rank mapped every peer before the first signal
        y = mf.moe_fwd(x, ids, w, lwg, lwu, lwd, C, ws)
        dx, dwg, dwu, dwd, ds = mf.moe_bwd(dy, x, ids, w, lwg, lwu, lwd, C, ws)
        status = mf.sync()
        out = {n: t.float().cpu().numpy() for n, t in (("y", y), ("dx", dx), ("ds", ds), ("dwg", dwg),
                                                         ("dwu", dwu), ("dwd", dwd))}
        out["status"] = np.array(status)
        out["counts"] = ch.numpy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
        dist.barrier()   # no rank unmaps / frees while a peer's kernels may still touch its memory
        mf.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("C,overlap", [(1, False), (2, False), (3, True)])
def test_ipc_p2p_two_processes_match_oracle(C, overlap, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), C, overlap, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for r in range(world):
        assert int(res[r]["status"]) == 0, (r, int(res[r]["status"]))
    routes = [synth.make_routing(T, E, K, rank=r, zipf_s=1.2, placement="contiguous") for r in range(world)]
    od1 = oracle.Dims(T=T, h=H, g=G, E=E, k=K)
    ref_counts = np.stack([oracle.route_counts(od1, routes[r][0], C)[0] for r in range(world)])
    for r in range(world):
        np.testing.assert_array_equal(res[r]["counts"], ref_counts)
    d = oracle.Dims(T=T, h=H, g=G, E=E, k=K, EP=world, in_dtype="bf16")
    bits = lambda t: t.contiguous().view(torch.int16).numpy().view(np.uint16)
    xa = np.concatenate([bits(synth.make_x(T, H, rank=r, dtype=torch.bfloat16)) for r in range(world)])
    dya = np.concatenate([bits(synth.make_dy(T, H, rank=r, dtype=torch.bfloat16)) for r in range(world)])
    ida = np.concatenate([rt[0] for rt in routes])
    wa = np.concatenate([rt[1] for rt in routes]).astype(np.float64)
    W = [bits(t) for t in synth.make_experts(range(E), H, G, dtype=torch.bfloat16)]
    y_ref, _, _ = oracle.fcda_forward(d, C, xa, ida, wa, *W)
    dx_ref, ds_ref, dwg_ref, dwu_ref, dwd_ref, _, _ = oracle.fcda_backward(d, C, dya, xa, ida, wa, *W)
    El = E // world
    t_ = tol(torch.bfloat16)
    for r in range(world):
        sl, es = slice(r * T, (r + 1) * T), slice(r * El, (r + 1) * El)
        errs = {"y": rel_err(res[r]["y"], y_ref[sl]), "dx": rel_err(res[r]["dx"], dx_ref[sl]),
                "dscore": rel_err(res[r]["ds"], ds_ref[sl]), "dw_gate": rel_err(res[r]["dwg"], dwg_ref[es]),
                "dw_up": rel_err(res[r]["dwu"], dwu_ref[es]), "dw_down": rel_err(res[r]["dwd"], dwd_ref[es])}
        assert all(v <= t_ for v in errs.values()), (r, errs)
