"""The N > 1 (expert-parallel) host logic on CPU with gloo, world_size 2 and 4:
every rank derives the same C from the all-gathered counts (reading R6), the all-to-allv
split tables agree pairwise (what a sends to b is what b expects from a), and the receive
layout is the canonical (local expert, src rank, token, slot) order of the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, errq):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2511_21431_b200 import capi, layer
        T, E, k, h, g = 301, 8, 2, 64, 128
        El = E // world
        ids_all = np.concatenate([synth.make_routing(T, E, k, rank=r, zipf_s=1.2, placement="contiguous")[0]
                                  for r in range(world)])
        od = oracle.Dims(T=T, h=h, g=g, E=E, k=k, EP=world)
        mine, _ = oracle.route_counts(oracle.Dims(T=T, h=h, g=g, E=E, k=k), ids_all[rank * T:(rank + 1) * T], 8)
        # C2 "first notification": all-gather the per-sub-chunk counts
        t = torch.from_numpy(mine.astype(np.int32))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        counts = torch.stack(parts).contiguous()
        dims = layer.make_dims(T, h, g, E, k, ep_size=world, ep_rank=rank)
        for budget in (10**6, 3 * 10**5, 10**5, 5 * 10**4):
            b = capi.make_budget(budget, 1.0, 1000, 0)
            p = layer.plan(counts, dims, b)
            vec = torch.tensor([p["status"], p["C"], p["c_theory"], p["hot_rank"], p["s_dd_max"]], dtype=torch.int64)
            allv = [torch.empty_like(vec) for _ in range(world)]
            dist.all_gather(allv, vec)
            assert all(torch.equal(v, vec) for v in allv), "ranks disagree on the plan"
            st, ro = oracle.plan(counts.numpy().astype(np.int64), od, budget_bytes=budget, static_bytes=1000,
                                 rule=1)   # the library default, rule EXACT
            assert st == p["status"]
            if st == 0:
                assert ro["C"] == p["C"] and ro["hot_rank"] == p["hot_rank"] and ro["s_dd_max"] == p["s_dd_max"]
        for C in (1, 2, 4, 8):
            for j in range(C):
                send, recv, off, rp = layer.a2a_plan(counts, dims, C, j)
                S = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
                R = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(S, torch.from_numpy(send))
                dist.all_gather(R, torch.from_numpy(recv))
                for a in range(world):
                    for b2 in range(world):
                        assert S[a][b2] == R[b2][a], (C, j, a, b2)
                # receive layout == canonical order (reading R3), padding per local expert to 128
                rows = []
                t0, t1 = oracle.chunk_begin(T, C, j), oracle.chunk_begin(T, C, j + 1)
                for el in range(El):
                    e = rank * El + el
                    seg_start = off[0, el]
                    assert seg_start % 128 == 0
                    for src in range(world):
                        qs = [(src * T + i) * k + s for i in range(t0, t1) for s in range(k)
                              if ids_all[src * T + i, s] == e]
                        assert off[src, el] == seg_start + sum(
                            int((ids_all[s2 * T + t0:s2 * T + t1] == e).sum()) for s2 in range(src))
                        rows += [(off[src, el] + n, q) for n, q in enumerate(qs)]
                rows.sort()
                ref = oracle.dispatch_order(od, ids_all, rank, C, j)
                np.testing.assert_array_equal(np.array([q for _, q in rows], np.int64), ref)
                assert rp % 128 == 0 and (not rows or rows[-1][0] < rp)
        # NCCL bootstrap: rank 0's unique id reaches every rank intact (gloo broadcast)
        import ctypes
        buf = (ctypes.c_uint8 * 128)()
        ok = torch.tensor([1])
        if rank == 0:
            ok[0] = int(capi.lib().memfine_nccl_unique_id(buf) == 0)
        dist.broadcast(ok, 0)
        if ok.item():
            obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0)
            if rank == 0:
                assert obj[0] == bytes(buf)
            assert len(obj[0]) == 128 and any(obj[0])
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_ep_host_logic_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, PORTS[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not q.empty():
        errs.append(q.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


PORTS = {2: _free_port(), 4: _free_port()}
