"""Torch-facing wrapper of the C ABI: device memory, streams and EP process groups only.

The names follow include/memfine.h: ``plan`` (memfine_plan), ``workspace_bytes``
(memfine_workspace_bytes), and on a ``MemFine`` handle ``route_counts``, ``moe_fwd``,
``moe_bwd``, ``sync``, ``last_stats``.  Nothing here computes any part of the layer.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import capi

_DT = {torch.bfloat16: capi.BF16, torch.float32: capi.FP32}


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_dims(tokens, hidden, ffn, num_experts, topk, ep_size=1, ep_rank=0, dtype=torch.bfloat16,
              mx: bool = False, overlap: bool = False, ep_path: bool = False, mx_wgrad: bool = False) -> capi.Dims:
    """mx=True: MEMFINE_MXFP8 (bf16 storage, MXFP8 expert-GEMM operands; dtype must be bf16).
    overlap=True: MEMFINE_FLAG_OVERLAP (EP > 1, C > 1: exchange of chunk j+-1 on a comm stream
    while chunk j's GEMMs run; two slots of exchanged rows in the workspace).
    ep_path=True (ep_size == 1): MEMFINE_FLAG_EP_PATH, the EP data path over a 1-rank NCCL comm.
    mx_wgrad=True (mx): MEMFINE_FLAG_MX_WGRAD, MXFP8 weight gradients (reading R28c)."""
    assert not mx or dtype == torch.bfloat16
    return capi.Dims(int(tokens), int(hidden), int(ffn), int(num_experts), int(topk), int(ep_size), int(ep_rank),
                     capi.MXFP8 if mx else _DT[dtype],
                     (capi.FLAG_OVERLAP if overlap else 0) | (capi.FLAG_EP_PATH if ep_path else 0) |
                     (capi.FLAG_MX_WGRAD if mx_wgrad else 0))


def mx_weights_bytes(dims: capi.Dims) -> int:
    out = C.c_uint64()
    capi.check(capi.lib().memfine_mx_weights_bytes(C.byref(dims), C.byref(out)), "memfine_mx_weights_bytes")
    return int(out.value)


def mx_quantize(src: torch.Tensor, stream=None):
    """memfine_mx_quantize: bf16 [rows][K] -> (E4M3 codes uint8 [rows][K], scale codes uint8 [rows*K/32])."""
    assert src.dtype == torch.bfloat16 and src.is_cuda and src.is_contiguous() and src.dim() == 2
    codes = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    scales = torch.empty(src.numel() // 32, dtype=torch.uint8, device=src.device)
    capi.check(capi.lib().memfine_mx_quantize(_ptr(src), src.shape[0], src.shape[1], _ptr(codes), _ptr(scales),
                                              _stream(stream)), "memfine_mx_quantize")
    return codes, scales


def m_g(v: int, p: int, r_pp: int, full_recompute: bool = False) -> int:
    """memfine_m_g: Eq. 2's m_g for pipeline stage r_pp (1 under full recomputation)."""
    out = C.c_int32()
    capi.check(capi.lib().memfine_m_g(int(v), int(p), int(r_pp), int(bool(full_recompute)), C.byref(out)),
               "memfine_m_g")
    return int(out.value)


def plan(counts: torch.Tensor, dims: capi.Dims, budget: capi.Budget, stream=False) -> dict:
    """memfine_plan: counts int32 [EP][nsub][E] on the host (CPU tensor) or the device.  stream: False =
    memfine_plan (synchronises the device); None or a torch stream = memfine_plan_stream on that stream
    (None: the current stream) - the caller's other streams keep running."""
    assert counts.dtype == torch.int32 and counts.dim() == 3 and counts.is_contiguous()
    info = capi.PlanInfo()
    if stream is False:
        st = capi.lib().memfine_plan(_ptr(counts), counts.shape[1], C.byref(dims), C.byref(budget), C.byref(info))
    else:
        st = capi.lib().memfine_plan_stream(_ptr(counts), counts.shape[1], C.byref(dims), C.byref(budget),
                                            C.byref(info), _stream(stream))
    d = info.as_dict()
    d["status"] = int(st)
    return d


def workspace_bytes(counts_host: Optional[torch.Tensor], dims: capi.Dims, C_: int, pass_: int) -> int:
    out = C.c_uint64()
    if counts_host is not None:
        assert counts_host.device.type == "cpu" and counts_host.dtype == torch.int32 and counts_host.is_contiguous()
        nsub = counts_host.shape[1]
    else:
        nsub = 0
    capi.check(capi.lib().memfine_workspace_bytes(_ptr(counts_host), nsub, C.byref(dims), C_, pass_, C.byref(out)),
               "memfine_workspace_bytes")
    return int(out.value)


def a2a_plan(counts_host: torch.Tensor, dims: capi.Dims, C_: int, chunk: int):
    """memfine_a2a_plan: (send_rows [EP], recv_rows [EP], recv_offsets [EP, E_l], rows_padded)."""
    import numpy as np
    assert counts_host.device.type == "cpu" and counts_host.dtype == torch.int32 and counts_host.is_contiguous()
    EP, El = dims.ep_size, dims.num_experts // dims.ep_size
    send = np.zeros(EP, np.int64)
    recv = np.zeros(EP, np.int64)
    off = np.zeros((EP, El), np.int64)
    rp = C.c_int64()
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    capi.check(capi.lib().memfine_a2a_plan(_ptr(counts_host), counts_host.shape[1], C.byref(dims), C_, chunk,
                                           vp(send), vp(recv), vp(off), C.byref(rp)), "memfine_a2a_plan")
    return send, recv, off, int(rp.value)


class LocalGroup:
    """memfine_local_group_create: ep_size ranks of one layer in this process on one device
    (one host thread per rank); used to validate the EP data path on a single GPU."""

    def __init__(self, nranks: int):
        g = C.c_void_p()
        capi.check(capi.lib().memfine_local_group_create(nranks, C.byref(g)), "memfine_local_group_create")
        self.g = g

    def close(self):
        if getattr(self, "g", None):
            capi.lib().memfine_local_group_destroy(self.g)
            self.g = None


class MemFine:
    """One handle = one EP rank of one MoE layer shape.  ``process_group``: the EP group
    (torch.distributed) used only to broadcast the NCCL unique id when ep_size > 1."""

    def __init__(self, tokens, hidden, ffn, num_experts, topk, ep_size=1, ep_rank=0, dtype=torch.bfloat16,
                 process_group=None, local_group=None, mx: bool = False, overlap: bool = False,
                 ep_path: bool = False, mx_wgrad: bool = False, ipc: bool = False):
        self.dims = make_dims(tokens, hidden, ffn, num_experts, topk, ep_size, ep_rank, dtype, mx, overlap, ep_path,
                              mx_wgrad)
        self.dtype = dtype
        self.mx = mx
        self._wq = None
        self.E_l = num_experts // ep_size
        self._ws = None
        if local_group is not None:
            h = C.c_void_p()
            capi.check(capi.lib().memfine_create_local(C.byref(self.dims), local_group.g, C.byref(h)),
                       "memfine_create_local")
            self.h = h
            return
        if ipc:   # memfine_create_ipc: P2P transport only, mappings exchanged by the caller (no NCCL)
            h = C.c_void_p()
            capi.check(capi.lib().memfine_create_ipc(C.byref(self.dims), C.byref(h)), "memfine_create_ipc")
            self.h = h
            return
        uid = None
        if ep_path and ep_size == 1:
            buf = (C.c_uint8 * 128)()
            capi.check(capi.lib().memfine_nccl_unique_id(buf), "memfine_nccl_unique_id")
            uid = buf
        elif ep_size > 1:
            import torch.distributed as dist
            buf = (C.c_uint8 * 128)()
            if ep_rank == 0:
                capi.check(capi.lib().memfine_nccl_unique_id(buf), "memfine_nccl_unique_id")
            obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(process_group, 0) if process_group else 0,
                                       group=process_group)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        capi.check(capi.lib().memfine_create(C.byref(self.dims), uid, C.byref(h)), "memfine_create")
        self.h = h
        self._ws = None

    def close(self):
        if getattr(self, "h", None):
            capi.lib().memfine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ A1 + A2
    def route_counts(self, ids: torch.Tensor, nsub: int = 8, stream=None) -> torch.Tensor:
        d = self.dims
        assert ids.dtype == torch.int32 and ids.is_cuda and ids.is_contiguous()
        counts = torch.empty((d.ep_size, nsub, d.num_experts), dtype=torch.int32, device=ids.device)
        capi.check(capi.lib().memfine_route_counts(self.h, _ptr(ids), nsub, _ptr(counts), _stream(stream)),
                   "memfine_route_counts")
        return counts

    def workspace(self, counts_host, C_: int, pass_: int, device=None) -> torch.Tensor:
        n = workspace_bytes(counts_host, self.dims, C_, pass_)
        return torch.empty(n, dtype=torch.uint8, device=device or torch.cuda.current_device())

    # ------------------------------------------------------------------ MXFP8 variant (N4)
    def mx_quantize_weights(self, w_gate, w_up, w_down, wq: Optional[torch.Tensor] = None, stream=None):
        """memfine_mx_quantize_weights: quantise and bind the local experts' weights (again after
        every weight update).  Returns the (kept-alive) quantised-weights buffer."""
        if wq is None:
            wq = torch.empty(mx_weights_bytes(self.dims), dtype=torch.uint8, device=w_gate.device)
        capi.check(capi.lib().memfine_mx_quantize_weights(self.h, _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(wq),
                                                          wq.numel(), _stream(stream)), "memfine_mx_quantize_weights")
        self._wq = wq
        return wq

    # ------------------------------------------------------------------ FCDA forward / backward
    def moe_fwd(self, x, ids, w, w_gate, w_up, w_down, C_: int, ws: torch.Tensor, y=None, stream=None):
        if y is None:
            y = torch.empty_like(x)
        capi.check(capi.lib().memfine_moe_fwd(self.h, _ptr(x), _ptr(ids), _ptr(w), _ptr(w_gate), _ptr(w_up),
                                              _ptr(w_down), C_, _ptr(y), _ptr(ws), ws.numel(), _stream(stream)),
                   "memfine_moe_fwd")
        return y

    def moe_bwd(self, dy, x, ids, w, w_gate, w_up, w_down, C_: int, ws: torch.Tensor, dx=None, dw_gate=None,
                dw_up=None, dw_down=None, dscore=None, accumulate_dw=False, want_dscore=True, stream=None):
        if dx is None:
            dx = torch.empty_like(x)
        f32 = dict(dtype=torch.float32, device=x.device)
        if dw_gate is None:
            dw_gate = torch.empty(w_gate.shape, **f32)
        if dw_up is None:
            dw_up = torch.empty(w_up.shape, **f32)
        if dw_down is None:
            dw_down = torch.empty(w_down.shape, **f32)
        if dscore is None and want_dscore:
            dscore = torch.empty(w.shape, **f32)
        capi.check(capi.lib().memfine_moe_bwd(self.h, _ptr(dy), _ptr(x), _ptr(ids), _ptr(w), _ptr(w_gate),
                                              _ptr(w_up), _ptr(w_down), C_, _ptr(dx), _ptr(dw_gate), _ptr(dw_up),
                                              _ptr(dw_down), _ptr(dscore), int(bool(accumulate_dw)), _ptr(ws),
                                              ws.numel(), _stream(stream)),
                   "memfine_moe_bwd")
        return dx, dw_gate, dw_up, dw_down, dscore

    # ------------------------------------------------------------------ router (N3)
    def router_fwd(self, x, w_router, logits=None, stream=None):
        T, k = x.shape[0], self.dims.topk
        ids = torch.empty((T, k), dtype=torch.int32, device=x.device)
        scores = torch.empty((T, k), dtype=torch.float32, device=x.device)
        capi.check(capi.lib().memfine_router_fwd(self.h, _ptr(x), _ptr(w_router), _ptr(ids), _ptr(scores),
                                                 _ptr(logits), _stream(stream)), "memfine_router_fwd")
        return ids, scores

    def router_bwd(self, x, w_router, ids, scores, dscore, dx=None, accumulate_dx=False, dw_router=None,
                   accumulate_dw=False, stream=None):
        if dx is None:
            dx = torch.empty_like(x)
        if dw_router is None:
            dw_router = torch.empty(w_router.shape, dtype=torch.float32, device=x.device)
        capi.check(capi.lib().memfine_router_bwd(self.h, _ptr(x), _ptr(w_router), _ptr(ids), _ptr(scores),
                                                 _ptr(dscore), _ptr(dx), int(bool(accumulate_dx)), _ptr(dw_router),
                                                 int(bool(accumulate_dw)), _stream(stream)), "memfine_router_bwd")
        return dx, dw_router

    def sync(self, stream=None) -> int:
        return int(capi.lib().memfine_sync(self.h, _stream(stream)))

    def last_stats(self) -> dict:
        s = capi.Stats()
        capi.check(capi.lib().memfine_last_stats(self.h, C.byref(s)), "memfine_last_stats")
        return s.as_dict()

    def profile_enable(self, on: bool = True):
        capi.check(capi.lib().memfine_profile_enable(self.h, int(on)), "memfine_profile_enable")

    def profile_read(self) -> dict:
        pr = capi.Profile()
        capi.check(capi.lib().memfine_profile_read(self.h, C.byref(pr)), "memfine_profile_read")
        return pr.as_dict()

    def set_ep_transport(self, transport: int):
        capi.check(capi.lib().memfine_set_ep_transport(self.h, int(transport)), "memfine_set_ep_transport")

    def set_comm_sms(self, n: int):
        """memfine_set_comm_sms: SMs the GEMMs leave to the comm stream while chunks overlap."""
        capi.check(capi.lib().memfine_set_comm_sms(self.h, int(n)), "memfine_set_comm_sms")

    def register_workspace(self, ws: torch.Tensor, stream=None):
        """memfine_register_workspace (collective for NCCL handles): map every rank's workspace
        for the fused peer-memory exchange."""
        capi.check(capi.lib().memfine_register_workspace(self.h, _ptr(ws), ws.numel(), _stream(stream)),
                   "memfine_register_workspace")

    def ipc_export(self, ws: torch.Tensor) -> bytes:
        """memfine_ipc_export: this rank's mapping record for workspace ws (IPC handles)."""
        rec = (C.c_uint8 * capi.IPC_RECORD_BYTES)()
        capi.check(capi.lib().memfine_ipc_export(self.h, _ptr(ws), ws.numel(), rec), "memfine_ipc_export")
        return bytes(rec)

    def ipc_import(self, records):
        """memfine_ipc_import: every rank's record (rank order); the caller barriers afterwards."""
        buf = (C.c_uint8 * (capi.IPC_RECORD_BYTES * len(records))).from_buffer_copy(b"".join(records))
        capi.check(capi.lib().memfine_ipc_import(self.h, buf), "memfine_ipc_import")

    def set_debug(self, on: bool = True):
        capi.check(capi.lib().memfine_set_debug(self.h, int(on)), "memfine_set_debug")

    def debug_perm(self, chunk: int):
        import numpy as np
        n = C.c_int64()
        capi.check(capi.lib().memfine_debug_perm(self.h, chunk, None, 0, C.byref(n)), "memfine_debug_perm")
        out = np.zeros(max(1, n.value), dtype=np.int64)
        capi.check(capi.lib().memfine_debug_perm(self.h, chunk, out.ctypes.data_as(C.c_void_p), out.size,
                                                 C.byref(n)), "memfine_debug_perm")
        return out[:n.value]

    def debug_rows(self, chunk: int):
        """The last call's chunk `chunk`: copy index (i*k + slot) of every expert-major padded row, -1 padding."""
        import numpy as np
        n = C.c_int64()
        capi.check(capi.lib().memfine_debug_rows(self.h, chunk, None, 0, C.byref(n)), "memfine_debug_rows")
        out = np.zeros(max(1, n.value), dtype=np.int32)
        capi.check(capi.lib().memfine_debug_rows(self.h, chunk, out.ctypes.data_as(C.c_void_p), out.size,
                                                 C.byref(n)), "memfine_debug_rows")
        return out[:n.value]

    def debug_mx(self, chunk: int, which: int):
        """MXFP8 decisions of the last call's chunk (memfine_debug_mx): (codes uint8 [rows][cols], scale
        bytes uint8 [rows*cols/32] in the scale-chunk layout with K = cols)."""
        import numpy as np
        r, c = C.c_int64(), C.c_int64()
        capi.check(capi.lib().memfine_debug_mx(self.h, chunk, which, None, None, 0, C.byref(r), C.byref(c)),
                   "memfine_debug_mx")
        q = np.zeros(max(1, r.value * c.value), dtype=np.uint8)
        sf = np.zeros(max(1, r.value * c.value // 32), dtype=np.uint8)
        capi.check(capi.lib().memfine_debug_mx(self.h, chunk, which, q.ctypes.data_as(C.c_void_p),
                                               sf.ctypes.data_as(C.c_void_p), q.size, C.byref(r), C.byref(c)),
                   "memfine_debug_mx")
        return q[:r.value * c.value].reshape(r.value, c.value), sf[:r.value * c.value // 32]
