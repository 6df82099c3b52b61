"""Thin ctypes binding of libmemfine.so (include/memfine.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.  There is no fallback — if the
library is missing or cannot load, import-time use raises."""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmemfine.so")

OK, ERR_INVALID_ARG, ERR_INFEASIBLE, ERR_ROUTING, ERR_CUDA, ERR_NCCL, ERR_WORKSPACE, ERR_UNSUPPORTED = range(8)
BF16, FP32, MXFP8 = 0, 1, 2
RULE_EXACT, RULE_EQ9 = 0, 1      # memfine_budget.rule: EXACT is the default (0)
MODEL_PAPER, MODEL_IMPL = 0, 1
EP_COPY, EP_P2P = 0, 1
FLAG_OVERLAP, FLAG_EP_PATH, FLAG_MX_WGRAD = 1, 2, 4
FWD, BWD = 0, 1
IPC_RECORD_BYTES = 256   # MEMFINE_IPC_RECORD_BYTES

# Every symbol include/memfine.h declares (checked by tests/test_abi.py).
SYMBOLS = ("memfine_abi_version", "memfine_status_str", "memfine_nccl_unique_id", "memfine_create",
           "memfine_destroy", "memfine_local_group_create", "memfine_local_group_destroy", "memfine_create_local", "memfine_create_ipc", "memfine_ipc_export", "memfine_ipc_import", "memfine_set_ep_transport", "memfine_set_comm_sms", "memfine_register_workspace", "memfine_route_counts", "memfine_plan", "memfine_plan_stream", "memfine_workspace_bytes", "memfine_a2a_plan",
           "memfine_moe_fwd", "memfine_moe_bwd", "memfine_router_fwd", "memfine_router_bwd", "memfine_sync", "memfine_last_stats",
           "memfine_profile_enable", "memfine_profile_read", "memfine_set_debug", "memfine_debug_perm",
           "memfine_debug_rows", "memfine_debug_mx",
           "memfine_mx_weights_bytes", "memfine_mx_quantize_weights", "memfine_mx_quantize", "memfine_m_g")

PROF_SLOTS = ("gemm_gateup_swiglu", "gemm_down", "gemm_dact_epilogue", "gemm_dx", "gemm_wgrad_down",
              "gemm_wgrad_gateup", "dispatch_permute", "combine_unpermute", "memset", "nccl_exchange",
              "mx_quant_colwise")


class MemfineError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_str(status)} (status {status})")


class Dims(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("hidden", C.c_int32), ("ffn", C.c_int32),
                ("num_experts", C.c_int32), ("topk", C.c_int32), ("ep_size", C.c_int32),
                ("ep_rank", C.c_int32), ("dtype", C.c_int32), ("flags", C.c_int32)]


class Budget(C.Structure):
    _fields_ = [("gpu_capacity_bytes", C.c_uint64), ("alpha", C.c_double), ("static_bytes", C.c_uint64),
                ("other_act_bytes", C.c_uint64), ("m_g", C.c_uint32), ("tp", C.c_uint32), ("cp", C.c_uint32),
                ("micro_batch", C.c_uint32), ("bins", C.POINTER(C.c_int32)), ("nbins", C.c_int32),
                ("rule", C.c_int32), ("model", C.c_int32), ("pass_", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("C", C.c_int32), ("c_theory", C.c_int32), ("clamped", C.c_int32), ("feasible", C.c_int32),
                ("hot_rank", C.c_int32), ("exact_peak", C.c_int32), ("s_dd_max", C.c_int64),
                ("s_prime_max", C.c_int64), ("s_chunk_max", C.c_int64), ("predicted_peak_bytes", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Stats(C.Structure):
    _fields_ = [("C", C.c_int32), ("pass_", C.c_int32), ("rows", C.c_int64 * 64), ("rows_padded", C.c_int64 * 64),
                ("workspace_used_bytes", C.c_uint64), ("workspace_given_bytes", C.c_uint64),
                ("device_error", C.c_int32), ("gemm_launches", C.c_int32), ("kernel_launches", C.c_int32),
                ("comm_ops", C.c_int32)]

    def as_dict(self):
        n = self.C
        return {"C": n, "pass": self.pass_, "rows": list(self.rows[:n]), "rows_padded": list(self.rows_padded[:n]),
                "workspace_used_bytes": self.workspace_used_bytes,
                "workspace_given_bytes": self.workspace_given_bytes, "device_error": self.device_error,
                "gemm_launches": self.gemm_launches, "kernel_launches": self.kernel_launches,
                "comm_ops": self.comm_ops}


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int32 * len(PROF_SLOTS)), ("ms", C.c_double * len(PROF_SLOTS))]

    def as_dict(self):
        return {PROF_SLOTS[i]: {"launches": self.launches[i], "ms": self.ms[i]} for i in range(len(PROF_SLOTS))}


_lib = None


def lib():
    """Load libmemfine.so (built by __graft_entry__.build() / paper_2511_21431_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        L.memfine_abi_version.restype = i32
        L.memfine_status_str.restype = C.c_char_p
        L.memfine_status_str.argtypes = [C.c_int]
        for name in SYMBOLS[2:]:
            getattr(L, name).restype = C.c_int
        L.memfine_nccl_unique_id.argtypes = [vp]
        L.memfine_create.argtypes = [C.POINTER(Dims), vp, C.POINTER(vp)]
        L.memfine_destroy.argtypes = [vp]
        L.memfine_local_group_create.argtypes = [i32, C.POINTER(vp)]
        L.memfine_local_group_destroy.argtypes = [vp]
        L.memfine_create_local.argtypes = [C.POINTER(Dims), vp, C.POINTER(vp)]
        L.memfine_set_ep_transport.argtypes = [vp, i32]
        L.memfine_set_comm_sms.argtypes = [vp, i32]
        L.memfine_register_workspace.argtypes = [vp, vp, u64, vp]
        L.memfine_create_ipc.argtypes = [C.POINTER(Dims), C.POINTER(vp)]
        L.memfine_ipc_export.argtypes = [vp, vp, u64, vp]
        L.memfine_ipc_import.argtypes = [vp, vp]
        L.memfine_route_counts.argtypes = [vp, vp, i32, vp, vp]
        L.memfine_plan.argtypes = [vp, i32, C.POINTER(Dims), C.POINTER(Budget), C.POINTER(PlanInfo)]
        L.memfine_plan_stream.argtypes = [vp, i32, C.POINTER(Dims), C.POINTER(Budget), C.POINTER(PlanInfo), vp]
        L.memfine_workspace_bytes.argtypes = [vp, i32, C.POINTER(Dims), i32, i32, C.POINTER(u64)]
        L.memfine_a2a_plan.argtypes = [vp, i32, C.POINTER(Dims), i32, i32, vp, vp, vp, vp]
        L.memfine_moe_fwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, u64, vp]
        L.memfine_moe_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, vp, u64, vp]
        L.memfine_router_fwd.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.memfine_router_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32, vp, i32, vp]
        L.memfine_sync.argtypes = [vp, vp]
        L.memfine_last_stats.argtypes = [vp, C.POINTER(Stats)]
        L.memfine_profile_enable.argtypes = [vp, i32]
        L.memfine_profile_read.argtypes = [vp, C.POINTER(Profile)]
        L.memfine_set_debug.argtypes = [vp, i32]
        L.memfine_debug_perm.argtypes = [vp, i32, vp, i64, C.POINTER(i64)]
        L.memfine_debug_rows.argtypes = [vp, i32, vp, i64, C.POINTER(i64)]
        L.memfine_debug_mx.argtypes = [vp, i32, i32, vp, vp, i64, C.POINTER(i64), C.POINTER(i64)]
        L.memfine_mx_weights_bytes.argtypes = [C.POINTER(Dims), C.POINTER(u64)]
        L.memfine_mx_quantize_weights.argtypes = [vp, vp, vp, vp, vp, u64, vp]
        L.memfine_mx_quantize.argtypes = [vp, i64, i32, vp, vp, vp]
        if L.memfine_abi_version() != 2:
            raise RuntimeError("libmemfine.so ABI mismatch")
        _lib = L
    return _lib


def status_str(s: int) -> str:
    return lib().memfine_status_str(int(s)).decode()


def check(status: int, where: str) -> None:
    if status != OK:
        raise MemfineError(status, where)


def make_budget(gpu_capacity_bytes: int, alpha: float = 1.0, static_bytes: int = 0, other_act_bytes: int = 0,
                m_g: int = 1, tp: int = 1, cp: int = 1, micro_batch: int = 1, bins=(1, 2, 4, 8),
                rule: int = RULE_EXACT, model: int = MODEL_PAPER, pass_: int = BWD):
    arr = (C.c_int32 * len(bins))(*bins) if bins is not None else None
    b = Budget(int(gpu_capacity_bytes), float(alpha), int(static_bytes), int(other_act_bytes), m_g, tp, cp,
               micro_batch, C.cast(arr, C.POINTER(C.c_int32)) if arr is not None else None,
               len(bins) if bins is not None else 0, rule, model, pass_)
    b._keep = arr  # keep the bins array alive
    return b
