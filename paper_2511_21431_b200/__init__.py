"""MemFine (arXiv 2511.21431) on B200: the chunked MoE layer behind libmemfine.so.

``capi``  — ctypes binding of include/memfine.h (marshalling only)
``layer`` — torch tensors / streams / process groups around the C ABI
``build`` — nvcc build of libmemfine.so for sm_100a (in-tree)
"""
from . import capi  # noqa: F401
from .layer import MemFine, make_dims, plan, workspace_bytes  # noqa: F401
