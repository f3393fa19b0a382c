"""ctypes binding of the C ABI in include/mcrdl_nvl.h (libmcrdl_nvl.so).

This is the reference-side binding a Python host uses: the reference itself
is pure Python, so ctypes is its natural FFI. Loading fails
loudly when the library is missing — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from ctypes import (CFUNCTYPE, POINTER, Structure, c_char_p, c_double, c_int, c_int64, c_size_t,
                    c_uint64, c_void_p)
from pathlib import Path
from typing import Optional

from ..errors import NativeBackendMissing, from_status

LIB_PATH = Path(__file__).resolve().parents[1] / "lib" / "libmcrdl_nvl.so"

ALLGATHER_FN = CFUNCTYPE(c_int, c_void_p, c_void_p, c_void_p, c_size_t)


class Caps(Structure):
    _fields_ = [
        ("rank", c_int), ("world", c_int), ("device", c_int), ("num_sms", c_int),
        ("nvls_supported", c_int), ("ranks_per_device", c_int),
        ("workspace_bytes", c_uint64), ("max_oneshot_bytes", c_uint64),
        ("max_twoshot_chunk", c_uint64),
    ]


_P = c_void_p
_I64P = POINTER(c_int64)
# name -> (restype, argtypes); every entry point declared in include/mcrdl_nvl.h
SIGNATURES = {
    "mcrdl_comm_init": (c_int, [POINTER(c_void_p), c_int, c_int, c_int, ALLGATHER_FN, c_void_p,
                                c_uint64, c_double]),
    "mcrdl_comm_destroy": (c_int, [_P]),
    "mcrdl_comm_caps": (c_int, [_P, POINTER(Caps)]),
    "mcrdl_comm_status": (c_int, [_P]),
    "mcrdl_comm_stream": (c_int, [_P, c_int, POINTER(c_void_p)]),
    "mcrdl_comm_set_tuning": (c_int, [_P, c_int, c_int, POINTER(c_uint64), POINTER(c_int)]),
    "mcrdl_comm_last_algo": (c_int, [_P, c_int]),
    "mcrdl_comm_log_id": (c_uint64, [_P]),
    "mcrdl_comm_op_time": (c_int, [_P, c_uint64, c_uint64, _I64P]),
    "mcrdl_comm_log_flush": (c_int, [_P]),
    "mcrdl_symm_alloc": (c_int, [_P, c_uint64, POINTER(c_void_p)]),
    "mcrdl_symm_free": (c_int, [_P, _P]),
    "mcrdl_pool_create": (c_int, [_P, c_uint64, POINTER(c_void_p)]),
    "mcrdl_pool_activate": (c_int, [_P]),
    "mcrdl_pool_stats": (c_int, [_P, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)]),
    "mcrdl_pool_destroy": (c_int, [_P]),
    "mcrdl_pool_malloc": (c_void_p, [c_int64, c_int, _P]),
    "mcrdl_pool_free": (None, [_P, c_size_t, c_int, _P]),
    "mcrdl_all_reduce": (c_int, [_P, _P, _P, c_uint64, c_int, c_int, c_int, c_uint64, _P]),
    "mcrdl_reduce_scatter": (c_int, [_P, _P, _P, c_uint64, c_int, c_int, c_int, c_uint64, _P]),
    "mcrdl_reduce": (c_int, [_P, _P, _P, c_uint64, c_int, c_int, c_int, c_int, c_uint64, _P]),
    "mcrdl_all_to_allv": (c_int, [_P, _P, _P, _I64P, _I64P, _I64P, _I64P, c_int, c_int, c_uint64, _P]),
    "mcrdl_all_to_allv_dev": (c_int, [_P, _P, c_uint64, _P, c_uint64, _P, c_int, c_int, c_uint64,
                                      _P]),
    "mcrdl_all_to_all_single": (c_int, [_P, _P, _P, c_uint64, c_int, c_int, c_uint64, _P]),
    "mcrdl_all_to_all_ptrs": (c_int, [_P, POINTER(c_void_p), _I64P, POINTER(c_void_p), _I64P, c_int,
                                      c_int, c_uint64, _P]),
    "mcrdl_all_gatherv": (c_int, [_P, _P, _P, _I64P, _I64P, c_int, c_int, c_uint64, _P]),
    "mcrdl_gatherv": (c_int, [_P, _P, _P, _I64P, _I64P, c_int, c_int, c_int, c_uint64, _P]),
    "mcrdl_all_gatherv_dev": (c_int, [_P, _P, c_uint64, _P, c_uint64, _P, _P, c_int, c_int,
                                      c_uint64, _P]),
    "mcrdl_gatherv_dev": (c_int, [_P, _P, c_uint64, _P, c_uint64, _P, _P, c_int, c_int, c_int,
                                  c_uint64, _P]),
    "mcrdl_bcast": (c_int, [_P, _P, c_uint64, c_int, c_int, c_int, c_uint64, _P]),
    "mcrdl_barrier": (c_int, [_P, c_uint64, _P]),
    "mcrdl_send": (c_int, [_P, _P, c_uint64, c_int, _P]),
    "mcrdl_recv": (c_int, [_P, _P, c_uint64, c_int, _P]),
    "mcrdl_fusion_pack": (c_int, [_P, _P, _P, c_int, _P, _P]),
    "mcrdl_fusion_unpack": (c_int, [_P, _P, _P, _P, c_int, _P]),
    "mcrdl_all_reduce_fused": (c_int, [_P, _P, _P, _P, _P, c_int, c_uint64, c_int, c_int, c_int,
                                       c_uint64, _P]),
    "mcrdl_last_error": (c_char_p, []),
    "mcrdl_status_kind": (c_char_p, [c_int]),
    "mcrdl_abi_version": (c_int, []),
    "mcrdl_launch_count": (c_uint64, []),
    "mcrdl_debug_trace": (c_int, [_P, POINTER(POINTER(c_uint64)), POINTER(c_uint64)]),
}

_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    """Load libmcrdl_nvl.so (built in-tree by paper_2303_08374_b200.build)."""
    global _lib, LIB_PATH
    if _lib is not None:
        return _lib
    import os

    if os.environ.get("MCRDL_TRACE_LIB", "0") not in ("", "0"):
        LIB_PATH = LIB_PATH.with_name("libmcrdl_nvl_trace.so")  # developer timeline build
    if not LIB_PATH.exists():
        raise NativeBackendMissing(
            f"{LIB_PATH} is not built; run `python -m paper_2303_08374_b200.build` "
            "(the NVLink backend has no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int) -> None:
    """Raise the mapped CommError for a non-zero status."""
    if code != 0:
        msg = load().mcrdl_last_error().decode(errors="replace")
        raise from_status(code, msg)


def i64_array(values) -> ctypes.Array:
    return (c_int64 * len(values))(*[int(v) for v in values])


def ptr_array(values) -> ctypes.Array:
    return (c_void_p * len(values))(*[int(v) if v else None for v in values])


def launch_count() -> int:
    return int(load().mcrdl_launch_count())
