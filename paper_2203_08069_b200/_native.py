"""ctypes binding of the C ABI in `include/distal_b200.h`.

The library (`libdistal_b200.so`, built in-tree by `make` /
`__graft_entry__.build()`) is the only compute path: there is no CPU
fallback.  `lib()` raises `DeviceUnavailable` if the library is missing, and
`check()` turns negative status codes into `NativeError` with the message
from `td_last_error()`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceUnavailable, NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdistal_b200.so")

_lock = threading.Lock()
_lib = None

vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int, C.c_void_p
_I64P = C.POINTER(C.c_int64)

_SIGNATURES = {
    "td_version": ([], i32),
    "td_last_error": ([], C.c_char_p),
    "td_device_count": ([], i32),
    "td_set_device": ([i32], i32),
    "td_launch_count": ([], C.c_longlong),
    "td_stream_device": ([vp], i32),
    "td_dgemm": ([vp, i64, i64, i64, dp, i64, dp, i64, dp, i64, i32], i32),
    "td_dgemm_config": ([vp, i32, i64, i64, i64, dp, i64, dp, i64, dp, i64, i32], i32),
    "td_dgemm_batched": ([vp, i64, i64, i64, i64, dp, i64, i64, dp, i64, i64, dp, i64, i64, i32], i32),
    "td_ttv": ([vp, i64, i64, i64, dp, i64, i64, dp, dp, i64, i64, i32], i32),
    "td_ttm": ([vp, i64, i64, i64, i64, dp, i64, i64, dp, i64, dp, i64, i64, i32], i32),
    "td_mttkrp": ([vp, i64, i64, i64, i64, dp, i64, i64, dp, i64, dp, i64, dp, i64, i32], i32),
    "td_mttkrp_config": ([vp, i32, i64, i64, i64, i64, dp, i64, i64, dp, i64, dp, i64, dp, i64, i32], i32),
    "td_innerprod": ([vp, i64, i64, dp, i64, dp, i64, dp, dp, i32], i32),
    "td_innerprod_work_size": ([], i64),
    "td_nest_eval": ([vp, vp, i64], i32),
    "td_copy_box": ([vp, i32, _I64P, dp, _I64P, dp, _I64P, i32], i32),
    "td_memcpy_2d": ([vp, dp, i64, dp, i64, i64, i64], i32),
    "td_fill": ([vp, dp, i64, C.c_double], i32),
    "td_generate": ([vp, i32, _I64P, _I64P, _I64P, dp, _I64P, C.c_uint64, C.c_uint64, i32], i32),
    "td_nccl_version": ([], i32),
    "td_comm_unique_id": ([C.c_char_p], i32),
    "td_comm_init_rank": ([C.POINTER(vp), i32, i32, C.c_char_p, i32], i32),
    "td_comm_init_all": ([C.POINTER(vp), i32, C.POINTER(C.c_int)], i32),
    "td_comm_destroy": ([vp], i32),
    "td_comm_split": ([vp, i32, i32, C.POINTER(vp)], i32),
    "td_group_start": ([], i32),
    "td_group_end": ([], i32),
    "td_send": ([vp, vp, dp, i64, i32], i32),
    "td_recv": ([vp, vp, dp, i64, i32], i32),
    "td_bcast": ([vp, vp, dp, i64, i32], i32),
    "td_reduce_sum": ([vp, vp, dp, dp, i64, i32], i32),
    "td_allreduce_sum": ([vp, vp, dp, dp, i64], i32),
    "td_peer_can_access": ([i32, i32], i32),
    "td_peer_enable": ([i32, i32], i32),
    "td_peer_alloc": ([i32, i64, C.POINTER(vp), C.c_char_p], i32),
    "td_peer_free": ([i32, vp], i32),
    "td_peer_open": ([i32, C.c_char_p, C.POINTER(vp)], i32),
    "td_peer_close": ([i32, vp], i32),
}

EXPORTED = tuple(_SIGNATURES)


def load(path: str = LIB_PATH):
    """Load and prototype the library (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceUnavailable(
                f"{path} is missing: build it with `make` (or __graft_entry__.build()); "
                "this package has no CPU fallback")
        lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def check(status: int, what: str = "") -> int:
    if status < 0:
        msg = lib().td_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'native call'} failed ({status}): {msg}")
    return status


def call(name: str, *args) -> int:
    return check(getattr(lib(), name)(*args), name)


def i64_array(values):
    vals = list(values) or [0]
    return (C.c_int64 * len(vals))(*vals)


def launch_count() -> int:
    return int(lib().td_launch_count())
