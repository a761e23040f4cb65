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
import struct
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
    "td_dgemm_grouped": ([vp, i32, vp, i32], i32),
    "td_event_create": ([i32, C.POINTER(vp)], i32),
    "td_event_destroy": ([vp], i32),
    "td_event_record": ([vp, vp, i32], i32),
    "td_stream_wait_event": ([vp, vp, i32], i32),
    "td_execute_plan": ([vp, i64], i32),
    "td_comm_wait": ([C.POINTER(vp), i32, C.POINTER(vp), i32, C.c_double], i32),
    "td_init": ([i32, C.POINTER(C.c_int)], i32),
    "td_finalize": ([], i32),
    "td_allgather": ([vp, vp, dp, dp, i64], i32),
    "td_shift": ([vp, vp, dp, dp, i64, i32], i32),
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
    rc = check(getattr(lib(), name)(*args), name)
    rec = _RECORDING
    if rec is not None:
        rec.add(name, args)
    return rc


# ------------------------------------------------------------- launch plans
# td_op kinds (include/distal_b200.h): the entry points a plan may replay
PLAN_OPS = {"td_dgemm": 1, "td_dgemm_batched": 2, "td_dgemm_grouped": 3, "td_ttv": 4, "td_ttm": 5,
            "td_mttkrp": 6, "td_innerprod": 7, "td_nest_eval": 8, "td_copy_box": 9, "td_memcpy_2d": 10,
            "td_fill": 11, "td_group_start": 12, "td_group_end": 13, "td_send": 14, "td_recv": 15,
            "td_bcast": 16, "td_reduce_sum": 17, "td_event_record": 18, "td_stream_wait_event": 19}
# calls with no device effect: harmless while recording
_QUERIES = {"td_version", "td_last_error", "td_device_count", "td_launch_count", "td_stream_device",
            "td_innerprod_work_size", "td_nccl_version", "td_peer_can_access"}
MAX_ARGS = 16


class TdOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nargs", C.c_int32), ("arg", C.c_int64 * MAX_ARGS)]


class TdGemmProblem(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("A", C.c_void_p), ("lda", C.c_int64),
                ("B", C.c_void_p), ("ldb", C.c_int64), ("C", C.c_void_p), ("ldc", C.c_int64),
                ("K2", C.c_int64), ("A2", C.c_void_p), ("lda2", C.c_int64), ("B2", C.c_void_p), ("ldb2", C.c_int64)]


_SIGNATURES["td_dgemm_grouped"] = ([vp, i32, C.POINTER(TdGemmProblem), i32], i32)

_RECORDING = None


def _word(arg, keep) -> int:
    """One argument as the 64-bit word td_execute_plan passes back."""
    if isinstance(arg, (C.Array, C.Structure)):
        keep.append(arg)
        return C.addressof(arg)
    if type(arg).__name__ == "CArgObject":          # C.byref(x)
        keep.append(arg._obj)
        return C.addressof(arg._obj)
    if isinstance(arg, (float, C.c_double)):
        v = arg.value if isinstance(arg, C.c_double) else arg
        return struct.unpack("<q", struct.pack("<d", v))[0]
    if isinstance(arg, C._SimpleCData):
        arg = arg.value or 0
    v = int(arg)
    return v - (1 << 64) if v >= (1 << 63) else v


class PlanRecorder:
    """Collects the plan ops of the native calls issued while it is active
    (they still run: recording is an eager run plus bookkeeping), the device
    buffers those ops touch (kept alive for the plan's lifetime), and the
    native events the plan owns."""

    def __init__(self):
        self.ops = []
        self.keep = []
        self.events = []
        self.valid = True
        self.reason = None

    def add(self, name, args):
        kind = PLAN_OPS.get(name)
        if kind is None:
            if name not in _QUERIES:
                self.invalidate(f"{name} is not replayable")
            return
        if len(args) > MAX_ARGS:
            self.invalidate(f"{name}: {len(args)} arguments")
            return
        self.ops.append((kind, [_word(a, self.keep) for a in args]))

    def invalidate(self, why):
        if self.valid:
            self.valid, self.reason = False, why

    def hold(self, obj):
        self.keep.append(obj)
        return obj

    def event(self, device_index: int) -> int:
        ev = C.c_void_p()
        check(lib().td_event_create(device_index, C.byref(ev)), "td_event_create")
        self.events.append(ev.value)
        return ev.value

    def finish(self) -> "Plan":
        return Plan(self.ops, self.keep, self.events)


class Plan:
    """A recorded launch: td_execute_plan replays every op in one call."""

    def __init__(self, ops, keep, events):
        self.n = len(ops)
        self.array = (TdOp * max(1, self.n))()
        for k, (kind, words) in enumerate(ops):
            self.array[k].kind = kind
            self.array[k].nargs = len(words)
            for j, w in enumerate(words):
                self.array[k].arg[j] = w
        self.keep = keep
        self.events = events
        self.extra = {}     # owner-specific state (e.g. the runtime's inbox credit events)

    def run(self) -> None:
        check(lib().td_execute_plan(C.addressof(self.array), self.n), "td_execute_plan")

    def __del__(self):
        try:
            for ev in self.events:
                lib().td_event_destroy(C.c_void_p(ev))
        except Exception:
            pass
        self.events = []


class recording:
    """Context: record the plan ops of the native calls issued inside it."""

    def __init__(self):
        self.rec = PlanRecorder()

    def __enter__(self) -> PlanRecorder:
        global _RECORDING
        if _RECORDING is not None:
            raise NativeError("plan recordings do not nest")
        _RECORDING = self.rec
        return self.rec

    def __exit__(self, *exc):
        global _RECORDING
        _RECORDING = None
        if exc[0] is not None:
            self.rec.invalidate(f"raised {exc[0].__name__}")
        return False


def recorder():
    """The active PlanRecorder, or None."""
    return _RECORDING


def i64_array(values):
    vals = list(values) or [0]
    return (C.c_int64 * len(vals))(*vals)


def launch_count() -> int:
    return int(lib().td_launch_count())
