"""Launch-plan recording on the host (no GPU needed): every replayable
entry point becomes a td_op of its kind with its arguments as 64-bit words
(pointers / integers as-is, doubles bit-cast, arrays and by-reference
structs by address and kept alive); anything else invalidates the plan."""

import ctypes as C
import struct

from paper_2203_08069_b200 import _native


def test_words_and_kinds():
    rec = _native.PlanRecorder()
    arr = _native.i64_array([3, 4])
    prog = _native.TdGemmProblem(1, 2, 3, 4, 5, 6, 7, 8, 9)
    rec.add("td_fill", (C.c_void_p(7), C.c_void_p(4096), 12, -1.5))
    rec.add("td_copy_box", (C.c_void_p(7), 2, arr, C.c_void_p(8), arr, C.c_void_p(16), arr, 1))
    rec.add("td_nest_eval", (C.c_void_p(7), C.byref(prog), C.sizeof(prog)))
    rec.add("td_group_start", ())
    rec.add("td_send", (C.c_void_p(99), C.c_void_p(7), C.c_void_p(4096), 10, 1))
    rec.add("td_group_end", ())
    rec.add("td_innerprod_work_size", ())        # a query: ignored, still valid
    assert rec.valid
    kinds = [k for k, _ in rec.ops]
    assert kinds == [_native.PLAN_OPS[n] for n in ("td_fill", "td_copy_box", "td_nest_eval", "td_group_start",
                                                   "td_send", "td_group_end")]
    fill = rec.ops[0][1]
    assert fill[:3] == [7, 4096, 12] and fill[3] == struct.unpack("<q", struct.pack("<d", -1.5))[0]
    box = rec.ops[1][1]
    assert box[2] == C.addressof(arr) and box[7] == 1 and arr in rec.keep
    assert rec.ops[2][1][1] == C.addressof(prog) and prog in rec.keep
    plan = rec.finish()
    assert plan.n == 6 and plan.array[4].kind == _native.PLAN_OPS["td_send"] and plan.array[4].nargs == 5
    assert plan.array[4].arg[0] == 99


def test_non_replayable_call_invalidates():
    rec = _native.PlanRecorder()
    rec.add("td_comm_split", (C.c_void_p(1), 0, 0, C.byref(C.c_void_p())))
    assert not rec.valid and "td_comm_split" in rec.reason


def test_recordings_do_not_nest():
    import pytest
    from paper_2203_08069_b200.errors import NativeError
    with _native.recording():
        with pytest.raises(NativeError):
            with _native.recording():
                pass
    assert _native.recorder() is None
