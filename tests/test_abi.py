"""The C-ABI library loads without a GPU and exports every entry point that
include/distal_b200.h declares (no compute calls here)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "distal_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|long long|const char\*)\s+(td_\w+)\s*\(", text, re.M)))


def test_header_declares_the_surface():
    names = declared()
    for want in ("td_dgemm", "td_ttv", "td_ttm", "td_mttkrp", "td_innerprod", "td_nest_eval",
                 "td_send", "td_recv", "td_bcast", "td_reduce_sum", "td_comm_init_rank", "td_comm_split",
                 "td_init", "td_finalize", "td_allgather", "td_shift", "td_execute_plan", "td_dgemm_grouped",
                 "td_comm_wait"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2203_08069_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run `make`)")
    lib = _native.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_native.EXPORTED)
    assert lib.td_version() == 10000
    assert lib.td_last_error() == b""
    assert lib.td_nccl_version() >= 22800


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: a missing library raises DeviceUnavailable."""
    from paper_2203_08069_b200 import _native
    from paper_2203_08069_b200.errors import DeviceUnavailable
    saved = _native._lib
    _native._lib = None
    try:
        with pytest.raises(DeviceUnavailable):
            _native.load(str(tmp_path / "nope.so"))
    finally:
        _native._lib = saved
