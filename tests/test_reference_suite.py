"""Drop-in check: the REFERENCE's own unit tests, run against this package.

The reference's own tests are staged by `make ref` into oracle/_ref/tests
(git-ignored, travels to the GPU box with the snapshot; read in place, never
committed).  Every test module, the CLI ones included (paper_2203_08069_b200.cli), is loaded with `tendist` and its
submodules aliased to `paper_2203_08069_b200`, and each test function is run
unmodified.  Tests that need values computed (run_statement, interpret,
sequential_evaluate) raise DeviceUnavailable on a GPU-less host and are
reported as skipped there; the `-m gpu` twin runs every case on the B200
and fails on DeviceUnavailable; everything else -- machines, tensors and their file
formats, the IR and parser, CIN structure and pretty-printing, distributions,
the scheduling language and its error taxonomy -- must pass as is.
Nothing is copied from the reference: its test files are read in place.
"""

import importlib.util
import inspect
import os
import sys

import pytest

from oracle.reference import tests_dir

REF_TESTS = tests_dir()
SKIP_FILES = set()


def _alias():
    import paper_2203_08069_b200 as pkg
    from paper_2203_08069_b200 import (cin, cli, distribution, errors, ir, machine, scheduling, tensors)
    mods = {"tendist": pkg, "tendist.cin": cin, "tendist.cli": cli, "tendist.distribution": distribution,
            "tendist.errors": errors, "tendist.ir": ir, "tendist.machine": machine,
            "tendist.scheduling": scheduling, "tendist.tensors": tensors}
    saved = {k: sys.modules.get(k) for k in mods}
    sys.modules.update(mods)
    return saved


def _restore(saved):
    for k, v in saved.items():
        if v is None:
            sys.modules.pop(k, None)
        else:
            sys.modules[k] = v


def _collect():
    if not REF_TESTS:
        return []
    saved = _alias()
    cases = []
    try:
        for fname in sorted(os.listdir(REF_TESTS)):
            if not fname.startswith("test_") or not fname.endswith(".py") or fname in SKIP_FILES:
                continue
            spec = importlib.util.spec_from_file_location(f"_reference_suite_{fname[:-3]}",
                                                          os.path.join(REF_TESTS, fname))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            for name, fn in vars(mod).items():
                if not (name.startswith("test_") and callable(fn)):
                    continue
                params = [m for m in getattr(fn, "pytestmark", []) if m.name == "parametrize"]
                if params:
                    argnames, values = params[0].args[0], params[0].args[1]
                    for k, v in enumerate(values):
                        cases.append((fname, f"{name}[{k}]", fn, {argnames: v}))
                else:
                    cases.append((fname, name, fn, {}))
    finally:
        _restore(saved)
    return cases


CASES = _collect()


def _run(case, tmp_path, capsys, monkeypatch, on_gpu):
    from paper_2203_08069_b200.errors import DeviceUnavailable
    fname, name, fn, kwargs = case
    kwargs = dict(kwargs)
    fixtures = {"tmp_path": tmp_path, "capsys": capsys, "monkeypatch": monkeypatch}
    wanted = inspect.signature(fn).parameters
    for p in wanted:
        if p not in kwargs:
            if p not in fixtures:
                pytest.skip(f"needs fixture {p}")
            kwargs[p] = fixtures[p]
    saved = _alias()
    try:
        fn(**kwargs)
    except DeviceUnavailable:
        if on_gpu:
            raise
        pytest.skip("computes values: runs on the GPU (test_reference_unit_test_on_b200)")
    finally:
        _restore(saved)


IDS = [f"{c[0][:-3]}::{c[1]}" for c in CASES] or None


@pytest.mark.skipif(not CASES, reason="reference tests not staged (make ref)")
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_reference_unit_test(case, tmp_path, capsys, monkeypatch):
    _run(case, tmp_path, capsys, monkeypatch, on_gpu=False)


@pytest.mark.gpu
@pytest.mark.skipif(not CASES, reason="reference tests not staged (make ref)")
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_reference_unit_test_on_b200(case, tmp_path, capsys, monkeypatch):
    """The same unmodified reference test, values computed by the B200 path."""
    _run(case, tmp_path, capsys, monkeypatch, on_gpu=True)
