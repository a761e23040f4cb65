"""Drop-in check: the REFERENCE's own unit tests, run against this package.

When the reference checkout is present (the build container), every test
module of `pkg/tests` except the CLI ones is loaded with `tendist` and its
submodules aliased to `paper_2203_08069_b200`, and each test function is run
unmodified.  Tests that need values computed (run_statement, interpret,
sequential_evaluate) raise DeviceUnavailable on a GPU-less host and are
reported as skipped; everything else -- machines, tensors and their file
formats, the IR and parser, CIN structure and pretty-printing, distributions,
the scheduling language and its error taxonomy -- must pass as is.
Nothing is copied from the reference: its test files are read in place.
"""

import importlib.util
import inspect
import os
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
SKIP_FILES = {"test_cli.py", "test_acceptance.py"}    # exercise the reference CLI (out of scope)


def _alias():
    import paper_2203_08069_b200 as pkg
    from paper_2203_08069_b200 import (cin, distribution, errors, ir, machine, scheduling, tensors)
    mods = {"tendist": pkg, "tendist.cin": cin, "tendist.distribution": distribution, "tendist.errors": errors,
            "tendist.ir": ir, "tendist.machine": machine, "tendist.scheduling": scheduling,
            "tendist.tensors": tensors}
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
    if not os.path.isdir(REF_TESTS):
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


@pytest.mark.skipif(not CASES, reason="reference checkout not present")
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0][:-3]}::{c[1]}" for c in CASES] or None)
def test_reference_unit_test(case, tmp_path, capsys, monkeypatch):
    from paper_2203_08069_b200.errors import DeviceUnavailable
    fname, name, fn, kwargs = case
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
        pytest.skip("computes values: runs on the GPU (see the -m gpu parity tests)")
    finally:
        _restore(saved)
