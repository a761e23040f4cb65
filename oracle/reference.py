"""Import the reference package `tendist` -- TEST / BASELINE INFRASTRUCTURE ONLY.

The reference is pure Python (nothing to compile).  `make ref` (part of
`__graft_entry__.build()`) stages it from the read-only checkout into
`oracle/_ref/tendist` (+ its own tests in `oracle/_ref/tests`); that staged
copy is git-ignored and travels to the GPU box, where `/root/reference`
does not exist.  In the build container the checkout itself is used if the
staged copy is missing.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
STAGED = os.path.join(HERE, "_ref")
CHECKOUT = "/root/reference/pkg/src"


def location():
    if os.path.isdir(os.path.join(STAGED, "tendist")):
        return STAGED
    if os.path.isdir(os.path.join(CHECKOUT, "tendist")):
        return CHECKOUT
    return None


def tests_dir():
    for d in (os.path.join(STAGED, "tests"), "/root/reference/pkg/tests"):
        if os.path.isdir(d):
            return d
    return None


def tendist():
    """The reference package (raises ImportError if it was never staged)."""
    where = location()
    if where is None:
        raise ImportError("the reference is not staged: run `make ref` where /root/reference exists")
    if where not in sys.path:
        sys.path.insert(0, where)
    import tendist as mod
    return mod
