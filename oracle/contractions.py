"""numpy restatement of the reference's leaf statements and oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* `gemm`, `ttv`, `ttm`, `innerprod`, `mttkrp`: the contractions of the
  reference bundles (pkg/src/tendist/algorithms.py:80-83 GEMM, :280-281 TTV,
  :300-301 TTM, :320 innerprod, :339-340 MTTKRP).  On integer-valued inputs
  every partial sum is an integer below 2**53, so any summation order --
  including BLAS's -- gives the exact value; with `exact=True` they are
  evaluated in longdouble for real-valued tolerance checks.
* `seq_eval`: restatement of `sequential_evaluate`
  (pkg/src/tendist/ir.py:197-229): free points outside, reduction points in
  lexicographic order of the reduction variables (first-appearance order),
  accumulated one at a time from +0.0 -- vectorised over free points only, so
  it reproduces the reference bit for bit on real-valued data too.
"""

from __future__ import annotations

import itertools
import re

import numpy as np


def _ld(x, exact):
    return np.asarray(x, dtype=np.longdouble) if exact else np.asarray(x, dtype=np.float64)


def gemm(a, b, exact=False):
    if exact:
        return np.einsum("ik,kj->ij", _ld(a, 1), _ld(b, 1))
    return np.asarray(a, np.float64) @ np.asarray(b, np.float64)


def ttv(b, c, exact=False):
    return np.einsum("ijk,k->ij", _ld(b, exact), _ld(c, exact))


def ttm(b, cm, exact=False):
    b = _ld(b, exact)
    i, j, k = b.shape
    if exact:
        return np.einsum("ijk,kl->ijl", b, _ld(cm, 1))
    return (b.reshape(i * j, k) @ np.asarray(cm, np.float64)).reshape(i, j, -1)


def innerprod(b, c, exact=False):
    return (_ld(b, exact) * _ld(c, exact)).sum() if exact else float(np.dot(
        np.asarray(b, np.float64).ravel(), np.asarray(c, np.float64).ravel()))


def mttkrp(b, cm, d, exact=False):
    b = _ld(b, exact)
    i, k, l = b.shape
    t = np.einsum("ikl,lj->ikj", b, _ld(d, exact))          # B(i,k,:) . D
    return np.einsum("ikj,kj->ij", t, _ld(cm, exact))       # Hadamard with C, sum over k


# ---------------------------------------------------------------- seq_eval
_TOK = re.compile(r"\s*([A-Za-z_]\w*|\d+(?:\.\d+)?|[()=+*,])")


def _parse(text):
    toks = _TOK.findall(text)
    pos = [0]

    def peek():
        return toks[pos[0]] if pos[0] < len(toks) else None

    def take(x=None):
        t = toks[pos[0]]
        if x is not None and t != x:
            raise ValueError(f"expected {x!r}, got {t!r}")
        pos[0] += 1
        return t

    def access():
        name = take()
        vs = []
        if peek() == "(":
            take("(")
            while peek() != ")":
                vs.append(take())
                if peek() == ",":
                    take(",")
            take(")")
        return ("acc", name, tuple(vs))

    def atom():
        t = peek()
        if t == "(":
            take("(")
            e = expr()
            take(")")
            return e
        if re.fullmatch(r"\d+(?:\.\d+)?", t):
            take()
            return ("const", float(t))
        return access()

    def term():
        e = atom()
        while peek() == "*":
            take("*")
            e = ("mul", e, atom())
        return e

    def expr():
        e = term()
        while peek() == "+":
            take("+")
            e = ("add", e, term())
        return e

    lhs = access()
    take("=")
    return lhs, expr()


def _accesses(e):
    if e[0] == "acc":
        return [e]
    if e[0] in ("add", "mul"):
        return _accesses(e[1]) + _accesses(e[2])
    return []


def seq_eval(text: str, extents: dict, inputs: dict) -> np.ndarray:
    """Reference-order evaluation of a statement (see module docstring)."""
    lhs, rhs = _parse(text)
    free = list(dict.fromkeys(lhs[2]))
    red = list(dict.fromkeys(v for a in _accesses(rhs) for v in a[2] if v not in free))
    fshape = tuple(extents[v] for v in free)
    grids = dict(zip(free, np.indices(fshape))) if free else {}

    def ev(e, point):
        if e[0] == "const":
            return np.float64(e[1])
        if e[0] == "acc":
            arr = np.asarray(inputs[e[1]], dtype=np.float64)
            if not e[2]:
                return arr.reshape(())[()]
            idx = tuple(grids[v] if v in grids else point[v] for v in e[2])
            return arr[idx]
        x, y = ev(e[1], point), ev(e[2], point)
        return x + y if e[0] == "add" else x * y

    if red:
        acc = np.zeros(fshape, dtype=np.float64)
        for pt in itertools.product(*(range(extents[v]) for v in red)):
            acc = acc + ev(rhs, dict(zip(red, pt)))
        val = acc
    else:
        val = np.broadcast_to(ev(rhs, {}), fshape).astype(np.float64)
    # lhs may repeat a variable (e.g. D(i, i)); scatter into the output box
    out_dims = tuple(extents[v] for v in lhs[2])
    out = np.zeros(out_dims, dtype=np.float64)
    if not lhs[2]:
        return np.asarray(val, dtype=np.float64).reshape(())
    idx = tuple(grids[v] for v in lhs[2])
    out[idx] = val
    return out
