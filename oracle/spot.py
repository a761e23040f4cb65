"""Sampled-point oracle for full-size configs -- TEST / BENCH CHECKER ONLY.

At BASELINE.json's full sizes (GEMM 16384^3, TTM 1024^3 x 64, MTTKRP 1024^3
r32, TTV 2048^3) the whole-statement oracle is out of reach, but any single
output point only needs the input slices its reduction sweeps.  For a
statement `lhs(free) = prod of rhs accesses` (sum over the reduction
variables, reference `ir.py:197-229`), `points()` regenerates exactly those
slices with the counter generator (oracle/generator.py, the twin of the
device generator the inputs came from) and evaluates each point

  * `exact`:  in Python integers (mode 0 inputs: every product and sum is an
    exact integer, so the B200 value must match bit for bit);
  * `value`, `bound`: in long double (64-bit significand) with the matching
    sum of absolute products, for the floating-point tolerance check
    |got - value| <= gamma_n * bound,  gamma_n = n u / (1 - n u), u = 2^-53,
    n = the number of products summed (+ the product depth).

Statement objects are duck-typed (`lhs.var_names`, `lhs.tensor`, the rhs a
product of accesses), so both this package's and the reference's work.
"""

from __future__ import annotations

import numpy as np

from oracle.generator import generate_box

U = 2.0 ** -53


def gamma(n: int) -> float:
    return n * U / (1.0 - n * U)


def _factors(expr, out):
    kind = type(expr).__name__
    if kind == "Access":
        out.append(expr)
    elif kind == "Mul":
        _factors(expr.lhs, out)
        _factors(expr.rhs, out)
    else:
        raise ValueError(f"spot oracle handles products of accesses only, got {kind}")
    return out


def points(stmt, coords, *, seed=0, mode=0, ids=None):
    """[(exact int or None, long double value, long double bound)] for each
    output coordinate in `coords` (tuples in lhs variable order)."""
    out_name = stmt.lhs.tensor.name
    names = sorted(n for n in stmt.tensors() if n != out_name)
    ids = ids or {n: k + 1 for k, n in enumerate(names)}
    accs = _factors(stmt.rhs, [])
    free = list(stmt.lhs.var_names)
    red = [v for v in stmt.reduction_vars]
    letters = {v: chr(ord("a") + k) for k, v in enumerate(free + red)}
    spec = ",".join("".join(letters[v] for v in a.var_names if v not in free) for a in accs)
    spec += "->"
    res = []
    for coord in coords:
        pin = dict(zip(free, coord))
        ops = []
        for a in accs:
            dims = a.tensor.dims
            origin = tuple(pin.get(v, 0) for v in a.var_names)
            shape = tuple(1 if v in pin else d for v, d in zip(a.var_names, dims))
            blk = generate_box(dims, origin, shape, seed, ids[a.tensor.name], mode)
            ops.append(blk.reshape([s for v, s in zip(a.var_names, shape) if v not in pin]))
        exact = None
        if mode == 0:
            exact = int(np.einsum(spec, *[o.astype(np.int64) for o in ops], dtype=np.int64))
        ld = [o.astype(np.longdouble) for o in ops]
        value = np.einsum(spec, *ld)
        bound = np.einsum(spec, *[np.abs(o) for o in ld])
        res.append((exact, value, bound))
    return res


def reduction_length(stmt) -> int:
    n = 1
    for v in stmt.reduction_vars:
        n *= stmt.extents[v]
    return n
