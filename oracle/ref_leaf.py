"""A numpy/BLAS leaf kernel written against the reference's plugin contract
-- TEST / BASELINE INFRASTRUCTURE ONLY.

The reference's leaf plugin API (`pkg/src/tendist/cin.py:344-379`) hands a
kernel a `LeafRuntime`: `loops` [(var, lo, hi)] of the substituted nest,
`stmt` (Assign / Reduce / Place), `env` (pinned outer variables), `defs`
(relation map), `read_store` (global canonical DenseTensors) and `out_store`
(a full-size zeroed DenseTensor per task, written in place).  This kernel
works out the iteration box of the nest -- which contiguous range of every
statement variable it sweeps -- and evaluates the leaf over that box with
one `np.einsum` (a BLAS GEMM for the GEMM-shaped leaves).  Nests that are
not boxes (a variable driven by two loops, strided or wrapping ranges, sums
of products) fall back to `rt.execute_point` per point, which is the
reference's own interpreter path.

Uses: the CPU-B baseline of SURVEY.md §8(d) (`bench.py --impl reference`,
tendist's `run_statement` with this leaf substituted through its own
`Schedule.substitute_leaf`), the golden fixtures of the G1 config
(`tests/golden/make_golden.py`), and the drop-in test that an unmodified
tendist plugin runs on this package (`tests/test_host_plugin_gpu.py`).
"""

from __future__ import annotations

import numpy as np

NAME = "numpy-einsum"


def _names_of(expr, out):
    """Access objects of a product-of-accesses expression, or None."""
    kind = type(expr).__name__
    if kind == "Access":
        out.append(expr)
        return out
    if kind == "Const":
        return out
    if kind == "Mul":
        if _names_of(expr.lhs, out) is None or _names_of(expr.rhs, out) is None:
            return None
        return out
    return None


def _consts(expr):
    kind = type(expr).__name__
    if kind == "Const":
        return float(expr.value)
    if kind == "Mul":
        return _consts(expr.lhs) * _consts(expr.rhs)
    return 1.0


def _walk_points(rt):
    import itertools
    vars_ = [v for v, _, _ in rt.loops]
    for pt in itertools.product(*[range(lo, hi) for _, lo, hi in rt.loops]):
        rt.execute_point({**rt.env, **dict(zip(vars_, pt))})


def box_of(rt):
    """{statement var: (lo, hi)} swept by the nest, or None if not a box."""
    stmt = rt.stmt
    accs = [stmt.lhs] + (_names_of(stmt.rhs, []) or [])
    names = sorted({v for a in accs for v in a.var_names})
    base = dict(rt.env)
    for v, lo, hi in rt.loops:
        if hi <= lo:
            return {}
        base[v] = lo
    r0 = rt.resolve(names, base)
    if r0 is None:
        return None
    rng = {n: (r0[n], r0[n] + 1) for n in names}
    driven = {}
    for v, lo, hi in rt.loops:
        count = 1
        moved = None
        for x in range(lo + 1, hi):
            r = rt.resolve(names, {**base, v: x})
            if r is None:
                break
            diff = [n for n in names if r[n] != r0[n]]
            if x == lo + 1:
                if len(diff) > 1 and len({r[n] - r0[n] for n in diff}) != 1:
                    return None
                moved = diff
            if diff != moved or any(r[n] - r0[n] != x - lo for n in diff):
                return None
            count += 1
        for n in moved or []:
            if n in driven:
                return None
            driven[n] = v
            rng[n] = (r0[n], r0[n] + count)
    return rng


def numpy_leaf(rt) -> None:
    """The leaf: one einsum over the nest's box, in place into out_store."""
    stmt = rt.stmt
    kind = type(stmt).__name__
    if kind == "Place":
        return
    accs = _names_of(stmt.rhs, [])
    box = box_of(rt) if accs is not None else None
    if box is None:
        _walk_points(rt)
        return
    if not box:
        return
    letters = {}
    for a in [stmt.lhs] + accs:
        for v in a.var_names:
            letters.setdefault(v, chr(ord("a") + len(letters)))

    def view(tensor, acc):
        idx = tuple(slice(*box[v]) for v in acc.var_names)
        return tensor.data[idx] if idx else tensor.data

    ops = [view(rt.read_store[a.tensor.name], a) for a in accs]
    spec = ",".join("".join(letters[v] for v in a.var_names) for a in accs)
    spec += "->" + "".join(letters[v] for v in stmt.lhs.var_names)
    val = np.einsum(spec, *ops, optimize=True) if ops else np.float64(1.0)
    c = _consts(stmt.rhs)
    if c != 1.0:
        val = val * c
    out = rt.out_store[stmt.lhs.tensor.name]
    idx = tuple(slice(*box[v]) for v in stmt.lhs.var_names)
    if kind == "Assign":
        if idx:
            out.data[idx] = val
        else:
            out.data[...] = val
    else:
        if idx:
            out.data[idx] += val
        else:
            out.data[...] += val


def innermost_vars(cin):
    """The innermost nest of a scheduled statement: the loops below the last
    loop that is distributed, communicated at, or a rotation result (what the
    survey's probe substitutes)."""
    node = cin
    chain, pinned = [], set()
    while type(node).__name__ in ("Forall", "Suchthat"):
        if type(node).__name__ == "Forall":
            chain.append(node.var)
        else:
            for rel in node.relations:
                kind = type(rel).__name__
                if kind in ("Distribute", "Communicate"):
                    pinned.add(rel.var)
                elif kind == "Rotate":
                    pinned.add(rel.result)
        node = node.body
    last = max((k for k, v in enumerate(chain) if v in pinned), default=-1)
    return tuple(chain[last + 1:])
