"""Leaf dispatch: from one step's loop nest to a native sm_100a kernel.

The reference evaluates a task's loop nest point by point (reference
`pkg/src/tendist/cin.py:399-477`) unless `substitute_leaf` routes it to a
registered plugin (`cin.py:459-463`; the paper's
``.substitute({ii, ji, ki}, CuBLAS::GeMM)``).  On B200 every
step of a task is first reduced to its *iteration box*: the interval each
statement variable sweeps when the launch and step loops are pinned
(`box_of`).  When the nest visits every point of that box exactly once, the
leaf statement is matched against the native contractions:

    GEMM      X(a,b) += Y(a,c) * Z(c,b)             -> td_dgemm
    TTV       X(a,b) += Y(a,b,c) * z(c)             -> td_ttv
    TTM       X(a,b,d) += Y(a,b,c) * Z(c,d)         -> td_ttm
    MTTKRP    X(a,b) += Y(a,c,d) * Z(c,b) * W(d,b)  -> td_mttkrp (fused)
    innerprod x += Y(v...) * Z(v...)                -> td_innerprod
    any other X += P * Q with a contracted index     -> (batched) td_dgemm after
              grouping the indices into batch / M / N / K (transposed GEMMs,
              GEMV, TTM/TTV on other modes; `_contract`)

Anything else -- or any nest under the ``"interpreter"`` leaf / the
``"exact"`` policy -- runs on the exact-order nest kernel (`interp.py`),
which reproduces the reference's accumulation order bit for bit.  The
native contractions reassociate sums (exact on integer-valued inputs,
within gamma_K |A||B| otherwise).

Builtin leaf names usable with `substitute_leaf`: ``"auto"`` (match, else
nest kernel), ``"dgemm"``/``"gemm"``, ``"ttv"``, ``"ttm"``, ``"mttkrp"``,
``"innerprod"`` (require that contraction) and ``"interpreter"``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from .cin import Divide, Reduce, Split
from .errors import ConfigError, TendistError
from .interp import DeviceTile, device_buffer, run_nest, stream_handle, torch_mod
from .ir import Access, Mul, accesses_of
from .distribution import HyperRect

BUILTIN_LEAVES = frozenset({"auto", "dgemm", "gemm", "ttv", "ttm", "mttkrp", "innerprod"})
_ENUM_LIMIT = 1 << 22

# counters for the bench / tests: which path each step took
STATS = {"dgemm": 0, "ttv": 0, "ttm": 0, "mttkrp": 0, "innerprod": 0, "contract": 0, "nest": 0, "grouped": 0,
         "k_merged": 0, "folded": 0}
# a tile's two remaining k-segments (after k-merging) go out as one two-segment
# grouped problem (td_gemm_problem.K2) instead of two rounds (a measurement switch)
FOLD_SEGMENTS = True


# optional per-launch device timing: set TIMING = [] to collect
# (kind, start_event, end_event) recorded on the launching stream
TIMING = None


def reset_stats():
    for k in STATS:
        STATS[k] = 0


# ------------------------------------------------------------ box analysis
def _deps(name, defs, ranges, cache) -> tuple:
    """Loop variables `name` depends on (ordered, unique)."""
    if name in cache:
        return cache[name]
    if name in ranges:
        out = (name,)
    else:
        rel = defs.get(name)
        if rel is None:
            raise TendistError(f"{name} is not resolvable")
        parts = [rel.outer, rel.inner] if isinstance(rel, (Split, Divide)) else [rel.result, *rel.over]
        seen = []
        for p in parts:
            for l in _deps(p, defs, ranges, cache):
                if l not in seen:
                    seen.append(l)
        out = tuple(seen)
    cache[name] = out
    return out


def _eval_grid(name, defs, grid):
    """Evaluate `name` on a dict of broadcast loop-value arrays; (value, phantom)."""
    if name in grid:
        return grid[name], np.zeros(grid[name].shape, dtype=bool)
    rel = defs[name]
    if isinstance(rel, (Split, Divide)):
        o, po = _eval_grid(rel.outer, defs, grid)
        i, pi = _eval_grid(rel.inner, defs, grid)
        v = o * rel.block + i
        return v, po | pi | (v >= rel.extent)
    r, pr = _eval_grid(rel.result, defs, grid)
    for x in rel.over:
        o, po = _eval_grid(x, defs, grid)
        r = r + o
        pr = pr | po
    return r % rel.extent, pr


def box_of(loops, leaf, defs):
    """Interval per statement variable if the nest visits each point of the
    box exactly once, else None.  loops: [(var, lo, hi)] incl. pinned ones."""
    ranges = {v: (lo, hi) for v, lo, hi in loops}
    names = list(dict.fromkeys(n for a in [leaf.lhs, *accesses_of(leaf.rhs)] for n in a.var_names))
    cache = {}
    owner = {}
    box = {}
    for n in names:
        deps = _deps(n, defs, ranges, cache)
        live = [d for d in deps if ranges[d][1] - ranges[d][0] > 1]
        for d in live:
            if d in owner and owner[d] != n:
                return None           # a loop feeds two variables: not a product box
            owner[d] = n
        size = 1
        for d in deps:
            size *= max(0, ranges[d][1] - ranges[d][0])
        if size == 0:
            return {}                 # empty nest
        if size > _ENUM_LIMIT:
            return None
        axes = [np.arange(*ranges[d], dtype=np.int64) for d in deps]
        mesh = np.meshgrid(*axes, indexing="ij") if axes else []
        grid = dict(zip(deps, mesh))
        val, ph = _eval_grid(n, defs, grid)
        vals = np.asarray(val)[~np.asarray(ph)].ravel()
        if vals.size == 0:
            return {}
        lo, hi = int(vals.min()), int(vals.max()) + 1
        if hi - lo != vals.size or np.unique(vals).size != vals.size:
            return None
        box[n] = (lo, hi)
    # every live loop must feed some variable, else points repeat
    for v, lo, hi in loops:
        if hi - lo > 1 and v not in owner:
            return None
    return box


# ------------------------------------------------------------ matching
def _factors(e):
    if isinstance(e, Mul):
        return _factors(e.lhs) + _factors(e.rhs)
    return [e]


@dataclass
class Match:
    kind: str
    roles: dict     # role -> index of the rhs access (accesses_of order)


def classify(leaf) -> Match | None:
    if not isinstance(leaf, Reduce):
        return None
    facs = _factors(leaf.rhs)
    if not all(isinstance(f, Access) for f in facs):
        return None
    accs = accesses_of(leaf.rhs)
    idx = {id(a): k for k, a in enumerate(accs)}
    out = leaf.lhs.var_names
    if len(set(out)) != len(out):
        return None
    vs = [f.var_names for f in facs]
    if any(len(set(v)) != len(v) for v in vs):
        return None
    if len(facs) == 2:
        p, q = facs
        for y, z in ((p, q), (q, p)):
            a_, b_ = y.var_names, z.var_names
            # GEMM X(a,b) += Y(a,c) Z(c,b)
            if len(out) == 2 and len(a_) == 2 and len(b_) == 2:
                a, b = out
                if a_[0] == a and b_[1] == b and a_[1] == b_[0] and a_[1] not in out:
                    return Match("dgemm", {"A": idx[id(y)], "B": idx[id(z)]})
            # TTV X(a,b) += Y(a,b,c) z(c)
            if len(out) == 2 and len(a_) == 3 and len(b_) == 1:
                if a_[:2] == out and a_[2] == b_[0] and b_[0] not in out:
                    return Match("ttv", {"B": idx[id(y)], "c": idx[id(z)]})
            # TTM X(a,b,d) += Y(a,b,c) Z(c,d)
            if len(out) == 3 and len(a_) == 3 and len(b_) == 2:
                if a_[:2] == out[:2] and b_ == (a_[2], out[2]) and a_[2] not in out:
                    return Match("ttm", {"B": idx[id(y)], "C": idx[id(z)]})
        # innerprod x += Y(v) Z(v)
        if len(out) == 0 and p.var_names == q.var_names:
            return Match("innerprod", {"B": idx[id(p)], "C": idx[id(q)]})
        # any other pairwise contraction: X(batch, m, n) += P(batch, m, k) Q(batch, k, n)
        # up to axis order (transposed GEMMs, GEMV, TTM/TTV on any mode, batched products)
        sp, sq, so = set(p.var_names), set(q.var_names), set(out)
        if so <= sp | sq and sp <= so | sq and sq <= so | sp and (sp & sq) - so:
            return Match("contract", {"P": idx[id(p)], "Q": idx[id(q)]})
        return None
    if len(facs) == 3 and len(out) == 2:
        a, b = out
        big = [f for f in facs if len(f.var_names) == 3]
        if len(big) != 1:
            return None
        y = big[0]
        if y.var_names[0] != a:
            return None
        c, d = y.var_names[1], y.var_names[2]
        if len({a, b, c, d}) != 4:
            return None
        rest = [f for f in facs if f is not y]
        z = next((f for f in rest if f.var_names == (c, b)), None)
        w = next((f for f in rest if f.var_names == (d, b)), None)
        if z is None or w is None or z is w:
            return None
        return Match("mttkrp", {"B": idx[id(y)], "C": idx[id(z)], "D": idx[id(w)]})
    return None


# ------------------------------------------------------------ launching
def _sub(tile: DeviceTile, acc: Access, box) -> DeviceTile:
    lo = tuple(box[v][0] for v in acc.var_names)
    hi = tuple(box[v][1] for v in acc.var_names)
    if lo == tile.rect.lo and hi == tile.rect.hi:
        return tile           # the tile already is the box (the common case): no new view
    return tile.view(HyperRect(lo, hi))


def _p(t: DeviceTile):
    return C.c_void_p(t.ptr())


def _launch_native(m: Match, leaf, box, out: DeviceTile, ins, stream, accumulate=1) -> bool:
    accs = accesses_of(leaf.rhs)
    o = _sub(out, leaf.lhs, box)
    v = {role: _sub(ins[k], accs[k], box) for role, k in m.roles.items()}
    s = stream_handle(stream)
    st = {r: t.strides() for r, t in v.items()}
    ost = o.strides()
    ext = {n: hi - lo for n, (lo, hi) in box.items()}
    if m.kind != "dgemm":
        flush_pending()
    if m.kind == "dgemm":
        a, b = leaf.lhs.var_names
        c = accs[m.roles["A"]].var_names[1]
        if st["A"][1] != 1 or st["B"][1] != 1 or ost[1] != 1:
            return False
        _dgemm(stream, ext[a], ext[b], ext[c], v["A"].ptr(), st["A"][0], v["B"].ptr(), st["B"][0], o.ptr(),
               ost[0], accumulate, keep=(v["A"].data, v["B"].data, o.data))
    elif m.kind == "ttv":
        a, b = leaf.lhs.var_names
        c = accs[m.roles["c"]].var_names[0]
        if st["B"][2] != 1 or st["c"][0] != 1:
            return False
        _timed_call("ttv", stream, "td_ttv", s, ext[a], ext[b], ext[c], _p(v["B"]), st["B"][0], st["B"][1],
                    _p(v["c"]), _p(o), ost[0], ost[1], accumulate)
    elif m.kind == "ttm":
        a, b, d = leaf.lhs.var_names
        c = accs[m.roles["B"]].var_names[2]
        if st["B"][2] != 1 or st["C"][1] != 1 or ost[2] != 1:
            return False
        _timed_call("ttm", stream, "td_ttm", s, ext[a], ext[b], ext[c], ext[d], _p(v["B"]), st["B"][0],
                    st["B"][1], _p(v["C"]), st["C"][0], _p(o), ost[0], ost[1], accumulate)
    elif m.kind == "mttkrp":
        a, b = leaf.lhs.var_names
        _, c, d = accs[m.roles["B"]].var_names
        if st["B"][2] != 1 or st["C"][1] != 1 or st["D"][1] != 1 or ost[1] != 1:
            return False
        _timed_call("mttkrp", stream, "td_mttkrp", s, ext[a], ext[c], ext[d], ext[b], _p(v["B"]), st["B"][0],
                    st["B"][1], _p(v["C"]), st["C"][0], _p(v["D"]), st["D"][0], _p(o), ost[0], accumulate)
    elif m.kind == "innerprod":
        ok = _innerprod(v["B"], v["C"], o, stream, accumulate)
        if not ok:
            return False
    elif m.kind == "contract":
        ev = _timing_start(stream)
        _contract(leaf.lhs.var_names, accs[m.roles["P"]].var_names, accs[m.roles["Q"]].var_names,
                  o, v["P"], v["Q"], ext, stream, accumulate)
        _timing_stop("contract", ev, stream)
    else:
        return False
    STATS[m.kind] += 1
    return True


# ------------------------------------------------------- generic contraction
def _group_strides(view, names, groups):
    """View strides regrouped as one stride per group of axes, if each group is
    a row-major-contiguous run (else None).  groups: list of var-name lists."""
    st = dict(zip(names, view.strides()))
    shape = dict(zip(names, view.rect.shape))
    out = []
    for g in groups:
        if not g:
            out.append(0)
            continue
        stride = st[g[-1]]
        expect = stride * shape[g[-1]]
        for v in reversed(g[:-1]):
            if shape[v] != 1 and st[v] != expect:
                return None
            expect = st[v] * shape[v] if shape[v] != 1 else expect
        out.append(stride)
    return out


def _packed(view, names, order, ext, stream):
    """Contiguous copy of `view` with its axes permuted into `order`."""
    torch = torch_mod()
    shape = [ext[v] for v in order]
    buf = device_buffer(shape, view.data.device, stream)
    st = dict(zip(names, view.strides()))
    if shape:
        _native.call("td_copy_box", stream_handle(stream), len(order), _native.i64_array(shape),
                     C.c_void_p(buf.data_ptr()), _native.i64_array(buf.stride()), C.c_void_p(view.ptr()),
                     _native.i64_array([st[v] for v in order]), 0)
    return buf


def _contract_layout(out_names, p_names, q_names, o, pv, qv, ext):
    """Groups and in-place strides for computing X = P . Q with M from P."""
    so, sp, sq = set(out_names), set(p_names), set(q_names)
    batch = [v for v in out_names if v in sp and v in sq]
    mvars = [v for v in out_names if v in sp and v not in sq]
    nvars = [v for v in out_names if v in sq and v not in sp]
    kvars = [v for v in p_names if v in sq and v not in so]
    gp = _group_strides(pv, p_names, [batch, mvars, kvars])
    if gp is None or gp[2] != 1 or list(p_names) != batch + mvars + kvars:
        gp = None
    gq = _group_strides(qv, q_names, [batch, kvars, nvars])
    if gq is None or (nvars and gq[2] != 1) or list(q_names) != batch + kvars + nvars:
        gq = None
    go = _group_strides(o, out_names, [batch, mvars, nvars])
    if go is None or (nvars and go[2] != 1) or list(out_names) != batch + mvars + nvars:
        go = None
    size = lambda vs: int(np.prod([ext[v] for v in vs])) if vs else 1
    # elements copied to re-layout operands / the output when not usable in place
    cost = ((0 if gp else size(p_names)) + (0 if gq else size(q_names)) + (0 if go else 2 * size(out_names)))
    return cost, (batch, mvars, nvars, kvars, gp, gq, go)


def _contract(out_names, p_names, q_names, o, pv, qv, ext, stream, accumulate):
    """X(b, m, n) (+)= P(b, m, k) Q(b, k, n) for any axis order.  Both operand
    roles are tried (X = P.Q or, as X's transpose, Q.P) and the one that needs
    the fewest re-layout copies wins; operands whose axes already form
    row-major (batch, M, K) / (batch, K, N) matrices are read in place, others
    are packed by one strided copy; the product is a (batched) DMMA GEMM; an
    output in another axis order is produced in a scratch matrix and added
    back with one strided copy."""
    torch = torch_mod()
    c1, lay1 = _contract_layout(out_names, p_names, q_names, o, pv, qv, ext)
    c2, lay2 = _contract_layout(out_names, q_names, p_names, o, qv, pv, ext)
    if c2 < c1:
        p_names, q_names, pv, qv, lay = q_names, p_names, qv, pv, lay2
    else:
        lay = lay1
    batch, mvars, nvars, kvars, gp, gq, go = lay
    size = lambda vs: int(np.prod([ext[v] for v in vs])) if vs else 1
    Bt, Mt, Nt, Kt = size(batch), size(mvars), size(nvars), size(kvars)
    keep = []
    if gp is None:
        buf = _packed(pv, p_names, batch + mvars + kvars, ext, stream)
        keep.append(buf)
        pptr, gp = buf.data_ptr(), [Mt * Kt, Kt, 1]
    else:
        pptr = pv.ptr()
    if gq is None:
        buf = _packed(qv, q_names, batch + kvars + nvars, ext, stream)
        keep.append(buf)
        qptr, gq = buf.data_ptr(), [Kt * Nt, Nt, 1]
    else:
        qptr = qv.ptr()
    direct_out = go is not None
    if direct_out:
        optr, ostr, acc = o.ptr(), go, accumulate
    else:
        scratch = device_buffer((Bt, Mt, Nt), o.data.device, stream)
        keep.append(scratch)
        optr, ostr, acc = scratch.data_ptr(), [Mt * Nt, Nt, 1], 0
    lda = gp[1] if mvars else Kt
    ldb = gq[1] if kvars else Nt
    ldc = ostr[1] if mvars else Nt
    s = stream_handle(stream)
    if Bt == 1:
        _native.call("td_dgemm", s, Mt, Nt, Kt, C.c_void_p(pptr), lda, C.c_void_p(qptr), ldb,
                     C.c_void_p(optr), ldc, acc)
    else:
        _native.call("td_dgemm_batched", s, Bt, Mt, Nt, Kt, C.c_void_p(pptr), lda, gp[0], C.c_void_p(qptr),
                     ldb, gq[0], C.c_void_p(optr), ldc, ostr[0], acc)
    if not direct_out:
        st = dict(zip(out_names, o.strides()))
        order = batch + mvars + nvars
        src_st = {}
        run = 1
        for v in reversed(order):
            src_st[v] = run
            run *= ext[v]
        _native.call("td_copy_box", s, len(out_names), _native.i64_array([ext[v] for v in out_names]),
                     C.c_void_p(o.ptr()), _native.i64_array([st[v] for v in out_names]),
                     C.c_void_p(optr), _native.i64_array([src_st[v] for v in out_names]), accumulate)
    for t in keep:
        t.record_stream(stream)


def _rows_view(t: DeviceTile):
    """(rows, n, row_stride) if the tile is a stack of equal-stride rows."""
    shape, st = t.rect.shape, t.strides()
    if not shape:
        return 1, 1, 1
    if st[-1] != 1:
        return None
    n = shape[-1]
    outer = list(zip(shape[:-1], st[:-1]))
    outer = [(e, s) for e, s in outer if e != 1]
    if not outer:
        return 1, n, n
    # merge outer axes into one stride
    rows = 1
    stride = outer[-1][1]
    expect = stride
    for e, s in reversed(outer):
        if s != expect:
            return None
        rows *= e
        expect = s * e
    return rows, n, stride


def _innerprod(b: DeviceTile, c: DeviceTile, out: DeviceTile, stream, accumulate) -> bool:
    rb, rc = _rows_view(b), _rows_view(c)
    if rb is None or rc is None or rb[:2] != rc[:2]:
        return False
    work = device_buffer((int(_native.lib().td_innerprod_work_size()),), out.data.device, stream)
    _timed_call("innerprod", stream, "td_innerprod", stream_handle(stream), rb[0], rb[1], _p(b), rb[2], _p(c),
                rc[2], _p(out), C.c_void_p(work.data_ptr()), accumulate)
    if stream is not None:
        work.record_stream(stream)
    return True


# ------------------------------------------------------------ GEMM batches
class gemm_batch:
    """Context: plain GEMM leaves issued inside it are deferred and launched
    at exit by `_flush_gemms` (k-continuations merged, then grouped launches
    of <= 8 independent output tiles, td_dgemm_grouped).  The executor wraps
    one step's leaves of the tasks co-located on a GPU in it, and the whole
    step loop of a GPU-local program (nothing moves between its steps: every
    transfer is an alias).  Merging a task's k-slab steps into one GEMM
    reassociates its k sum: exact on integer data, within gamma_K otherwise
    (the "exact" policy never reaches here).  Inactive while leaves are
    timed (TIMING), since the timing events bracket single launches."""

    def __enter__(self):
        global _GEMM_BATCH
        self.outer = _GEMM_BATCH
        if self.outer is None and TIMING is None:
            _GEMM_BATCH = []
        return self

    def __exit__(self, *exc):
        global _GEMM_BATCH
        if self.outer is None and _GEMM_BATCH is not None:
            pending, _GEMM_BATCH = _GEMM_BATCH, None
            if exc[0] is None:
                _flush_gemms(pending)
        return False


_GEMM_BATCH = None


def _dgemm(stream, M, N, K, a, lda, b, ldb, c, ldc, accumulate, keep=()) -> None:
    """td_dgemm, or deferred into the active gemm_batch (holding `keep`, the
    operand tensors, until the grouped launch is issued: temporaries such
    as assembled operands must not return to the allocator before that)."""
    if _GEMM_BATCH is not None and M > 0 and N > 0 and K > 0:
        _GEMM_BATCH.append((stream, accumulate, (M, N, K, a, lda, b, ldb, c, ldc), keep))
        return
    _timed_call("dgemm", stream, "td_dgemm", stream_handle(stream), M, N, K, C.c_void_p(a), lda, C.c_void_p(b),
                ldb, C.c_void_p(c), ldc, accumulate)


def _k_adjacent(first, nxt) -> bool:
    """Does GEMM `nxt` continue `first` along k (same C, same operand
    layouts, A and B advanced by exactly first's K)?"""
    m, n, k, a, lda, b, ldb, c, ldc = first
    return (nxt[0] == m and nxt[1] == n and nxt[7] == c and nxt[8] == ldc and nxt[4] == lda
            and nxt[6] == ldb and nxt[3] == a + 8 * k and nxt[5] == b + 8 * k * ldb)


def _same_tile(first, nxt) -> bool:
    """Do two GEMMs write the same output tile (M, N, C, ldc)?"""
    return first[0] == nxt[0] and first[1] == nxt[1] and first[7] == nxt[7] and first[8] == nxt[8]


def _flush_gemms(pending) -> None:
    """Issue deferred GEMMs: per output tile, consecutive GEMMs continuing
    each other along k (a task's steps reading k-slabs of the same resident
    pieces) merge into one longer-k GEMM; then round r launches the r-th
    GEMM of every output tile, grouped 8 per launch.  Output tiles are
    independent, and each tile's GEMMs keep their order."""
    by_stream = {}
    for stream, acc, prob, _keep in pending:
        by_stream.setdefault(id(stream), (stream, {}))[1].setdefault(prob[7], []).append([acc, prob])
    for stream, per_c in by_stream.values():
        for seq in per_c.values():
            merged = [seq[0]]
            for acc, prob in seq[1:]:
                last = merged[-1]
                if acc == 1 and _k_adjacent(last[1], prob):
                    last[1] = last[1][:2] + (last[1][2] + prob[2],) + last[1][3:]
                    STATS["k_merged"] += 1
                else:
                    merged.append([acc, prob])
            if FOLD_SEGMENTS and len(merged) == 2 and merged[1][0] == 1 and _same_tile(merged[0][1], merged[1][1]):
                # two k-segments of one tile from different pieces: one problem, the
                # second accumulated after the first in the same registers
                _, _, k2, a2, lda2, b2, ldb2, _, _ = merged[1][1]
                merged = [[merged[0][0], merged[0][1] + (k2, a2, lda2, b2, ldb2)]]
                STATS["folded"] += 1
            seq[:] = merged
        depth = max(len(seq) for seq in per_c.values())
        for r in range(depth):
            items = [seq[r] for seq in per_c.values() if r < len(seq)]
            for acc in (0, 1):
                probs = [p for a, p in items if a == acc]
                for lo in range(0, len(probs), GROUP_MAX):
                    _launch_group(stream, probs[lo:lo + GROUP_MAX], acc)
    for stream, _acc, _prob, keep in pending:   # operands stay allocated until the launches ran
        for t in keep:
            if getattr(t, "is_cuda", False):
                t.record_stream(stream)


def flush_pending() -> None:
    """Issue the deferred GEMMs now (the batch stays open): called before any
    write that is not deferred, so per-tile write order is kept."""
    global _GEMM_BATCH
    if _GEMM_BATCH:
        pending, _GEMM_BATCH = _GEMM_BATCH, []
        _flush_gemms(pending)


def _launch_group(stream, chunk, acc) -> None:
    if len(chunk) == 1 and len(chunk[0]) == 9:
        m, n, k, a, lda, b, ldb, c, ldc = chunk[0]
        _native.call("td_dgemm", stream_handle(stream), m, n, k, C.c_void_p(a), lda, C.c_void_p(b), ldb,
                     C.c_void_p(c), ldc, acc)
        return
    arr = (_native.TdGemmProblem * len(chunk))(*[_native.TdGemmProblem(*p) for p in chunk])
    _native.call("td_dgemm_grouped", stream_handle(stream), len(chunk), arr, acc)
    STATS["grouped"] += 1


GROUP_MAX = 8


def _timed_call(kind, stream, name, *args) -> None:
    """A leaf's native call, bracketed by CUDA events when TIMING collects
    them: recorded right around the call, after the host-side preparation,
    so a GPU idling while Python prepares the launch is not counted."""
    ev = _timing_start(stream)
    _native.call(name, *args)
    _timing_stop(kind, ev, stream)


def _timing_start(stream):
    if TIMING is None:
        return None
    rec = _native.recorder()
    if rec is not None:
        rec.invalidate("leaf timing is on")
    torch = torch_mod()
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(stream)
    return ev


def _timing_stop(kind, ev, stream):
    if ev is None:
        return
    torch = torch_mod()
    end = torch.cuda.Event(enable_timing=True)
    end.record(stream)
    TIMING.append((kind, ev, end))


_MEMO: dict = {}


def _classify_cached(leaf):
    hit = _MEMO.get(("cls", id(leaf)))
    if hit is not None and hit[0] is leaf:
        return hit[1]
    m = classify(leaf)
    _MEMO[("cls", id(leaf))] = (leaf, m)
    return m


def _box_cached(loops, leaf, defs):
    """box_of memoised on (nest bounds, leaf, relation map): the bounds of a
    task's step nest repeat across steps and across repeated executes."""
    key = ("box", tuple(loops), id(leaf), id(defs))
    hit = _MEMO.get(key)
    if hit is not None and hit[0] is leaf and hit[1] is defs:
        return hit[2]
    if len(_MEMO) > 65536:
        _MEMO.clear()
    box = box_of(loops, leaf, defs)
    _MEMO[key] = (leaf, defs, box)
    return box


def native_plan(policy: str, loops, leaf, defs):
    """(Match, box) when this step nest runs as one native contraction over
    the iteration box `box`, else None (nest kernel, empty box, plugins)."""
    if not isinstance(leaf, Reduce) or policy in ("interpreter", "exact"):
        return None
    m = _classify_cached(leaf)
    want = {"gemm": "dgemm"}.get(policy, policy)
    if m is None or not (want == "auto" or want == m.kind):
        return None
    box = _box_cached(loops, leaf, defs)
    if not box:
        return None
    return m, box


def contracted_var(m, leaf):
    """The summed statement variable of a native GEMM leaf (k of C(i,j) += A(i,k) B(k,j))."""
    if m.kind != "dgemm":
        return None
    return accesses_of(leaf.rhs)[m.roles["A"]].var_names[1]


def run_native_box(m, leaf, box, out: DeviceTile, ins, stream, accumulate: int = 1) -> None:
    """Launch the native contraction `m` over `box` (a sub-box of the nest's
    iteration box: the pipelined first step runs its k-range in pieces)."""
    if not _launch_native(m, leaf, box, out, ins, stream, accumulate):
        raise TendistError(f"native {m.kind} leaf cannot address its operands on the box {box}")


def _zero_tile(out: DeviceTile, stream) -> None:
    """out = +0.0 on `stream` (contiguous tiles, including peer inboxes)."""
    flush_pending()
    data = out.data
    if not data.is_contiguous():
        raise TendistError(f"cannot zero the strided output tile {out!r}")
    _native.call("td_fill", stream_handle(stream), C.c_void_p(data.data_ptr()), data.numel(), 0.0)


def run_leaf(policy: str, loops, leaf, defs, out: DeviceTile, ins, stream, accumulate: int = 1) -> str:
    """Execute one step nest; returns the path taken ("dgemm", ..., "nest").

    policy: "auto" | a builtin contraction name | "interpreter" / "exact".
    accumulate=0: `out` holds garbage and this nest is its only writer (a
    peer-memory inbox, `peer.py`): a native leaf covering the whole tile
    overwrites it (0 + x = x, so the bits equal accumulating into zeros);
    anything else zeroes it first."""
    zeroed = bool(accumulate)
    if isinstance(leaf, Reduce) and policy not in ("interpreter", "exact"):
        m = _classify_cached(leaf)
        want = {"gemm": "dgemm"}.get(policy, policy)
        if m is not None and (want == "auto" or want == m.kind):
            box = _box_cached(loops, leaf, defs)
            if box == {}:
                if not zeroed:
                    _zero_tile(out, stream)
                return "empty"
            if box is not None:
                acc = accumulate
                if not zeroed and _sub(out, leaf.lhs, box).rect != out.rect:
                    _zero_tile(out, stream)
                    zeroed, acc = True, 1
                if _launch_native(m, leaf, box, out, ins, stream, acc):
                    return m.kind
        if want not in ("auto",):
            raise ConfigError(f"leaf kernel {policy!r} does not apply to {leaf!r} on this nest")
    elif policy not in ("auto", "interpreter", "exact"):
        raise ConfigError(f"leaf kernel {policy!r} needs a reduction statement")
    if not zeroed:
        _zero_tile(out, stream)
    flush_pending()
    run_nest(loops, leaf, defs, out, ins, stream)
    STATS["nest"] += 1
    return "nest"
