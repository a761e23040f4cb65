"""Exact-order loop-nest evaluation on the GPU (host side of `csrc/interp.cu`).

The reference executes every leaf by walking the loop nest in Python and
evaluating one iteration point at a time (`pkg/src/tendist/cin.py:420-477`,
`_run_leaf` :399-417).  Here a nest is compiled into a `td_nest_prog` (loop
bounds, derived-variable program, access views, postfix expression) and
evaluated by one CUDA kernel: loops that determine the output coordinate
become threads, each thread walks the remaining loops lexicographically and
accumulates ``out += value`` point by point, so every output element sees
exactly the reference's sequence of floating-point additions.

Also here: `DeviceTile` (an HBM buffer holding a global box of a tensor),
`interpret_on_device` (the single-memory `interpret`) and
`evaluate_statement` (`sequential_evaluate`), both on the GPU.
"""

from __future__ import annotations

import ctypes as C
import itertools

from . import _native
from .cin import (Assign, Divide, Forall, LeafKernel, Place, Reduce, Seq, Split, Suchthat,
                  INTERPRETER_KERNEL, LeafRuntime, body_of, leaf_statements, lookup_leaf_kernel,
                  relation_defs, relations_of)
from .distribution import HyperRect, full_rect
from .errors import DeviceUnavailable, OOBAccess, TendistError, UnboundVariable
from .ir import Access, Add, Const, Mul, accesses_of
from .tensors import DenseTensor

MAX_LOOPS, MAX_VARS, MAX_ACC, MAX_DIMS, MAX_CODE, MAX_OVER = 16, 48, 8, 8, 64, 4
VAR_LOOP, VAR_STRIP, VAR_ROTATE = 0, 1, 2
OP_CONST, OP_LOAD, OP_ADD, OP_MUL = 0, 1, 2, 3


class _VarDef(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("nover", C.c_int32),
                ("over", C.c_int32 * MAX_OVER), ("block", C.c_int64), ("extent", C.c_int64)]


class _Access(C.Structure):
    _fields_ = [("base", C.c_void_p), ("ndim", C.c_int32), ("pad", C.c_int32),
                ("slot", C.c_int32 * MAX_DIMS), ("origin", C.c_int64 * MAX_DIMS),
                ("stride", C.c_int64 * MAX_DIMS)]


class NestProg(C.Structure):
    _fields_ = [("nloops", C.c_int32), ("nvars", C.c_int32), ("nacc", C.c_int32), ("ncode", C.c_int32),
                ("reduce", C.c_int32), ("serial", C.c_int32), ("npar", C.c_int32), ("pad", C.c_int32),
                ("lo", C.c_int64 * MAX_LOOPS), ("hi", C.c_int64 * MAX_LOOPS),
                ("par", C.c_int32 * MAX_LOOPS), ("vars", _VarDef * MAX_VARS), ("out", _Access),
                ("acc", _Access * MAX_ACC), ("op", C.c_int32 * MAX_CODE), ("arg", C.c_int32 * MAX_CODE),
                ("konst", C.c_double * MAX_CODE)]


def torch_mod():
    try:
        import torch
    except Exception as exc:  # pragma: no cover
        raise DeviceUnavailable(f"PyTorch is required for device memory: {exc}") from exc
    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device is visible; the B200 path has no CPU fallback")
    return torch


def stream_handle(stream) -> C.c_void_p:
    return C.c_void_p(stream.cuda_stream if stream is not None else 0)


class DeviceTile:
    """An HBM buffer holding the global box `rect` of tensor `name`.

    ``data`` is a (possibly strided) CUDA float64 tensor of shape
    ``rect.shape``; the element at global coordinate x is ``data[x - rect.lo]``.
    """

    __slots__ = ("name", "rect", "data", "dims")

    def __init__(self, name, rect: HyperRect, data, dims=None):
        self.name = name
        self.rect = rect
        self.data = data
        self.dims = tuple(dims) if dims is not None else tuple(rect.hi)

    @property
    def origin(self) -> tuple:
        return self.rect.lo

    def strides(self) -> tuple:
        return tuple(self.data.stride())

    def ptr(self) -> int:
        return self.data.data_ptr()

    def view(self, box: HyperRect) -> "DeviceTile":
        """Sub-tile covering `box` (must lie inside this tile)."""
        if not self.rect.contains(box):
            raise OOBAccess(f"{self.name}: {box} is outside the resident box {self.rect}")
        if not box.lo:
            return DeviceTile(self.name, box, self.data, self.dims)
        idx = tuple(slice(a - o, b - o) for a, b, o in zip(box.lo, box.hi, self.rect.lo))
        return DeviceTile(self.name, box, self.data[idx], self.dims)

    def __repr__(self):
        return f"DeviceTile({self.name}, {self.rect}, device={self.data.device})"


# ------------------------------------------------------------------- compiler
def _closure(names, defs):
    """Derived variables needed by `names`, dependencies first."""
    order, seen = [], set()

    def visit(n):
        if n in seen:
            return
        seen.add(n)
        rel = defs.get(n)
        if rel is None:
            return
        deps = (rel.outer, rel.inner) if isinstance(rel, (Split, Divide)) else (rel.result, *rel.over)
        for d in deps:
            visit(d)
        order.append(n)

    for n in names:
        visit(n)
    return order


def _tree_loops(name, defs, loop_ext, acc):
    """Multiset of loop variables under `name`'s defining tree."""
    if name in loop_ext:
        acc.append(name)
        return
    rel = defs.get(name)
    if rel is None:
        raise UnboundVariable(f"{name} is neither loop-bound nor derivable")
    if isinstance(rel, (Split, Divide)):
        _tree_loops(rel.outer, defs, loop_ext, acc)
        _tree_loops(rel.inner, defs, loop_ext, acc)
    else:
        _tree_loops(rel.result, defs, loop_ext, acc)
        for v in rel.over:
            sub = []
            _tree_loops(v, defs, loop_ext, sub)
            if any(isinstance(x, tuple) or loop_ext[x] > 1 for x in sub):
                acc.append(("__rotate_over__", v))  # offsets over live loops: not injective-safe
            acc.extend(sub)


def compile_nest(loops, leaf, defs, out_tile: DeviceTile, in_tiles) -> NestProg:
    """loops: [(var, lo, hi)] in nest order (pinned variables as 1-trip loops).
    in_tiles: one DeviceTile per rhs access (accesses_of order)."""
    if not isinstance(leaf, (Assign, Reduce)):
        raise TendistError(f"cannot evaluate leaf {leaf!r}")
    rhs_acc = accesses_of(leaf.rhs)
    if len(loops) > MAX_LOOPS or len(rhs_acc) > MAX_ACC:
        raise TendistError(f"nest too large for the GPU evaluator ({len(loops)} loops, "
                           f"{len(rhs_acc)} accesses)")
    p = NestProg()
    loop_ext = {}
    slot = {}
    for q, (v, lo, hi) in enumerate(loops):
        p.lo[q], p.hi[q] = lo, hi
        loop_ext[v] = hi - lo
        slot[v] = q
        d = p.vars[q]
        d.kind, d.a = VAR_LOOP, q
    p.nloops = len(loops)
    names = list(dict.fromkeys(n for acc in [leaf.lhs, *rhs_acc] for n in acc.var_names))
    derived = [n for n in _closure(names, defs) if n not in slot]
    for n in names:
        if n not in slot and n not in derived:
            raise UnboundVariable(f"{n} is neither loop-bound nor derivable")
    if len(slot) + len(derived) > MAX_VARS:
        raise TendistError("too many variables for the GPU evaluator")
    for n in derived:
        q = len(slot)
        slot[n] = q
        rel = defs[n]
        d = p.vars[q]
        if isinstance(rel, (Split, Divide)):
            d.kind, d.a, d.b, d.block, d.extent = VAR_STRIP, slot[rel.outer], slot[rel.inner], rel.block, rel.extent
        else:
            if len(rel.over) > MAX_OVER:
                raise TendistError("rotate over too many loops for the GPU evaluator")
            d.kind, d.a, d.nover, d.extent = VAR_ROTATE, slot[rel.result], len(rel.over), rel.extent
            for k, v in enumerate(rel.over):
                d.over[k] = slot[v]
    p.nvars = len(slot)

    def fill(acc_struct, access: Access, tile: DeviceTile):
        nd = len(access.indices)
        acc_struct.ndim = nd
        acc_struct.base = tile.ptr()
        st = tile.strides() if nd else ()
        for ax, v in enumerate(access.var_names):
            acc_struct.slot[ax] = slot[v]
            acc_struct.origin[ax] = tile.rect.lo[ax]
            acc_struct.stride[ax] = st[ax]

    fill(p.out, leaf.lhs, out_tile)
    for k, (acc, tile) in enumerate(zip(rhs_acc, in_tiles)):
        fill(p.acc[k], acc, tile)
    p.nacc = len(rhs_acc)

    code = []
    index = {id(a): k for k, a in enumerate(rhs_acc)}

    def emit(e):
        if isinstance(e, Const):
            code.append((OP_CONST, 0, float(e.value)))
        elif isinstance(e, Access):
            code.append((OP_LOAD, index[id(e)], 0.0))
        elif isinstance(e, (Add, Mul)):
            emit(e.lhs)
            emit(e.rhs)
            code.append((OP_ADD if isinstance(e, Add) else OP_MUL, 0, 0.0))
        else:
            raise TendistError(f"cannot compile {e!r}")

    emit(leaf.rhs)
    if len(code) > MAX_CODE:
        raise TendistError("expression too long for the GPU evaluator")
    for k, (op, arg, kv) in enumerate(code):
        p.op[k], p.arg[k], p.konst[k] = op, arg, kv
    p.ncode = len(code)
    p.reduce = 1 if isinstance(leaf, Reduce) else 0

    # parallel loops: live loops under the output coordinate, if injective
    used = []
    for n in dict.fromkeys(leaf.lhs.var_names):
        _tree_loops(n, defs, loop_ext, used)
    live = [u for u in used if isinstance(u, tuple) or loop_ext[u] > 1]
    injective = all(not isinstance(u, tuple) for u in live) and len(set(live)) == len(live)
    if injective:
        par = [slot[v] for v, _, _ in loops if v in set(live)]
        p.serial = 0
        p.npar = len(par)
        for k, q in enumerate(par):
            p.par[k] = q
    else:
        p.serial = 1
        p.npar = 0
    return p


def launch_nest(prog: NestProg, stream) -> None:
    _native.call("td_nest_eval", stream_handle(stream), C.byref(prog), C.sizeof(prog))


def run_nest(loops, leaf, defs, out_tile, in_tiles, stream) -> None:
    launch_nest(compile_nest(loops, leaf, defs, out_tile, in_tiles), stream)


# ------------------------------------------------------- single-memory API
def device_buffer(shape, device, stream=None, *, zero: bool = False):
    """float64 HBM buffer for a launch's temporaries.  While a launch plan is
    being recorded (`_native.recording`) the buffer is kept alive by the plan
    (its ops hold raw pointers into it), and a zero fill is a plan op
    (td_fill) so replays zero it again."""
    torch = torch_mod()
    if stream is not None:
        with torch.cuda.stream(stream):
            t = torch.empty(tuple(shape), dtype=torch.float64, device=device)
    else:
        t = torch.empty(tuple(shape), dtype=torch.float64, device=device)
    rec = _native.recorder()
    if rec is not None:
        rec.hold(t)
    if zero and t.numel():
        st = stream if stream is not None else torch.cuda.current_stream(t.device)
        _native.call("td_fill", stream_handle(st), C.c_void_p(t.data_ptr()), t.numel(), 0.0)
    return t


def _upload(name, t: DenseTensor, device):
    torch = torch_mod()
    data = torch.from_numpy(t.data).to(device)
    return DeviceTile(name, full_rect(t.dims), data, t.dims)


def _zeros_tile(name, dims, device):
    torch = torch_mod()
    return DeviceTile(name, full_rect(dims), torch.zeros(tuple(dims), dtype=torch.float64, device=device),
                      dims)


def _download(tile: DeviceTile) -> DenseTensor:
    return DenseTensor(tile.dims, tile.data.detach().cpu().numpy())


def _nest_of(node):
    loops = []
    while isinstance(node, (Forall, Suchthat)):
        if isinstance(node, Forall):
            loops.append((node.var, node.lo, node.hi))
        node = node.body
    return loops, node


def _plugins(relations) -> dict:
    out = {}
    for rel in relations:
        if isinstance(rel, LeafKernel) and rel.kernel != INTERPRETER_KERNEL:
            fn = lookup_leaf_kernel(rel.kernel)
            if fn is None:
                from .leaves import BUILTIN_LEAVES
                if rel.kernel in BUILTIN_LEAVES:
                    continue  # native leaves: the nest itself runs on the GPU
                raise TendistError(f"leaf kernel {rel.kernel!r} is not registered")
            out[rel.vars[0]] = fn
    return out


def execute_chain(loops, leaf, env, defs, read_tiles, out_tiles, plugins, stream, device):
    """Run one Forall chain ending at `leaf`: Python-iterate loops above a
    plugin-substituted nest (reference semantics, cin.py:459-467) and
    evaluate everything else with the GPU nest kernel."""
    if isinstance(leaf, Place):
        return
    cut = next((k for k, (v, _, _) in enumerate(loops) if v in plugins), None)
    pinned = [(v, x, x + 1) for v, x in env.items()]
    if cut is None:
        ins = [read_tiles[a.tensor.name] for a in accesses_of(leaf.rhs)]
        run_nest(pinned + list(loops), leaf, defs, out_tiles[leaf.lhs.tensor.name], ins, stream)
        return
    outer, inner = loops[:cut], loops[cut:]
    fn = plugins[inner[0][0]]
    for point in itertools.product(*(range(lo, hi) for _, lo, hi in outer)):
        penv = dict(env)
        penv.update({v: x for (v, _, _), x in zip(outer, point)})
        if getattr(fn, "device", True):
            fn(LeafRuntime(list(inner), leaf, penv, defs, read_tiles, out_tiles, device, stream))
        else:
            _call_host_plugin(fn, list(inner), leaf, penv, defs, read_tiles, out_tiles, stream, device)


def _box_index(rect: HyperRect) -> tuple:
    return tuple(slice(a, b) for a, b in zip(rect.lo, rect.hi))


def _call_host_plugin(fn, inner, leaf, env, defs, read_tiles, out_tiles, stream, device):
    """The reference's plugin contract (`cin.py:359-379, 441-446`) for a
    plugin registered without ``device=True``: ``read_store`` holds full-size
    host DenseTensors in GLOBAL coordinates (the boxes this task-step reads,
    copied out of HBM -- a leaf only reads inside its iteration box) and
    ``out_store`` one full-size host tensor holding the task's partial so far
    (zero at the task's start, as the reference's per-task zeroed output),
    which the plugin updates in place; the output box is then written back
    to HBM.  ``execute_point`` evaluates one point with the GPU nest kernel
    against that host state, so a plugin mixing its own arithmetic with
    interpreter points sees the reference's order of writes."""
    torch = torch_mod()
    name = leaf.lhs.tensor.name
    out_tile = out_tiles[name]
    out_box = _box_index(out_tile.rect)
    with torch.cuda.stream(stream):
        read = {}
        for tname, tile in read_tiles.items():
            full = DenseTensor(tile.dims)
            full.data[_box_index(tile.rect)] = tile.data.cpu().numpy()
            read[tname] = full
        host_out = DenseTensor(out_tile.dims)
        host_out.data[out_box] = out_tile.data.cpu().numpy()
        ins = [read_tiles[a.tensor.name] for a in accesses_of(leaf.rhs)]

        def point(penv):
            out_tile.data.copy_(torch.from_numpy(host_out.data[out_box]))
            run_nest([(v, x, x + 1) for v, x in penv.items()], leaf, defs, out_tile, ins, stream)
            host_out.data[out_box] = out_tile.data.cpu().numpy()

        fn(LeafRuntime(inner, leaf, env, defs, read, {name: host_out}, device, stream, point))
        out_tile.data.copy_(torch.from_numpy(host_out.data[out_box]))


def interpret_on_device(stmt, store: dict) -> dict:
    torch = torch_mod()
    _native.load()
    device = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(device)
    read = {n: _upload(n, t, device) for n, t in store.items()}
    produced: dict = {}
    rels = relations_of(stmt)
    plugins = _plugins(rels)

    def outputs_for(node):
        outs = {}
        for leaf in leaf_statements(node):
            if isinstance(leaf, (Assign, Reduce)):
                t = leaf.lhs.tensor
                outs.setdefault(t.name, _zeros_tile(t.name, t.dims, device))
        return outs

    def walk(node, defs, outs):
        if isinstance(node, Suchthat):
            walk(node.body, relation_defs(node.relations) | defs, outs)
        elif isinstance(node, Seq):
            for s in node.stmts:
                local = outputs_for(s)
                walk(s, defs, local)
                read.update(local)
                produced.update(local)
        else:
            loops, leaf = _nest_of(node)
            execute_chain(loops, leaf, {}, defs, read, outs, plugins, stream, device)

    top = body_of(stmt)
    outs = {} if isinstance(top, Seq) else outputs_for(top)
    walk(top, relation_defs(rels), outs)
    produced.update(outs)
    torch.cuda.synchronize(device)
    result = dict(store)
    result.update({n: _download(t) for n, t in produced.items()})
    return result


def evaluate_statement(stmt, inputs: dict) -> DenseTensor:
    from .cin import lower_to_cin
    out = interpret_on_device(lower_to_cin(stmt), {n: inputs[n] for n in inputs})
    return out[stmt.lhs.tensor.name]


# ---------------------------------------------------------- LeafRuntime hooks
def run_point(rt: LeafRuntime, env) -> None:
    loops = [(v, x, x + 1) for v, x in env.items()]
    ins = [rt.read_store[a.tensor.name] for a in accesses_of(rt.stmt.rhs)]
    run_nest(loops, rt.stmt, rt.defs, rt.out_store[rt.stmt.lhs.tensor.name], ins, rt.stream)


def run_leaf_nest(rt: LeafRuntime) -> None:
    pinned = [(v, x, x + 1) for v, x in rt.env.items()]
    ins = [rt.read_store[a.tensor.name] for a in accesses_of(rt.stmt.rhs)]
    run_nest(pinned + list(rt.loops), rt.stmt, rt.defs, rt.out_store[rt.stmt.lhs.tensor.name], ins,
             rt.stream)
