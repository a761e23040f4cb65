"""Execution on B200s: HBM tile store, NCCL transfer program, leaf launches.

Drop-in for the reference's runtime (`pkg/src/tendist/simulator.py`):

* `RegionStore` / `Region` (reference `simulator.py:274-314`): the host
  bookkeeping (distribution, residency) plus the *HBM tile map*: one
  contiguous row-major float64 buffer per (GPU, piece), shared by every
  processor placed on that GPU.  ``Region.tensor`` gathers the canonical
  value back to the host on demand.
* `execute` (reference `simulator.py:537-663`): `planner.build_program`
  reproduces the reference ledger and emits the buffer program; this module
  runs it.  Per step: the step's transfers are issued as one NCCL group on
  each GPU's communication stream (same-GPU transfers alias the source
  tile), the compute stream waits for them, then every task's step nest runs
  as a native leaf (`leaves.run_leaf`).  Because step s+1's group is queued
  on the communication stream while step s's leaves run on the compute
  stream, communication overlaps computation (the reference's double
  buffering of temporaries across one step boundary, `simulator.py:607-613`).
  Write-backs (`simulator.py:624-654`) are NCCL transfers into the home GPU
  followed by an in-order accumulation, so reductions combine in machine
  enumeration order exactly as the reference does.
* `run_statement`, `RunResult`, `verify_result`, `redistribute`
  (reference `simulator.py:317-357, 668-726`).
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native, peer
from .cin import (Forall, INTERPRETER_KERNEL, LeafKernel, Suchthat,
                  leaf_accesses, leaf_statements, lookup_leaf_kernel, lower_to_cin)
from .comm import world as current_world
from .distribution import HyperRect, TensorDistribution, check_redistributable, subtract_rects
from .errors import (ConfigError, ExtentMismatch, MissingDistribution, MissingInput, TendistError,
                     VerifyFail)
from .interp import DeviceTile, device_buffer, execute_chain, stream_handle, torch_mod
from .ir import TensorIndexStmt, accesses_of
from .leaves import BUILTIN_LEAVES, contracted_var, flush_pending, native_plan, run_leaf, run_native_box
from .machine import Machine
from .planner import build_program
from .tensors import DenseTensor
from .trace import CommEvent, ExecutionTrace

LEAF_POLICIES = ("auto", "exact")
# lower one-to-many fetches to ncclBroadcast on GPU sub-communicators (else p2p fan-out)
USE_BROADCAST = True
# issue step s+1's NCCL group while step s's leaves run (False serialises every
# step: a measurement switch for the overlap, used by bench.py).  Even when True,
# a step whose NCCL transfers are large (>= SERIAL_MIN_BYTES into one GPU) yet
# take < SERIAL_FRACTION of the previous step's leaf time (at NVLINK_GBS / FP64
# peak) is serialised: NCCL's copy kernels would only hold SM slots the DMMA
# waves need for gigabytes' worth of transfer (Cannon 2x2 at 26112^3 on 4 B200s:
# 249.0 ms per step serialised on every box, 251-276 ms overlapped).  Copy-engine
# shifts (peer.CE_SHIFTS) hold no SM slot and stay overlapped.
OVERLAP_COMM = True
SERIAL_MIN_BYTES = 64 << 20
SERIAL_FRACTION = 0.1
NVLINK_GBS = 400.0
# pipeline the first step: its cross-GPU transfers go in two k-pieces (1/8, 7/8)
# and the GEMM leaves start on the first piece while the rest is in flight
# (nothing earlier can hide step 0's transfers: Cannon's skew, Johnson's faces)
SPLIT_FIRST_STEP = True
SPLIT_MIN_BYTES = 32 << 20


def _k_cuts(lo: int, hi: int, pieces: int = 2) -> list:
    """Pieces of a k-range for the pipelined first step: a short head
    (1/8, rounded up to 64) that arrives quickly, then the rest; or, with
    pieces > 2 (inputs still uploading, RegionStore.first_step_pieces),
    `pieces` equal parts cut like the upload slabs (RegionStore.upload)."""
    n = hi - lo
    if pieces > 2 and n >= 64 * pieces:
        return [(lo + (q * n) // pieces, lo + ((q + 1) * n) // pieces) for q in range(pieces)]
    head = min(n, -(-max(1, n // 8) // 64) * 64)
    if n < 256 or head >= n:
        return [(lo, hi)]
    return [(lo, lo + head), (lo + head, hi)]


def _with_range(rect: HyperRect, axis: int, lo: int, hi: int) -> HyperRect:
    return HyperRect(tuple(lo if a == axis else x for a, x in enumerate(rect.lo)),
                     tuple(hi if a == axis else x for a, x in enumerate(rect.hi)))


def _strides(t):
    return _native.i64_array(t.stride())


def _copy_box(stream, dst, src, accumulate=False):
    """dst (+)= src for two same-shape CUDA views on one device."""
    shape = tuple(dst.shape)
    if not shape:
        shape, ds, ss = (1,), _native.i64_array([1]), _native.i64_array([1])
    else:
        ds, ss = _strides(dst), _strides(src)
    _native.call("td_copy_box", stream_handle(stream), len(shape), _native.i64_array(shape),
                 C.c_void_p(dst.data_ptr()), ds, C.c_void_p(src.data_ptr()), ss, int(accumulate))


def _slice(buf, rect: HyperRect, box: HyperRect):
    """View of the part `box` of a buffer that holds `rect`."""
    if not box.lo or (box.lo == rect.lo and box.hi == rect.hi):
        return buf
    return buf[tuple(slice(a - o, b - o) for a, b, o in zip(box.lo, box.hi, rect.lo))]


# ------------------------------------------------------------------ regions
class Region:
    """One tensor: distribution, residency (host bookkeeping) and HBM pieces."""

    def __init__(self, store, name: str, dist: TensorDistribution):
        self._store = weakref.ref(store)     # no store<->region cycle: HBM frees on `del store`
        self.name = name
        self.dist = dist
        self.residency = dist.residency()
        self.pieces = {}          # (gpu, color) -> CUDA tensor holding piece_bounds(color)
        self.zeroed = False       # every piece is known to hold +0.0 (fresh output)
        # pieces that are +0.0 by contract but not yet in memory (RegionStore.zero is lazy:
        # the first leaf writing a whole piece overwrites it; anything else fills it first)
        self.pending_zero = set()

    def materialize(self) -> None:
        """Write the zeros `RegionStore.zero` deferred (before any read)."""
        if not self.pending_zero:
            return
        torch = torch_mod()
        for key in sorted(self.pending_zero, key=repr):
            buf = self.pieces.get(key)
            if buf is not None:
                _native.call("td_fill", stream_handle(torch.cuda.current_stream(buf.device)),
                             C.c_void_p(buf.data_ptr()), buf.numel(), 0.0)
        self.pending_zero = set()

    @property
    def store(self):
        return self._store()

    @property
    def dims(self):
        return self.dist.tensor_dims

    def held_at(self, coord) -> list:
        return self.residency.get(coord, [])

    def volume_at(self, coord) -> int:
        return sum(r.volume for r in self.held_at(coord))

    def gpus_of(self, color) -> list:
        box = self.dist.piece_bounds(color)
        m, W = self.store.machine, self.store.world.ngpus
        out = []
        for p in self.dist.processors_of(color):
            if box in self.residency.get(p, ()):
                g = m.device_of(p, W)
                if g not in out:
                    out.append(g)
        return out

    def piece(self, g, color):
        return self.pieces[(g, color)]

    @property
    def tensor(self) -> DenseTensor:
        return self.store.gather(self.name)


class RegionStore:
    """All regions of one machine, resident in the HBM of the job's GPUs."""

    def __init__(self, machine: Machine, world=None):
        self.machine = machine
        self.world = world or current_world()
        self.regions: dict = {}
        self.ready: dict = {}     # (tensor, gpu, color) -> [(box, CUDA event)] of slabs still arriving
        self.done: dict = {}      # (tensor, gpu, color) -> CUDA event after the last write of a launch
        self.pending: dict = {}   # (tensor, gpu, color) -> [box, buf, host, slabs left] deferred uploads
        # output streaming (e2e): the last step's GEMM leaves of a directly written
        # home piece run in `stream_rows` row pieces, each followed by an event in
        # row_done[(tensor, gpu, color)] = [(row lo, row hi, event)] (piece-local rows),
        # so a caller can start the D2H of finished rows while later rows compute
        self.stream_rows: int = 0
        self.row_done: dict = {}
        # k-pieces of the pipelined first step (runtime._k_cuts): 2 = head + rest;
        # with inputs uploading in k-slabs, set it to the slab count so every piece
        # waits only for its own slabs.  Must be equal on every rank (it shapes the
        # NCCL groups).
        self.first_step_pieces: int = 2

    def __contains__(self, name) -> bool:
        return name in self.regions

    def __getitem__(self, name) -> Region:
        return self.regions[name]

    def persistent_volume(self, coord) -> int:
        return sum(r.volume_at(coord) for r in self.regions.values())

    def _check(self, name, dims, dist):
        if dist.machine != self.machine:
            raise ConfigError(f"distribution machine {dist.machine} is not the store's {self.machine}")
        if tuple(dims) != dist.tensor_dims:
            raise ConfigError(f"{name} has dims {tuple(dims)}, distribution wants {dist.tensor_dims}")

    def _alloc(self, name, dist, fill):
        """Create the region and one buffer per (owned GPU, piece); fill(g, color, box, buf)."""
        torch = torch_mod()
        region = Region(self, name, dist)
        for color, box, _ in dist.pieces():
            for g in region.gpus_of(color):
                if not self.world.owns(g):
                    continue
                dev = self.world.device(g)
                with torch.cuda.device(dev):
                    buf = torch.empty(box.shape, dtype=torch.float64, device=dev)
                    fill(g, color, box, buf)
                region.pieces[(g, color)] = buf
        self.regions[name] = region
        return region

    def place(self, name: str, tensor: DenseTensor, dist: TensorDistribution) -> Region:
        """Copy a host tensor into its pieces (reference `simulator.py:297-305`)."""
        self._check(name, tensor.dims, dist)
        torch = torch_mod()
        host = tensor.data

        def fill(g, color, box, buf):
            src = host[box.slices()] if box.lo else host
            buf.copy_(torch.from_numpy(np.ascontiguousarray(src)), non_blocking=False)

        return self._alloc(name, dist, fill)

    def place_file(self, name: str, path, dist: TensorDistribution) -> Region:
        """Load a tensor saved in the reference's binary format (little-endian
        u64 order, u64 extents, row-major <f8 payload; reference
        `tensors.py:72-92`) straight into the pieces this process holds: the
        file is memory-mapped and only each piece's box is read, so no host
        copy of the whole tensor is ever made."""
        import struct
        torch = torch_mod()
        with open(path, "rb") as fh:
            head = fh.read(8)
            (order,) = struct.unpack("<Q", head)
            dims = struct.unpack("<" + "Q" * order, fh.read(8 * order)) if order else ()
        self._check(name, dims, dist)
        need = 8 * (1 + order) + 8 * (int(np.prod(dims, dtype=np.int64)) if dims else 1)
        have = os.path.getsize(path)
        if have != need:     # as the reference's from_bytes (tensors.py:84-92): short or long payloads fail
            raise ExtentMismatch(f"{path}: {have} bytes, but a tensor of dims {tuple(dims)} needs {need}")
        payload = np.memmap(path, dtype="<f8", mode="r", offset=8 * (1 + order),
                            shape=tuple(dims) if dims else (1,))

        def fill(g, color, box, buf):
            src = payload[box.slices()] if box.lo else payload.reshape(())
            buf.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)))

        region = self._alloc(name, dist, fill)
        del payload
        return region

    def save_file(self, name: str, path) -> None:
        """Write a region's canonical value in the reference's binary format."""
        from .tensors import save_tensor
        save_tensor(self.gather(name), path)

    def place_zeros(self, name: str, dist: TensorDistribution) -> Region:
        region = self._alloc(name, dist, lambda g, c, b, buf: buf.zero_())
        region.zeroed = True
        return region

    def place_host(self, name: str, host: np.ndarray, dist: TensorDistribution, streams=None) -> Region:
        """Upload from (ideally pinned) host memory with async copies; `streams`
        maps GPU -> stream (default: that GPU's compute stream)."""
        self._check(name, host.shape, dist)
        torch = torch_mod()

        def fill(g, color, box, buf):
            st = (streams or {}).get(g) or self.world.streams(g)[0]
            src = torch.from_numpy(host[box.slices()] if box.lo else host)
            with torch.cuda.stream(st):
                if src.is_contiguous():
                    buf.copy_(src, non_blocking=True)
                else:
                    _h2d_box(st, buf, src)
                buf.record_stream(st)

        return self._alloc(name, dist, fill)

    def local_colors(self, dist: TensorDistribution):
        """(color, box) of the pieces some GPU of this process must hold."""
        probe = Region(self, "?", dist)
        for color, box, _ in dist.pieces():
            if any(self.world.owns(g) for g in probe.gpus_of(color)):
                yield color, box

    def place_local(self, name: str, dist: TensorDistribution, host_pieces: dict, *, slabs: int = 1,
                    axis: int = 0, copy_stream: int = 0, defer: bool = False) -> Region:
        """Upload per-piece host arrays (pinned for async H2D): host_pieces maps
        color -> array of that piece's box.  Only this process's pieces are
        needed -- the e2e path of the benchmark.

        With ``slabs > 1`` each piece arrives in that many slabs along `axis`
        on the GPU's copy stream, each with its own event; `execute` makes a
        leaf (or a send) wait only for the slabs its box touches, so the
        upload of later k-slabs overlaps the leaves of earlier steps.  With
        ``defer=True`` only the buffers are allocated and the caller orders
        the copies itself with `upload` (all before `execute`)."""
        torch = torch_mod()

        def fill(g, color, box, buf):
            src = torch.from_numpy(host_pieces[color])
            if defer:
                self.pending[(name, g, color)] = [box, buf, src, None]
            elif slabs <= 1 or not box.lo:
                st = self.world.streams(g)[0]
                with torch.cuda.stream(st):
                    buf.copy_(src, non_blocking=True)
                buf.record_stream(st)
            else:
                self.pending[(name, g, color)] = [box, buf, src, None]
                self.upload(name, color, slabs=slabs, axis=axis, copy_stream=copy_stream)

        region = self._alloc(name, dist, fill)
        if slabs <= 1 and not defer:
            for g in self.world.owned:
                torch.cuda.current_stream(self.world.device(g)).wait_stream(self.world.streams(g)[0])
        return region

    def upload(self, name: str, color, *, slabs: int = 1, axis: int = 0, copy_stream: int = 0,
               only=None) -> None:
        """Enqueue the H2D copy of (some slabs of) a deferred piece on every
        owned GPU holding it; `only` selects slab indices (default: all)."""
        torch = torch_mod()
        for (n, g, c), rec in list(self.pending.items()):
            if n != name or c != color:
                continue
            box, buf, src, left = rec
            if left is None:
                left = rec[3] = set(range(slabs))
            st = self.world.copy_stream(g, copy_stream)
            size = box.shape[axis] if box.lo else 1
            cuts = [(q * size) // slabs for q in range(slabs + 1)]
            events = self.ready.setdefault((name, g, color), [])
            for q in sorted(left if only is None else set(only) & left):
                a, b = cuts[q], cuts[q + 1]
                left.discard(q)
                if b <= a:
                    continue
                if box.lo:
                    idx = tuple(slice(a, b) if d == axis else slice(None) for d in range(len(box.lo)))
                    _copy_any(st, buf[idx], src[idx])
                    lo, hi = list(box.lo), list(box.hi)
                    lo[axis], hi[axis] = box.lo[axis] + a, box.lo[axis] + b
                    part = HyperRect(lo, hi)
                else:
                    _copy_any(st, buf, src)
                    part = box
                ev = torch.cuda.Event()
                ev.record(st)
                events.append((part, ev))
            buf.record_stream(st)
            if not left:
                del self.pending[(n, g, c)]

    def wait_ready(self, stream, name, g, color, rect) -> None:
        """Make `stream` wait for the slabs of piece (name, g, color) that `rect` touches."""
        if (name, g, color) in self.pending:
            raise ConfigError(f"{name} piece {color} still has slabs that were never uploaded")
        for box, ev in self.ready.get((name, g, color), ()):
            if not rect.lo or box.intersect(rect) is not None:
                stream.wait_event(ev)

    def zero(self, name: str) -> None:
        """Reset every resident piece of a region to +0.0 (a fresh output).

        Lazy: the pieces are only marked.  The next launch writing the region
        lets the first leaf of each task that owns a whole piece overwrite it
        (0 + x = x: the same bits as accumulating into zeros, without the fill
        pass or the epilogue's read of the old values) and fills the rest;
        every read path (gather, local_pieces, redistribute, ...) fills first."""
        region = self.regions[name]
        region.pending_zero = set(region.pieces)
        region.zeroed = True

    def place_generated(self, name: str, dist: TensorDistribution, *, seed=0, tensor_id=0,
                        mode=0) -> Region:
        """Synthetic inputs generated in HBM (values per oracle/generator.py)."""
        dims = dist.tensor_dims

        def fill(g, color, box, buf):
            shape = box.shape or (1,)
            _native.call("td_generate", stream_handle(_torch_current(buf)), len(dims),
                         _native.i64_array(dims), _native.i64_array(box.lo or (0,)),
                         _native.i64_array(shape), C.c_void_p(buf.data_ptr()),
                         _native.i64_array(buf.stride() or (1,)), seed, tensor_id, mode)

        return self._alloc(name, dist, fill)

    # ---- host views
    def gather(self, name: str) -> DenseTensor:
        """Canonical value of a region on the host (D2H of the home pieces).

        COLLECTIVE in SPMD jobs (one process per GPU): every piece is
        broadcast from its holder, so every rank must call gather (or read
        `RunResult.output`) at the same point -- calling it on rank 0 only
        would leave rank 0 waiting for the others; the World.wait watchdog
        then aborts NCCL and raises CommError after TD_NCCL_TIMEOUT seconds
        instead of hanging.  Use `local_pieces` for rank-local reads."""
        torch = torch_mod()
        region = self.regions[name]
        region.materialize()
        out = np.zeros(region.dims, dtype=np.float64)
        W = self.world
        if W.multi_gpu:
            W.wait()
        for color, box, procs in region.dist.pieces():
            gpus = region.gpus_of(color)
            if not gpus:
                continue
            src_g = gpus[0]
            if W.owns(src_g):
                buf = region.pieces[(src_g, color)]
                with torch.cuda.device(buf.device):
                    torch.cuda.current_stream().wait_stream(W.streams(src_g)[0])
                    arr = buf.cpu().numpy()
            else:
                arr = None
            if W.nprocs > 1:
                arr = _bcast_piece(W, src_g, box, arr)
            if box.lo:
                out[box.slices()] = arr
            else:
                out[...] = arr
        return DenseTensor(region.dims, out)

    def local_pieces(self, name: str):
        """(box, CUDA tensor) for the home pieces of `name` on this process's GPUs."""
        region = self.regions[name]
        region.materialize()
        for color, box, procs in region.dist.pieces():
            gpus = region.gpus_of(color)
            if gpus and self.world.owns(gpus[0]):
                yield box, region.pieces[(gpus[0], color)]


def _torch_current(buf):
    import torch
    return torch.cuda.current_stream(buf.device)


def _h2d_box(stream, dst, src):
    """Host (strided) -> device box copy."""
    _copy_any(stream, dst, src)


def _copy_any(stream, dst, src):
    """Async copy between two same-shape views (host pinned <-> device or
    device <-> device) with pitched 2-D DMA copies: the views' trailing axes
    must be unit-stride; leading axes are collapsed when possible and looped
    otherwise."""
    shape = tuple(dst.shape)
    if not shape:
        dst.copy_(src, non_blocking=True)
        return
    if dst.is_contiguous() and src.is_contiguous():
        n = dst.numel()
        _native.call("td_memcpy_2d", stream_handle(stream), C.c_void_p(dst.data_ptr()), n,
                     C.c_void_p(src.data_ptr()), n, n, 1)
        return
    if dst.stride()[-1] != 1 or src.stride()[-1] != 1:
        raise ConfigError("pitched copies need unit-stride rows")
    if len(shape) == 1:
        _native.call("td_memcpy_2d", stream_handle(stream), C.c_void_p(dst.data_ptr()), shape[0],
                     C.c_void_p(src.data_ptr()), shape[0], shape[0], 1)
        return
    # collapse leading axes that are uniformly strided on both sides
    def rows_of(t):
        st, sh = t.stride(), t.shape
        pitch = st[-2]
        for d in range(len(sh) - 2, 0, -1):
            if st[d - 1] != st[d] * sh[d]:
                return None
        return pitch
    pd, ps = rows_of(dst), rows_of(src)
    if pd is not None and ps is not None:
        rows = 1
        for e in shape[:-1]:
            rows *= e
        _native.call("td_memcpy_2d", stream_handle(stream), C.c_void_p(dst.data_ptr()), pd,
                     C.c_void_p(src.data_ptr()), ps, shape[-1], rows)
        return
    for q in range(shape[0]):
        _copy_any(stream, dst[q], src[q])


def _bcast_piece(W, root_g, box, arr):
    """SPMD: every process obtains the piece held by GPU root_g."""
    torch = torch_mod()
    g = W.owned[0]
    dev = W.device(g)
    buf = torch.from_numpy(arr).to(dev) if arr is not None else torch.empty(box.shape, dtype=torch.float64,
                                                                           device=dev)
    st = torch.cuda.current_stream(dev)
    _native.call("td_bcast", W.comm(g), stream_handle(st), C.c_void_p(buf.data_ptr()),
                 max(1, box.volume), root_g)
    W.wait()       # watchdog: a rank that never joins aborts the job instead of hanging it
    return buf.cpu().numpy()


# ----------------------------------------------------------------- execute
def _loops_of(node):
    loops = []
    while isinstance(node, (Forall, Suchthat)):
        if isinstance(node, Forall):
            loops.append((node.var, node.lo, node.hi))
        node = node.body
    return loops, node


def _leaf_choice(relations, loop_vars, policy):
    """(policy, python plugin or None) for a nest, from its LeafKernel relations."""
    for rel in relations:
        if isinstance(rel, LeafKernel) and rel.vars[0] in loop_vars:
            if rel.kernel == INTERPRETER_KERNEL:
                return "exact", None
            fn = lookup_leaf_kernel(rel.kernel)
            if fn is not None:
                return policy, {rel.vars[0]: fn}
            if rel.kernel in BUILTIN_LEAVES:
                return (rel.kernel if policy == "auto" else policy), None
            raise TendistError(f"leaf kernel {rel.kernel!r} is not registered")
    return policy, None


# NVTX ranges around each step's transfers / leaves and the commit phase
# (TD_NVTX=1): host-side ranges a profiler (ncu --nvtx, nsys) attributes the
# launches to; off by default (they cost a few microseconds each)
NVTX = os.environ.get("TD_NVTX", "0") == "1"


class _nvtx:
    __slots__ = ("name",)

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if NVTX:
            torch_mod().cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if NVTX:
            torch_mod().cuda.nvtx.range_pop()
        return False


class _NoBatch:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class _NativeEvent:
    """A plan-owned cudaEvent (td_event_create), usable where torch events are."""

    __slots__ = ("handle",)

    def __init__(self, handle: int):
        self.handle = handle


def g_index(world, g) -> int:
    return world.device(g).index


class _Executor:
    shift: dict = {}            # id(Transfer) -> copy-engine shift buffer (set per launch by run)

    def __init__(self, prog, store: RegionStore, policy: str):
        self.prog = prog
        self.plan = prog.plan
        self.store = store
        self.W = store.world
        self.policy = policy
        self.m = store.machine
        self.use_bcast = USE_BROADCAST and self.W.multi_gpu
        self.buffers = {}            # hid -> CUDA tensor (owned GPUs only)
        self.alias_origin = {}       # temp hid aliasing a piece -> (tensor, gpu, color)
        self.out_bufs = {}           # task coord -> CUDA tensor of out_rect
        self.torch = torch_mod()
        self.gpus = sorted({self.gpu(t.coord) for t in self.plan.tasks} |
                           {g for g in self.W.owned})
        self.owned = [g for g in self.gpus if self.W.owns(g)]
        self.credits = {}            # id(inbox) -> plan-owned credit event (while recording)

    def gpu(self, p) -> int:
        cache = self.__dict__.setdefault("_gpu_of", {})
        g = cache.get(p)
        if g is None:
            g = cache[p] = self.m.device_of(p, self.W.ngpus)
        return g

    def cstream(self, g):
        return self.W.streams(g)[0]

    def xstream(self, g):
        return self.W.streams(g)[1]

    # ---- buffers
    def holding_buf(self, hid):
        h = self.prog.holdings[hid]
        if h.kind == "piece":
            return self.store[h.tensor].piece(self.gpu(h.proc), h.color)
        return self.buffers[hid]

    def origin(self, hid):
        """(tensor, gpu, color) of the resident piece a holding views, if any."""
        h = self.prog.holdings[hid]
        if h.kind == "piece":
            return (h.tensor, self.gpu(h.proc), h.color)
        return self.alias_origin.get(hid)

    def wait_piece(self, stream, hid, rect):
        """Progressive placement: wait for the slabs of the underlying piece."""
        o = self.origin(hid)
        if o is not None and (self.store.ready or self.store.pending):
            self.store.wait_ready(stream, o[0], o[1], o[2], rect)

    def _sync(self, waiter, producer):
        self._after(waiter, self._mark(producer))

    def _mark(self, stream):
        """An event on `stream` at this point (a plan-owned native event and a
        plan op while a launch plan is being recorded)."""
        rec = _native.recorder()
        if rec is None:
            ev = self.torch.cuda.Event()
            ev.record(stream)
            return ev
        dev = stream.device.index
        h = rec.event(dev)
        _native.call("td_event_record", C.c_void_p(h), stream_handle(stream), dev)
        return _NativeEvent(h)

    @staticmethod
    def _after(stream, ev, record=True):
        """`stream` waits for `ev` (torch or native event)."""
        if isinstance(ev, _NativeEvent):
            dev = stream.device.index
            if record:
                _native.call("td_stream_wait_event", stream_handle(stream), C.c_void_p(ev.handle), dev)
            else:
                _native.check(_native.lib().td_stream_wait_event(stream_handle(stream), C.c_void_p(ev.handle),
                                                                 dev))
        else:
            stream.wait_event(ev)

    # ---- phases
    def run(self):
        torch = self.torch
        for g in self.owned:
            cur = torch.cuda.current_stream(self.W.device(g))
            self._sync(self.cstream(g), cur)
            self._sync(self.xstream(g), cur)
        out_region = self.store[self.plan.out_name]
        self.store.row_done = {k: v for k, v in self.store.row_done.items() if k[0] != self.plan.out_name}
        self.direct = self._direct_commits(out_region)
        self.inbox = self._inboxes()
        self.shift = self._shifts()
        self.overwrite = self._lazy_zeros(out_region)
        for t in self.plan.tasks:
            g = self.gpu(t.coord)
            if t.out_rect is not None and self.W.owns(g):
                if t.coord in self.direct:
                    color = self.direct[t.coord]
                    self.out_bufs[t.coord] = out_region.piece(g, color)
                    continue
                ib = self.inbox.get(t.coord)
                if ib is not None:
                    if ib.credit is not None and not _CAPTURING:   # the home has released the inbox
                        self._after(self.cstream(g), ib.credit, record=False)
                    rec = _native.recorder()
                    if rec is not None:
                        # a replay's leaf waits for the previous replay's release of the inbox
                        h = self.credits[id(ib)] = rec.event(g_index(self.W, g))
                        _native.call("td_stream_wait_event", stream_handle(self.cstream(g)), C.c_void_p(h),
                                     g_index(self.W, g))
                    self.out_bufs[t.coord] = ib.writer_view()
                    continue
                self.out_bufs[t.coord] = device_buffer(t.out_rect.shape, self.W.device(g), self.cstream(g),
                                                       zero=True)
        nsteps = self.plan.num_steps
        local = self._local_only()
        if local and self._early_outputs():
            self._run_task_major(out_region)
        else:
            from .leaves import gemm_batch
            batch = gemm_batch() if local and not self._reads_output() else _NoBatch()
            with batch:
                self._steps(nsteps)
            if not self.prog.stepwise:
                self.compute(self.prog.work[-1], -1)
            self._fill_unwritten()
            self._shift_credits()
            with _nvtx("commit"):
                self.commit(out_region)
            self._mark_done(out_region, self.prog.commits)
        for g in self.owned:
            cur = torch.cuda.current_stream(self.W.device(g))
            self._sync(cur, self.cstream(g))
            self._sync(cur, self.xstream(g))
        self.buffers.clear()
        self.out_bufs.clear()

    def _lazy_zeros(self, out_region) -> set:
        """Resolve `RegionStore.zero`'s deferred zeros for this launch: the
        tasks writing a whole pending output piece directly get their first
        leaf as an overwrite (returned); every other pending piece, of the
        output or of any region the launch reads, is filled now."""
        overwrite = set()
        task_loops, _ = _loops_of(self.plan.task_body)
        _, plugins = _leaf_choice(self.plan.relations, [v for v, _, _ in task_loops], self.policy)
        if out_region.pending_zero and not plugins and not self._reads_output():
            for t in self.plan.tasks:
                color = self.direct.get(t.coord)
                key = (self.gpu(t.coord), color)
                if color is not None and key in out_region.pending_zero:
                    overwrite.add(t.coord)
                    out_region.pending_zero.discard(key)
        for region in self.store.regions.values():
            if not region.pending_zero:
                continue
            for key in sorted(region.pending_zero, key=repr):
                g = key[0]
                if self.W.owns(g) and key in region.pieces:
                    buf = region.pieces[key]
                    _native.call("td_fill", stream_handle(self.cstream(g)), C.c_void_p(buf.data_ptr()),
                                 buf.numel(), 0.0)
            region.pending_zero = set()
        return overwrite

    def _fill_unwritten(self, coords=None) -> None:
        """A task granted the first-leaf overwrite that ran no leaf at all
        (no iteration points) still owes its piece the zeros."""
        for coord in sorted(self.overwrite if coords is None else self.overwrite & set(coords)):
            self.overwrite.discard(coord)
            buf = self.out_bufs.get(coord)
            if buf is not None:
                from .leaves import flush_pending
                flush_pending()
                _native.call("td_fill", stream_handle(self.cstream(self.gpu(coord))), C.c_void_p(buf.data_ptr()),
                             buf.numel(), 0.0)

    def _acc_of(self, coord) -> int:
        """0: this task's leaf overwrites its output tile (a peer inbox, or the
        first leaf into a lazily zeroed piece; run_leaf zero-fills when the
        leaf does not cover the tile), else 1 (accumulate)."""
        if coord in self.inbox:
            return 0
        if coord in self.overwrite:
            self.overwrite.discard(coord)
            return 0
        return 1

    def _reads_output(self) -> bool:
        return self.plan.out_name in {a.tensor.name for leaf in leaf_statements(self.plan.task_body)
                                      for a in accesses_of(leaf.rhs)}

    def _serial_steps(self) -> frozenset:
        """Steps whose transfers wait for the previous step's leaves (see
        OVERLAP_COMM); decided from the program alone, so every rank agrees."""
        ce = bool(self.shift)
        cached = self.prog.__dict__.get("_serial_steps")
        if cached is not None and cached[0] == ce:
            return cached[1]
        out = set()
        for s in range(self.plan.num_steps):
            # step 0 overlaps the previous launch's leaves (back-to-back launches): the
            # same contention, measured against its own leaves (Johnson 2x2x2 on 4 GPUs:
            # 492 ms per step serialised, 506-579 ms overlapped on the same box)
            inbound = {}
            for t in self.prog.transfers[s]:
                gs, gd = self.gpu(t.src), self.gpu(t.dst)
                if gs != gd and id(t) not in self.shift:   # copy-engine shifts hold no SM slots
                    inbound[gd] = inbound.get(gd, 0) + 8 * t.part.volume
            flops = {}
            for w in self.prog.work[max(s - 1, 0)]:
                ext = {}
                for names, (_, rect, _) in w.operands.items():
                    if rect is not None:
                        ext.update(zip(names, rect.shape))
                vol = 1
                for e in ext.values():
                    vol *= e
                g = self.gpu(w.task.coord)
                flops[g] = flops.get(g, 0) + 2 * vol
            big = max(inbound.values(), default=0)
            comm_s = big / (NVLINK_GBS * 1e9)
            compute_s = min(flops.values(), default=0) / (FP64_PEAK_GFLOPS * 1e9)
            if big >= SERIAL_MIN_BYTES and comm_s < SERIAL_FRACTION * compute_s:
                out.add(s)
        self.prog._serial_steps = (ce, frozenset(out))
        return self.prog._serial_steps[1]

    def _steps(self, nsteps):
        serial = self._serial_steps() if OVERLAP_COMM else frozenset()
        for s in range(nsteps):
            if not OVERLAP_COMM or s in serial:   # step s's transfers wait for step s-1's leaves
                for g in self.owned:
                    self._sync(self.xstream(g), self.cstream(g))
            split = self._split_plan(s) if s == 0 and self.prog.stepwise else None
            if split is not None:
                with _nvtx(f"step {s} pipelined"):
                    self.compute_split(self.prog.work[s], s, split,
                                       self.transfers_split(self.prog.transfers[s], split))
                self.release(s)
                continue
            with _nvtx(f"step {s} transfers"):
                self.transfers(self.prog.transfers[s])
            for g in self.owned:
                self._sync(self.cstream(g), self.xstream(g))
            if self.prog.stepwise:
                with _nvtx(f"step {s} leaves"):
                    self.compute(self.prog.work[s], s)
            self.release(s)

    def _inboxes(self) -> dict:
        """{task coord: peer.Inbox} of the write-backs that go through peer
        memory (leaf epilogue stores into the home GPU, `peer.py`)."""
        if not (peer.PEER_REDUCE and self.W.multi_gpu) or not self.prog.commits:
            return {}
        task_loops, _ = _loops_of(self.plan.task_body)
        _, plugins = _leaf_choice(self.plan.relations, [v for v, _, _ in task_loops], self.policy)
        if plugins:             # user leaf kernels are handed PyTorch tensors
            return {}
        return peer.inbox_set(self.prog, self.W, self.gpu).by_task()

    def _shifts(self) -> dict:
        """{id(Transfer): peer.Inbox} of the transfers that go by copy engine
        into a persistent buffer on the receiving GPU (`peer.CE_SHIFTS`)."""
        if not (self.W.multi_gpu and self.prog.stepwise) or not peer._shifts_apply(self.W):
            return {}
        task_loops, _ = _loops_of(self.plan.task_body)
        _, plugins = _leaf_choice(self.plan.relations, [v for v, _, _ in task_loops], self.policy)
        if plugins:             # user leaf kernels are handed PyTorch tensors
            return {}
        return peer.inbox_set(self.prog, self.W, self.gpu).by_transfer()

    def _shift_credits(self) -> None:
        """End of launch: every receiver has read its shift buffers (its
        compute stream is done) -- an 8-byte NCCL credit per shift lets the
        sender's next copy (stream-ordered after it on the sender's
        communication stream) overwrite the buffer."""
        if not self.shift:
            return
        for g in self.owned:
            self._sync(self.xstream(g), self.cstream(g))
        sends, recvs = [], []
        for ib in self.shift.values():
            if self.W.owns(ib.home_gpu):
                sends.append((ib.home_gpu, ib.writer_gpu, self._token(ib.home_gpu)))
            if self.W.owns(ib.writer_gpu):
                recvs.append((ib.writer_gpu, ib.home_gpu, self._token(ib.writer_gpu)))
        self._nccl(sends, recvs)

    def _local_only(self) -> bool:
        """No transfer or commit crosses GPUs (e.g. every single-GPU run)."""
        if not self.prog.stepwise:
            return False
        for moves in self.prog.transfers:
            for t in moves:
                if self.gpu(t.src) != self.gpu(t.dst):
                    return False
        return all(self.gpu(c.task.coord) == self.gpu(c.home) for c in self.prog.commits)

    def _early_outputs(self) -> bool:
        """Does a caller consume output pieces as they finish (e2e: inputs
        still uploading, rows streamed out)?  Then GPU-local programs run
        task-major; otherwise step-major, where one step's leaves of all the
        co-located tasks go out as grouped launches."""
        st = self.store
        return bool(st.ready or st.pending or st.stream_rows >= 2)

    def _run_task_major(self, region):
        """Task-major order for GPU-local programs: each task runs all its
        steps and commits before the next task starts.  Every transfer is an
        HBM alias, each task's step order and the task-order commits are
        unchanged, so results are identical to the step-major order -- but a
        task's output pieces are final early, and `store.done` events let a
        caller start their download while later tasks still compute."""
        for s, moves in enumerate(self.prog.transfers):
            self.transfers(moves)
        by_task = {}
        for s, works in enumerate(self.prog.work):
            for w in works:
                by_task.setdefault(w.task.coord, []).append((s, w))
        commits = {}
        for c in self.prog.commits:
            commits.setdefault(c.task.coord, []).append(c)
        for task in self.plan.tasks:
            for s, w in by_task.get(task.coord, []):
                self.compute([w], s)
            self._fill_unwritten([task.coord])
            mine = commits.get(task.coord, [])
            self._apply_commits(region, [(c, None) for c in mine])
            self._mark_done(region, mine, upto=task.coord)

    def _mark_done(self, region, commits, upto=None):
        """Record, per output piece, an event after its last commit (eager
        runs only: replayed plans clear `store.done` for their output)."""
        if _native.recorder() is not None:
            return
        last = {}
        for c in self.prog.commits:
            last[(self.gpu(c.home), c.color)] = c.task.coord
        for c in commits:
            key = (self.gpu(c.home), c.color)
            if not self.W.owns(key[0]) or (upto is not None and last[key] != upto):
                continue
            ev = self.torch.cuda.Event()
            ev.record(self.cstream(key[0]))
            self.store.done[(self.plan.out_name,) + key] = ev

    def _apply_commits(self, region, items):
        """Apply (commit, staged buffer or None) in order on the home GPUs."""
        acc = self.plan.out_kind == "reduce"
        for c, staged in items:
            gh = self.gpu(c.home)
            if not self.W.owns(gh) or c.task.coord in self.direct:
                continue
            piece = region.piece(gh, c.color)
            dst = _slice(piece, region.dist.piece_bounds(c.color), c.part)
            src = staged if staged is not None else _slice(self.out_bufs[c.task.coord], c.task.out_rect,
                                                           c.part)
            _copy_box(self.cstream(gh), dst, src, accumulate=acc)

    def _direct_commits(self, region) -> dict:
        """Tasks whose leaves may write straight into their home piece.

        Valid when the output region is a fresh +0.0 region, the task's only
        commit targets a piece on its own GPU whose box is exactly the task's
        output box, no other task commits into that piece, and the statement
        does not read its own output.  Then "leaf into a zero buffer, then
        canon (+)= buffer" and "leaf into canon" produce the same bits (the
        reference's commit, `simulator.py:624-634`, adds to +0.0 exactly)."""
        if not region.zeroed:
            return {}
        rhs = {a.tensor.name for leaf in leaf_statements(self.plan.task_body)
               for a in accesses_of(leaf.rhs)}
        if self.plan.out_name in rhs:
            return {}
        by_task, first = {}, {}
        for c in self.prog.commits:
            by_task.setdefault(c.task.coord, []).append(c)
            first.setdefault((self.gpu(c.home), c.color), c)
        out = {}
        for t in self.plan.tasks:
            cs = by_task.get(t.coord, [])
            if len(cs) != 1 or t.out_rect is None:
                continue
            c = cs[0]
            g = self.gpu(t.coord)
            # the first committer of a zeroed piece may write it in place: later
            # reductions (Johnson's depth partials) still add in task order
            if (self.gpu(c.home) == g and self.W.owns(g) and first[(g, c.color)] is c
                    and c.part == t.out_rect == region.dist.piece_bounds(c.color)
                    and (g, c.color) in region.pieces):
                out[t.coord] = c.color
        return out

    def transfers(self, moves):
        """One NCCL group per relay wave (planner.Transfer.wave): a temp
        forwarded in the step it arrives is sent only after its receive, by
        stream order on the communication stream."""
        for wave in sorted({t.wave for t in moves}):
            self._transfer_group([t for t in moves if t.wave == wave])

    def _send_view(self, gs, t, part=None):
        """Contiguous device view of a transfer's part (or a sub-box of it) on its source GPU."""
        torch = self.torch
        part = t.part if part is None else part
        src_h = self.prog.holdings[t.src_hid]
        self.wait_piece(self.xstream(gs), t.src_hid, part)
        view = _slice(self.holding_buf(t.src_hid), src_h.rect, part)
        if not view.is_contiguous():
            st = self.xstream(gs)
            packed = device_buffer(part.shape, view.device, st)
            _copy_box(st, packed, view)
            view = packed
        return view

    def _recv_buf(self, gd, part):
        buf = device_buffer(part.shape, self.W.device(gd), self.xstream(gd))
        buf.record_stream(self.cstream(gd))
        return buf

    def _transfer_group(self, moves):
        """One NCCL group: same-GPU moves become aliases; a box sent from one
        holding to >= 2 other GPUs (SUMMA / COSMA panel fan-out, Johnson face
        broadcast at g > 2) becomes one ncclBroadcast over the sub-communicator
        of those GPUs; everything else is an ncclSend/ncclRecv pair (Cannon's
        cyclic shifts, relays, single-destination fetches)."""
        fan = {}
        for t in moves:
            gs, gd = self.gpu(t.src), self.gpu(t.dst)
            if gs != gd:
                fan.setdefault((gs, t.src_hid, t.part), []).append(t)
        bkeys = [k for k, ms in fan.items() if len({self.gpu(m.dst) for m in ms}) >= 2] \
            if self.use_bcast else []
        for k in bkeys:     # sub-communicators first: collective over every rank, same order
            self.W.group_comm({k[0]} | {self.gpu(m.dst) for m in fan[k]})
        bset = set(bkeys)
        sends, recvs, bcasts = [], [], []
        for t in moves:
            gs, gd = self.gpu(t.src), self.gpu(t.dst)
            if gs == gd:
                if self.W.owns(gs):
                    src_h = self.prog.holdings[t.src_hid]
                    self.buffers[t.dst_hid] = _slice(self.holding_buf(t.src_hid), src_h.rect, t.part)
                    o = self.origin(t.src_hid)
                    if o is not None:
                        self.alias_origin[t.dst_hid] = o
                continue
            if (gs, t.src_hid, t.part) in bset:
                continue
            ib = self.shift.get(id(t)) if self.shift else None
            if ib is not None:
                # copy engine into the receiver's buffer, then an 8-byte token in the group
                if self.W.owns(gs):
                    view = self._send_view(gs, t)
                    n = max(1, view.numel())
                    _native.call("td_memcpy_2d", stream_handle(self.xstream(gs)), C.c_void_p(ib.writer_ptr), n,
                                 C.c_void_p(view.data_ptr()), n, n, 1)
                    sends.append((gs, gd, self._token(gs)))
                if self.W.owns(gd):
                    self.buffers[t.dst_hid] = ib.home_view()
                    recvs.append((gd, gs, self._token(gd)))
                continue
            if self.W.owns(gs):
                sends.append((gs, gd, self._send_view(gs, t)))
            if self.W.owns(gd):
                buf = self._recv_buf(gd, t.part)
                self.buffers[t.dst_hid] = buf
                recvs.append((gd, gs, buf))
        for k in bkeys:
            gs, _, part = k
            dsts = sorted({self.gpu(m.dst) for m in fan[k]})
            members = tuple(sorted({gs, *dsts}))
            comms = self.W.group_comm(members)
            root = members.index(gs)
            if self.W.owns(gs):
                bcasts.append((comms[gs], gs, self._send_view(gs, fan[k][0]), root))
            for gd in dsts:
                if not self.W.owns(gd):
                    continue
                buf = self._recv_buf(gd, part)
                for m in fan[k]:
                    if self.gpu(m.dst) == gd:
                        self.buffers[m.dst_hid] = buf
                bcasts.append((comms[gd], gd, buf, root))
        self._nccl(sends, recvs, bcasts)

    def _nccl(self, sends, recvs, bcasts=()):
        if not sends and not recvs and not bcasts:
            return
        _native.call("td_group_start")
        try:
            for g, peer, view in sends:
                _native.call("td_send", self.W.comm(g), stream_handle(self.xstream(g)),
                             C.c_void_p(view.data_ptr()), max(1, view.numel()), peer)
            for g, peer, buf in recvs:
                _native.call("td_recv", self.W.comm(g), stream_handle(self.xstream(g)),
                             C.c_void_p(buf.data_ptr()), max(1, buf.numel()), peer)
            for comm, g, buf, root in bcasts:
                _native.call("td_bcast", C.c_void_p(comm), stream_handle(self.xstream(g)),
                             C.c_void_p(buf.data_ptr()), max(1, buf.numel()), root)
        finally:
            _native.call("td_group_end")

    def operand(self, g, name, rect, hids):
        """A CUDA view holding `rect` of tensor `name` on GPU g."""
        torch = self.torch
        st = self.cstream(g)
        for hid in hids:
            self.wait_piece(st, hid, rect)
        if len(hids) == 1 and self.prog.holdings[hids[0]].rect.contains(rect):
            h = self.prog.holdings[hids[0]]
            return _slice(self.holding_buf(hids[0]), h.rect, rect)
        buf = device_buffer(rect.shape, self.W.device(g), st, zero=True)
        for hid in hids:
            h = self.prog.holdings[hid]
            part = h.rect.intersect(rect) if rect.lo else rect
            if part is None:
                continue
            _copy_box(st, _slice(buf, rect, part), _slice(self.holding_buf(hid), h.rect, part))
        return buf

    # ---- pipelined first step
    def _work_loops(self, w, s, task_loops):
        plan = self.plan
        loops = [(v, c, c + 1) for v, c in w.task.env.items()]
        for v, lo, hi in task_loops:
            if s >= 0 and plan.step_var is not None and v == plan.step_var.var:
                lo, hi = s, s + 1
            loops.append((v, lo, hi))
        return loops

    def _split_plan(self, s):
        """{"kv", "axis": {tensor: axis}} when step s may run pipelined, else None.

        Decided from the program alone (identical on every rank: it shapes the
        NCCL groups): every leaf of the step is a native GEMM over its whole
        iteration box, every cross-GPU transfer is a single-destination p2p
        move of an operand along whose k axis the receiving task's box spans
        exactly the transferred range, and enough bytes move to matter."""
        if not (SPLIT_FIRST_STEP and self.W.multi_gpu):
            return None
        moves = self.prog.transfers[s]
        cross = [t for t in moves if self.gpu(t.src) != self.gpu(t.dst)]
        if not cross or any(t.wave for t in moves):
            return None
        if 8 * max(t.part.volume for t in cross) < SPLIT_MIN_BYTES:
            return None
        fan = {}
        for t in cross:
            fan.setdefault((self.gpu(t.src), t.src_hid, t.part), set()).add(self.gpu(t.dst))
        if self.use_bcast and any(len(d) >= 2 for d in fan.values()):
            return None
        plan = self.plan
        task_loops, leaf = _loops_of(plan.task_body)
        policy, plugins = _leaf_choice(plan.relations, [v for v, _, _ in task_loops], self.policy)
        if plugins:
            return None
        rhs = accesses_of(leaf.rhs)
        dst_of = {t.dst_hid: t for t in cross}
        kv, axis = None, {}
        for w in self.prog.work[s]:
            np_ = native_plan(policy, self._work_loops(w, s, task_loops), leaf, plan.defs)
            if np_ is None:
                return None
            m, box = np_
            k = contracted_var(m, leaf)
            if k is None or (kv is not None and k != kv):
                return None
            kv = k
            for a in rhs:
                if kv in a.var_names:
                    axis[a.tensor.name] = a.var_names.index(kv)
            for key, (name, rect, hids) in w.operands.items():
                fed = [h for h in hids if h in dst_of]
                if not fed:
                    continue
                if len(hids) != 1 or rect is None or name not in axis:
                    return None
                ax = axis[name]
                t = dst_of[hids[0]]
                if (rect.lo[ax], rect.hi[ax]) != box[kv] or (t.part.lo[ax], t.part.hi[ax]) != box[kv]:
                    return None
        if kv is None or any(t.tensor not in axis for t in cross):
            return None
        return {"kv": kv, "axis": axis}

    def transfers_split(self, moves, split):
        """Step-0 transfers in k-pieces: one NCCL group per piece, an event per
        owned GPU after each.  Column pieces of row-major tiles are packed on
        the sender and unpacked on the receiver by strided copies."""
        torch = self.torch
        cross = [t for t in moves if self.gpu(t.src) != self.gpu(t.dst)]
        self._transfer_group([t for t in moves if self.gpu(t.src) == self.gpu(t.dst)])   # aliases
        full = {}
        for t in cross:
            gd = self.gpu(t.dst)
            if self.W.owns(gd):
                full[t.dst_hid] = self.buffers[t.dst_hid] = self._recv_buf(gd, t.part)
        kp = self.store.first_step_pieces
        npieces = max(len(_k_cuts(t.part.lo[split["axis"][t.tensor]], t.part.hi[split["axis"][t.tensor]], kp))
                      for t in cross)
        events = {g: [] for g in self.owned}
        for c in range(npieces):
            sends, recvs, unpack = [], [], []
            for t in cross:
                ax = split["axis"][t.tensor]
                cuts = _k_cuts(t.part.lo[ax], t.part.hi[ax], kp)
                if c >= len(cuts):
                    continue
                sub = _with_range(t.part, ax, *cuts[c])
                gs, gd = self.gpu(t.src), self.gpu(t.dst)
                if self.W.owns(gs):
                    sends.append((gs, gd, self._send_view(gs, t, sub)))
                if self.W.owns(gd):
                    dst = _slice(full[t.dst_hid], t.part, sub)
                    if not dst.is_contiguous():
                        stage = device_buffer(sub.shape, self.W.device(gd), self.xstream(gd))
                        unpack.append((gd, dst, stage))
                        dst = stage
                    recvs.append((gd, gs, dst))
            self._nccl(sends, recvs)
            for gd, dst, stage in unpack:
                _copy_box(self.xstream(gd), dst, stage)
            for g in self.owned:
                events[g].append(self._mark(self.xstream(g)))
        return events

    def compute_split(self, works, s, split, events):
        """Step-0 GEMM leaves in the k-pieces of `transfers_split`: piece c
        waits only for the transfers of pieces <= c."""
        plan = self.plan
        task_loops, leaf = _loops_of(plan.task_body)
        policy, _ = _leaf_choice(plan.relations, [v for v, _, _ in task_loops], self.policy)
        kv = split["kv"]
        for w in works:
            g = self.gpu(w.task.coord)
            if not self.W.owns(g) or w.task.out_rect is None:
                continue
            st = self.cstream(g)
            self._after(st, events[g][0])
            acc = self._acc_of(w.task.coord)
            if any(rect is None for _, rect, _ in w.operands.values()):
                if not acc:   # an empty access: the partial is all zeros
                    _native.call("td_fill", stream_handle(st), C.c_void_p(self.out_bufs[w.task.coord].data_ptr()),
                                 self.out_bufs[w.task.coord].numel(), 0.0)
                continue
            self._run_k_pieces(w, s, g, st, acc, self._work_loops(w, s, task_loops), leaf, policy, kv,
                               events[g])

    def _run_k_pieces(self, w, s, g, st, acc, loops, leaf, policy, kv, events=None) -> None:
        """One native GEMM leaf in the k-pieces of `_k_cuts` (first_step_pieces):
        operand views are taken without waiting, and piece c waits only for the
        input slabs it touches (progressive placement) and, when `events` is
        given, for the transfers of pieces <= c."""
        plan = self.plan
        rhs = accesses_of(leaf.rhs)
        m, box = native_plan(policy, loops, leaf, plan.defs)
        out_tile = DeviceTile(plan.out_name, w.task.out_rect, self.out_bufs[w.task.coord],
                              plan.out_access.tensor.dims)
        kaxis = {a.tensor.name: a.var_names.index(kv) for a in rhs if kv in a.var_names}
        tiles, lazy = {}, []
        for key, (name, rect, hids) in w.operands.items():
            h = self.prog.holdings[hids[0]]
            if len(hids) == 1 and h.rect.contains(rect) and name in kaxis:
                # a view; input slabs still uploading are waited for piece by piece below
                buf = _slice(self.holding_buf(hids[0]), h.rect, rect)
                lazy.append((hids[0], rect, kaxis[name]))
            else:
                buf = self.operand(g, name, rect, hids)
            tiles[key] = DeviceTile(name, rect, buf, self.store[name].dims)
        ins = [tiles[(a.tensor.name, a.var_names)] for a in rhs]
        for c, (a, b) in enumerate(_k_cuts(*box[kv], self.store.first_step_pieces)):
            if c and events:
                self._after(st, events[min(c, len(events) - 1)])
            for hid, rect, ax in lazy:
                self.wait_piece(st, hid, _with_range(rect, ax, a, b))
            sub = dict(box)
            sub[kv] = (a, b)
            run_native_box(m, leaf, sub, out_tile, ins, st, acc if c == 0 else 1)
        for e in (events or [])[1:]:
            self._after(st, e)

    def compute(self, works, s):
        from .leaves import gemm_batch
        with gemm_batch() if not self._early_outputs() else _NoBatch():
            self._compute(works, s)

    def _compute(self, works, s):
        plan = self.plan
        task_loops, leaf = _loops_of(plan.task_body)
        loop_vars = [v for v, _, _ in task_loops]
        policy, plugins = _leaf_choice(plan.relations, loop_vars, self.policy)
        rhs = accesses_of(leaf.rhs)
        for w in works:
            g = self.gpu(w.task.coord)
            if not self.W.owns(g) or w.task.out_rect is None:
                continue
            st = self.cstream(g)
            acc = self._acc_of(w.task.coord)
            if any(rect is None for _, rect, _ in w.operands.values()):
                if not acc:   # some access is empty on this step: the partial is all zeros
                    _native.call("td_fill", stream_handle(st), C.c_void_p(self.out_bufs[w.task.coord].data_ptr()),
                                 self.out_bufs[w.task.coord].numel(), 0.0)
                continue      # no iteration points
            loops = [(v, c, c + 1) for v, c in w.task.env.items()]
            for v, lo, hi in task_loops:
                if s >= 0 and plan.step_var is not None and v == plan.step_var.var:
                    lo, hi = s, s + 1
                loops.append((v, lo, hi))
            if (not plugins and s == 0 and self.store.first_step_pieces > 2 and self.store.ready
                    and w.task.coord == self._first_task(g) and self._progressive_gemm(loops, leaf, policy)):
                # inputs still arriving in k-slabs (e2e): the GPU's first GEMM in k-pieces, each
                # waiting only for its own slabs
                self._run_k_pieces(w, s, g, st, acc, loops, leaf, policy,
                                   contracted_var(native_plan(policy, loops, leaf, plan.defs)[0], leaf))
                continue
            out_tile = DeviceTile(plan.out_name, w.task.out_rect, self.out_bufs[w.task.coord],
                                  plan.out_access.tensor.dims)
            tiles = {}
            for key, (name, rect, hids) in w.operands.items():
                tiles[key] = DeviceTile(name, rect, self.operand(g, name, rect, hids),
                                        self.store[name].dims)
            ins = [tiles[(a.tensor.name, a.var_names)] for a in rhs]
            if not plugins and acc and self._stream_rows(w, s, g, loops, leaf, policy, out_tile, ins, st):
                continue
            if plugins:
                read = {a.tensor.name: tiles[(a.tensor.name, a.var_names)] for a in rhs}
                flush_pending()
                execute_chain(loops[len(w.task.env):], leaf, dict(w.task.env), plan.defs, read,
                              {plan.out_name: out_tile}, plugins, st, self.W.device(g))
            else:
                run_leaf(policy, loops, leaf, plan.defs, out_tile, ins, st, accumulate=acc)

    def _first_task(self, g):
        for t in self.plan.tasks:
            if self.gpu(t.coord) == g and t.out_rect is not None:
                return t.coord
        return None

    def _progressive_gemm(self, loops, leaf, policy) -> bool:
        np_ = native_plan(policy, loops, leaf, self.plan.defs)
        return np_ is not None and contracted_var(np_[0], leaf) is not None

    def _stream_rows(self, w, s, g, loops, leaf, policy, out_tile, ins, st) -> bool:
        """Last step of a task that writes its home piece directly (and alone):
        run the native GEMM leaf in row pieces with an event after each
        (RegionStore.stream_rows / row_done).  False: not applicable."""
        n = self.store.stream_rows
        if n < 2 or s != self.plan.num_steps - 1 or w.task.coord not in self.direct:
            return False
        color = self.direct[w.task.coord]
        if sum(1 for c in self.prog.commits if self.gpu(c.home) == g and c.color == color) != 1:
            return False
        np_ = native_plan(policy, loops, leaf, self.plan.defs)
        if np_ is None or contracted_var(np_[0], leaf) is None:
            return False
        m, box = np_
        rv = leaf.lhs.var_names[0]
        lo, hi = box[rv]
        step = -(-max(1, (hi - lo) // n) // 64) * 64
        if hi - lo < 2 * step:
            return False
        key = (self.plan.out_name, g, color)
        base = out_tile.rect.lo[0]
        marks = []
        for a in range(lo, hi, step):
            b = min(hi, a + step)
            sub = dict(box)
            sub[rv] = (a, b)
            run_native_box(m, leaf, sub, out_tile, ins, st, 1)
            ev = self.torch.cuda.Event()
            ev.record(st)
            marks.append((a - base, b - base, ev))
        self.store.row_done[key] = marks
        return True

    def release(self, s):
        for hid, last in self.prog.last_use.items():
            if last == s:
                self.buffers.pop(hid, None)

    def commit(self, region):
        torch = self.torch
        plan = self.plan
        # senders must see finished leaves
        for g in self.owned:
            self._sync(self.xstream(g), self.cstream(g))
        sends, recvs, staged = [], [], {}
        tokens = []           # (inbox, writer token, home token) of peer-memory write-backs
        for k, c in enumerate(self.prog.commits):
            gt, gh = self.gpu(c.task.coord), self.gpu(c.home)
            if gt == gh:
                continue
            ib = self.inbox.get(c.task.coord)
            if ib is not None:
                # the partial is already in the home's inbox: an 8-byte token orders
                # the home's accumulation after the writer's leaf
                tw = self._token(gt) if self.W.owns(gt) else None
                th = self._token(gh) if self.W.owns(gh) else None
                if tw is not None:
                    sends.append((gt, gh, tw))
                if th is not None:
                    recvs.append((gh, gt, th))
                    staged[k] = ib.home_view()
                tokens.append((ib, tw, th))
                continue
            if self.W.owns(gt):
                self.out_bufs[c.task.coord].record_stream(self.xstream(gt))
                view = _slice(self.out_bufs[c.task.coord], c.task.out_rect, c.part)
                if not view.is_contiguous():
                    st = self.xstream(gt)
                    packed = device_buffer(c.part.shape, view.device, st)
                    _copy_box(st, packed, view)
                    view = packed
                sends.append((gt, gh, view))
            if self.W.owns(gh):
                buf = device_buffer(c.part.shape, self.W.device(gh), self.xstream(gh))
                buf.record_stream(self.cstream(gh))
                staged[k] = buf
                recvs.append((gh, gt, buf))
        self._nccl(sends, recvs)
        for g in self.owned:
            self._sync(self.cstream(g), self.xstream(g))
        self._apply_commits(region, [(c, staged.get(k)) for k, c in enumerate(self.prog.commits)])
        if tokens:
            # credit: the home has read its inboxes; the writers' next leaves may overwrite them
            for g in self.owned:
                self._sync(self.xstream(g), self.cstream(g))
            sends, recvs = [], []
            for ib, tw, th in tokens:
                if th is not None:
                    sends.append((ib.home_gpu, ib.writer_gpu, th))
                if tw is not None:
                    recvs.append((ib.writer_gpu, ib.home_gpu, tw))
            self._nccl(sends, recvs)
            for ib, tw, th in tokens:
                if tw is not None and not _CAPTURING:
                    h = self.credits.get(id(ib))
                    if h is not None:       # recording: the plan's own credit event
                        _native.call("td_event_record", C.c_void_p(h), stream_handle(self.xstream(ib.writer_gpu)),
                                     g_index(self.W, ib.writer_gpu))
                        ib.credit = _NativeEvent(h)
                    else:
                        ev = self.torch.cuda.Event()
                        ev.record(self.xstream(ib.writer_gpu))
                        ib.credit = ev

    def _token(self, g):
        return device_buffer((1,), self.W.device(g), self.xstream(g))


_PLAN_CACHE: dict = {}


def _plan_cached(stmt, store, trace, record_requirements):
    """build_program, memoised per (statement object, store layout): repeated
    executes of one scheduled statement on one store (benchmark steps,
    iterative solvers) skip the Python planning and replay its ledger."""
    # the program depends on the distributions and residency only, not on the
    # store object or its values: key on those so fresh stores (e2e steps) hit
    from .machine import placement
    layout = (store.machine, store.world.ngpus, placement(),
              tuple((n, r.dist, tuple(len(v) for v in r.residency.values()))
                    for n, r in sorted(store.regions.items())))
    cache = _PLAN_CACHE
    key = (id(stmt), bool(record_requirements))
    hit = cache.get(key)
    if hit is not None and hit[0] is stmt and hit[1] == layout:
        _, _, prog, events, reqs, memory = hit
        trace.events.extend(events)
        trace.requirements.extend(reqs)
        for p, v in memory.items():
            trace.bump_memory(p, v)
        return prog
    scratch = ExecutionTrace(store.machine)
    prog = build_program(stmt, store, scratch, record_requirements=record_requirements)
    trace.events.extend(scratch.events)
    trace.requirements.extend(scratch.requirements)
    for p, v in scratch.memory.items():
        trace.bump_memory(p, v)
    if len(cache) > 256:
        cache.clear()
    cache[key] = (stmt, layout, prog, list(scratch.events), list(scratch.requirements), dict(scratch.memory))
    return prog


# roofline denominators of `execute(timed=True)` (bench.py uses the same figures):
# the FP64 DMMA peak measured on this pool's B200s (profiles/peaks_r01.json) and
# the copy bandwidth of MEASURED_PEAKS.json
FP64_PEAK_GFLOPS = 37070.0
HBM_PEAK_GBS = 6544.3


def _algorithmic_work(plan):
    """(flop, bytes) of one launch of the statement: every iteration point of
    the leaf does (#factors - 1) multiplications (+1 addition for a Reduce);
    bytes = each distinct tensor read or written once."""
    leaf = leaf_statements(plan.task_body)[0]
    accs = [leaf.lhs, *accesses_of(leaf.rhs)]
    ext = {}
    for a in accs:
        for v, d in zip(a.var_names, a.tensor.dims):
            ext[v] = d
    points = 1
    for d in ext.values():
        points *= d
    nf = len(accesses_of(leaf.rhs))
    flop = float(points) * (nf - 1 + (1 if plan.out_kind == "reduce" else 0))
    vols = {}
    for a in accs:
        vol = 1
        for d in a.tensor.dims:
            vol *= d
        vols[a.tensor.name] = vol
    return flop, 8.0 * sum(vols.values())


def execute(stmt, store: RegionStore, *, trace: ExecutionTrace = None, workers: int = 1,
            label: str = None, record_requirements: bool = True, leaf_policy: str = "auto",
            timed: bool = False):
    """Run one scheduled statement on the GPUs (reference `simulator.py:537-663`).

    `workers` is accepted for signature compatibility and has no effect: the
    reference's thread pool over tasks (`simulator.py:617-620`) is replaced by
    the GPUs themselves, and results do not depend on it (as in the
    reference).  `leaf_policy` is ``"auto"`` (native contractions where they
    apply) or ``"exact"`` (the nest kernel everywhere: bitwise identical to
    the reference on any input).  `timed=True` brackets the launch with CUDA
    events on every owned GPU, waits for it, and appends a record to
    `trace.timings` (device ms, max over GPUs and ranks; algorithmic flop /
    bytes; rate vs the FP64 or HBM roof), which `trace.stats()` reports under
    "measured".  Collective under SPMD, like execute itself."""
    if leaf_policy not in LEAF_POLICIES:
        raise ConfigError(f"leaf_policy must be one of {LEAF_POLICIES}")
    if trace is None:
        trace = ExecutionTrace(store.machine)
    prog = _plan_cached(stmt, store, trace, record_requirements)
    W = store.world
    marks = None
    if timed:
        torch = torch_mod()
        marks = {}
        for g in W.owned:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(W.device(g)))
            marks[g] = ev
    _launch(prog, store, leaf_policy)
    plan = prog.plan
    if marks is not None:
        ms = 0.0
        for g, ev in marks.items():
            end = torch.cuda.Event(enable_timing=True)
            end.record(torch.cuda.current_stream(W.device(g)))
            if W.multi_gpu:
                W.wait()
            end.synchronize()
            ms = max(ms, ev.elapsed_time(end))
        if W.nprocs > 1:
            ms = max(W.all_gather_object(ms))
        flop, nbytes = _algorithmic_work(plan)
        tensor_bound = nbytes == 0 or flop / nbytes > FP64_PEAK_GFLOPS / HBM_PEAK_GBS
        trace.record_timing(label or plan.out_name, ms, flops=flop, nbytes=nbytes,
                            bound="tensor" if tensor_bound else "hbm",
                            peak=FP64_PEAK_GFLOPS if tensor_bound else HBM_PEAK_GBS, gpus=W.ngpus)
    out_region = store[plan.out_name]
    out_region.zeroed = False
    if plan.out_kind == "reduce" and out_region.dist.replicated:
        for color in out_region.dist.colors():
            procs = out_region.dist.processors_of(color)
            bounds = out_region.dist.piece_bounds(color)
            for q in procs[1:]:
                out_region.residency[q] = [r for r in out_region.residency.get(q, []) if r != bounds]
        keep = {(g, c) for (g, c) in out_region.pieces if g in out_region.gpus_of(c)}
        out_region.pieces = {k: v for k, v in out_region.pieces.items() if k in keep}
    trace.num_steps = max(trace.num_steps, plan.num_steps)
    trace.launches.append({"phase": "compute", "label": label or plan.out_name,
                           "tasks": len(plan.tasks), "steps": plan.num_steps})
    return trace


_CAPTURING = False      # inside CapturedLaunch's capture: no cross-launch events

# ---------------------------------------------------------------- launch plans
# Repeated launches of one program on one store (benchmark steps, iterative
# solvers) replay a recorded plan: the second execute of a (program, store
# layout, streams) runs eagerly while `_native.recording` collects every
# native call it issues -- leaves, box copies, fills, NCCL groups, event
# edges -- with their device pointers; from the third on, `td_execute_plan`
# issues that op array in one C++ call (csrc/plan.cu), so the per-step loop
# no longer runs in Python.  Temporaries of the recorded run stay allocated
# for the plan's lifetime.  Not recorded: Python leaf plugins, progressive
# uploads / row streaming (e2e hooks that hand events to the caller), leaf
# timing, CUDA-graph capture.
PLANS = True
PLAN_MAX_BYTES_PER_GPU = 24 << 30
PLANS_PER_STORE = 8


def _plannable(prog, store, policy) -> bool:
    from . import leaves as _leaves
    if not PLANS or _CAPTURING or _leaves.TIMING is not None or _native.recorder() is not None:
        return False
    if store.ready or store.pending or store.stream_rows >= 2:
        return False
    task_loops, _ = _loops_of(prog.plan.task_body)
    _, plugins = _leaf_choice(prog.plan.relations, [v for v, _, _ in task_loops], policy)
    return not plugins


def _plan_key(prog, store, policy):
    torch = torch_mod()
    W = store.world
    out = store[prog.plan.out_name]
    pieces = tuple((n, tuple((k, b.data_ptr()) for k, b in r.pieces.items())) for n, r in store.regions.items())
    streams = tuple(torch.cuda.current_stream(W.device(g)).cuda_stream for g in W.owned)
    pending = tuple(bool(r.pending_zero) for r in store.regions.values())
    return (id(prog), policy, out.zeroed, pending, pieces, streams)


def _launch(prog, store, policy) -> None:
    """Run one launch: eagerly, recording a plan, or replaying one."""
    if not _plannable(prog, store, policy):
        _Executor(prog, store, policy).run()
        return
    cache = store.__dict__.setdefault("_launch_plans", {})
    key = _plan_key(prog, store, policy)
    hit = cache.get(key)
    if isinstance(hit, tuple) and hit[0] is prog:
        _replay(hit[1], prog, store)
        return
    if hit != "seen":
        if hit is None:
            cache[key] = "seen"
        _Executor(prog, store, policy).run()
        return
    with _native.recording() as rec:
        ex = _Executor(prog, store, policy)
        ex.run()
    per_gpu = {}
    for t in rec.keep:
        if hasattr(t, "data_ptr") and t.is_cuda:
            per_gpu[t.device.index] = per_gpu.get(t.device.index, 0) + t.numel() * 8
    if not rec.valid or max(per_gpu.values(), default=0) > PLAN_MAX_BYTES_PER_GPU:
        cache[key] = "never"
        return
    plan = rec.finish()
    sets = [] if not (ex.inbox or ex.shift) else [peer.inbox_set(prog, store.world, ex.gpu)]
    plan.extra["credits"] = [(ib, h) for ib in ex.inbox.values() for i, h in ex.credits.items() if i == id(ib)]
    plan.extra["inbox_sets"] = sets
    for st in sets:
        st.pin()
        weakref.finalize(plan, st.unpin)
    while len(cache) >= PLANS_PER_STORE:
        cache.pop(next(iter(cache)))
    cache[key] = (prog, plan)


def _replay(plan, prog, store) -> None:
    W = store.world
    for ib, h in plan.extra["credits"]:
        # an eager launch in between left a torch credit event the plan does not know
        if ib.credit is not None and not isinstance(ib.credit, _NativeEvent):
            W.streams(ib.writer_gpu)[0].wait_event(ib.credit)
    plan.run()
    for region in store.regions.values():    # the plan's fills / overwrites resolved them, as when recorded
        region.pending_zero = set()
    for ib, h in plan.extra["credits"]:
        ib.credit = _NativeEvent(h)
    out = prog.plan.out_name
    store.done = {k: v for k, v in store.done.items() if k[0] != out}
    store.row_done = {k: v for k, v in store.row_done.items() if k[0] != out}


class CapturedLaunch:
    """One `execute` of a scheduled statement on a store, captured once into a
    CUDA graph and replayed: every leaf, copy, NCCL send / receive /
    broadcast, event fork/join and stream-ordered allocation of the launch
    becomes one `graph.replay()`, removing the host issue cost that dominates
    small launches (SUMMA 1024^3 on 2x2: 8 steps x 4 tasks) -- the step loop
    no longer runs in Python.  Inputs are read in place, so refresh them
    between replays by writing into their pieces; with ``reset_output`` the
    output pieces are zeroed inside the graph (a fresh run_statement
    output).  Jobs on one GPU, or SPMD jobs with one GPU per process
    (`configure_distributed`): every rank captures its own GPU's part of the
    same program, so the captured NCCL calls pair up at every replay; replays
    must then be issued by every rank, like `execute`.  Replays on one stream
    are ordered, so the peer-inbox credit (`peer.py`) needs no event across
    replays."""

    def __init__(self, stmt, store: RegionStore, *, leaf_policy: str = "auto", reset_output: bool = True):
        global _CAPTURING
        torch = torch_mod()
        W = store.world
        if W.ngpus > 1 and not (W.nprocs == W.ngpus and len(W.owned) == 1):
            raise ConfigError("CapturedLaunch supports one-GPU jobs and SPMD jobs with one GPU per process")
        self.stmt, self.store = stmt, store
        plan_trace = ExecutionTrace(store.machine)
        prog = _plan_cached(stmt, store, plan_trace, False)
        self.out = prog.plan.out_name
        # warm-up outside the capture: plan cache, kernel attributes, pools
        if reset_output:
            store.zero(self.out)
        execute(stmt, store, record_requirements=False, leaf_policy=leaf_policy)
        torch.cuda.synchronize()
        self.trace = plan_trace
        if not _touches_owned(prog, store):
            # this rank's GPUs hold no task, transfer or commit of the program: nothing
            # to capture (an empty graph); replay() is a no-op here
            self.graph = None
            return
        self.graph = torch.cuda.CUDAGraph()
        _CAPTURING = True
        try:
            with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                if reset_output:
                    for buf in store[self.out].pieces.values():
                        buf.zero_()
                    store[self.out].pending_zero = set()
                store[self.out].zeroed = reset_output
                execute(stmt, store, record_requirements=False, leaf_policy=leaf_policy)
        finally:
            _CAPTURING = False
        self.trace = plan_trace
        # the graph holds raw peer-inbox pointers: keep their InboxSet alive
        # (not evicted by later programs) for the graph's lifetime
        iset = W.inbox_sets.get(id(prog)) if hasattr(W, "inbox_sets") else None
        if iset is not None and iset.prog is prog and getattr(iset, "inboxes", None):
            iset.pin()
            weakref.finalize(self, iset.unpin)

    def replay(self) -> None:
        if self.graph is not None:
            self.graph.replay()


def _touches_owned(prog, store) -> bool:
    """Does any task, transfer or commit of the program run on this process's GPUs?"""
    W, m = store.world, store.machine

    def mine(p):
        return W.owns(m.device_of(p, W.ngpus))
    if any(mine(t.coord) for t in prog.plan.tasks if t.out_rect is not None):
        return True
    if any(mine(t.src) or mine(t.dst) for moves in prog.transfers for t in moves):
        return True
    return any(mine(c.home) or mine(c.task.coord) for c in prog.commits)


@dataclass
class RunResult:
    output_name: str
    trace: ExecutionTrace
    store: RegionStore
    _output: DenseTensor = None

    @property
    def output(self) -> DenseTensor:
        """The output on the host (collective under SPMD: see RegionStore.gather)."""
        if self._output is None:
            self._output = self.store.gather(self.output_name)
        return self._output


def _scheduled(stmt, schedule):
    cin = lower_to_cin(stmt) if isinstance(stmt, TensorIndexStmt) else stmt
    return schedule.apply(cin) if schedule is not None else cin


def prepare_store(cin, machine, distributions, inputs=None, *, world=None, generated=None):
    """Place inputs (host tensors, or synthetic `generated={name: (seed, id, mode)}`)
    and a zero output; validation follows reference `simulator.py:691-711`."""
    leaves = leaf_statements(cin)
    out_name = leaves[0].lhs.tensor.name
    dims = {}
    for leaf in leaves:
        for acc in leaf_accesses(leaf):
            dims[acc.tensor.name] = acc.tensor.dims
    store = RegionStore(machine, world)
    for name in sorted(dims):
        if name not in distributions:
            raise MissingDistribution(f"no distribution for {name}")
        if name == out_name:
            continue
        if generated is not None and name in generated:
            seed, tid, mode = generated[name]
            store.place_generated(name, distributions[name], seed=seed, tensor_id=tid, mode=mode)
            continue
        if inputs is None or name not in inputs:
            raise MissingInput(f"no input tensor for {name}")
        if inputs[name].dims != dims[name]:
            raise ExtentMismatch(f"{name}: statement wants dims {dims[name]}, input has {inputs[name].dims}")
        store.place(name, inputs[name], distributions[name])
    store.place_zeros(out_name, distributions[out_name])
    return store, out_name


def run_statement(stmt, machine: Machine, distributions: dict, inputs: dict, schedule=None, *,
                  workers: int = 1, label: str = None, leaf_policy: str = "auto",
                  timed: bool = False) -> RunResult:
    """Place inputs in HBM, apply the schedule, execute, return the output
    (reference `simulator.py:676-715`).  `timed`: see `execute`."""
    cin = _scheduled(stmt, schedule)
    store, out_name = prepare_store(cin, machine, distributions, inputs)
    trace = ExecutionTrace(machine)
    execute(cin, store, trace=trace, workers=workers, label=label, leaf_policy=leaf_policy, timed=timed)
    return RunResult(out_name, trace, store)


def verify_result(stmt, inputs: dict, result: RunResult, atol: float = 1e-9) -> None:
    """Compare a run with the single-memory evaluation (reference `simulator.py:718-726`);
    the reference evaluation itself runs on the GPU's exact-order nest kernel."""
    from .ir import sequential_evaluate
    expected = sequential_evaluate(stmt, inputs)
    got = result.output
    if expected.dims != got.dims:
        raise VerifyFail(f"output dims {got.dims} != reference {expected.dims}")
    err = float(np.max(np.abs(expected.data - got.data))) if expected.volume else 0.0
    if err > atol:
        raise VerifyFail(f"max deviation {err} above {atol}")


def redistribute(store: RegionStore, name: str, new_dist: TensorDistribution,
                 trace: ExecutionTrace) -> None:
    """Move a region to a new distribution (reference `simulator.py:317-357`):
    every piece a processor must newly hold is fetched from the
    lowest-enumeration other holder, as placement-phase events; the data
    moves over NCCL (or stays in place on a shared GPU)."""
    torch = torch_mod()
    region = store.regions[name]
    region.materialize()
    check_redistributable(region.dist, new_dist)
    old = region.residency
    new = new_dist.residency()
    old_colors = [(region.dist.piece_bounds(c), region.dist.processors_of(c), c)
                  for c in region.dist.colors()]
    moved = 0
    fetched = {p: 0 for p in store.machine.enumerate()}
    moves = []   # (src proc, dst proc, part, old color)
    for p in store.machine.enumerate():
        for rect in new.get(p, []):
            for piece in subtract_rects([rect], old.get(p, [])):
                for bounds, procs, color in old_colors:
                    part = piece.intersect(bounds)
                    if part is None:
                        continue
                    src = next((q for q in procs if q != p), None)
                    if src is None:
                        continue
                    trace.events.append(CommEvent(0, src, p, name, part, part.volume, "copy", "placement"))
                    moves.append((src, p, part, color))
                    moved += part.volume
                    fetched[p] += part.volume
    for p in store.machine.enumerate():
        trace.bump_memory(p, store.persistent_volume(p) + fetched[p])
    # data: build the new pieces from old pieces (local copies) and NCCL moves
    W = store.world
    for g in W.owned:   # pieces may still be landing on the store's compute stream (place_host)
        torch.cuda.current_stream(W.device(g)).wait_stream(W.streams(g)[0])
    old_region = region
    new_region = Region(store, name, new_dist)
    sends, recvs = [], []
    for color, box, _ in new_dist.pieces():
        for g in new_region.gpus_of(color):
            if not W.owns(g):
                continue
            dev = W.device(g)
            buf = torch.zeros(box.shape, dtype=torch.float64, device=dev)
            new_region.pieces[(g, color)] = buf
            st = torch.cuda.current_stream(dev)
            for ocolor, obox, oprocs in region.dist.pieces():
                part = box.intersect(obox) if box.lo else box
                if part is None:
                    continue
                og = [x for x in old_region.gpus_of(ocolor)]
                if g in og:
                    _copy_box(st, _slice(buf, box, part),
                              _slice(old_region.piece(g, ocolor), obox, part))
                else:
                    src_g = og[0]
                    staging = torch.empty(part.shape, dtype=torch.float64, device=dev)
                    recvs.append((g, src_g, staging, buf, box, part))
    for color, box, _ in new_dist.pieces():
        for g in new_region.gpus_of(color):
            for ocolor, obox, oprocs in region.dist.pieces():
                part = box.intersect(obox) if box.lo else box
                if part is None:
                    continue
                og = old_region.gpus_of(ocolor)
                if g in og or not W.owns(og[0]):
                    continue
                view = _slice(old_region.piece(og[0], ocolor), obox, part).contiguous()
                sends.append((og[0], g, view))
    if sends or recvs:
        _native.call("td_group_start")
        for g, peer, view in sends:
            _native.call("td_send", W.comm(g), stream_handle(torch.cuda.current_stream(W.device(g))),
                         C.c_void_p(view.data_ptr()), max(1, view.numel()), peer)
        for g, peer, staging, _, _, _ in recvs:
            _native.call("td_recv", W.comm(g), stream_handle(torch.cuda.current_stream(W.device(g))),
                         C.c_void_p(staging.data_ptr()), max(1, staging.numel()), peer)
        _native.call("td_group_end")
        for g, _, staging, buf, box, part in recvs:
            _copy_box(torch.cuda.current_stream(W.device(g)), _slice(buf, box, part), staging)
    region.dist = new_dist
    region.residency = new
    region.pieces = new_region.pieces
    trace.launches.append({"phase": "placement", "kind": "redistribute", "tensor": name,
                           "elements": moved, "to": new_dist.describe()})
