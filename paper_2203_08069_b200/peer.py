"""Peer-memory write-backs: a leaf stores its partial straight into the home GPU.

The reference's commit phase (`pkg/src/tendist/simulator.py:624-654`) adds
each task's partial output into the home piece in task order; tasks on other
processors ship the partial first (the `reduce` write-back events,
`simulator.py:635-645`).  On one NVSwitch box the shipping does not need to
follow the math: when a task's *whole* partial goes to one home piece on
another GPU (Johnson-3D's depth partials `algorithms.py:169-172`, COSMA's
k-split), the task's leaf writes it into an **inbox** in the home GPU's HBM
(`csrc/peer.cu`).  The DMMA GEMM epilogue then stores every finished tile
over NVLink while the remaining tiles still compute -- the GEMM and the
reduction's transfer are one kernel.  Ordering across GPUs is two 8-byte
NCCL messages per inbox and execute:

* *token* (writer -> home) after the leaf: the home's task-order
  accumulation (unchanged, so results are those of the NCCL path bit for
  bit) reads the inbox only after it;
* *credit* (home -> writer) after that accumulation: the writer's next leaf
  into the same inbox waits for it (no write-after-read race across
  executes).

Eligibility is decided from the program alone, identically on every rank:
the commit crosses GPUs, it is the task's only commit, it covers the task's
whole output box, and the task runs exactly one leaf (so the leaf can
*overwrite* the inbox instead of accumulating into zeros).

The same buffers carry **copy-engine shifts** in SPMD jobs: a big
single-destination transfer after step 0 (Cannon's per-step A / B shifts,
`algorithms.py:109-132`) is a `cudaMemcpy` by the sender straight into the
receiver's buffer over NVLink -- no NCCL kernel holding SM slots while the
DMMA waves run -- followed by an 8-byte NCCL token the receiver's step waits
for; an 8-byte credit at the end of the launch orders the next launch's copy
(stream-ordered behind it on the sender's communication stream) after the
receiver's reads.
"""

from __future__ import annotations

import ctypes as C
import os
import math
from collections import Counter

from . import _native

# leaves whose whole partial is reduced into another GPU's piece write it there
# directly (False: leaf into a local buffer, then an NCCL send; a measurement switch)
PEER_REDUCE = True
# big single-destination transfers after step 0 (Cannon's shifts) go GPU to GPU by
# copy engine into a persistent buffer on the receiver, ordered by 8-byte NCCL
# tokens: no SM slot is held while the DMMA waves run (SPMD jobs; False: NCCL
# send/recv, then serialised behind the leaves, runtime._serial_steps)
CE_SHIFTS = os.environ.get("TD_CE_SHIFTS", "1") != "0"
SHIFT_MIN_BYTES = 64 << 20

IPC_HANDLE_BYTES = 64


class RawView:
    """Strided float64 view of device memory the process does not own through
    PyTorch (a peer GPU's inbox).  Offers the slice of the tensor interface the
    leaves and commit copies use: shape, stride(), data_ptr(), basic slicing."""

    __slots__ = ("ptr", "shape", "_stride", "device")

    def __init__(self, ptr: int, shape, stride=None, device=None):
        self.ptr = int(ptr)
        self.shape = tuple(int(s) for s in shape)
        if stride is None:
            st, acc = [], 1
            for s in reversed(self.shape):
                st.append(acc)
                acc *= max(1, s)
            stride = tuple(reversed(st))
        self._stride = tuple(int(s) for s in stride)
        self.device = device

    def data_ptr(self) -> int:
        return self.ptr

    def stride(self) -> tuple:
        return self._stride

    def numel(self) -> int:
        return math.prod(self.shape)

    def dim(self) -> int:
        return len(self.shape)

    def is_contiguous(self) -> bool:
        acc = 1
        for s, st in zip(reversed(self.shape), reversed(self._stride)):
            if s != 1 and st != acc:
                return False
            acc *= s
        return True

    def record_stream(self, stream) -> None:   # lifetime is the inbox's, not the allocator's
        pass

    def __getitem__(self, idx):
        if not isinstance(idx, tuple):
            idx = (idx,)
        if len(idx) > len(self.shape):
            raise IndexError("too many indices for RawView")
        off, shape = 0, []
        for k, sl in enumerate(idx):
            if not isinstance(sl, slice) or sl.step not in (None, 1):
                raise TypeError("RawView supports unit-step slices only")
            lo, hi, _ = sl.indices(self.shape[k])
            hi = max(lo, hi)
            off += lo * self._stride[k]
            shape.append(hi - lo)
        shape.extend(self.shape[len(idx):])
        return RawView(self.ptr + 8 * off, shape, self._stride, self.device)

    def __repr__(self):
        return f"RawView(0x{self.ptr:x}, shape={self.shape}, stride={self._stride}, device={self.device})"


def eligible_commits(prog, gpu_of) -> dict:
    """{commit index: Commit} that may be written through a peer inbox."""
    works = Counter(w.task.coord for ws in prog.work for w in ws)
    commits = Counter(c.task.coord for c in prog.commits)
    out = {}
    for k, c in enumerate(prog.commits):
        t = c.task
        if gpu_of(t.coord) == gpu_of(c.home) or t.out_rect is None:
            continue
        if commits[t.coord] != 1 or works[t.coord] != 1 or c.part != t.out_rect:
            continue
        out[k] = c
    return out


def eligible_shifts(prog, gpu_of) -> dict:
    """{(step, index): Transfer} of the transfers that go by copy engine: after
    step 0 (step 0's are pipelined with its leaves), cross-GPU, not relayed,
    one destination GPU for their source box, >= SHIFT_MIN_BYTES."""
    out = {}
    for s, moves in enumerate(prog.transfers):
        if s == 0:
            continue
        dsts = {}
        for t in moves:
            gs, gd = gpu_of(t.src), gpu_of(t.dst)
            if gs != gd:
                dsts.setdefault((gs, t.src_hid, t.part), set()).add(gd)
        for i, t in enumerate(moves):
            gs, gd = gpu_of(t.src), gpu_of(t.dst)
            if gs == gd or t.wave != 0 or len(dsts[(gs, t.src_hid, t.part)]) != 1:
                continue
            if 8 * t.part.volume >= SHIFT_MIN_BYTES:
                out[(s, i)] = t
    return out


def _shifts_apply(world) -> bool:
    """Copy-engine shifts run in SPMD jobs (one GPU per process)."""
    return CE_SHIFTS and world.nprocs > 1 and world.nprocs == world.ngpus


class Inbox:
    """One write-back buffer in the home GPU's HBM, mapped on the writer GPU
    (a commit's partial, or -- `transfer` set -- a copy-engine shift's box)."""

    def __init__(self, commit, home_gpu, writer_gpu, shape, transfer=None):
        self.commit = commit
        self.transfer = transfer
        self.home_gpu = home_gpu
        self.writer_gpu = writer_gpu
        self.shape = tuple(shape)
        self.home_ptr = None       # set where the home GPU is owned
        self.writer_ptr = None     # set where the writer GPU is owned
        self.opened = False        # writer_ptr came from td_peer_open (close, not free)
        self.home_dev = None
        self.writer_dev = None
        self.credit = None         # writer side: event after the home released the inbox

    def home_view(self):
        return RawView(self.home_ptr, self.shape, device=self.home_dev)

    def writer_view(self):
        return RawView(self.writer_ptr, self.shape, device=self.writer_dev)

    def close_mapping(self):
        """Writer side: unmap another process's inbox (phase 1 of a release)."""
        try:
            if self.writer_ptr and self.opened:
                _native.call("td_peer_close", self.writer_dev.index, C.c_void_p(self.writer_ptr))
        except Exception:
            pass
        if self.opened:
            self.writer_ptr = None

    def free_home(self):
        """Home side: free the allocation (phase 2, after every writer unmapped it)."""
        try:
            if self.home_ptr:
                _native.call("td_peer_free", self.home_dev.index, C.c_void_p(self.home_ptr))
        except Exception:
            pass
        self.home_ptr = self.writer_ptr = None

    def free(self):
        self.close_mapping()
        self.free_home()


class InboxSet:
    """The inboxes of one program on one World (built once, reused by every
    execute of that program)."""

    def __init__(self, prog, world, gpu_of):
        self.prog = prog
        self.inboxes = {}
        self.pins = 0          # captured graphs / recorded plans holding raw inbox pointers
        cand = eligible_commits(prog, gpu_of)
        shifts = eligible_shifts(prog, gpu_of) if _shifts_apply(world) else {}
        if not cand and not shifts:
            return
        W = world
        multi = W.nprocs > 1
        boxes = {}
        handles = {}
        ok = True
        for k, c in sorted(cand.items()):
            boxes[("c", k)] = Inbox(c, gpu_of(c.home), gpu_of(c.task.coord), c.part.shape)
        for (s, i), t in sorted(shifts.items()):
            boxes[("x", s, i)] = Inbox(None, gpu_of(t.dst), gpu_of(t.src), t.part.shape, transfer=t)
        for ib in boxes.values():
            if W.owns(ib.home_gpu):
                ib.home_dev = W.device(ib.home_gpu)
            if W.owns(ib.writer_gpu):
                ib.writer_dev = W.device(ib.writer_gpu)
        # single process: both ends owned -> plain peer access
        for k, ib in boxes.items():
            if ib.home_dev is not None and ib.writer_dev is not None:
                if _native.call("td_peer_can_access", ib.writer_dev.index, ib.home_dev.index) != 1:
                    ok = False
                    break
                _native.call("td_peer_enable", ib.writer_dev.index, ib.home_dev.index)
        if ok:
            for k, ib in boxes.items():
                if ib.home_dev is None:
                    continue
                ptr = C.c_void_p()
                nbytes = 8 * max(1, math.prod(ib.shape))
                h = C.create_string_buffer(IPC_HANDLE_BYTES) if multi and ib.writer_dev is None else None
                try:
                    _native.call("td_peer_alloc", ib.home_dev.index, nbytes, C.byref(ptr), h)
                except Exception:
                    # PyTorch's cache may hold the free memory: release it once, then
                    # fall back to the NCCL write-back if there is still no room
                    import torch
                    with torch.cuda.device(ib.home_dev):
                        torch.cuda.empty_cache()
                    try:
                        _native.call("td_peer_alloc", ib.home_dev.index, nbytes, C.byref(ptr), h)
                    except Exception:
                        ok = False
                        break
                ib.home_ptr = ptr.value
                if ib.writer_dev is not None:
                    ib.writer_ptr = ib.home_ptr
                else:
                    handles[k] = bytes(h.raw)
        if multi:
            # collective: every rank walks the same program, so every rank is here
            allh = {}
            for part in W.all_gather_object(handles if ok else None):
                if part is None:
                    ok = False
                else:
                    allh.update(part)
            if ok:
                for k, ib in boxes.items():
                    if ib.writer_dev is None or ib.writer_ptr:
                        continue
                    ptr = C.c_void_p()
                    try:
                        _native.call("td_peer_open", ib.writer_dev.index, C.c_char_p(allh[k]), C.byref(ptr))
                        ib.writer_ptr = ptr.value
                        ib.opened = True
                    except Exception:
                        ok = False
            ok = all(W.all_gather_object(ok))
        if not ok:
            for ib in boxes.values():
                ib.free()
            return
        self.inboxes = boxes

    def by_task(self) -> dict:
        return {ib.commit.task.coord: ib for ib in self.inboxes.values() if ib.commit is not None}

    def by_transfer(self) -> dict:
        return {id(ib.transfer): ib for ib in self.inboxes.values() if ib.transfer is not None}

    def pin(self):
        self.pins += 1

    def unpin(self):
        self.pins = max(0, self.pins - 1)

    def free(self):
        for ib in self.inboxes.values():
            ib.free()
        self.inboxes = {}

    def release(self, world):
        """Free after the owned GPUs drained (no leaf still writes an inbox,
        every token was received).  Collective in SPMD jobs, in two phases:
        every writer unmaps its IPC mappings, all ranks meet, and only then
        do the homes free the memory (freeing an exported allocation while
        another process still maps it is undefined)."""
        release_sets([self], world)


def release_sets(sets, world) -> None:
    """Two-phase release of several InboxSets (see InboxSet.release)."""
    sets = [s for s in sets if getattr(s, "inboxes", None)]
    if world.nprocs == 1 and not sets:
        return
    import torch
    for g in world.owned:
        torch.cuda.synchronize(world.device(g))
    for st in sets:
        for ib in st.inboxes.values():
            ib.close_mapping()
    world.all_gather_object(None)          # barrier: every writer has unmapped
    for st in sets:
        for ib in st.inboxes.values():
            ib.free_home()
        st.inboxes = {}


# InboxSets kept per World (most recent programs); older ones are released
MAX_SETS = 2


class _Empty:
    inboxes: dict = {}

    def by_task(self) -> dict:
        return {}

    def by_transfer(self) -> dict:
        return {}


_NO_INBOXES = _Empty()


def inbox_set(prog, world, gpu_of) -> InboxSet:
    """The InboxSet of (prog, world), created on first use.  Creation is
    collective in SPMD jobs (handle exchange): every rank reaches it at the
    same execute because every rank runs the same program sequence, and the
    least recently created sets are released in the same order everywhere."""
    reg = world.inbox_sets
    hit = reg.get(id(prog))
    if hit is not None and hit.prog is prog:
        return hit
    if not eligible_commits(prog, gpu_of) and not (_shifts_apply(world) and eligible_shifts(prog, gpu_of)):
        return _NO_INBOXES                     # nothing to map: do not evict a useful set
    while len(reg) >= MAX_SETS:
        # the least recently created set no rank pins (a CUDA graph or launch plan
        # holding its raw pointers keeps it alive; then the registry grows); the
        # pin states are exchanged so every rank evicts the same set
        pinned = [[k for k, v in reg.items() if getattr(v, "pins", 0)]]
        if world.nprocs > 1:
            pinned = world.all_gather_object(pinned[0])
        held = {k for part in pinned for k in part}
        victim = next((k for k in reg if k not in held), None)
        if victim is None:
            break
        reg.pop(victim).release(world)
    s = InboxSet(prog, world, gpu_of)
    reg[id(prog)] = s
    return s
