"""The GPU job: which B200s take part, which ones this process drives, NCCL.

Two process models, both mapping the reference's processor grid onto GPUs
with `Machine.device_of` (rank-order blocks; identity when the grid has one
processor per GPU):

* single process (default): this process drives ``devices`` (default: the
  current CUDA device only); several GPUs share one NCCL clique built with
  ``ncclCommInitAll``;
* SPMD (``torchrun``, one process per GPU): `configure_distributed()` takes
  RANK / LOCAL_RANK / WORLD_SIZE from `torch.distributed`, exchanges an NCCL
  unique id over it, and builds one communicator with ``ncclCommInitRank``.

Every process plans the same launch program (planning is deterministic) and
issues only the NCCL calls and kernels of the GPUs it owns, in one global
order, so sends and receives pair up without any extra handshake.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _native
from .errors import CommError, ConfigError, DeviceUnavailable

#: seconds World.wait lets the GPUs go without progress before aborting NCCL
NCCL_TIMEOUT_S = float(os.environ.get("TD_NCCL_TIMEOUT", "600"))


class World:
    def __init__(self, ngpus, owned, rank=0, nprocs=1, comms=None, torch_devices=None):
        self.ngpus = ngpus              # GPUs in the job
        self.owned = list(owned)        # global GPU indices this process drives
        self.rank = rank
        self.nprocs = nprocs
        self.comms = comms or {}        # global GPU index -> ncclComm_t (as int)
        self.torch_devices = torch_devices or {}   # global GPU index -> torch.device
        self._streams = {}
        self._groups = {}               # sorted GPU tuple -> {owned GPU: sub-communicator}
        self.inbox_sets = {}            # id(program) -> peer.InboxSet (peer-memory write-backs)

    def owns(self, g: int) -> bool:
        return g in self.torch_devices

    def device(self, g: int):
        return self.torch_devices[g]

    def streams(self, g: int):
        """(compute stream, communication stream) of an owned GPU."""
        if g not in self._streams:
            import torch
            dev = self.torch_devices[g]
            self._streams[g] = (torch.cuda.Stream(device=dev, priority=0),
                                torch.cuda.Stream(device=dev, priority=-1))
        return self._streams[g]

    def copy_stream(self, g: int, k: int = 0):
        """Host<->device copy stream k of an owned GPU (progressive placement;
        independent streams let several inputs upload concurrently)."""
        key = ("h2d", g, k)
        if key not in self._streams:
            import torch
            self._streams[key] = torch.cuda.Stream(device=self.torch_devices[g])
        return self._streams[key]

    def comm(self, g: int):
        if g not in self.comms:
            raise ConfigError(f"GPU {g} has no NCCL communicator (job of {self.ngpus} GPU(s))")
        return C.c_void_p(self.comms[g])

    @property
    def multi_gpu(self) -> bool:
        return self.ngpus > 1

    def all_gather_object(self, obj) -> list:
        """obj of every process, in rank order (torch.distributed; [obj] alone)."""
        if self.nprocs == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.nprocs
        dist.all_gather_object(out, obj)
        return out

    def group_comm(self, gpus):
        """{owned GPU: communicator} over the GPU set `gpus` (ranked by GPU
        index), created on first use with ncclCommSplit.  Collective: every
        process of the job must request the same sets in the same order --
        the SPMD executor does, because all ranks walk the same program."""
        key = tuple(sorted(set(gpus)))
        if key not in self._groups:
            color = 0  # every split below is its own call; one color per member set
            made = {}
            grouped = len(self.comms) > 1   # one thread splitting several comms must group them
            if grouped:
                _native.call("td_group_start")
            try:
                for g in sorted(self.comms):
                    h = C.c_void_p()
                    member = g in key
                    _native.call("td_comm_split", C.c_void_p(self.comms[g]), color if member else -1,
                                 key.index(g) if member else 0, C.byref(h))
                    made[g] = h
            finally:
                if grouped:
                    _native.call("td_group_end")
            out = {}
            for g, h in made.items():
                if g in key:
                    if not h.value:
                        raise ConfigError(f"ncclCommSplit gave no communicator for GPU {g} in {key}")
                    out[g] = h.value
            self._groups[key] = out
        return self._groups[key]

    def all_comms(self) -> list:
        return list(self.comms.values()) + [h for grp in self._groups.values() for h in grp.values()]

    def wait(self, timeout: float = None) -> None:
        """Block until this process's GPUs finished the launches issued so far,
        with a watchdog instead of an unbounded sync: NCCL async errors are
        polled while waiting, and on one -- or after `timeout` seconds without
        completion (default TD_NCCL_TIMEOUT, 600 s) -- every communicator is
        aborted (ncclCommAbort) and CommError is raised (td_comm_wait)."""
        import torch
        streams = []
        for g in self.owned:
            streams += [s.cuda_stream for s in self.streams(g)]
            cur = torch.cuda.current_stream(self.device(g)).cuda_stream
            if cur:
                streams.append(cur)
        comms = self.all_comms()
        ca = (C.c_void_p * max(1, len(comms)))(*comms)
        sa = (C.c_void_p * max(1, len(streams)))(*streams)
        t = NCCL_TIMEOUT_S if timeout is None else float(timeout)
        rc = _native.lib().td_comm_wait(ca, len(comms), sa, len(streams), t)
        if rc < 0:
            msg = _native.lib().td_last_error().decode(errors="replace")
            self.comms, self._groups = {}, {}     # aborted: never destroy them again
            self.broken = True
            raise CommError(msg)
        for g in self.owned:                      # the legacy default streams too
            torch.cuda.synchronize(self.device(g))

    def close(self):
        if getattr(self, "broken", False):
            self.inbox_sets = {}
            return
        from .peer import release_sets
        release_sets(list(self.inbox_sets.values()), self)
        self.inbox_sets = {}
        for grp in self._groups.values():
            for h in grp.values():
                try:
                    _native.call("td_comm_destroy", C.c_void_p(h))
                except Exception:
                    pass
        self._groups = {}
        for h in self.comms.values():
            try:
                _native.call("td_comm_destroy", C.c_void_p(h))
            except Exception:
                pass
        self.comms = {}


_WORLD = None


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device is visible; the B200 path has no CPU fallback")
    return torch


def world() -> World:
    global _WORLD
    if _WORLD is None:
        torch = _torch()
        _native.load()
        dev = torch.cuda.current_device()
        _WORLD = World(1, [0], torch_devices={0: torch.device("cuda", dev)})
    return _WORLD


def configure(devices=None) -> World:
    """Single process driving `devices` (CUDA ordinals; default all visible)."""
    global _WORLD
    torch = _torch()
    _native.load()
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = list(devices)
    if _WORLD is not None:
        _WORLD.close()
    comms = {}
    if len(devices) > 1:
        arr = (C.c_void_p * len(devices))()
        ids = (C.c_int * len(devices))(*devices)
        _native.call("td_comm_init_all", arr, len(devices), ids)
        comms = {g: arr[g] for g in range(len(devices))}
    _WORLD = World(len(devices), range(len(devices)), comms=comms,
                   torch_devices={g: torch.device("cuda", d) for g, d in enumerate(devices)})
    return _WORLD


def configure_distributed() -> World:
    """One process per GPU under torch.distributed (torchrun)."""
    global _WORLD
    torch = _torch()
    import torch.distributed as dist
    _native.load()
    if not dist.is_initialized():
        raise ConfigError("torch.distributed is not initialised")
    rank, size = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank % max(1, torch.cuda.device_count())))
    torch.cuda.set_device(local)
    comms = {}
    if size > 1:
        uid = C.create_string_buffer(128)
        if rank == 0:
            _native.call("td_comm_unique_id", uid)
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0)
        handle = C.c_void_p()
        _native.call("td_comm_init_rank", C.byref(handle), size, rank, C.c_char_p(box[0]), local)
        comms = {rank: handle.value}
    if _WORLD is not None:
        _WORLD.close()
    _WORLD = World(size, [rank], rank=rank, nprocs=size, comms=comms,
                   torch_devices={rank: torch.device("cuda", local)})
    return _WORLD


def reset():
    global _WORLD
    if _WORLD is not None:
        _WORLD.close()
    _WORLD = None
