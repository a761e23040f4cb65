"""The communication ledger: events, launches, memory high-water, timings.

`CommEvent` and the `ExecutionTrace` query/stats surface keep the
reference's record types and its stats JSON schema (reference
`pkg/src/tendist/simulator.py:113-269`) -- the schema is the contract the
reference's anchor tests and tools read.  The implementation is a small
group-by engine: every aggregate in the stats (totals, phases, per edge, per
step, per machine level) is `_rollup(events, key)` over one event filter,
and `stats()` is assembled from the `_SECTIONS` table.

On the B200 path every compute-phase `CommEvent` is a real transfer:
`runtime.py` issues one NCCL send/recv (or a zero-copy same-GPU alias) per
event, so the ledger describes the bytes that crossed NVLink.  When a run
is timed (`execute(..., timed=True)`), `timings` holds one record per
launch measured with CUDA events on the executing streams, and `stats()`
adds a ``"measured"`` section (device milliseconds, GFLOP/s or GB/s, and
the fraction of the B200 roof) beside the reference's keys.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

from .distribution import HyperRect
from .machine import Machine

_record = dataclass(frozen=True)


@_record
class CommEvent:
    """One aggregate transfer: ``src`` sends box ``rect`` of ``tensor`` to ``dst``."""

    timestep: int
    src: tuple
    dst: tuple
    tensor: str
    rect: HyperRect
    elements: int
    kind: str    # copy (fetch / write-back) or reduce (accumulated into the home)
    phase: str   # compute (inside a launch) or placement (redistribute)


@_record
class TaskInfo:
    coord: tuple
    rank: int
    env: dict = field(hash=False, compare=False, default_factory=dict)
    out_rect: object = None


@_record
class Requirement:
    """What one task needed for one step before sourcing (debug record)."""

    coord: tuple
    step: int
    tensor: str
    rect: HyperRect
    scope: str   # fetched once per launch, or again every step


def _rollup(events, key=None) -> dict:
    """{key(e): [messages, elements]} in first-seen order (key None: one bucket)."""
    acc: dict = {}
    for e in events:
        slot = acc.setdefault(None if key is None else key(e), [0, 0])
        slot[0] += 1
        slot[1] += e.elements
    return acc


def _pair(counts) -> dict:
    messages, elements = counts or (0, 0)
    return {"messages": messages, "elements": elements}


_FILTER_FIELDS = {"kind": "kind", "phase": "phase", "tensor": "tensor", "step": "timestep"}


class ExecutionTrace:
    """Events, launch records, and per-processor memory high-water (elements)."""

    def __init__(self, machine: Machine):
        self.machine = machine
        # the ledger: transfers, launch records, per-task needs (debug)
        self.events, self.launches, self.requirements = [], [], []
        self.num_steps = 0
        self.memory = dict.fromkeys(machine.enumerate(), 0)
        self.timings: list = []

    # -- recording ----------------------------------------------------------
    def bump_memory(self, coord, elements: int) -> None:
        self.memory[coord] = max(self.memory[coord], elements)

    def record_timing(self, label: str, device_ms: float, *, flops: float = 0.0, nbytes: float = 0.0,
                      bound: str = "tensor", peak: float = 0.0, gpus: int = 1) -> None:
        """One timed launch: device time (max over the GPUs that ran it) and
        its algorithmic work, from which the measured rates follow."""
        self.timings.append({"label": label, "device_ms": device_ms, "flops": flops, "bytes": nbytes,
                             "bound": bound, "peak": peak, "gpus": gpus})

    # -- queries ----------------------------------------------------------------
    @property
    def high_water(self) -> int:
        """Largest per-processor resident element count."""
        return max([0, *self.memory.values()])

    def events_of(self, kind=None, phase=None, tensor=None, step=None) -> list:
        wanted = [(_FILTER_FIELDS[k], v) for k, v in
                  (("kind", kind), ("phase", phase), ("tensor", tensor), ("step", step)) if v is not None]
        return [e for e in self.events if all(getattr(e, f) == v for f, v in wanted)]

    @property
    def total_messages(self) -> int:
        return _pair(_rollup(self.events).get(None))["messages"]

    @property
    def total_elements(self) -> int:
        return _pair(_rollup(self.events).get(None))["elements"]

    def per_edge(self) -> list:
        groups = _rollup(self.events, key=lambda e: (e.src, e.dst))
        order = sorted(groups, key=lambda edge: tuple(map(self.machine.rank_of, edge)))
        return [{"src": list(src), "dst": list(dst), **_pair(groups[(src, dst)])} for src, dst in order]

    def per_step(self) -> list:
        groups = _rollup(self.events_of(phase="compute"), key=lambda e: e.timestep)
        return [{"step": s, **_pair(groups.get(s))} for s in range(self.num_steps)]

    # -- stats ------------------------------------------------------------------
    def _totals(self) -> dict:
        by_kind = _rollup(self.events, key=lambda e: e.kind)
        out = {"messages": self.total_messages, "elements": self.total_elements}
        for kind in ("copy", "reduce"):
            m, n = by_kind.get(kind, (0, 0))
            out[f"{kind}_messages"], out[f"{kind}_elements"] = m, n
        return out

    def _phases(self) -> dict:
        by_phase = _rollup(self.events, key=lambda e: e.phase)
        return {ph: _pair(by_phase.get(ph)) for ph in ("placement", "compute")}

    def _memory(self) -> dict:
        return {"overall": self.high_water,
                "per_processor": [{"processor": list(p), "elements": self.memory[p]}
                                  for p in self.machine.enumerate()]}

    def _levels(self):
        if self.machine.num_levels <= 1:
            return None
        cut = self.machine.level_slices()[0][1]
        split = _rollup(self.events, key=lambda e: e.src[:cut] == e.dst[:cut])
        return {"intra_node": _pair(split.get(True)), "inter_node": _pair(split.get(False))}

    def _measured(self):
        if not self.timings:
            return None
        rows = []
        for t in self.timings:
            sec = t["device_ms"] * 1e-3
            rate = (t["flops"] / sec / 1e9 if t["bound"] == "tensor" else t["bytes"] / sec / 1e9) if sec > 0 else 0.0
            rows.append({**t, "rate": rate, "rate_unit": "GFLOP/s" if t["bound"] == "tensor" else "GB/s",
                         "frac_of_peak": rate / (t["peak"] * t["gpus"]) if t["peak"] else None})
        total_ms = sum(t["device_ms"] for t in self.timings)
        return {"launches": rows, "device_ms": total_ms,
                "flops": sum(t["flops"] for t in self.timings),
                "bytes": sum(t["bytes"] for t in self.timings)}

    _SECTIONS = (("totals", _totals), ("phases", _phases), ("per_edge", per_edge),
                 ("per_step", per_step), ("memory_high_water", _memory))

    def stats(self, config=None) -> dict:
        out = {"schema": 1, "config": dict(config or {}), "machine": str(self.machine),
               "num_steps": self.num_steps}
        for name, build in self._SECTIONS:
            out[name] = build(self)
        out["launches"] = list(self.launches)
        for name, build in (("levels", ExecutionTrace._levels), ("measured", ExecutionTrace._measured)):
            section = build(self)
            if section is not None:
                out[name] = section
        return out


def write_edge_csv(trace: ExecutionTrace, path) -> None:
    """The per_edge table as CSV (header src,dst,messages,elements; grid
    coordinates joined with "x")."""
    rows = [["src", "dst", "messages", "elements"]]
    rows += [["x".join(map(str, r["src"])), "x".join(map(str, r["dst"])), r["messages"], r["elements"]]
             for r in trace.per_edge()]
    with open(path, "w", newline="") as fh:
        csv.writer(fh).writerows(rows)
