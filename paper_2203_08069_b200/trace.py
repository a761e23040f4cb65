"""The communication ledger: events, launches and memory high-water.

`CommEvent` / `ExecutionTrace` keep the reference's record types and
statistics (reference `pkg/src/tendist/simulator.py:113-269`).  On the
B200 path every compute-phase `CommEvent` is a real transfer: `runtime.py`
issues one NCCL send/recv (or a zero-copy same-GPU alias) per event, so the
ledger is a faithful description of the bytes that crossed NVLink, and the
reference's traffic anchors double as tests of the collective lowering.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

from .distribution import HyperRect
from .machine import Machine


@dataclass(frozen=True)
class CommEvent:
    """One aggregate transfer: ``src`` sends box ``rect`` of ``tensor`` to ``dst``."""

    timestep: int
    src: tuple
    dst: tuple
    tensor: str
    rect: HyperRect
    elements: int
    kind: str    # "copy" | "reduce"
    phase: str   # "compute" | "placement"


@dataclass(frozen=True)
class TaskInfo:
    coord: tuple
    rank: int
    env: dict = field(hash=False, compare=False, default_factory=dict)
    out_rect: object = None


@dataclass(frozen=True)
class Requirement:
    """What one task needed for one step before sourcing (debug record)."""

    coord: tuple
    step: int
    tensor: str
    rect: HyperRect
    scope: str   # "launch" | "step"


def _tally(events) -> dict:
    return {"messages": len(events), "elements": sum(e.elements for e in events)}


class ExecutionTrace:
    """Events, launch records, and per-processor memory high-water (elements)."""

    def __init__(self, machine: Machine):
        self.machine = machine
        self.events: list = []
        self.launches: list = []
        self.requirements: list = []
        self.num_steps = 0
        self.memory = {p: 0 for p in machine.enumerate()}
        self.timings: list = []   # B200 addition: per-launch device timings (ms)

    def bump_memory(self, coord, elements: int) -> None:
        if elements > self.memory[coord]:
            self.memory[coord] = elements

    @property
    def high_water(self) -> int:
        return max(self.memory.values(), default=0)

    def events_of(self, kind=None, phase=None, tensor=None, step=None) -> list:
        want = {"kind": kind, "phase": phase, "tensor": tensor, "timestep": step}
        want = {k: v for k, v in want.items() if v is not None}
        return [e for e in self.events if all(getattr(e, k) == v for k, v in want.items())]

    @property
    def total_messages(self) -> int:
        return len(self.events)

    @property
    def total_elements(self) -> int:
        return sum(e.elements for e in self.events)

    def per_edge(self) -> list:
        agg: dict = {}
        for e in self.events:
            m, n = agg.get((e.src, e.dst), (0, 0))
            agg[(e.src, e.dst)] = (m + 1, n + e.elements)
        rank = self.machine.rank_of
        return [{"src": list(s), "dst": list(d), "messages": agg[(s, d)][0],
                 "elements": agg[(s, d)][1]}
                for s, d in sorted(agg, key=lambda sd: (rank(sd[0]), rank(sd[1])))]

    def per_step(self) -> list:
        agg: dict = {}
        for e in self.events:
            if e.phase == "compute":
                m, n = agg.get(e.timestep, (0, 0))
                agg[e.timestep] = (m + 1, n + e.elements)
        return [{"step": s, "messages": agg.get(s, (0, 0))[0], "elements": agg.get(s, (0, 0))[1]}
                for s in range(self.num_steps)]

    def stats(self, config=None) -> dict:
        copies, reduces = self.events_of(kind="copy"), self.events_of(kind="reduce")
        out = {
            "schema": 1,
            "config": dict(config or {}),
            "machine": str(self.machine),
            "num_steps": self.num_steps,
            "totals": {
                "messages": self.total_messages,
                "elements": self.total_elements,
                "copy_messages": len(copies),
                "copy_elements": sum(e.elements for e in copies),
                "reduce_messages": len(reduces),
                "reduce_elements": sum(e.elements for e in reduces),
            },
            "phases": {"placement": _tally(self.events_of(phase="placement")),
                       "compute": _tally(self.events_of(phase="compute"))},
            "per_edge": self.per_edge(),
            "per_step": self.per_step(),
            "memory_high_water": {
                "overall": self.high_water,
                "per_processor": [{"processor": list(p), "elements": self.memory[p]}
                                  for p in self.machine.enumerate()],
            },
            "launches": list(self.launches),
        }
        if self.machine.num_levels > 1:
            cut = self.machine.level_slices()[0][1]
            same = [e for e in self.events if e.src[:cut] == e.dst[:cut]]
            cross = [e for e in self.events if e.src[:cut] != e.dst[:cut]]
            out["levels"] = {"intra_node": _tally(same), "inter_node": _tally(cross)}
        return out


def write_edge_csv(trace: ExecutionTrace, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["src", "dst", "messages", "elements"])
        for row in trace.per_edge():
            w.writerow(["x".join(map(str, row["src"])), "x".join(map(str, row["dst"])),
                        row["messages"], row["elements"]])
