"""Processor grids and their mapping onto GPUs.

A `Machine` is a tuple of levels, each a tuple of positive extents
(reference `pkg/src/tendist/machine.py:21-85`).  Processors are flat
coordinate tuples; `enumerate()` lists them lexicographically and that order
is the deterministic tie-break used everywhere (task order, reduction
combine order, source choice).  `rank_of` is the row-major linearisation.

B200 mapping: one NVSwitch box is a single flat level, so a hierarchical
machine executes as its flattened grid (levels only matter for the stats
split).  `device_of` places processor ``rank`` on GPU
``rank * ndev // size`` -- identity when the grid has exactly one processor
per GPU, contiguous blocks of processors per GPU when oversubscribed
(placement "block", the default).  `set_placement("cyclic")` deals the
processors round robin instead (``rank % ndev``), which e.g. puts Johnson's
depth pairs on different GPUs; choose it before placing data (it decides
where every piece lives).
"""

from __future__ import annotations

import itertools
from functools import reduce

from .errors import ConfigError, EmptyGrid

PLACEMENTS = ("block", "cyclic")
_PLACEMENT = "block"


def set_placement(policy: str) -> None:
    """Processor -> GPU mapping of oversubscribed grids: "block" or "cyclic"."""
    global _PLACEMENT
    if policy not in PLACEMENTS:
        raise ConfigError(f"placement must be one of {PLACEMENTS}, got {policy!r}")
    _PLACEMENT = policy


def placement() -> str:
    return _PLACEMENT


class Machine:
    __slots__ = ("levels", "_procs", "_flat", "_size", "_rank")

    def __init__(self, levels):
        lv = tuple(tuple(int(d) for d in level) for level in levels)
        if not lv or any(len(level) == 0 for level in lv):
            raise EmptyGrid(f"every machine level needs a dimension: {lv}")
        if any(d <= 0 for level in lv for d in level):
            raise EmptyGrid(f"machine extents must be positive: {lv}")
        object.__setattr__(self, "levels", lv)
        flat = tuple(d for level in lv for d in level)
        procs = tuple(itertools.product(*map(range, flat)))
        object.__setattr__(self, "_procs", procs)
        object.__setattr__(self, "_flat", flat)
        object.__setattr__(self, "_size", reduce(lambda a, b: a * b, flat, 1))
        # rank lookups sit on every executor step (processor -> GPU): precomputed
        object.__setattr__(self, "_rank", {p: r for r, p in enumerate(procs)})

    def __setattr__(self, name, value):
        raise AttributeError("Machine is immutable")

    def __eq__(self, other):
        return isinstance(other, Machine) and other.levels == self.levels

    def __hash__(self):
        return hash(self.levels)

    def __repr__(self):
        return f"Machine(levels={self.levels})"

    def __str__(self):
        return "/".join("x".join(map(str, level)) for level in self.levels)

    @property
    def flat_dims(self) -> tuple:
        return self._flat

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def size(self) -> int:
        return self._size

    def enumerate(self) -> tuple:
        """Processors in lexicographic order of their flat coordinates."""
        return self._procs

    def rank_of(self, coord) -> int:
        r = self._rank.get(tuple(coord))
        if r is not None:
            return r
        r = 0
        for extent, c in zip(self._flat, coord):
            r = r * extent + c
        return r

    def coord_of(self, rank: int) -> tuple:
        return self._procs[rank]

    def level_slices(self):
        out, at = [], 0
        for level in self.levels:
            out.append((at, at + len(level)))
            at += len(level)
        return out

    def flatten(self) -> "Machine":
        return Machine((self.flat_dims,))

    def device_of(self, coord, ndev: int) -> int:
        """GPU ordinal (in the job's device list) that runs processor coord."""
        r = self.rank_of(coord)
        if ndev >= self.size:
            return r
        return r % ndev if _PLACEMENT == "cyclic" else r * ndev // self.size


def make_machine(levels) -> Machine:
    return Machine(levels)


def grid(*dims) -> Machine:
    return Machine([dims])


def parse_machine(text: str) -> Machine:
    """``"3x3"`` -> flat grid, ``"2x2/4"`` -> two levels."""
    try:
        return Machine([[int(tok) for tok in part.split("x")] for part in text.strip().split("/")])
    except ValueError as exc:
        raise ConfigError(f"cannot parse machine {text!r}") from exc
