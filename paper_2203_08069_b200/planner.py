"""Launch planning: scheduled CIN -> task grid, step loop, transfer program.

This is the integer-only half of the path.  It restates the reference's task
lowering and ledger phase (reference `pkg/src/tendist/simulator.py:59-108`
bounds analysis, `:398-505` `lower_to_tasks`, `:514-525` source choice,
`:557-613` phase one, `:624-654` commit events) but, instead of only
recording `CommEvent`s, it also emits the *buffer program* the GPUs execute:

* `Holding`   -- a box of one tensor resident on one processor: either a
  distribution piece (shared HBM tile per GPU) or a fetched temporary;
* `Transfer`  -- one event = move `part` from a holding on `src` into a new
  temporary holding on `dst` (NCCL send/recv across GPUs, an alias of the
  source tile when both processors sit on the same GPU);
* `StepWork`  -- for one task and one step: the pinned loop nest to run and,
  for every access, which holdings cover the box it reads;
* `Commit`    -- write-back of a task's output box into the home piece
  (``copy``) or accumulation in task order (``reduce``).

Events, requirements and memory high-water are produced exactly as the
reference does, so ledger parity with `tendist` is testable on the CPU.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

from .cin import (Communicate, Distribute, Forall, Place, Reduce, Seq, Suchthat, body_of,
                  leaf_accesses, leaf_statements, relation_defs, relations_of)
from .distribution import HyperRect, subtract_rects
from .errors import (ConfigError, GridMismatch, MissingDistribution, NonAffineAccess,
                     OOBAccess, OverlappingWrites, UnboundVariable, WriteToReplica)
from .ir import Access, IndexVar
from .trace import CommEvent, ExecutionTrace, Requirement, TaskInfo


# ------------------------------------------------------------ bounds analysis
def var_interval(name: str, env: dict, defs: dict) -> tuple:
    """Half-open range of values `name` takes when every loop variable ranges
    over its interval in env (reference `simulator.py:59-89`)."""
    if name in env:
        return env[name]
    rel = defs.get(name)
    if rel is None:
        raise UnboundVariable(f"no range for {name}")
    if hasattr(rel, "outer"):                        # Split / Divide
        olo, ohi = var_interval(rel.outer, env, defs)
        ilo, ihi = var_interval(rel.inner, env, defs)
        if olo >= ohi or ilo >= ihi:
            return (0, 0)
        b = rel.block
        return (min(olo * b + ilo, rel.extent), min((ohi - 1) * b + ihi, rel.extent))
    rlo, rhi = var_interval(rel.result, env, defs)   # Rotate
    offs = [var_interval(v, env, defs) for v in rel.over]
    if rlo >= rhi or any(a >= b for a, b in offs):
        return (0, 0)
    if rhi - rlo == 1 and all(b - a == 1 for a, b in offs):
        v = (rlo + sum(a for a, _ in offs)) % rel.extent
        return (v, v + 1)
    return (0, rel.extent)


def access_rect(access: Access, env: dict, defs: dict):
    """Box an access touches under interval env; None if empty."""
    lo, hi = [], []
    for v in access.indices:
        if not isinstance(v, IndexVar):
            raise NonAffineAccess(f"access index {v!r} is not a plain variable")
        a, b = var_interval(v.name, env, defs)
        lo.append(a)
        hi.append(b)
    box = HyperRect(lo, hi)
    if box.lo and box.is_empty:
        return None
    for a, b, d in zip(box.lo, box.hi, access.tensor.dims):
        if a < 0 or b > d:
            raise OOBAccess(f"{access.tensor.name} rows {box} outside dims {access.tensor.dims}")
    return box


# ------------------------------------------------------------------- plan
@dataclass
class LaunchPlan:
    machine: object
    launch_vars: list
    task_body: object
    relations: tuple
    defs: dict
    intervals: dict
    step_var: object
    num_steps: int
    fetch_plan: list
    out_name: str
    out_kind: str
    out_access: Access
    tasks: list


def _intervals(node, acc: dict) -> dict:
    if isinstance(node, Forall):
        acc[node.var] = (node.lo, node.hi)
        _intervals(node.body, acc)
    elif isinstance(node, Seq):
        for s in node.stmts:
            _intervals(s, acc)
    elif isinstance(node, Suchthat):
        _intervals(node.body, acc)
    return acc


def lower_to_tasks(stmt, store) -> LaunchPlan:
    """Leading distributed loops -> one task per processor (reference
    `simulator.py:398-505`); also picks the step loop and fetch scopes."""
    machine = store.machine
    rels = relations_of(stmt)
    defs = relation_defs(rels)
    body = body_of(stmt)
    distributed = {r.var for r in rels if isinstance(r, Distribute)}

    launch, node = [], body
    while isinstance(node, Forall) and node.var in distributed:
        launch.append(node)
        node = node.body
    task_body = node
    if not launch:
        raise GridMismatch("statement has no leading distributed loops")
    inner = set(_intervals(task_body, {}))
    if distributed & inner:
        raise GridMismatch(f"distributed loops {sorted(distributed & inner)} are not outermost")
    dims = machine.flat_dims
    if len(launch) != len(dims):
        raise GridMismatch(f"{len(launch)} distributed loops for machine {machine} with "
                           f"{len(dims)} dimensions")
    for f, d in zip(launch, dims):
        if not ((f.lo == 0 and f.hi == d) or (f.extent == 1 and 0 <= f.lo < d)):
            raise GridMismatch(f"loop {f.var} spans [{f.lo},{f.hi}) over a machine "
                               f"dimension of extent {d}")

    leaves = leaf_statements(stmt)
    if any(isinstance(l, Place) for l in leaves):
        raise ConfigError("placement statements run through place()/redistribute()")
    if isinstance(task_body, Seq):
        raise ConfigError("tasks must be single loop nests")
    outs = {l.lhs.tensor.name for l in leaves}
    if len(outs) != 1:
        raise ConfigError(f"one output tensor per launch, got {sorted(outs)}")
    out_name = next(iter(outs))
    out_kind = "reduce" if any(isinstance(l, Reduce) for l in leaves) else "copy"
    out_access = leaves[0].lhs

    names = sorted({a.tensor.name for l in leaves for a in leaf_accesses(l)})
    for n in names:
        if n not in store:
            raise MissingDistribution(f"tensor {n} has no placed region")
    if out_kind == "copy" and store[out_name].dist.replicated:
        raise WriteToReplica(f"{out_name} is replicated; plain writes would diverge the copies")

    comms = [r for r in rels if isinstance(r, Communicate)]
    step_candidates = {c.var for c in comms} - distributed
    step_var, cur = None, task_body
    while isinstance(cur, Forall):
        if cur.var in step_candidates:
            step_var = cur
            break
        cur = cur.body
    num_steps = step_var.extent if step_var is not None else 1
    intervals = _intervals(body, {})

    by_tensor: dict = {}
    for leaf in leaves:
        for acc in leaf_accesses(leaf):
            lst = by_tensor.setdefault(acc.tensor.name, [])
            if all(a.var_names != acc.var_names for a in lst):
                lst.append(acc)
    fetch_plan = []
    for n in names:
        if n == out_name:
            continue
        named = [c for c in comms if n in c.tensors]
        if named and named[0].var in distributed:
            scope = "launch"
        else:
            scope = "step" if step_var is not None else "launch"
        fetch_plan.append((n, tuple(by_tensor[n]), scope))

    tasks = []
    for coord in itertools.product(*(range(f.lo, f.hi) for f in launch)):
        env = {f.var: c for f, c in zip(launch, coord)}
        iv = dict(intervals)
        iv.update({v: (c, c + 1) for v, c in env.items()})
        tasks.append(TaskInfo(coord, machine.rank_of(coord), env,
                              access_rect(out_access, iv, defs)))
    if out_kind == "copy":
        for a, b in itertools.combinations(tasks, 2):
            if a.out_rect is not None and b.out_rect is not None:
                both = a.out_rect.intersect(b.out_rect)
                if both is not None:
                    raise OverlappingWrites(f"tasks {a.coord} and {b.coord} both write "
                                            f"{both} of {out_name}")
    return LaunchPlan(machine, launch, task_body, rels, defs, intervals, step_var,
                      num_steps, fetch_plan, out_name, out_kind, out_access, tasks)


# -------------------------------------------------------- buffer program
@dataclass
class Holding:
    hid: int
    proc: tuple
    tensor: str
    rect: HyperRect
    kind: str                  # "piece" | "temp"
    color: tuple = None        # pieces only
    step: int = -1             # temps: creation step
    scope: str = ""            # temps: "launch" | "step"


@dataclass
class Transfer:
    step: int
    src: tuple
    dst: tuple
    tensor: str
    part: HyperRect
    src_hid: int
    dst_hid: int
    wave: int = 0      # > 0: relays a temp received earlier in the same step



@dataclass
class StepWork:
    task: TaskInfo
    step: int                  # -1: whole task nest after all steps (fallback)
    operands: dict             # access var_names key -> (tensor, rect, [hid, ...])


@dataclass
class Commit:
    task: TaskInfo
    tensor: str
    part: HyperRect
    home: tuple
    color: tuple
    kind: str                  # "copy" | "reduce"


@dataclass
class Program:
    plan: LaunchPlan
    holdings: dict = field(default_factory=dict)       # hid -> Holding
    piece_hid: dict = field(default_factory=dict)      # (proc, tensor, color) -> hid
    transfers: list = field(default_factory=list)      # per step: [Transfer]
    work: list = field(default_factory=list)           # per step: [StepWork]
    commits: list = field(default_factory=list)        # [Commit] in task order
    stepwise: bool = True
    last_use: dict = field(default_factory=dict)       # temp hid -> last step it is read


def _key(acc) -> tuple:
    return (acc.tensor.name, acc.var_names)


def build_program(stmt, store, trace: ExecutionTrace, *, record_requirements=True) -> Program:
    """Phase one of execute (ledger) plus the buffer program for the GPUs."""
    plan = lower_to_tasks(stmt, store)
    prog = Program(plan)
    machine = store.machine
    order = list(machine.enumerate())
    events = trace.events
    nid = itertools.count()

    def new_holding(**kw) -> Holding:
        h = Holding(next(nid), **kw)
        prog.holdings[h.hid] = h
        return h

    # resident pieces of every tensor the launch touches
    for name in sorted({n for n, _, _ in plan.fetch_plan} | {plan.out_name}):
        dist = store[name].dist
        held = store[name].residency
        for color, box, procs in dist.pieces():
            for p in procs:
                if box in held.get(p, ()):
                    h = new_holding(proc=p, tensor=name, rect=box, kind="piece", color=color)
                    prog.piece_hid[(p, name, color)] = h.hid

    def pieces_at(p, name) -> list:
        dist = store[name].dist
        out = []
        for color in dist.colors():
            hid = prog.piece_hid.get((p, name, color))
            if hid is not None:
                out.append(hid)
        return out

    # step-pinned execution keeps the reference's per-point accumulation
    # order only when the step loop heads the task nest
    prog.stepwise = plan.step_var is None or plan.task_body is plan.step_var

    launch_temps: dict = {}     # proc -> [hid]
    prev_temps: dict = {}
    persist = {p: store.persistent_volume(p) for p in order}
    out_buf = {t.coord: (t.out_rect.volume if t.out_rect is not None else 0) for t in plan.tasks}
    all_temps: dict = {}        # proc -> [hid] (fallback mode keeps everything)

    def temps_with(table, q, name):
        return [hid for hid in table.get(q, []) if prog.holdings[hid].tensor == name]

    def source_for(name, part, p, homes):
        """(proc, hid) serving `part` (reference `_pick_source`, `simulator.py:514-525`)."""
        for table in (prev_temps, launch_temps):
            for q in order:
                if q == p:
                    continue
                for hid in temps_with(table, q, name):
                    if prog.holdings[hid].rect.contains(part):
                        return q, hid
        for q in homes:
            if q != p:
                return q, None
        return None, None

    def holder_hid(q, name, part, color):
        hid = prog.piece_hid.get((q, name, color))
        if hid is not None and prog.holdings[hid].rect.contains(part):
            return hid
        for hid in pieces_at(q, name):
            if prog.holdings[hid].rect.contains(part):
                return hid
        raise ConfigError(f"no resident copy of {name} {part} on {q}")

    for s in range(plan.num_steps):
        cur_temps: dict = {}
        moves: list = []
        wave_of: dict = {}      # temp hid made this step -> wave of the transfer making it
        for task in plan.tasks:
            p = task.coord
            launch_iv = dict(plan.intervals)
            launch_iv.update({v: (c, c + 1) for v, c in task.env.items()})
            step_iv = dict(launch_iv)
            if plan.step_var is not None:
                step_iv[plan.step_var.var] = (s, s + 1)
            for name, accs, scope in plan.fetch_plan:
                if scope == "launch" and s > 0:
                    continue
                iv = launch_iv if scope == "launch" else step_iv
                seen = []
                for acc in accs:
                    box = access_rect(acc, iv, plan.defs)
                    if box is None or box in seen:
                        continue
                    seen.append(box)
                    if record_requirements:
                        trace.requirements.append(Requirement(p, s, name, box, scope))
                    region = store[name]
                    held = list(region.held_at(p))
                    for table in (launch_temps, prev_temps, cur_temps):
                        held += [prog.holdings[h].rect for h in temps_with(table, p, name)]
                    sink = launch_temps if scope == "launch" else cur_temps
                    for piece in subtract_rects([box], held):
                        for color in region.dist.colors():
                            part = piece.intersect(region.dist.piece_bounds(color))
                            if part is None:
                                continue
                            src, src_hid = source_for(name, part, p,
                                                      region.dist.processors_of(color))
                            if src is None:
                                raise ConfigError(f"{name} {part} has no source for {p}")
                            if src_hid is None:
                                src_hid = holder_hid(src, name, part, color)
                            events.append(CommEvent(s, src, p, name, part, part.volume,
                                                    "copy", "compute"))
                            h = new_holding(proc=p, tensor=name, rect=part, kind="temp",
                                            step=s, scope=scope)
                            # a source that is itself a temp received this step
                            # (launch-scope relay, e.g. MTTKRP's D 00->01->10) must
                            # be forwarded in a later NCCL group than its arrival
                            wave = wave_of[src_hid] + 1 if src_hid in wave_of else 0
                            wave_of[h.hid] = wave
                            moves.append(Transfer(s, src, p, name, part, src_hid, h.hid, wave))
                            sink.setdefault(p, []).append(h.hid)
                            all_temps.setdefault(p, []).append(h.hid)
        for p in order:
            vol = persist[p] + out_buf.get(p, 0)
            for table in (launch_temps, prev_temps, cur_temps):
                vol += sum(prog.holdings[h].rect.volume for h in table.get(p, []))
            trace.bump_memory(p, vol)
        prog.transfers.append(moves)

        # what each task reads this step
        step_work = []
        if prog.stepwise:
            for task in plan.tasks:
                step_work.append(_operands(prog, plan, task, s, store, pieces_at,
                                           [launch_temps, prev_temps, cur_temps]))
        prog.work.append(step_work)
        prev_temps = cur_temps

    if not prog.stepwise:
        prog.work.append([_operands(prog, plan, task, -1, store, pieces_at, [all_temps])
                          for task in plan.tasks])

    # commit / write-back (reference `simulator.py:624-645`)
    last = plan.num_steps - 1
    out_dist = store[plan.out_name].dist
    for task in plan.tasks:
        if task.out_rect is None:
            continue
        for color in out_dist.colors():
            part = task.out_rect.intersect(out_dist.piece_bounds(color))
            if part is None:
                continue
            procs = out_dist.processors_of(color)
            targets = procs if plan.out_kind == "copy" else procs[:1]
            for h in targets:
                prog.commits.append(Commit(task, plan.out_name, part, h, color, plan.out_kind))
                if h != task.coord:
                    events.append(CommEvent(last, task.coord, h, plan.out_name, part,
                                            part.volume, plan.out_kind, "compute"))

    # temp lifetimes: last step whose work or transfers read the holding
    for s, moves in enumerate(prog.transfers):
        for t in moves:
            prog.last_use[t.src_hid] = max(prog.last_use.get(t.src_hid, -1), s)
    for s, works in enumerate(prog.work):
        step = s if prog.stepwise else plan.num_steps
        for w in works:
            for _, _, hids in w.operands.values():
                for hid in hids:
                    prog.last_use[hid] = max(prog.last_use.get(hid, -1), step)
    return prog


def _operands(prog, plan, task, s, store, pieces_at, tables) -> StepWork:
    p = task.coord
    iv = dict(plan.intervals)
    iv.update({v: (c, c + 1) for v, c in task.env.items()})
    if s >= 0 and plan.step_var is not None:
        iv[plan.step_var.var] = (s, s + 1)
    ops = {}
    for leaf in leaf_statements(plan.task_body):
        for acc in leaf_accesses(leaf)[1:]:
            key = _key(acc)
            if key in ops:
                continue
            box = access_rect(acc, iv, plan.defs)
            name = acc.tensor.name
            if box is None:
                ops[key] = (name, None, [])
                continue
            cands = pieces_at(p, name)
            for table in tables:
                cands += [h for h in table.get(p, []) if prog.holdings[h].tensor == name]
            cover = [h for h in cands if prog.holdings[h].rect.intersect(box) is not None]
            whole = [h for h in cover if prog.holdings[h].rect.contains(box)]
            ops[key] = (name, box, whole[:1] if whole else cover)
    return StepWork(task, s, ops)



# ------------------------------------------------ host-only planning (no GPU)
class _HostRegion:
    def __init__(self, name, dist):
        self.name = name
        self.dist = dist
        self.residency = dist.residency()

    def held_at(self, coord) -> list:
        return self.residency.get(coord, [])

    def volume_at(self, coord) -> int:
        return sum(r.volume for r in self.held_at(coord))


class HostStore:
    """Bookkeeping-only region store: plans and ledgers without touching a GPU
    (the reference's RegionStore minus values, `simulator.py:274-314`)."""

    def __init__(self, machine):
        self.machine = machine
        self.regions: dict = {}

    def declare(self, name, dist):
        self.regions[name] = _HostRegion(name, dist)
        return self.regions[name]

    def __contains__(self, name):
        return name in self.regions

    def __getitem__(self, name):
        return self.regions[name]

    def persistent_volume(self, coord) -> int:
        return sum(r.volume_at(coord) for r in self.regions.values())


def plan_statement(stmt, machine, distributions, schedule=None, *, record_requirements=True, label=None):
    """(Program, ExecutionTrace) of a statement: the full ledger and buffer
    program, computed on the host only."""
    from .cin import lower_to_cin
    from .errors import MissingDistribution
    from .ir import TensorIndexStmt
    cin = lower_to_cin(stmt) if isinstance(stmt, TensorIndexStmt) else stmt
    if schedule is not None:
        cin = schedule.apply(cin)
    store = HostStore(machine)
    names = sorted({a.tensor.name for l in leaf_statements(cin) for a in leaf_accesses(l)})
    for n in names:
        if n not in distributions:
            raise MissingDistribution(f"no distribution for {n}")
        store.declare(n, distributions[n])
    trace = ExecutionTrace(machine)
    prog = build_program(cin, store, trace, record_requirements=record_requirements)
    trace.num_steps = prog.plan.num_steps
    trace.launches.append({"phase": "compute", "label": label or prog.plan.out_name,
                           "tasks": len(prog.plan.tasks), "steps": prog.plan.num_steps})
    return prog, trace


def comm_schedule(prog: Program, machine, ngpus: int) -> list:
    """Cross-GPU traffic of a program in issue order: one entry
    (phase, step, wave, src_gpu, dst_gpu, elements) per NCCL send/recv pair.
    Every SPMD rank derives the same list (planning is deterministic), takes
    the sends and receives of its own GPU, and NCCL pairs them in this order;
    same-GPU transfers are HBM aliases and do not appear."""
    out = []
    for s, moves in enumerate(prog.transfers):
        for wave in sorted({t.wave for t in moves}):
            for t in moves:
                if t.wave != wave:
                    continue
                gs, gd = machine.device_of(t.src, ngpus), machine.device_of(t.dst, ngpus)
                if gs != gd:
                    out.append(("fetch", s, wave, gs, gd, t.part.volume))
    last = prog.plan.num_steps - 1
    for c in prog.commits:
        gs, gd = machine.device_of(c.task.coord, ngpus), machine.device_of(c.home, ngpus)
        if gs != gd:
            out.append(("commit", last, 0, gs, gd, c.part.volume))
    return out
