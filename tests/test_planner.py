"""Ledger parity (CPU): the planner's CommEvents, memory high-water, step
counts and requirement records equal the reference's, event for event, for
every golden case (fixtures made by running `tendist`: tests/golden/make_golden.py).
The ledger is also the NCCL transfer program, so this pins the collective
lowering's pattern (who sends which box to whom at which step)."""

import pytest

import paper_2203_08069_b200 as td
from paper_2203_08069_b200.planner import plan_statement

from _cases import build, case_id, load

LEDGERS = load("ledgers.json")


def _box(r):
    return [list(r.lo), list(r.hi)]


@pytest.mark.parametrize("fix", LEDGERS, ids=[case_id(f["case"]) for f in LEDGERS])
def test_ledger_matches_reference(fix):
    b = build(td, fix["case"])
    prog, tr = plan_statement(b.statement, b.machine, b.distributions, b.schedule, label=b.name)
    got = [[e.timestep, list(e.src), list(e.dst), e.tensor, _box(e.rect), e.elements, e.kind, e.phase]
           for e in tr.events]
    assert got == fix["events"]
    assert [[list(p), v] for p, v in tr.memory.items()] == fix["memory"]
    assert tr.num_steps == fix["num_steps"]
    assert [[list(r.coord), r.step, r.tensor, _box(r.rect), r.scope] for r in tr.requirements] == \
        fix["requirements"]
    st = tr.stats()
    assert st["totals"] == fix["totals"]
    assert st["per_step"] == fix["per_step"]
    assert st["per_edge"] == fix["per_edge"]
    assert st["launches"] == fix["launches"]
    if fix["signature"] is not None:
        assert b.signature(tr) == fix["signature"]


@pytest.mark.parametrize("fix", LEDGERS, ids=[case_id(f["case"]) for f in LEDGERS])
def test_buffer_program_is_consistent(fix):
    """Every transfer reads a holding that contains its part, every task
    operand is covered by its holdings, and each temp dies after its last use."""
    b = build(td, fix["case"])
    prog, _ = plan_statement(b.statement, b.machine, b.distributions, b.schedule)
    n_events = sum(len(m) for m in prog.transfers)
    assert n_events == sum(1 for e in fix["events"] if e[6] == "copy" and e[0] >= 0) - sum(
        1 for c in prog.commits if c.kind == "copy" and c.home != c.task.coord)
    for moves in prog.transfers:
        for t in moves:
            src = prog.holdings[t.src_hid]
            assert src.proc == t.src and src.rect.contains(t.part)
            dst = prog.holdings[t.dst_hid]
            assert dst.proc == t.dst and dst.rect == t.part
    for works in prog.work:
        for w in works:
            for name, rect, hids in w.operands.values():
                if rect is None:
                    continue
                covered = td.subtract_rects([rect], [prog.holdings[h].rect for h in hids])
                if name != prog.plan.out_name:
                    assert covered == [], (name, rect)
                assert all(prog.holdings[h].proc == w.task.coord for h in hids)


def test_placement_policies_map_processors_to_gpus():
    """block: contiguous runs of processors per GPU; cyclic: round robin;
    identity whenever there is a GPU per processor."""
    from paper_2203_08069_b200 import machine as mach
    m = td.grid(2, 2, 2)
    procs = list(m.enumerate())
    assert [m.device_of(p, 4) for p in procs] == [0, 0, 1, 1, 2, 2, 3, 3]
    mach.set_placement("cyclic")
    try:
        assert [m.device_of(p, 4) for p in procs] == [0, 1, 2, 3, 0, 1, 2, 3]
        assert [m.device_of(p, 8) for p in procs] == list(range(8))
    finally:
        mach.set_placement("block")
    with pytest.raises(td.ConfigError):
        mach.set_placement("random")
