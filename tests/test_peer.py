"""Peer-memory write-backs (paper_2203_08069_b200/peer.py), host side on CPU:
the RawView used for inbox pointers and which commits qualify."""

import pytest

import paper_2203_08069_b200 as td
from paper_2203_08069_b200.peer import RawView, eligible_commits
from paper_2203_08069_b200.planner import plan_statement


def test_rawview_slicing_and_strides():
    v = RawView(0x1000, (6, 8))
    assert v.stride() == (8, 1) and v.numel() == 48 and v.is_contiguous()
    s = v[2:5, 3:7]
    assert s.shape == (3, 4) and s.stride() == (8, 1)
    assert s.data_ptr() == 0x1000 + 8 * (2 * 8 + 3)
    assert not s.is_contiguous()
    assert v[1:3].is_contiguous() and v[1:3].shape == (2, 8)
    assert v[4:2].shape == (0, 8)
    with pytest.raises(TypeError):
        v[::2]


def _gpu_of(machine, ngpus):
    return lambda p: machine.device_of(p, ngpus)


def _eligible(bundle, ngpus):
    prog, _ = plan_statement(bundle.statement, bundle.machine, bundle.distributions, bundle.schedule)
    return prog, eligible_commits(prog, _gpu_of(bundle.machine, ngpus))


def test_johnson_depth_partials_qualify_at_eight_gpus():
    b = td.johnson(2, 2, 2, dims=(16, 12, 20))
    prog, el = _eligible(b, 8)
    # the four k=1 tasks ship their whole partial to (i, j, 0)
    assert sorted(c.task.coord for c in el.values()) == [(0, 0, 1), (0, 1, 1), (1, 0, 1), (1, 1, 1)]
    for c in el.values():
        assert c.home == c.task.coord[:2] + (0,) and c.part == c.task.out_rect
    # at 2 or 4 GPUs the depth pairs share a GPU: nothing crosses
    assert _eligible(b, 4)[1] == {} and _eligible(b, 2)[1] == {}


def test_cosma_k_split_qualifies_and_multi_step_does_not():
    _, el = _eligible(td.cosma_like((1, 1, 2), (1, 1, 1), dims=(12, 10, 14)), 2)
    assert [c.task.coord for c in el.values()] == [(0, 0, 1)]
    # two sequential k-steps per task: the leaf cannot overwrite the inbox
    _, el = _eligible(td.cosma_like((1, 1, 2), (1, 1, 2), dims=(12, 10, 14)), 2)
    assert el == {}


@pytest.mark.parametrize("bundle", [td.cannon(2, 2, dims=(8, 8, 8)), td.summa(2, 1, dims=(8, 8, 8), chunk=2),
                                    td.ttv(4, dims=(8, 4, 6))])
def test_no_cross_gpu_reduction_no_inbox(bundle):
    assert _eligible(bundle, bundle.machine.size)[1] == {}


# ---- pipelined first step (runtime._split_plan / _k_cuts), host side
class _FakeWorld:
    def __init__(self, ngpus):
        self.ngpus = ngpus
        self.multi_gpu = ngpus > 1


def _executor(bundle, ngpus, policy="auto"):
    from paper_2203_08069_b200.runtime import _Executor
    prog, _ = plan_statement(bundle.statement, bundle.machine, bundle.distributions, bundle.schedule)
    ex = object.__new__(_Executor)
    ex.prog, ex.plan, ex.W, ex.m, ex.policy, ex.use_bcast = prog, prog.plan, _FakeWorld(ngpus), bundle.machine, \
        policy, True
    return ex


def test_k_cuts():
    from paper_2203_08069_b200.runtime import _k_cuts
    assert _k_cuts(0, 13056) == [(0, 1664), (1664, 13056)]
    assert _k_cuts(100, 300) == [(100, 300)]          # too short to split
    cuts = _k_cuts(5, 16389)
    assert cuts[0][0] == 5 and cuts[-1][1] == 16389 and (cuts[0][1] - 5) % 64 == 0


@pytest.mark.parametrize("bundle,ngpus", [(td.cannon(2, 2, dims=(4096, 4096, 4096)), 4),
                                          (td.johnson(2, 2, 2, dims=(4096, 4096, 4096)), 8),
                                          (td.johnson(2, 2, 2, dims=(4096, 4096, 4096)), 4)])
def test_first_step_pipelines_for_the_gemm_sweeps(bundle, ngpus):
    split = _executor(bundle, ngpus)._split_plan(0)
    assert split == {"kv": "k", "axis": {"A": 1, "B": 0}}


def test_first_step_stays_whole_when_it_must():
    # the exact policy (nest kernel), small transfers, single GPU
    assert _executor(td.cannon(2, 2, dims=(4096,) * 3), 4, policy="exact")._split_plan(0) is None
    assert _executor(td.cannon(2, 2, dims=(256,) * 3), 4)._split_plan(0) is None
    assert _executor(td.cannon(2, 2, dims=(4096,) * 3), 1)._split_plan(0) is None
    # MTTKRP is not a GEMM leaf
    assert _executor(td.mttkrp(2, 2, dims=(512, 32, 512, 512)), 4)._split_plan(0) is None
