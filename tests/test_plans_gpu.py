"""Launch plans (csrc/plan.cu, runtime._launch): repeated executes of one
program on one store are recorded once and replayed by td_execute_plan in
one C++ call.  Replays must give exactly the eager results (integer inputs:
bit-exact against the oracle; real inputs: bitwise equal to the eager run,
since a replay issues the same kernels on the same buffers), across the
algorithm bundles, and the C ABI must run a hand-built op array."""

import ctypes as C

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from paper_2203_08069_b200 import _native, runtime
from oracle.contractions import seq_eval

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

BUNDLES = {
    "summa": lambda: td.summa(2, 2, dims=(96, 80, 112), chunk=16),
    "cannon": lambda: td.cannon(2, 2, dims=(64, 48, 80)),
    "johnson": lambda: td.johnson(2, 2, 2, dims=(40, 36, 44)),
    "pumma": lambda: td.pumma(2, 2, dims=(48, 40, 56)),
    "solomonik": lambda: td.solomonik(2, 2, 2, dims=(32, 40, 48)),
    "cosma": lambda: td.cosma_like((2, 1, 2), (1, 1, 2), dims=(40, 32, 48)),
    "ttv": lambda: td.ttv(3, dims=(30, 20, 40)),
    "ttm2d": lambda: td.ttm2d(2, 2, dims=(16, 12, 20, 8)),
    "innerprod3": lambda: td.innerprod3(3, dims=(20, 12, 16)),
    "mttkrp": lambda: td.mttkrp(2, 2, dims=(20, 8, 16, 12)),
}


def _runs(bundle, ins, n=5):
    cin = bundle.scheduled()
    store, _ = runtime.prepare_store(cin, bundle.machine, bundle.distributions, ins)
    outs = []
    for _ in range(n):
        store.zero(bundle.statement.lhs.tensor.name)
        td.execute(cin, store)
        outs.append(store.gather(bundle.statement.lhs.tensor.name).data.copy())
    plans = [v for v in store.__dict__.get("_launch_plans", {}).values() if isinstance(v, tuple)]
    return outs, plans


@pytest.mark.parametrize("name", sorted(BUNDLES))
def test_replayed_plans_are_exact(name):
    b = BUNDLES[name]()
    ins = td.random_inputs(b.statement, 21)
    want = seq_eval(td.format_statement(b.statement), b.statement.extents, {k: v.data for k, v in ins.items()})
    outs, plans = _runs(b, ins)
    assert plans, "no plan was recorded"
    for o in outs:
        assert np.array_equal(o, np.asarray(want).reshape(o.shape))


@pytest.mark.parametrize("name", ["summa", "johnson", "mttkrp"])
def test_replay_bitwise_equals_eager_on_real_data(name):
    from oracle.generator import generate
    b = BUNDLES[name]()
    out = b.statement.lhs.tensor.name
    ins = {n: td.DenseTensor(t.dims, generate(t.dims, 9, k + 1, 1))
           for k, (n, t) in enumerate(sorted(b.statement.tensors().items())) if n != out}
    outs, plans = _runs(b, ins)
    assert plans
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_g1_replay_matches_reference_golden():
    import hashlib
    from _cases import load
    g1 = load("g1.json")
    b = td.summa(2, 2, dims=(1024,) * 3, chunk=128)
    ins = td.random_inputs(b.statement, 0)
    outs, plans = _runs(b, ins, n=4)
    assert plans
    for o in outs:
        assert hashlib.sha256(np.ascontiguousarray(o, dtype="<f8").tobytes()).hexdigest() == g1["int"]["output_sha256"]


def test_td_execute_plan_from_a_hand_built_op_array():
    """The ABI a non-Python host binds: fill C with 1, then C += A.B, as two
    td_op records in one td_execute_plan call."""
    lib = _native.load()
    m, n, k = 96, 64, 128
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = torch.empty(m, n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ops = (_native.TdOp * 2)()
    fill = [st, c.data_ptr(), m * n, _native._word(1.0, [])]
    gemm = [st, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, 1]
    for op, kind, words in ((ops[0], _native.PLAN_OPS["td_fill"], fill), (ops[1], _native.PLAN_OPS["td_dgemm"], gemm)):
        op.kind, op.nargs = kind, len(words)
        for j, w in enumerate(words):
            op.arg[j] = w
    assert lib.td_execute_plan(C.addressof(ops), 2) == 0
    torch.cuda.synchronize()
    want = 1.0 + a.cpu().numpy() @ b.cpu().numpy()
    assert np.allclose(c.cpu().numpy(), want, rtol=1e-12, atol=1e-12)
    bad = (_native.TdOp * 1)()
    bad[0].kind = 999
    assert lib.td_execute_plan(C.addressof(bad), 1) < 0
    assert b"op 0" in lib.td_last_error()


def test_grouped_gemm_equals_separate_launches():
    """td_dgemm_grouped: several GEMMs of different shapes in one launch give
    bitwise the results of separate td_dgemm calls."""
    lib = _native.load()
    shapes = [(512, 512, 128), (256, 384, 96), (64, 128, 512), (200, 120, 64)]
    st = torch.cuda.current_stream().cuda_stream
    probs = (_native.TdGemmProblem * len(shapes))()
    keep, sep = [], []
    for q, (m, n, k) in enumerate(shapes):
        a = torch.rand(m, k, dtype=torch.float64, device="cuda") - 0.5
        b = torch.rand(k, n, dtype=torch.float64, device="cuda") - 0.5
        c0 = torch.rand(m, n, dtype=torch.float64, device="cuda")
        c1 = c0.clone()
        keep += [a, b, c0, c1]
        probs[q].M, probs[q].N, probs[q].K = m, n, k
        probs[q].A, probs[q].lda, probs[q].B, probs[q].ldb = a.data_ptr(), k, b.data_ptr(), n
        probs[q].C, probs[q].ldc = c0.data_ptr(), n
        assert lib.td_dgemm(C.c_void_p(st), m, n, k, C.c_void_p(a.data_ptr()), k, C.c_void_p(b.data_ptr()), n,
                            C.c_void_p(c1.data_ptr()), n, 1) == 0
        sep.append((c0, c1))
    assert lib.td_dgemm_grouped(C.c_void_p(st), len(shapes), probs, 1) == 0
    torch.cuda.synchronize()
    for c0, c1 in sep:
        assert torch.equal(c0, c1)


@pytest.mark.parametrize("shapes", [
    [(512, 512, 512, 512)],                                        # one problem: still one folded launch
    [(512, 512, 512, 512), (512, 512, 128, 0), (256, 384, 96, 200), (200, 120, 64, 36)],
    [(300, 32, 64, 48), (128, 24, 40, 16)],                        # N <= 32 tiles
    [(128, 128, 64, 33)],                                          # K2 odd: TMA cannot take it -> two launches
])
def test_grouped_gemm_two_segments_exact(shapes):
    """td_dgemm_grouped with td_gemm_problem.K2: C (+)= A.B + A2.B2 with the
    two k-segments from unrelated buffers (a tile's two steps in different
    pieces, folded into one problem), exact on integer data, mixed with
    single-segment problems, ragged K / K2, and the fallback for operands the
    copy engine cannot address."""
    lib = _native.load()
    st = torch.cuda.current_stream().cuda_stream
    probs = (_native.TdGemmProblem * len(shapes))()
    keep, want = [], []
    g = torch.Generator(device="cuda").manual_seed(5)
    ints = lambda *s: torch.randint(-4, 5, s, generator=g, device="cuda").to(torch.float64)  # noqa: E731
    for q, (m, n, k, k2) in enumerate(shapes):
        a, b, c = ints(m, k), ints(k, n), ints(m, n)
        a2, b2 = ints(m, max(k2, 1)), ints(max(k2, 1), n)
        keep += [a, b, c, a2, b2]
        want.append(c.cpu().numpy() + a.cpu().numpy() @ b.cpu().numpy()
                    + (a2.cpu().numpy() @ b2.cpu().numpy() if k2 else 0))
        probs[q].M, probs[q].N, probs[q].K = m, n, k
        probs[q].A, probs[q].lda, probs[q].B, probs[q].ldb = a.data_ptr(), k, b.data_ptr(), n
        probs[q].C, probs[q].ldc = c.data_ptr(), n
        if k2:
            probs[q].K2, probs[q].A2, probs[q].lda2 = k2, a2.data_ptr(), a2.shape[1]
            probs[q].B2, probs[q].ldb2 = b2.data_ptr(), n
    assert lib.td_dgemm_grouped(C.c_void_p(st), len(shapes), probs, 1) == 0, lib.td_last_error()
    torch.cuda.synchronize()
    for q, w in enumerate(want):
        assert np.array_equal(keep[5 * q + 2].cpu().numpy(), w), shapes[q]


def test_plan_cache_follows_the_store_and_switches():
    """A plan is keyed on the program, the output's freshness, the pieces'
    addresses and the streams: re-placing an input (new buffers) records a
    new plan; PLANS = False runs the Python loop; a Python plugin is never
    recorded; all give the oracle's values."""
    b = BUNDLES["summa"]()
    ins = td.random_inputs(b.statement, 3)
    want = seq_eval(td.format_statement(b.statement), b.statement.extents, {k: v.data for k, v in ins.items()})
    cin = b.scheduled()
    store, _ = runtime.prepare_store(cin, b.machine, b.distributions, ins)

    def run():
        store.zero("C")
        td.execute(cin, store)
        return store.gather("C").data

    for _ in range(3):
        assert np.array_equal(run(), want)
    plans = lambda: [v for v in store.__dict__["_launch_plans"].values() if isinstance(v, tuple)]  # noqa: E731
    assert len(plans()) == 1
    ins2 = td.random_inputs(b.statement, 4)
    store.place("A", ins2["A"], b.distributions["A"])          # new buffers for A
    want2 = seq_eval(td.format_statement(b.statement), b.statement.extents,
                     {"A": ins2["A"].data, "B": ins["B"].data})
    for _ in range(3):
        assert np.array_equal(run(), want2)
    assert len(plans()) == 2
    runtime.PLANS = False
    try:
        assert np.array_equal(run(), want2)
    finally:
        runtime.PLANS = True

    from oracle.ref_leaf import NAME, innermost_vars, numpy_leaf
    td.register_leaf_kernel(NAME, numpy_leaf)
    cin3 = b.schedule.substitute_leaf(innermost_vars(cin), NAME).apply(td.lower_to_cin(b.statement))
    store3, _ = runtime.prepare_store(cin3, b.machine, b.distributions, ins)
    for _ in range(3):
        store3.zero("C")
        td.execute(cin3, store3)
        assert np.array_equal(store3.gather("C").data, want)
    assert not any(isinstance(v, tuple) for v in store3.__dict__.get("_launch_plans", {}).values())
