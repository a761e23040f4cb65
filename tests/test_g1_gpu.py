"""BASELINE config G1 on the B200 against the reference's own output.

G1 = SUMMA 1024^3 on a 2x2 grid, chunk 128 (reference `algorithms.py:88-106`),
the "results oracle" configuration.  tests/golden/g1.json holds what the
reference's `run_statement` produced for it (tests/golden/make_g1.py):
  * integer inputs (the reference's `random_inputs(stmt, 0)`): the B200 output
    must have the same sha256 -- bit-exact, in both leaf policies, eagerly and
    replayed from a captured CUDA graph;
  * real inputs (uniform(-1,1), oracle/generator.py): the sampled rows must be
    within 2*gamma_K*(|A||B|) of the reference's (K = 1024; both sides carry
    at most gamma_K of rounding error) and within the north star's 1e-10*K.
"""

import hashlib

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from oracle.generator import generate

from _cases import load

pytestmark = pytest.mark.gpu
G1 = load("g1.json")
U = 2.0 ** -53


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def _bundle():
    cfg = G1["config"]
    return td.summa(*cfg["grid"], dims=tuple(cfg["dims"]), chunk=cfg["chunk"])


@pytest.mark.parametrize("policy", ["auto", "exact"])
def test_g1_integer_output_is_the_references(policy):
    res, ins = _bundle().run(seed=0, leaf_policy=policy)
    assert {n: _sha(t.data) for n, t in ins.items()} == G1["int"]["input_sha256"]
    assert _sha(res.output.data) == G1["int"]["output_sha256"]
    assert len(res.trace.events) == G1["int"]["events"]


def test_g1_integer_graph_replay_is_the_references():
    from paper_2203_08069_b200.runtime import CapturedLaunch, prepare_store
    b = _bundle()
    ins = td.random_inputs(b.statement, 0)
    cin = b.scheduled()
    store, out = prepare_store(cin, b.machine, b.distributions, ins)
    cap = CapturedLaunch(cin, store)
    for _ in range(3):
        cap.replay()
    assert _sha(store.gather(out).data) == G1["int"]["output_sha256"]


def test_g1_real_within_gamma_of_the_reference():
    n = G1["config"]["dims"][0]
    a, b = generate((n, n), 0, 1, 1), generate((n, n), 0, 2, 1)
    res, _ = _bundle().run(inputs={"A": td.DenseTensor((n, n), a), "B": td.DenseTensor((n, n), b)})
    rows = G1["real"]["rows"]
    got = res.output.data[rows]
    ref = np.array([[float.fromhex(x) for x in r] for r in G1["real"]["row_hex"]])
    bound = np.abs(a[rows]) @ np.abs(b)
    gam = n * U / (1 - n * U)
    err = np.abs(got - ref)
    assert np.all(err <= 2 * gam * bound)
    assert np.all(err <= 1e-10 * n * bound)


def test_g1_reference_contract_plugin_runs_unchanged():
    """The drop-in boundary: a leaf written against the REFERENCE's plugin
    contract (oracle/ref_leaf.py: host DenseTensors in global coordinates,
    in-place writes into a full-size out_store; reference cin.py:359-379) is
    registered with the plain `register_leaf_kernel(name, fn)` call and
    substituted with `Schedule.substitute_leaf` exactly as on tendist -- and
    reproduces the reference's own G1 output bit for bit."""
    from oracle.ref_leaf import NAME, innermost_vars, numpy_leaf
    td.register_leaf_kernel(NAME, numpy_leaf)
    b = _bundle()
    sched = b.schedule.substitute_leaf(innermost_vars(b.scheduled()), NAME)
    ins = td.random_inputs(b.statement, 0)
    res = td.run_statement(b.statement, b.machine, b.distributions, ins, sched)
    assert _sha(res.output.data) == G1["int"]["output_sha256"]
    assert len(res.trace.events) == G1["int"]["events"]


@pytest.mark.parametrize("case", ["summa", "cannon", "johnson", "ttv", "mttkrp"])
def test_reference_contract_plugin_on_bundles(case):
    """Same host-contract plugin on other bundles (ragged shapes), against the
    GPU's exact-order interpreter."""
    from oracle.ref_leaf import NAME, innermost_vars, numpy_leaf
    td.register_leaf_kernel(NAME, numpy_leaf)
    b = {"summa": lambda: td.summa(2, 2, dims=(13, 11, 17), chunk=3),
         "cannon": lambda: td.cannon(2, 2, dims=(10, 9, 7)),
         "johnson": lambda: td.johnson(2, 2, 2, dims=(9, 7, 11)),
         "ttv": lambda: td.ttv(3, dims=(7, 5, 6)),
         "mttkrp": lambda: td.mttkrp(2, 2, dims=(6, 5, 7, 3))}[case]()
    ins = td.random_inputs(b.statement, 11)
    sched = b.schedule.substitute_leaf(innermost_vars(b.scheduled()), NAME)
    got = td.run_statement(b.statement, b.machine, b.distributions, ins, sched).output.data
    want = td.sequential_evaluate(b.statement, ins).data
    assert np.array_equal(got, want)
