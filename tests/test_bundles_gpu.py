"""End-to-end parity on the B200: every golden bundle runs through
`AlgorithmBundle.run` (placement in HBM, NCCL/alias transfers, native leaves,
ordered commits) and must reproduce the reference.

* integer inputs (the reference's own random_inputs, seed 13): bit-exact in
  both leaf policies ("auto" = native DMMA/stream kernels, "exact" = nest kernel);
* real-valued inputs (oracle/generator.py, uniform(-1,1)): the "exact" policy
  matches the reference's output bit for bit -- same per-point accumulation
  order and the same task-order reduction commits -- and the "auto" policy is
  within gamma_K * (|A||B|)-style bounds of a longdouble evaluation.
"""

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from oracle.contractions import seq_eval
from oracle.generator import generate

from _cases import build, case_id, load

pytestmark = pytest.mark.gpu
BUNDLES = load("bundles.json")
U = 2.0 ** -53


def _digest(inputs):
    import hashlib
    h = hashlib.sha256()
    for name in sorted(inputs):
        h.update(name.encode())
        h.update(np.ascontiguousarray(inputs[name].data).tobytes())
    return h.hexdigest()


def _real_inputs(b, seed=13):
    out = {}
    for k, name in enumerate(b.input_names):
        dims = b.statement.tensors()[name].dims
        out[name] = td.DenseTensor(dims, generate(dims, seed, k + 1, 1))
    return out


@pytest.mark.parametrize("fix", BUNDLES, ids=[case_id(f["case"]) for f in BUNDLES])
@pytest.mark.parametrize("policy", ["auto", "exact"])
def test_bundle_integer_bit_exact(fix, policy):
    b = build(td, fix["case"])
    res, inputs = b.run(seed=13, leaf_policy=policy)
    assert _digest(inputs) == fix["input_digest"]          # same inputs as the reference
    want = np.asarray(fix["output"], dtype=np.float64).reshape(fix["dims"])
    assert np.array_equal(res.output.data, want)
    if b.signature is not None:
        b.signature(res.trace)  # runs; the ledger itself is pinned in test_planner


@pytest.mark.parametrize("fix", BUNDLES, ids=[case_id(f["case"]) for f in BUNDLES])
def test_bundle_real_exact_policy_bitwise(fix):
    b = build(td, fix["case"])
    res, _ = b.run(inputs=_real_inputs(b), leaf_policy="exact")
    want = np.array([float.fromhex(x) for x in fix["real_output_hex"]]).reshape(fix["dims"])
    assert np.array_equal(res.output.data, want)


@pytest.mark.parametrize("fix", BUNDLES, ids=[case_id(f["case"]) for f in BUNDLES])
def test_bundle_real_auto_policy_tolerance(fix):
    b = build(td, fix["case"])
    ins = _real_inputs(b)
    res, _ = b.run(inputs=ins, leaf_policy="auto")
    stmt = b.statement
    from paper_2203_08069_b200.ir import format_statement
    arrays = {n: t.data for n, t in ins.items()}
    want = seq_eval(format_statement(stmt), stmt.extents, arrays)
    absval = seq_eval(format_statement(stmt), stmt.extents, {n: np.abs(a) for n, a in arrays.items()})
    K = 1
    for v in stmt.reduction_vars:
        K *= stmt.extents[v]
    gam = 2 * (K + 2) * U / (1 - (K + 2) * U)   # both evaluations carry rounding error
    assert np.all(np.abs(res.output.data - want) <= gam * absval + 1e-300)


def test_kats_sequential_evaluate():
    for kat in load("kats.json"):
        stmt = td.parse_statement(kat["statement"], kat["extents"])
        ins = {n: td.DenseTensor(np.asarray(v, float).shape, np.asarray(v, float))
               for n, v in kat["inputs"].items()}
        got = td.sequential_evaluate(stmt, ins)
        assert np.array_equal(got.data, np.asarray(kat["output"], float)), kat["statement"]


CHAINS = load("chains.json")


@pytest.mark.parametrize("k", range(0, len(CHAINS), 1))
def test_schedule_chain_interpret_bitwise(k):
    """The reference's schedule fuzz (test_acceptance.py:67-119): any chain
    of split/divide/reorder/rotate evaluated by the GPU nest kernel gives
    the reference interpreter's bits on real-valued inputs."""
    ch = CHAINS[k]
    stmt = td.parse_statement(ch["statement"], ch["extents"])
    cin = td.lower_to_cin(stmt)
    for kind, args in ch["commands"]:
        if kind == "split":
            cin = td.split(cin, *args)
        elif kind == "divide":
            cin = td.divide(cin, *args)
        elif kind == "reorder":
            cin = td.reorder(cin, args[0])
        else:
            cin = td.rotate(cin, args[0], tuple(args[1]), args[2])
    ins = {}
    for q, name in enumerate(sorted(n for n in stmt.tensors() if n != stmt.lhs.tensor.name)):
        dims = stmt.tensors()[name].dims
        ins[name] = td.DenseTensor(dims, generate(dims, ch["seed"], q + 1, 1))
    got = td.interpret(cin, ins)[stmt.lhs.tensor.name]
    want = np.array([float.fromhex(x) for x in ch["output_hex"]]).reshape(ch["dims"])
    assert np.array_equal(got.data, want)
