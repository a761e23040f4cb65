"""Generic pairwise contractions on the DMMA GEMM (leaves._contract).

Any statement X(...) = P(...) * Q(...) with at least one contracted index --
transposed GEMMs, GEMV in either orientation, batched products, TTM / TTV on
any mode, scalar bilinear forms -- runs as a (batched) GEMM with operands read
in place or packed by one strided copy.  Integer inputs: results must equal
the oracle bit for bit, on one processor and distributed over a 2x2 grid."""

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from oracle.contractions import seq_eval

pytestmark = pytest.mark.gpu

STATEMENTS = [
    ("C(i, j) = A(k, i) * B(k, j)", {"i": 37, "j": 29, "k": 41}),
    ("C(i, j) = A(i, k) * B(j, k)", {"i": 33, "j": 70, "k": 19}),
    ("y(i) = A(i, j) * x(j)", {"i": 65, "j": 47}),
    ("y(j) = A(i, j) * x(i)", {"i": 65, "j": 47}),
    ("C(b, i, j) = A(b, i, k) * B(b, k, j)", {"b": 5, "i": 17, "j": 23, "k": 11}),
    ("Y(i, l, k) = B(i, j, k) * C(j, l)", {"i": 6, "j": 9, "k": 7, "l": 5}),
    ("A(j, k) = B(i, j, k) * c(i)", {"i": 13, "j": 8, "k": 10}),
    ("a = A(i, j) * B(j, i)", {"i": 21, "j": 17}),
    ("Y(l, i) = C(k, l) * B(i, k)", {"i": 31, "j": 1, "k": 25, "l": 9}),
]


def _inputs(stmt, seed):
    rng = np.random.default_rng(seed)
    out = stmt.lhs.tensor.name
    return {n: td.DenseTensor(t.dims, rng.integers(-4, 5, size=t.dims).astype(float))
            for n, t in stmt.tensors().items() if n != out}


@pytest.mark.parametrize("text,ext", STATEMENTS, ids=[s for s, _ in STATEMENTS])
def test_contraction_single_processor(text, ext):
    from paper_2203_08069_b200 import leaves
    stmt = td.parse_statement(text, ext)
    ins = _inputs(stmt, 1)
    machine = td.grid(1)
    dists = {n: td.TensorDistribution(t.dims, machine, [(tuple("xyzw"[:len(t.dims)]),
                                                         ("x",) if t.dims else (0,))])
             for n, t in stmt.tensors().items()}
    first = stmt.var_order[0]
    sched = td.schedule().divide(first, "t_o", "t_i", 1).distribute("t_o")
    leaves.reset_stats()
    res = td.run_statement(stmt, machine, dists, ins, sched)
    assert leaves.STATS["contract"] + leaves.STATS["dgemm"] + leaves.STATS["ttv"] + leaves.STATS["ttm"] \
        + leaves.STATS["innerprod"] >= 1 and leaves.STATS["nest"] == 0, leaves.STATS
    want = seq_eval(text, ext, {n: t.data for n, t in ins.items()})
    assert np.array_equal(res.output.data, np.asarray(want))


@pytest.mark.parametrize("text,ext", STATEMENTS[:7], ids=[s for s, _ in STATEMENTS[:7]])
def test_contraction_distributed_views(text, ext):
    """2x2 grid, the first two output variables distributed: leaves read
    strided sub-views of the resident tiles and of fetched temporaries."""
    from paper_2203_08069_b200 import leaves
    stmt = td.parse_statement(text, ext)
    ins = _inputs(stmt, 2)
    machine = td.grid(2, 2)
    out = stmt.lhs.tensor.name
    f = stmt.free_vars
    if len(f) < 2:
        pytest.skip("needs two free variables to distribute")
    dists = {}
    for n, t in stmt.tensors().items():
        names = tuple("xyzw"[:len(t.dims)])
        ys = ("x", "y") if len(names) >= 2 else (("x", "*") if names else (0, 0))
        dists[n] = td.TensorDistribution(t.dims, machine, [(names, ys)])
    sched = (td.schedule().divide(f[0], "fo", "fi", 2).divide(f[1], "go", "gi", 2)
             .reorder("fo", "go", "fi", "gi").distribute("fo").distribute("go")
             .communicate([n for n in stmt.tensors() if n != out], "go"))
    leaves.reset_stats()
    res = td.run_statement(stmt, machine, dists, ins, sched)
    want = seq_eval(text, ext, {n: t.data for n, t in ins.items()})
    assert np.array_equal(res.output.data, np.asarray(want))
    assert leaves.STATS["nest"] == 0, leaves.STATS
