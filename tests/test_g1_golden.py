"""CPU pins of the G1 golden fixture (tests/golden/g1.json, made by running
the reference: tests/golden/make_g1.py).

* this package's `random_inputs(stmt, 0)` reproduces the reference's inputs
  (same Mersenne-Twister stream, reference `algorithms.py:54-68`) byte for byte;
* the fixture's sampled rows / column sums equal A @ B of those inputs
  (integers: exact), and its real-valued rows are within gamma_K of a
  longdouble product of the generator's inputs -- so the fixture itself is
  consistent before the GPU tests compare against it.
"""

import hashlib

import numpy as np

import paper_2203_08069_b200 as td
from oracle.generator import generate

from _cases import load

G1 = load("g1.json")
U = 2.0 ** -53


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def test_g1_inputs_are_the_references():
    cfg = G1["config"]
    b = td.summa(*cfg["grid"], dims=tuple(cfg["dims"]), chunk=cfg["chunk"])
    ins = td.random_inputs(b.statement, 0)
    assert {n: _sha(t.data) for n, t in ins.items()} == G1["int"]["input_sha256"]
    c = ins["A"].data @ ins["B"].data
    assert _sha(c) == G1["int"]["output_sha256"]
    for r, row in zip(G1["int"]["rows"], G1["int"]["row_values"]):
        assert np.array_equal(c[r], np.asarray(row))
    assert np.array_equal(c.sum(axis=0), np.asarray(G1["int"]["col_sums"]))


def test_g1_real_rows_within_gamma():
    n = G1["config"]["dims"][0]
    a, b = generate((n, n), 0, 1, 1), generate((n, n), 0, 2, 1)
    assert _sha(a) == G1["real"]["input_sha256"]["A"] and _sha(b) == G1["real"]["input_sha256"]["B"]
    rows = G1["real"]["rows"]
    exact = a[rows].astype(np.longdouble) @ b.astype(np.longdouble)
    bound = np.abs(a[rows]) @ np.abs(b)
    gam = n * U / (1 - n * U)
    got = np.array([[float.fromhex(x) for x in r] for r in G1["real"]["row_hex"]])
    assert np.all(np.abs(got - exact).astype(np.float64) <= gam * bound)
