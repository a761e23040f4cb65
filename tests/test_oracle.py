"""The CPU oracle is pinned before it is trusted (CPU only):
* reference known answers (pkg/tests/test_ir.py:65-103) -> kats.json;
* integer outputs of every golden bundle (made by running `tendist`);
* the input generator's numpy twin is self-consistent;
* random_inputs reproduces the reference's Mersenne-Twister stream."""

import hashlib

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from oracle import contractions as ref
from oracle.generator import generate, generate_box, values

from _cases import build, case_id, load

BUNDLES = load("bundles.json")


def test_kats():
    for kat in load("kats.json"):
        got = ref.seq_eval(kat["statement"], kat["extents"], kat["inputs"])
        assert np.array_equal(np.asarray(got), np.asarray(kat["output"], float)), kat["statement"]


@pytest.mark.parametrize("fix", BUNDLES, ids=[case_id(f["case"]) for f in BUNDLES])
def test_oracle_matches_reference_bundle_outputs(fix):
    b = build(td, fix["case"])
    ins = td.random_inputs(b.statement, seed=13)
    h = hashlib.sha256()
    for name in sorted(ins):
        h.update(name.encode())
        h.update(np.ascontiguousarray(ins[name].data).tobytes())
    assert h.hexdigest() == fix["input_digest"]
    got = ref.seq_eval(td.format_statement(b.statement), b.statement.extents,
                       {n: t.data for n, t in ins.items()})
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(fix["output"]))


def test_contractions_agree_with_seq_eval():
    rng = np.random.default_rng(0)
    a, b = rng.integers(-4, 5, (5, 7)).astype(float), rng.integers(-4, 5, (7, 3)).astype(float)
    assert np.array_equal(ref.gemm(a, b), ref.seq_eval("C(i,j) = A(i,k) * B(k,j)",
                                                       {"i": 5, "j": 3, "k": 7}, {"A": a, "B": b}))
    t, c = rng.integers(-4, 5, (3, 4, 5)).astype(float), rng.integers(-4, 5, (5,)).astype(float)
    assert np.array_equal(ref.ttv(t, c), ref.seq_eval("A(i,j) = B(i,j,k) * c(k)",
                                                      {"i": 3, "j": 4, "k": 5}, {"B": t, "c": c}))
    m = rng.integers(-4, 5, (5, 2)).astype(float)
    assert np.array_equal(ref.ttm(t, m), ref.seq_eval("Y(i,j,l) = B(i,j,k) * C(k,l)",
                                                      {"i": 3, "j": 4, "k": 5, "l": 2}, {"B": t, "C": m}))
    d = rng.integers(-4, 5, (5, 2)).astype(float)
    cm = rng.integers(-4, 5, (4, 2)).astype(float)
    assert np.array_equal(ref.mttkrp(t, cm, d), ref.seq_eval(
        "A(i,j) = B(i,k,l) * C(k,j) * D(l,j)", {"i": 3, "j": 2, "k": 4, "l": 5},
        {"B": t, "C": cm, "D": d}))
    assert ref.innerprod(t, t) == ref.seq_eval("a = B(i,j,k) * C(i,j,k)", {"i": 3, "j": 4, "k": 5},
                                               {"B": t, "C": t})


def test_generator_twin():
    full = generate((5, 6, 7), 3, 9, 0)
    assert full.min() >= -4 and full.max() <= 4 and set(np.unique(full)) <= set(range(-4, 5))
    box = generate_box((5, 6, 7), (1, 2, 3), (2, 3, 4), 3, 9, 0)
    assert np.array_equal(box, full[1:3, 2:5, 3:7])
    u = generate((1000,), 1, 1, 1)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.1
    assert values(np.arange(4), 3, 9, 0).tolist() == full.reshape(-1)[:4].tolist()
    assert not np.array_equal(generate((64,), 3, 9, 0), generate((64,), 3, 8, 0))
