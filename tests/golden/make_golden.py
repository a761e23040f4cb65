"""Generate golden fixtures by running the REFERENCE (`tendist`) itself.

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes (committed, small):
  * ledgers.json  -- for every case: the reference's full CommEvent ledger,
    memory high-water per processor, step count, requirement records, stats
    totals / per-step aggregates (pins planner.py's ledger to the reference);
  * bundles.json  -- bundle outputs of `AlgorithmBundle.run(seed)` on the
    reference's own integer inputs, plus a digest of those inputs (pins the
    GPU results and random_inputs), and reference outputs on real-valued
    inputs from oracle/generator.py (pins the exact-order path bit for bit);
  * chains.json   -- random schedule chains (the reference's criterion-02
    fuzz, test_acceptance.py:67-119) with the reference interpreter's output
    for each, for the GPU nest evaluator.
Nothing in the GPU tests, smoke() or bench.py reads /root/reference.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import tendist  # noqa: E402  (the reference, read-only)
from tendist.cin import interpret, lower_to_cin  # noqa: E402
from tendist.errors import ConfigError, NotContiguousNest  # noqa: E402
from tendist.scheduling import divide, reorder, rotate, split  # noqa: E402

from oracle.generator import generate  # noqa: E402

# (bundle function name, positional args, keyword args)
CASES = [
    ("summa", [2, 2], {"dims": [8, 8, 8], "chunk": 2}),
    ("summa", [2, 2], {"dims": [5, 7, 6], "chunk": 2}),
    ("summa", [4, 2], {"dims": [8, 8, 8], "chunk": 2}),
    ("summa", [2, 1], {"dims": [12, 10, 16], "chunk": 2}),
    ("summa", [2, 2], {"dims": [32, 24, 40], "chunk": 8}),
    ("cannon", [2, 2], {"dims": [8, 8, 8]}),
    ("cannon", [2, 2], {"dims": [4, 4, 4]}),
    ("cannon", [3, 3], {"dims": [7, 7, 5]}),
    ("cannon", [3, 3], {"dims": [6, 6, 6]}),
    ("cannon", [1, 1], {"dims": [9, 11, 7]}),
    ("pumma", [2, 2], {"dims": [8, 8, 8]}),
    ("pumma", [2, 2], {"dims": [5, 5, 3]}),
    ("pumma", [3, 3], {"dims": [6, 6, 6]}),
    ("johnson", [2, 2, 2], {"dims": [8, 8, 8]}),
    ("johnson", [2, 2, 2], {"dims": [7, 5, 3]}),
    ("johnson", [1, 1, 1], {"dims": [5, 6, 7]}),
    ("solomonik", [2, 2, 2], {"dims": [8, 8, 8]}),
    ("solomonik", [2, 2, 2], {"dims": [5, 7, 9]}),
    ("solomonik", [4, 4, 1], {"dims": [8, 8, 8]}),
    ("solomonik", [4, 4, 2], {"dims": [8, 8, 8]}),
    ("solomonik", [4, 4, 4], {"dims": [8, 8, 8]}),
    ("cosma_like", [[2, 2, 1], [1, 1, 2]], {"dims": [8, 8, 8]}),
    ("cosma_like", [[2, 2, 1], [1, 1, 2]], {"dims": [5, 4, 7]}),
    ("cosma_like", [[1, 1, 2], [1, 1, 1]], {"dims": [6, 5, 8]}),
    ("summa_hier", [], {"dims": [8, 8, 8], "chunk": 2}),
    ("summa_hier", [], {"dims": [7, 6, 5], "chunk": 3}),
    ("ttv", [2], {}),
    ("ttv", [3], {"dims": [7, 5, 4]}),
    ("ttv", [4], {"dims": [9, 6, 8]}),
    ("ttm", [2], {}),
    ("ttm", [3], {"dims": [5, 4, 7, 3]}),
    ("innerprod", [2], {}),
    ("innerprod", [3], {"dims": [7, 5]}),
    ("innerprod", [4], {"dims": [8, 6]}),
    ("mttkrp", [2, 2], {}),
    ("mttkrp", [2, 2], {"dims": [5, 3, 7, 2]}),
    ("mttkrp", [2, 1], {"dims": [6, 5, 4, 3]}),
    ("mttkrp", [1, 1], {"dims": [4, 5, 6, 7]}),
    # empty trailing blocks / idle processors (ceil-division blocks)
    ("summa", [4, 1], {"dims": [5, 7, 6], "chunk": 4}),
    ("cannon", [3, 3], {"dims": [4, 4, 4]}),
    ("johnson", [2, 2, 2], {"dims": [3, 1, 1]}),
    ("ttv", [4], {"dims": [3, 2, 5]}),
    ("innerprod", [4], {"dims": [2, 3]}),
    ("mttkrp", [3, 2], {"dims": [2, 3, 1, 4]}),
    ("ttm", [4], {"dims": [3, 1, 2, 2]}),
]

SEED = 13


def _box(r):
    return [list(r.lo), list(r.hi)]


def _ev(e):
    return [e.timestep, list(e.src), list(e.dst), e.tensor, _box(e.rect), e.elements, e.kind, e.phase]


def _digest(inputs):
    h = hashlib.sha256()
    for name in sorted(inputs):
        h.update(name.encode())
        h.update(np.ascontiguousarray(inputs[name].data).tobytes())
    return h.hexdigest()


def ledgers_and_outputs():
    ledgers, outputs = [], []
    for fn, args, kw in CASES:
        bundle = getattr(tendist, fn)(*[tuple(a) if isinstance(a, list) else a for a in args],
                                      **{k: tuple(v) if isinstance(v, list) else v for k, v in kw.items()})
        res, inputs = bundle.run(seed=SEED)
        tr = res.trace
        st = tr.stats()
        ledgers.append({
            "case": [fn, args, kw],
            "events": [_ev(e) for e in tr.events],
            "memory": [[list(p), v] for p, v in tr.memory.items()],
            "num_steps": tr.num_steps,
            "requirements": [[list(r.coord), r.step, r.tensor, _box(r.rect), r.scope] for r in tr.requirements],
            "totals": st["totals"],
            "per_step": st["per_step"],
            "per_edge": st["per_edge"],
            "launches": st["launches"],
            "residency_out": [[list(p), [_box(r) for r in rs]]
                              for p, rs in res.store[res.output_name].residency.items()],
            "signature": (bundle.signature(tr) if bundle.signature else None),
        })
        # real-valued inputs from the shared generator: reference bits to match exactly
        real_inputs = {}
        for k, name in enumerate(bundle.input_names):
            dims = bundle.statement.tensors()[name].dims
            real_inputs[name] = tendist.DenseTensor(dims, generate(dims, SEED, k + 1, 1)) if dims else \
                tendist.DenseTensor((), generate((), SEED, k + 1, 1))
        res_real, _ = bundle.run(inputs=real_inputs)
        outputs.append({
            "case": [fn, args, kw],
            "input_digest": _digest(inputs),
            "dims": list(res.output.dims),
            "output": res.output.data.reshape(-1).tolist(),
            "real_output_hex": [float(x).hex() for x in res_real.output.data.reshape(-1)],
        })
    return ledgers, outputs


def _chain_vars(cin):
    from tendist.cin import body_of
    node = body_of(cin)
    out = []
    while hasattr(node, "var"):
        out.append(node.var)
        node = node.body
    return out


STATEMENTS = [
    ("C(i, j) = A(i, k) * B(k, j)", {"i": 4, "j": 5, "k": 6}),
    ("A(i, j) = B(i, j, k) * c(k)", {"i": 3, "j": 4, "k": 5}),
    ("Y(i, j, l) = B(i, j, k) * C(k, l)", {"i": 3, "j": 2, "k": 4, "l": 3}),
    ("A(i, j) = B(i, k, l) * C(k, j) * D(l, j)", {"i": 3, "j": 2, "k": 4, "l": 3}),
    ("D(i, j) = A(i, j) + B(i, j) * 2", {"i": 5, "j": 3}),
]


def _encode_cmd(cmd):
    return cmd


def chains(n_rounds=60):
    """Random split/divide/reorder/rotate chains (reference test_acceptance.py:67-119)."""
    rng = random.Random(20261018)
    out = []
    for round_ in range(n_rounds):
        for text, ext in STATEMENTS:
            stmt = tendist.parse_statement(text, ext)
            real = {}
            for k, name in enumerate(sorted(n for n in stmt.tensors() if n != stmt.lhs.tensor.name)):
                dims = stmt.tensors()[name].dims
                real[name] = tendist.DenseTensor(dims, generate(dims, round_, k + 1, 1))
            cin = lower_to_cin(stmt)
            cmds = []
            fresh = itertools.count()
            for _ in range(rng.randint(1, 5)):
                names = _chain_vars(cin)
                kind = rng.choice(["split", "divide", "reorder", "rotate"])
                try:
                    if kind in ("split", "divide"):
                        n = next(fresh)
                        args = [rng.choice(names), f"{kind[0]}{n}o", f"{kind[0]}{n}i", rng.randint(1, 3)]
                        cin = (split if kind == "split" else divide)(cin, *args)
                    elif kind == "reorder":
                        if len(names) < 2:
                            continue
                        take = rng.randint(2, min(3, len(names)))
                        at = rng.randrange(len(names) - take + 1)
                        win = names[at:at + take]
                        rng.shuffle(win)
                        args = [win]
                        cin = reorder(cin, win)
                    else:
                        if len(names) < 2:
                            continue
                        at = rng.randrange(1, len(names))
                        n = next(fresh)
                        over = rng.sample(names[:at], rng.randint(1, min(2, at)))
                        args = [names[at], over, f"r{n}"]
                        cin = rotate(cin, *args)
                    cmds.append([kind, args])
                except (NotContiguousNest, ConfigError):
                    continue
            got = interpret(cin, real)[stmt.lhs.tensor.name]
            out.append({"statement": text, "extents": ext, "seed": round_, "commands": cmds,
                        "output_hex": [float(x).hex() for x in got.data.reshape(-1)],
                        "dims": list(got.dims)})
    return out


KATS = [
    # reference pkg/tests/test_ir.py:65-103 known answers
    {"statement": "C(i, j) = A(i, k) * B(k, j)", "extents": {"i": 2, "j": 2, "k": 2},
     "inputs": {"A": [[1, 2], [3, 4]], "B": [[5, 6], [7, 8]]}, "output": [[19, 22], [43, 50]]},
    {"statement": "A(i, j) = B(i, j, k) * c(k)", "extents": {"i": 2, "j": 2, "k": 2},
     "inputs": {"B": [[[0, 1], [2, 3]], [[4, 5], [6, 7]]], "c": [1, 2]}, "output": [[2, 8], [14, 20]]},
    {"statement": "a = A(i, j) * B(i, j)", "extents": {"i": 2, "j": 2},
     "inputs": {"A": [[1, 2], [3, 4]], "B": [[5, 6], [7, 8]]}, "output": 70},
    {"statement": "a = c(k) * o(k)", "extents": {"k": 3},
     "inputs": {"c": [1e16, -1e16, 1.5], "o": [1, 1, 1]}, "output": 1.5},
    {"statement": "D(i) = A(i) + B(i) * C(i)", "extents": {"i": 2},
     "inputs": {"A": [1, 2], "B": [3, 4], "C": [5, 6]}, "output": [16, 26]},
    {"statement": "D(i) = (A(i) + B(i)) * C(i)", "extents": {"i": 2},
     "inputs": {"A": [1, 2], "B": [3, 4], "C": [5, 6]}, "output": [20, 36]},
    {"statement": "D(i) = A(i) * 2 + 1", "extents": {"i": 3}, "inputs": {"A": [0, 1, 2]},
     "output": [1, 3, 5]},
]


def main():
    ledgers, outputs = ledgers_and_outputs()
    with open(os.path.join(HERE, "ledgers.json"), "w") as fh:
        json.dump(ledgers, fh, separators=(",", ":"))
    with open(os.path.join(HERE, "bundles.json"), "w") as fh:
        json.dump(outputs, fh, separators=(",", ":"))
    with open(os.path.join(HERE, "chains.json"), "w") as fh:
        json.dump(chains(), fh, separators=(",", ":"))
    # verify the KATs against the reference too, then store them
    for kat in KATS:
        stmt = tendist.parse_statement(kat["statement"], kat["extents"])
        ins = {n: tendist.DenseTensor(np.asarray(v, float).shape, np.asarray(v, float))
               for n, v in kat["inputs"].items()}
        got = tendist.sequential_evaluate(stmt, ins)
        assert np.array_equal(got.data, np.asarray(kat["output"], float)), kat
    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(KATS, fh, indent=1)
    print("wrote", len(ledgers), "ledgers,", len(outputs), "bundle outputs")


if __name__ == "__main__":
    main()
