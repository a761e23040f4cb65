"""Golden fixture of BASELINE config G1 made by running the REFERENCE itself.

G1 = SUMMA 1024^3 on a 2x2 grid, chunk 128 (reference `algorithms.py:88-106`),
the reference's "results oracle" configuration.  The reference's shipped leaf
(the per-point interpreter, `cin.py:399-417`) would need ~4 h here, so the
run substitutes the numpy/BLAS leaf of `oracle/ref_leaf.py` through the
reference's own plugin API (`register_leaf_kernel` + `Schedule.substitute_leaf`,
`cin.py:344-379`, `scheduling.py:263-299`); everything else -- placement,
task grid, steps, commits in task order -- is tendist's `run_statement`.

Two input sets:
  * "int":  the reference's own `random_inputs(stmt, seed=0)` (integers in
    [-4, 4], `algorithms.py:54-68`): every partial sum is exact, so the B200
    output must match this output's sha256 bit for bit;
  * "real": uniform(-1, 1) from `oracle/generator.py` (seed 0, tensor ids 1/2
    for A/B, mode 1): the B200 output must lie within 2*gamma_K*(|A||B|) of
    the sampled rows stored here (gamma_K = K u / (1 - K u), u = 2^-53, K = 1024).

Run in the build container (the staged reference in oracle/_ref or the
checkout):   python tests/golden/make_g1.py      -> tests/golden/g1.json
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.generator import generate  # noqa: E402
from oracle.ref_leaf import NAME, innermost_vars, numpy_leaf  # noqa: E402
from oracle.reference import tendist  # noqa: E402

N, CHUNK = 1024, 128
ROWS = [0, 1, 255, 256, 511, 512, 700, 767, 768, 1023]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def run(td, inputs):
    b = td.summa(2, 2, dims=(N, N, N), chunk=CHUNK)
    cin = b.schedule.apply(td.lower_to_cin(b.statement))
    sched = b.schedule.substitute_leaf(innermost_vars(cin), NAME)
    t0 = time.perf_counter()
    res = td.run_statement(b.statement, b.machine, b.distributions, inputs, sched)
    return res, time.perf_counter() - t0


def main():
    td = tendist()
    td.register_leaf_kernel(NAME, numpy_leaf)
    b = td.summa(2, 2, dims=(N, N, N), chunk=CHUNK)
    ints = td.random_inputs(b.statement, 0)
    res, secs = run(td, ints)
    c = res.output.data
    assert np.array_equal(c, ints["A"].data @ ints["B"].data), "integer G1 is not exact"
    out = {
        "config": {"bundle": "summa", "grid": [2, 2], "dims": [N, N, N], "chunk": CHUNK},
        "how": "tendist run_statement + oracle/ref_leaf.py numpy leaf via register_leaf_kernel/substitute_leaf",
        "int": {
            "input_sha256": {n: sha(ints[n].data) for n in sorted(ints)},
            "output_sha256": sha(c),
            "rows": ROWS,
            "row_values": [c[r].tolist() for r in ROWS],
            "col_sums": c.sum(axis=0).tolist(),
            "total": float(c.sum()),
            "events": len(res.trace.events),
            "seconds": secs,
        },
    }
    real = {"A": td.DenseTensor((N, N), generate((N, N), 0, 1, 1)),
            "B": td.DenseTensor((N, N), generate((N, N), 0, 2, 1))}
    res_r, secs_r = run(td, real)
    cr = res_r.output.data
    out["real"] = {
        "generator": {"seed": 0, "ids": {"A": 1, "B": 2}, "mode": 1},
        "input_sha256": {n: sha(real[n].data) for n in sorted(real)},
        "output_sha256": sha(cr),
        "rows": ROWS,
        "row_hex": [[float(x).hex() for x in cr[r]] for r in ROWS],
        "seconds": secs_r,
    }
    with open(os.path.join(HERE, "g1.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"G1 golden written: int {secs:.2f} s, real {secs_r:.2f} s, output sha {out['int']['output_sha256'][:16]}")


if __name__ == "__main__":
    main()
