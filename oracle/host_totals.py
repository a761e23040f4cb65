"""Exact / long-double host reductions over generated tensors -- TEST
INFRASTRUCTURE ONLY.

The full-size inner product (BASELINE config V: 2 x 2048^3 fp64, 137 GB) is
far beyond a single-process numpy oracle, but its value is checkable
independently of the GPU: the inputs come from the counter-based generator
(oracle/generator.py), so any slab can be regenerated on the host.  This
module sums `B . C` slab by slab in worker processes ("spawn": the workers
import only numpy and the generator, never CUDA):
  * integer mode (values in [-4, 4]): int64 per slab, a Python int overall --
    exact, so the GPU's fp64 total must match it bit for bit (every partial
    sum of integers < 2^53 is exact in any order);
  * real mode (uniform(-1, 1)): long double per slab (64-bit significand),
    plus the sum of |b||c| for the error bound.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np


def _slab(args):
    from oracle.generator import generate_box
    dims, i0, i1, seed, ids, mode = args
    shape = (i1 - i0,) + tuple(dims[1:])
    origin = (i0,) + (0,) * (len(dims) - 1)
    b = generate_box(dims, origin, shape, seed, ids[0], mode).ravel()
    c = generate_box(dims, origin, shape, seed, ids[1], mode).ravel()
    if mode == 0:
        return int(np.dot(b.astype(np.int64), c.astype(np.int64))), 0.0
    prod = b.astype(np.longdouble) * c.astype(np.longdouble)
    return prod.sum(), float(np.abs(b) @ np.abs(c))


def innerprod_total(dims, seed, ids, mode, *, slab_rows=None, workers=None):
    """sum_x B(x) C(x) over a generated tensor pair of shape dims, split into
    row slabs of the leading mode.  mode 0 -> (exact int, 0.0); mode 1 ->
    (long double total, float sum |B||C|)."""
    n0 = dims[0]
    per_row = 1
    for d in dims[1:]:
        per_row *= d
    rows = slab_rows or max(1, (1 << 22) // max(1, per_row))
    jobs = [(tuple(dims), i, min(n0, i + rows), seed, tuple(ids), mode) for i in range(0, n0, rows)]
    workers = workers or max(1, min(32, os.cpu_count() or 1))
    ctx = mp.get_context("spawn")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    old = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = root + (os.pathsep + old if old else "")
    try:
        with ctx.Pool(workers) as pool:
            parts = pool.map(_slab, jobs, chunksize=4)
    finally:
        os.environ["PYTHONPATH"] = old
    if mode == 0:
        return sum(p[0] for p in parts), 0.0
    total = np.longdouble(0)
    absum = 0.0
    for v, a in parts:
        total += v
        absum += a
    return total, absum
