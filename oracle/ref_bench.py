"""The REFERENCE arm: tendist itself, timed on the host -- BASELINE
INFRASTRUCTURE ONLY (bench.py `--impl reference` and the in-line
`cpu_baseline`; never imported by the package).

What runs is the unmodified reference package staged in oracle/_ref
(`oracle/reference.py`): its `run_statement` (placement, ledger, per-task
numerics, commits; reference `simulator.py:668-715`) on the same bundle
(statement, machine, distributions, schedule) the B200 run uses, with one
leaf substituted through the reference's own plugin API
(`register_leaf_kernel` + `Schedule.substitute_leaf`, reference
`cin.py:344-379`, `scheduling.py:263-299`):

  * "numpy" -- `oracle/ref_leaf.py`'s numpy/BLAS leaf (SURVEY.md §8(d)
    CPU-B: all host cores through OpenBLAS);
  * "interpreter" -- the reference as shipped, its per-point Python leaf
    (CPU-A, one core), only ever on small shapes.

`to_reference(bundle)` rebuilds one of this package's bundles as tendist
objects (statement text, machine levels, distribution levels, schedule
commands replayed one by one), so both arms run literally the same
algorithm; the weak-scaling GEMM layouts are tendist's own bundles too.
"""

from __future__ import annotations

import os
import time

import numpy as np

from oracle.generator import generate
from oracle.ref_leaf import NAME, innermost_vars, numpy_leaf
from oracle.reference import tendist


def to_reference(td, bundle):
    """(statement, machine, distributions, schedule) of `bundle` as tendist objects."""
    from paper_2203_08069_b200.ir import format_statement
    machine = td.make_machine([tuple(lvl) for lvl in bundle.machine.levels])
    stmt = td.parse_statement(format_statement(bundle.statement), dict(bundle.statement.extents))
    dists = {name: td.TensorDistribution(d.tensor_dims, machine, d.levels)
             for name, d in bundle.distributions.items()}
    sched = td.schedule()
    for step in bundle.schedule.commands:
        method = {"leaf": "substitute_leaf"}.get(step.name, step.name)
        sched = getattr(sched, method)(*step.args)
    return stmt, machine, dists, sched


def inputs_for(td, stmt, *, mode=0, seed=0):
    """Integer-valued (mode 0) or uniform(-1,1) (mode 1) inputs from the
    counter generator, tensor ids in sorted-name order (bundle.prepare's)."""
    out_name = stmt.lhs.tensor.name
    names = sorted(n for n in stmt.tensors() if n != out_name)
    return {n: td.DenseTensor(stmt.tensors()[n].dims, generate(stmt.tensors()[n].dims, seed, k + 1, mode))
            for k, n in enumerate(names)}


def run_reference(bundle, inputs=None, *, leaf="numpy", mode=0, seed=0):
    """One tendist `run_statement` of `bundle`; returns (output ndarray,
    wall seconds of run_statement, trace)."""
    td = tendist()
    stmt, machine, dists, sched = to_reference(td, bundle)
    if leaf == "numpy":
        td.register_leaf_kernel(NAME, numpy_leaf)
        sched = sched.substitute_leaf(innermost_vars(sched.apply(td.lower_to_cin(stmt))), NAME)
    if inputs is None:
        inputs = inputs_for(td, stmt, mode=mode, seed=seed)
    else:
        inputs = {n: td.DenseTensor(t.dims, t.data) for n, t in inputs.items()}
    t0 = time.perf_counter()
    res = td.run_statement(stmt, machine, dists, inputs, sched)
    secs = time.perf_counter() - t0
    return res.output.data, secs, res.trace


def blas_threads() -> int:
    """Threads OpenBLAS will use (all host cores unless pinned by the env)."""
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return os.cpu_count() or 1


def gemm_rows_exact(out: np.ndarray, n: int, rows=(0, 1)) -> bool:
    """Sampled rows of an integer-input GEMM output against A[rows] @ B."""
    a = generate((n, n), 0, 1, 0)[list(rows)]
    b = generate((n, n), 0, 2, 0)
    return bool(np.array_equal(out[list(rows)], a @ b))
