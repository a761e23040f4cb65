"""numpy restatement of the reference's distributed execution for the bundles
timed on the host -- TEST / BASELINE INFRASTRUCTURE ONLY.

The reference CPU path is `run_statement` -> `execute` (pkg/src/tendist/
simulator.py:537-663): one task per processor, each computing its partial
output over its iteration box step by step, then partials committed in task
order.  Its shipped leaf is the per-point Python interpreter (cin.py:399-417,
~1e5 points/s); the survey's "CPU-B" variant plugs a BLAS leaf in through the
reference's own plugin API (register_leaf_kernel / substitute_leaf).  This
module is that CPU-B path restated for the benchmark algorithms: the same
task grid and step structure, numpy/OpenBLAS for every leaf block, commits in
task order.  `bench.py --impl reference` and the `cpu_baseline` key time it
on the GPU box's host cores.
"""

from __future__ import annotations

import numpy as np


def _blocks(n, parts):
    b = -(-n // parts)
    return [(min(q * b, n), min((q + 1) * b, n)) for q in range(parts)]


def summa(a, b, g1, g2, chunk):
    """SUMMA on a g1 x g2 grid (reference algorithms.py:88-106): task (x,y)
    owns C block (x,y); per k chunk it adds A[xblk, chunk] @ B[chunk, yblk]."""
    m, k = a.shape
    n = b.shape[1]
    c = np.zeros((m, n))
    for (i0, i1) in _blocks(m, g1):
        for (j0, j1) in _blocks(n, g2):
            acc = np.zeros((i1 - i0, j1 - j0))
            for k0 in range(0, k, chunk):
                k1 = min(k, k0 + chunk)
                acc += a[i0:i1, k0:k1] @ b[k0:k1, j0:j1]
            c[i0:i1, j0:j1] = acc
    return c


def cannon(a, b, g):
    """Cannon on g x g (reference algorithms.py:109-132): task (x,y) at step s
    multiplies k block (x + y + s) mod g."""
    m, k = a.shape
    n = b.shape[1]
    c = np.zeros((m, n))
    kb = _blocks(k, g)
    for x, (i0, i1) in enumerate(_blocks(m, g)):
        for y, (j0, j1) in enumerate(_blocks(n, g)):
            acc = np.zeros((i1 - i0, j1 - j0))
            for s in range(g):
                k0, k1 = kb[(x + y + s) % g]
                acc += a[i0:i1, k0:k1] @ b[k0:k1, j0:j1]
            c[i0:i1, j0:j1] = acc
    return c


def johnson(a, b, g):
    """Johnson 3D (reference algorithms.py:160-180): task (x,y,z) computes one
    block product; partials reduced into z = 0 in task order."""
    m, k = a.shape
    n = b.shape[1]
    c = np.zeros((m, n))
    kb = _blocks(k, g)
    for (i0, i1) in _blocks(m, g):
        for (j0, j1) in _blocks(n, g):
            for (k0, k1) in kb:
                c[i0:i1, j0:j1] += a[i0:i1, k0:k1] @ b[k0:k1, j0:j1]
    return c


def gemm_for_gpus(p, a, b):
    """The weak-scaling sweep's algorithm at p processors."""
    n = a.shape[0]
    if p == 1:
        return cannon(a, b, 1)
    if p == 2:
        return summa(a, b, 2, 1, -(-n // 8))
    if p == 4:
        return cannon(a, b, 2)
    return johnson(a, b, 2)


def ttv_rows(bt, c, g):
    """ttv bundle (algorithms.py:275-292): row slabs, c replicated."""
    out = np.zeros(bt.shape[:2])
    for (i0, i1) in _blocks(bt.shape[0], g):
        out[i0:i1] = np.tensordot(bt[i0:i1], c, axes=([2], [0]))
    return out


def innerprod_rows(bt, ct, g):
    """3-order innerprod: per-slab partials, fanned in to processor 0 in order."""
    total = 0.0
    for (i0, i1) in _blocks(bt.shape[0], g):
        total += float(np.dot(bt[i0:i1].ravel(), ct[i0:i1].ravel()))
    return total


def ttm_rows(bt, cm, g):
    i, j, k = bt.shape
    out = np.zeros((i, j, cm.shape[1]))
    for (i0, i1) in _blocks(i, g):
        out[i0:i1] = (bt[i0:i1].reshape(-1, k) @ cm).reshape(i1 - i0, j, -1)
    return out


def mttkrp_grid(bt, cm, d, g1, g2):
    """mttkrp bundle (algorithms.py:334-354): task (x,y) owns B[xblk, yblk, :],
    partial A rows reduced into column 0 in task order."""
    i, k, l = bt.shape
    out = np.zeros((i, cm.shape[1]))
    for (i0, i1) in _blocks(i, g1):
        for (k0, k1) in _blocks(k, g2):
            t = (bt[i0:i1, k0:k1].reshape(-1, l) @ d).reshape(i1 - i0, k1 - k0, -1)
            out[i0:i1] += np.einsum("ikj,kj->ij", t, cm[k0:k1])
    return out
