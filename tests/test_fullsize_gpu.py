"""Parity at the BASELINE.json full sizes, through the public runtime.

The CPU oracle cannot evaluate these shapes whole, so each test checks
size-independent properties on integer-valued inputs from the device
generator (values in [-4, 4]; every sum is an integer < 2^53, so all
comparisons are exact):
  * sampled output rows against the oracle on the same generated rows;
  * Freivalds' identity C.x == A.(B.x) for the full GEMM (x integer);
  * linearity of the inner product over slabs (checksum of checksums).
"""

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from oracle.generator import generate_box

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _gather_rows(store, name, rows):
    """rows of a 2-D region from its home pieces (device -> host)."""
    out = {}
    for box, buf in store.local_pieces(name):
        for r in rows:
            if box.lo[0] <= r < box.hi[0]:
                out.setdefault(r, {})[box.lo[1]] = buf[r - box.lo[0]].cpu().numpy()
    return {r: np.concatenate([parts[k] for k in sorted(parts)]) for r, parts in out.items()}


def test_gemm_16384_cannon_rows_and_freivalds():
    n = 16384
    b = td.cannon(1, 1, dims=(n, n, n))
    cin, store = b.prepare(seed=0, mode=0)
    td.execute(cin, store)
    rows = [0, 1234, n - 1]
    got = _gather_rows(store, "C", rows)
    bmat = generate_box((n, n), (0, 0), (n, n), 0, 2, 0)
    for r in rows:
        a_row = generate_box((n, n), (r, 0), (1, n), 0, 1, 0)
        assert np.array_equal(got[r], (a_row @ bmat).ravel())
    # Freivalds on the device: x in {-1,0,1}^n, products stay exact
    x = torch.from_numpy(np.random.default_rng(0).integers(-1, 2, n).astype(np.float64)).cuda()
    (box, cbuf), = store.local_pieces("C")
    (_, abuf), = store.local_pieces("A")
    (_, bbuf), = store.local_pieces("B")
    lhs = cbuf @ x
    rhs = abuf @ (bbuf @ x)
    assert torch.equal(lhs, rhs)


def test_ttv_2048_sampled_rows():
    n = 2048
    b = td.ttv(1, dims=(n, n, n))
    cin, store = b.prepare(seed=0, mode=0)
    td.execute(cin, store)
    (box, abuf), = store.local_pieces("A")
    c = generate_box((n,), (0,), (n,), 0, 2, 0)   # input names sorted: B -> id 1, c -> id 2
    for i in (0, 777, n - 1):
        bi = generate_box((n, n, n), (i, 0, 0), (1, n, n), 0, 1, 0)[0]
        assert np.array_equal(abuf[i].cpu().numpy(), bi @ c)


def test_innerprod_2048_slab_linearity():
    n = 2048
    b = td.innerprod3(1, dims=(n, n, n))
    cin, store = b.prepare(seed=0, mode=0)
    td.execute(cin, store)
    total = store.gather("a").data.item()
    (_, bb), = store.local_pieces("B")
    (_, cc), = store.local_pieces("C")
    from paper_2203_08069_b200 import _native
    import ctypes as C
    work = torch.empty(int(_native.lib().td_innerprod_work_size()), dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    slabs = 8
    step = n // slabs
    for s in range(slabs):   # accumulate the 8 slab partials: must equal the one-shot value exactly
        _native.call("td_innerprod", st, 1, step * n * n, C.c_void_p(bb[s * step:].data_ptr()), step * n * n,
                     C.c_void_p(cc[s * step:].data_ptr()), step * n * n, C.c_void_p(out.data_ptr()),
                     C.c_void_p(work.data_ptr()), 1)
    assert out.item() == total
    # and one slab against the host oracle
    b0 = generate_box((n, n, n), (5, 0, 0), (1, n, n), 0, 1, 0)
    c0 = generate_box((n, n, n), (5, 0, 0), (1, n, n), 0, 2, 0)
    _native.call("td_innerprod", st, 1, n * n, C.c_void_p(bb[5:].data_ptr()), n * n,
                 C.c_void_p(cc[5:].data_ptr()), n * n, C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()), 0)
    assert out.item() == float(np.dot(b0.ravel(), c0.ravel()))


def test_ttm_1024x64_sampled_rows():
    m = 1024
    b = td.ttm2d(1, 1, dims=(m, m, m, 64))
    cin, store = b.prepare(seed=0, mode=0)
    td.execute(cin, store)
    (box, y), = store.local_pieces("Y")
    cm = generate_box((m, 64), (0, 0), (m, 64), 0, 2, 0)   # names: B -> 1, C -> 2
    for i in (0, 511, m - 1):
        bi = generate_box((m, m, m), (i, 0, 0), (1, m, m), 0, 1, 0)[0]
        assert np.array_equal(y[i].cpu().numpy(), bi @ cm)


def test_mttkrp_1024_r32_sampled_rows():
    m, r = 1024, 32
    b = td.mttkrp(1, 1, dims=(m, r, m, m))
    cin, store = b.prepare(seed=0, mode=0)
    td.execute(cin, store)
    (box, a), = store.local_pieces("A")
    cm = generate_box((m, r), (0, 0), (m, r), 0, 2, 0)     # names: B -> 1, C -> 2, D -> 3
    dm = generate_box((m, r), (0, 0), (m, r), 0, 3, 0)
    for i in (0, 300, m - 1):
        bi = generate_box((m, m, m), (i, 0, 0), (1, m, m), 0, 1, 0)[0]
        want = ((bi @ dm) * cm).sum(axis=0)
        assert np.array_equal(a[i].cpu().numpy(), want)
