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


# ---------------------------------------------------------------- real-valued, full size
# uniform(-1, 1) inputs (generator mode 1): sampled output points against a
# long-double evaluation of the same generated slices (oracle/spot.py).  Two
# bounds, both written here: the rounding-error bound |got - exact| <=
# gamma_n * sum|products| (n = reduction length + product depth, u = 2^-53),
# and the north star's "1e-10 scaled by the reduction length" relative to the
# same magnitude.
def _point_values(store, name, coords):
    got = []
    pieces = list(store.local_pieces(name))
    for c in coords:
        for box, buf in pieces:
            if all(a <= x < b for x, a, b in zip(c, box.lo, box.hi)):
                got.append(float(buf[tuple(x - a for x, a in zip(c, box.lo))].item()))
                break
        else:
            raise AssertionError(f"{name}{c} is not resident")
    return got


def _check_real(bundle, depth, seed=3):
    from oracle.spot import gamma, points, reduction_length
    torch.cuda.empty_cache()
    cin, store = bundle.prepare(seed=seed, mode=1)
    td.execute(cin, store)
    stmt = bundle.statement
    out = stmt.lhs.tensor.name
    dims = stmt.lhs.tensor.dims
    rng = np.random.default_rng(seed)
    coords = [tuple(0 for _ in dims), tuple(d - 1 for d in dims)]
    coords += [tuple(int(rng.integers(0, d)) for d in dims) for _ in range(6)]
    got = _point_values(store, out, coords)
    k = reduction_length(stmt)
    g = gamma(k + depth)
    for c, x, (_, exact, bound) in zip(coords, got, points(stmt, coords, seed=seed, mode=1)):
        err = abs(np.longdouble(x) - exact)
        assert err <= g * bound, (c, float(err), float(g * bound))
        assert err <= 1e-10 * k * bound, (c, float(err))
    del store
    torch.cuda.empty_cache()


def test_real_gemm_16384_within_gamma():
    n = 16384
    _check_real(td.cannon(1, 1, dims=(n, n, n)), depth=1)


def test_real_ttv_2048_within_gamma():
    n = 2048
    _check_real(td.ttv(1, dims=(n, n, n)), depth=1)


def test_real_ttm_1024x64_within_gamma():
    m = 1024
    _check_real(td.ttm2d(1, 1, dims=(m, m, m, 64)), depth=1)


def test_real_mttkrp_1024_r32_within_gamma():
    m = 1024
    _check_real(td.mttkrp(1, 1, dims=(m, 32, m, m)), depth=2)


def test_innerprod_2048_total_exact_against_host():
    """The full 2 x 2048^3 inner product (137 GB in HBM) against an exact
    integer total computed independently on the host from the generator,
    slab by slab on every host core (oracle/host_totals.py)."""
    from oracle.host_totals import innerprod_total
    n = 2048
    torch.cuda.empty_cache()
    b = td.innerprod3(1, dims=(n, n, n))
    cin, store = b.prepare(seed=4, mode=0)
    td.execute(cin, store)
    got = store.gather("a").data.item()
    del store
    torch.cuda.empty_cache()
    want, _ = innerprod_total((n, n, n), 4, (1, 2), 0)
    assert got == float(want) and abs(want) < 2 ** 53


def test_real_innerprod_1024_within_gamma():
    from oracle.host_totals import innerprod_total
    from oracle.spot import gamma
    n = 1024
    b = td.innerprod3(1, dims=(n, n, n))
    cin, store = b.prepare(seed=5, mode=1)
    td.execute(cin, store)
    got = np.longdouble(store.gather("a").data.item())
    want, absum = innerprod_total((n, n, n), 5, (1, 2), 1)
    k = n ** 3
    assert abs(got - want) <= gamma(k + 1) * absum
    assert abs(got - want) <= 1e-10 * k * absum


@pytest.mark.parametrize("case", ["gemm", "ttm", "mttkrp", "ttv"])
def test_real_ragged_large_within_gamma(case):
    """Large shapes that are not multiples of any tile (TMA zero-filled edges,
    ragged last blocks of every distributed dimension), multi-task layouts on
    one GPU, uniform(-1,1) inputs, against the long-double point oracle."""
    b = {"gemm": lambda: td.summa(2, 2, dims=(4099, 3071, 5003), chunk=1023),
         "ttm": lambda: td.ttm2d(2, 1, dims=(301, 257, 1021, 61)),
         "mttkrp": lambda: td.mttkrp(2, 2, dims=(203, 29, 517, 1021)),
         "ttv": lambda: td.ttv(3, dims=(513, 1027, 2051))}[case]()
    depth = {"gemm": 1, "ttm": 1, "mttkrp": 2, "ttv": 1}[case]
    _check_real(b, depth, seed=7)
