import ctypes as C, sys, time, json
sys.path.insert(0, ".")
import torch
from paper_2203_08069_b200 import _native as nat
nat.load()
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())
def gen(shape, tid):
    t = torch.empty(shape, dtype=torch.float64, device="cuda")
    nat.call("td_generate", st(), len(shape), nat.i64_array(shape), nat.i64_array([0]*len(shape)), nat.i64_array(shape), P(t), nat.i64_array(t.stride()), 0, tid, 0)
    return t
def bench(fn, it=5):
    fn(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    ts=[]
    for _ in range(it):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts), sorted(ts)[len(ts)//2]
res = {}
which = sys.argv[1:] or ["gemm", "ttv", "innerprod", "ttm", "mttkrp"]
if "gemm" in which:
    for n in (4096, 8192, 16384):
        a, b = gen((n, n), 1), gen((n, n), 2); c = torch.empty(n, n, dtype=torch.float64, device="cuda")
        best, med = bench(lambda: nat.call("td_dgemm", st(), n, n, n, P(a), n, P(b), n, P(c), n, 0), 3 if n == 16384 else 5)
        ok = torch.equal(c[:64], a[:64] @ b)
        res[f"dgemm_{n}"] = dict(ms=best, tflops=2*n**3/best/1e9, exact_rows=bool(ok))
        print(res[f"dgemm_{n}"], flush=True)
        del a, b, c
if "ttv" in which:
    n = 2048
    b = gen((n, n, n), 1); cv = gen((n,), 2); a = torch.empty(n, n, dtype=torch.float64, device="cuda")
    best, med = bench(lambda: nat.call("td_ttv", st(), n, n, n, P(b), n*n, n, P(cv), P(a), n, 1, 0))
    byts = 8*(n**3 + n + n*n)
    res["ttv_2048"] = dict(ms=best, gbs=byts/best/1e6, exact=bool(torch.equal(a[:4], torch.einsum('ijk,k->ij', b[:4], cv))))
    print(res["ttv_2048"], flush=True)
    del b, a
if "innerprod" in which:
    n = 2048
    b = gen((n, n, n), 1); c2 = gen((n, n, n), 3)
    out = torch.zeros(1, dtype=torch.float64, device="cuda"); work = torch.empty(8192, dtype=torch.float64, device="cuda")
    best, med = bench(lambda: nat.call("td_innerprod", st(), 1, n**3, P(b), n**3, P(c2), n**3, P(out), P(work), 0))
    res["innerprod_2048"] = dict(ms=best, gbs=16*n**3/best/1e6, value=out.item())
    print(res["innerprod_2048"], flush=True)
    del b, c2
if "ttm" in which:
    n, L = 1024, 64
    b = gen((n, n, n), 1); cm = gen((n, L), 2); y = torch.empty(n, n, L, dtype=torch.float64, device="cuda")
    best, med = bench(lambda: nat.call("td_ttm", st(), n, n, n, L, P(b), n*n, n, P(cm), L, P(y), n*L, L, 0))
    res["ttm_1024_64"] = dict(ms=best, tflops=2*n**3*L/best/1e9, exact=bool(torch.equal(y[:2], torch.einsum('ijk,kl->ijl', b[:2], cm))))
    print(res["ttm_1024_64"], flush=True)
    del b, y
if "mttkrp" in which:
    n, R = 1024, 32
    b = gen((n, n, n), 1); cm = gen((n, R), 2); d = gen((n, R), 3); a = torch.empty(n, R, dtype=torch.float64, device="cuda")
    best, med = bench(lambda: nat.call("td_mttkrp", st(), n, n, n, R, P(b), n*n, n, P(cm), R, P(d), R, P(a), R, 0))
    want = torch.einsum('ikj,kj->ij', torch.einsum('ikl,lj->ikj', b[:2], d), cm)
    res["mttkrp_1024_32"] = dict(ms=best, tflops=(2*n**3*R + 2*n*n*R)/best/1e9, gbs=8*n**3/best/1e6, exact=bool(torch.equal(a[:2], want)))
    print(res["mttkrp_1024_32"], flush=True)
json.dump(res, open("gpurun_out/kperf.json", "w"), indent=1)
