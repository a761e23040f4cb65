"""N = 64 (TTM) and square GEMM tile sweep."""
import ctypes as C, sys, json
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
    return min(ts)
cfgs = [int(x) for x in sys.argv[1].split(",")]
M, N, K = 1024*1024, 64, 1024
a, b = gen((M, K), 1), gen((K, N), 2); c = torch.empty(M, N, dtype=torch.float64, device="cuda")
for cfg in cfgs:
    ms = bench(lambda: nat.call("td_dgemm_config", st(), cfg, M, N, K, P(a), K, P(b), N, P(c), N, 0))
    print("n64", cfg, round(2*M*N*K/ms/1e9, 1), bool(torch.equal(c[:64], a[:64] @ b)), flush=True)
del a, b, c
n = 16384
a, b = gen((n, n), 1), gen((n, n), 2); c = torch.empty(n, n, dtype=torch.float64, device="cuda")
for cfg in cfgs:
    ms = bench(lambda: nat.call("td_dgemm_config", st(), cfg, n, n, n, P(a), n, P(b), n, P(c), n, 0), 2)
    print("sq", cfg, round(2*n**3/ms/1e9, 1), bool(torch.equal(c[:32], a[:32] @ b)), flush=True)
