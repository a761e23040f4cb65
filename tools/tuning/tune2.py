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
def bench(fn, it=3):
    fn(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    ts=[]
    for _ in range(it):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts)
gcfgs = [int(x) for x in sys.argv[1].split(",")]
tcfgs = [int(x) for x in sys.argv[2].split(",")]
mcfgs = [int(x) for x in sys.argv[3].split(",")]
res = {}
for n in (16384,):
    a, b = gen((n, n), 1), gen((n, n), 2); c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for cfg in gcfgs:
        ms = bench(lambda: nat.call("td_dgemm_config", st(), cfg, n, n, n, P(a), n, P(b), n, P(c), n, 0), 2)
        res[f"gemm{n}_cfg{cfg}"] = (round(2*n**3/ms/1e9, 1), bool(torch.equal(c[:32], a[:32] @ b)))
        print(n, cfg, res[f"gemm{n}_cfg{cfg}"], flush=True)
    del a, b, c
M, N, K = 1024*1024, 64, 1024
a, b = gen((M, K), 1), gen((K, N), 2); c = torch.empty(M, N, dtype=torch.float64, device="cuda")
for cfg in tcfgs:
    ms = bench(lambda: nat.call("td_dgemm_config", st(), cfg, M, N, K, P(a), K, P(b), N, P(c), N, 0))
    res[f"ttm_cfg{cfg}"] = (round(2*M*N*K/ms/1e9, 1), bool(torch.equal(c[:32], a[:32] @ b)))
    print("ttm", cfg, res[f"ttm_cfg{cfg}"], flush=True)
del a, c
n, R = 1024, 32
bt = gen((n, n, n), 1); cm = gen((n, R), 2); d = gen((n, R), 3); a = torch.empty(n, R, dtype=torch.float64, device="cuda")
want = torch.einsum('ikj,kj->ij', torch.einsum('ikl,lj->ikj', bt[:2], d), cm)
for cfg in mcfgs:
    ms = bench(lambda: nat.call("td_mttkrp_config", st(), cfg, n, n, n, R, P(bt), n*n, n, P(cm), R, P(d), R, P(a), R, 0))
    res[f"mttkrp_cfg{cfg}"] = (round((2*n**3*R + 2*n*n*R)/ms/1e9, 1), round(8*n**3/ms/1e6), bool(torch.equal(a[:2], want)))
    print("mttkrp", cfg, res[f"mttkrp_cfg{cfg}"], flush=True)
json.dump(res, open("gpurun_out/tune2.json", "w"), indent=1)
