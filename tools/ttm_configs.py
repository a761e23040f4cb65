"""TTM-shape (M = 2^20, N = 64, K = 1024) DGEMM device rate per td_dgemm_config tile.
    python tools/ttm_configs.py 47 50 40"""
import ctypes as C, os, sys
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
import torch
from paper_2203_08069_b200 import _native
lib = _native.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: C.c_void_p(t.data_ptr())
M, N, K = 1 << 20, 64, 1024
a = torch.randint(-4, 5, (M, K), dtype=torch.float64, device="cuda")
b = torch.randint(-4, 5, (K, N), dtype=torch.float64, device="cuda")
c = torch.empty(M, N, dtype=torch.float64, device="cuda")
ref = None
for cfg in [int(x) for x in sys.argv[1:]]:
    f = lambda: _native.check(lib.td_dgemm_config(st, cfg, M, N, K, p(a), K, p(b), N, p(c), N, 0))
    f(); torch.cuda.synchronize()
    if ref is None: ref = c.clone()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): f()
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"config {cfg}: {ms:.4f} ms {2.0*M*N*K/ms/1e9:.2f} TFLOP/s same {torch.equal(c, ref)}", flush=True)
