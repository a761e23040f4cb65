"""MTTKRP 1024^3 r32 device time per td_mttkrp_config configuration.
    python tools/mttkrp_configs.py 18 19 20"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_08069_b200 import _native  # noqa: E402

lib = _native.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
I = K = L = 1024
R = 32
B = torch.randint(-4, 5, (I, K, L), dtype=torch.float64, device="cuda")
Cm = torch.randint(-4, 5, (K, R), dtype=torch.float64, device="cuda")
D = torch.randint(-4, 5, (L, R), dtype=torch.float64, device="cuda")
ref = None
for cfg in [int(x) for x in sys.argv[1:]]:
    A = torch.zeros(I, R, dtype=torch.float64, device="cuda")

    def f():
        _native.check(lib.td_mttkrp_config(st, cfg, I, K, L, R, p(B), K * L, L, p(Cm), R, p(D), R, p(A), R, 0))
    f()
    torch.cuda.synchronize()
    if ref is None:
        ref = A.clone()
    ok = torch.equal(A, ref)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"config {cfg}: {ms:.4f} ms, {(2.0 * I * K * L * R + 2.0 * I * K * R) / ms / 1e9:.2f} TFLOP/s, "
          f"same bits {ok}", flush=True)
