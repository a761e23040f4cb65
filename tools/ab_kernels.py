"""A/B device rates of the headline leaves through the C ABI of one library
build (TD_LIB, default the in-tree .so): DGEMM 16384^3, TTM 1024^3 x 64,
MTTKRP 1024^3 r32 (default selection and configs 19 / 22).
    TD_LIB=build/alt_old.so python tools/ab_kernels.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_08069_b200 import _native  # noqa: E402

lib = _native.load(os.environ.get("TD_LIB", _native.LIB_PATH))
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
tag = os.path.basename(os.environ.get("TD_LIB", "in-tree"))


def rate(name, flop, f, reps):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{tag} {name}: {ms:.4f} ms {flop / ms / 1e9:.2f} TFLOP/s", flush=True)


n = 16384
a = torch.randint(-4, 5, (n, n), dtype=torch.float64, device="cuda")
b = torch.randint(-4, 5, (n, n), dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
rate("dgemm 16384^3", 2.0 * n ** 3, lambda: _native.check(lib.td_dgemm(st, n, n, n, p(a), n, p(b), n, p(c), n, 0)), 3)
del a, b, c
m, r = 1024, 64
B = torch.randint(-4, 5, (m, m, m), dtype=torch.float64, device="cuda")
Cm = torch.randint(-4, 5, (m, r), dtype=torch.float64, device="cuda")
Y = torch.empty(m, m, r, dtype=torch.float64, device="cuda")
rate("ttm 1024^3x64", 2.0 * m ** 3 * r,
     lambda: _native.check(lib.td_ttm(st, m, m, m, r, p(B), m * m, m, p(Cm), r, p(Y), m * r, r, 0)), 20)
del Y
R = 32
Cr = torch.randint(-4, 5, (m, R), dtype=torch.float64, device="cuda")
D = torch.randint(-4, 5, (m, R), dtype=torch.float64, device="cuda")
A = torch.empty(m, R, dtype=torch.float64, device="cuda")
for cfg in (-1, 19, 22):
    rate(f"mttkrp r32 config {cfg}", 2.0 * m ** 3 * R + 2.0 * m * m * R,
         lambda: _native.check(lib.td_mttkrp_config(st, cfg, m, m, m, R, p(B), m * m, m, p(Cr), R, p(D), R, p(A), R,
                                                    0)), 20)
