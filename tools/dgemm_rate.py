"""Device rate of one td_dgemm at n^3 (default 16384), CUDA events over 3 launches.
    python tools/dgemm_rate.py [n]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_08069_b200 import _native as nat  # noqa: E402

nat.load(os.environ.get("TD_LIB", nat.LIB_PATH))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = torch.rand(n, n, dtype=torch.float64, device="cuda")
b = torch.rand(n, n, dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def f():
    nat.call("td_dgemm", st, n, n, n, C.c_void_p(a.data_ptr()), n, C.c_void_p(b.data_ptr()), n,
             C.c_void_p(c.data_ptr()), n, 0)


f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    f()
e.record()
e.synchronize()
print(f"dgemm {n}^3: {3 * 2 * n ** 3 / (s.elapsed_time(e) / 1e3) / 1e12:.2f} TFLOP/s")
