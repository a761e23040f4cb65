"""Device-time probe of single leaf kernels through the C ABI (no runtime):
MTTKRP and TTM at several batch sizes, to separate the per-CTA efficiency
from the last-wave tail.   python tools/kernel_probe.py
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_08069_b200 import _native  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def main():
    lib = _native.load()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    K = L = 1024
    R = 32
    for I in [int(x) for x in (sys.argv[1:] or ["999", "1024", "1110", "2048", "4096"])]:
        B = torch.randint(-4, 5, (I, K, L), dtype=torch.float64, device="cuda")
        Cm = torch.randint(-4, 5, (K, R), dtype=torch.float64, device="cuda")
        D = torch.randint(-4, 5, (L, R), dtype=torch.float64, device="cuda")
        A = torch.zeros(I, R, dtype=torch.float64, device="cuda")
        ms = timed(lambda: _native.check(lib.td_mttkrp(st, I, K, L, R, p(B), K * L, L, p(Cm), R, p(D), R, p(A), R, 0)))
        flop = 2.0 * I * K * L * R + 2.0 * I * K * R
        print(json.dumps({"kernel": "mttkrp", "I": I, "ms": ms, "tflops": flop / ms / 1e9,
                          "waves_at_3_per_sm": I * 8 / 444}), flush=True)
        del B
        torch.cuda.empty_cache()
    for I in (1024, 2048):
        B = torch.randint(-4, 5, (I, 1024, 1024), dtype=torch.float64, device="cuda")
        Cm = torch.randint(-4, 5, (1024, 64), dtype=torch.float64, device="cuda")
        Y = torch.zeros(I, 1024, 64, dtype=torch.float64, device="cuda")
        ms = timed(lambda: _native.check(lib.td_ttm(st, I, 1024, 1024, 64, p(B), 1024 * 1024, 1024, p(Cm), 64, p(Y),
                                                     1024 * 64, 64, 0)))
        flop = 2.0 * I * 1024 * 1024 * 64
        print(json.dumps({"kernel": "ttm", "I": I, "ms": ms, "tflops": flop / ms / 1e9}), flush=True)
        del B, Y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
