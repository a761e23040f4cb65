"""SM clock / power while one MTTKRP configuration runs back to back (~2 s).
    python tools/mttkrp_clocks.py 18 19 26"""
import ctypes as C
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_08069_b200 import _native  # noqa: E402

lib = _native.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
I = int(os.environ.get("MK_I", 1024))
K = L = 1024
R = 32
B = torch.randint(-4, 5, (I, K, L), dtype=torch.float64, device="cuda")
Cm = torch.randint(-4, 5, (K, R), dtype=torch.float64, device="cuda")
D = torch.randint(-4, 5, (L, R), dtype=torch.float64, device="cuda")
A = torch.zeros(I, R, dtype=torch.float64, device="cuda")
flop = 2.0 * I * K * L * R + 2.0 * I * K * R


def sample(stop, out):
    while not stop.is_set():
        q = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        out.append(q)
        time.sleep(0.05)


for cfg in [int(x) for x in sys.argv[1:]]:
    def f():
        _native.check(lib.td_mttkrp_config(st, cfg, I, K, L, R, p(B), K * L, L, p(Cm), R, p(D), R, p(A), R, 0))
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    n = max(20, int(2.0 / (flop / 35e12)))
    stop, samples = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, samples))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    s.record()
    for _ in range(n):
        f()
    e.record()
    e.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    mhz = sorted(int(x.split(",")[0]) for x in samples if x)
    pw = sorted(float(x.split(",")[1]) for x in samples if x)
    reasons = sorted({x.split(",")[2].strip() for x in samples if x})
    print(f"config {cfg}: {ms:.4f} ms, {flop / ms / 1e9:.2f} TFLOP/s over {n} launches; sm MHz median "
          f"{mhz[len(mhz) // 2]} (min {mhz[0]}, max {mhz[-1]}), power median {pw[len(pw) // 2]:.0f} W, "
          f"reasons {reasons}", flush=True)
