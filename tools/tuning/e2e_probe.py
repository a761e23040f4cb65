import sys, time, torch
sys.path.insert(0, ".")
import paper_2203_08069_b200 as td
from paper_2203_08069_b200 import _native
from paper_2203_08069_b200.runtime import _copy_any
n = 16384
# pitched vs contiguous H2D
h = torch.empty((4096, n), dtype=torch.float64, pin_memory=True); h.fill_(1)
d = torch.empty((4096, n), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for w in (2048, 4096, 16384):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    _copy_any(st, d[:, :w], h[:, :w]); torch.cuda.synchronize()
    s.record(); _copy_any(st, d[:, :w], h[:, :w]); e.record(); e.synchronize()
    print("h2d width", w, 8 * 4096 * w / s.elapsed_time(e) / 1e6, "GB/s")
