"""Per-launch latency of small programs: eager Python step loop vs recorded
launch plans (td_execute_plan) vs a captured CUDA graph.

    python tools/launch_latency.py            (1 GPU; prints one JSON line per config)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from paper_2203_08069_b200 import runtime  # noqa: E402


def timed(fn, n=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


def main():
    configs = {
        "G1 summa 2x2 1024^3 chunk 128": (td.summa(2, 2, dims=(1024,) * 3, chunk=128), 2.0 * 1024 ** 3),
        "mttkrp 1x1 1024^3 r32": (td.mttkrp(1, 1, dims=(1024, 32, 1024, 1024)), 2.0 * 1024 ** 3 * 32),
        "ttm2d 1x1 1024^3 x 64": (td.ttm2d(1, 1, dims=(1024, 1024, 1024, 64)), 2.0 * 1024 ** 3 * 64),
    }
    for name, (b, flop) in configs.items():
        cin, store = b.prepare(seed=0, mode=0)
        out = b.statement.lhs.tensor.name

        def step():
            store.zero(out)
            td.execute(cin, store, record_requirements=False)

        runtime.PLANS = False
        eager = timed(step)
        runtime.PLANS = True
        planned = timed(step)
        cap = runtime.CapturedLaunch(cin, store)
        graph = timed(cap.replay)
        print(json.dumps({"config": name, "eager_ms": eager, "plan_ms": planned, "graph_ms": graph,
                          "plan_gflops": flop / planned / 1e6, "graph_gflops": flop / graph / 1e6}), flush=True)
        del cap, store


if __name__ == "__main__":
    main()
