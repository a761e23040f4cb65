"""Replays the G1 launch plan (SUMMA 1024^3 on 2x2, chunk 128, one GPU) a few
times; run under `ncu --metrics gpu__time_duration.sum` for its kernel list.
    python tools/g1_plan_kernels.py [replays]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402

b = td.summa(2, 2, dims=(1024,) * 3, chunk=128)
cin, store = b.prepare(seed=0, mode=0)
for _ in range(3 + int(sys.argv[1] if len(sys.argv) > 1 else 2)):
    store.zero("C")
    td.execute(cin, store, record_requirements=False)
torch.cuda.synchronize()
