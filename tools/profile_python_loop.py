"""cProfile of the Python step loop (launch plans off) on G1, to find host
overhead hot spots.   python tools/profile_python_loop.py"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from paper_2203_08069_b200 import runtime  # noqa: E402

runtime.PLANS = False
b = td.summa(2, 2, dims=(1024,) * 3, chunk=128)
cin, store = b.prepare(seed=0, mode=0)


def step():
    store.zero("C")
    td.execute(cin, store, record_requirements=False)


for _ in range(5):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(25)
