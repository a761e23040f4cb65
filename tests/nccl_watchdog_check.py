"""NCCL watchdog check (2 ranks): rank 0 posts a send that rank 1 never
receives.  World.wait must not hang: it polls ncclCommGetAsyncError, gives
up after the timeout, aborts the communicators (ncclCommAbort) and raises
CommError.  Run:  timeout 180 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/nccl_watchdog_check.py
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from paper_2203_08069_b200 import _native  # noqa: E402
from paper_2203_08069_b200.errors import CommError  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    world = td.configure_distributed()
    rank = dist.get_rank()
    ok = True
    if rank == 0:
        g = world.owned[0]
        buf = torch.ones(1 << 20, dtype=torch.float64, device=world.device(g))
        st = world.streams(g)[1]
        _native.call("td_send", world.comm(g), C.c_void_p(st.cuda_stream), C.c_void_p(buf.data_ptr()),
                     buf.numel(), 1)
        t0 = time.time()
        try:
            world.wait(timeout=5)
            ok = False
            print("watchdog: wait returned although the send has no receiver", flush=True)
        except CommError as exc:
            print(f"watchdog: CommError after {time.time() - t0:.1f} s: {exc}", flush=True)
            ok = world.__dict__.get("broken", False)
    flags = [None, None]
    dist.all_gather_object(flags, ok)
    if rank == 0:
        print(f"nccl_watchdog_check: {'OK' if all(flags) else 'FAIL'}", flush=True)
    dist.barrier()
    os._exit(0 if all(flags) else 1)


if __name__ == "__main__":
    main()
