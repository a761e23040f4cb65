"""NCCL watchdog check (2 ranks): rank 0 posts a receive that rank 1 never
sends.  World.wait must not hang: it polls ncclCommGetAsyncError, gives
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
    g = world.owned[0]
    buf = torch.ones(1 << 20, dtype=torch.float64, device=world.device(g))
    st = world.streams(g)[1]
    # a matched pair first: NCCL connects peers lazily, and connection setup
    # blocks on the host (not covered by the watchdog; NCCL_RUNTIME_CONNECT=0
    # moves it into communicator creation)
    for sender in (0, 1):       # both directions are separate connections
        op = "td_send" if rank == sender else "td_recv"
        _native.call(op, world.comm(g), C.c_void_p(st.cuda_stream), C.c_void_p(buf.data_ptr()), buf.numel(),
                     1 - rank)
        world.wait(timeout=60)
    print(f"watchdog: rank {rank} warm-up pair done", flush=True)
    if rank == 0:     # a receive whose data never comes: its NCCL kernel cannot finish
        _native.call("td_recv", world.comm(g), C.c_void_p(st.cuda_stream), C.c_void_p(buf.data_ptr()),
                     buf.numel(), 1)
        t0 = time.time()
        print("watchdog: waiting", flush=True)
        try:
            world.wait(timeout=5)
            ok = False
            print("watchdog: wait returned although the receive has no sender", flush=True)
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
