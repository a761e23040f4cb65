"""MTTKRP weak-scaled step time under torchrun: where the multi-GPU overhead goes.

    torchrun --nproc-per-node 4 tools/tuning/mttkrp_mp.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from paper_2203_08069_b200 import leaves, peer  # noqa: E402
from paper_2203_08069_b200 import runtime as rt  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = td.configure_distributed()
    size = dist.get_world_size()
    g1, g2 = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}[size]
    b = td.mttkrp(g1, g2, dims=(1024 * g1, 32, 1024 * g2, 1024))
    cin, store = b.prepare(seed=0, world=world)

    def step():
        store.zero("A")
        td.execute(cin, store, record_requirements=False)

    def timed(label, steps=20):
        for _ in range(3):
            step()
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        leaves.TIMING = []
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        s.record()
        for _ in range(steps):
            step()
        e.record()
        host = (time.perf_counter() - h0) * 1e3 / steps
        e.synchronize()
        ks = [a.elapsed_time(z) for k, a, z in leaves.TIMING if k == "mttkrp"]
        leaves.TIMING = None
        t = torch.tensor([s.elapsed_time(e) / steps, host, sum(ks) / max(1, len(ks))], device="cuda",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if dist.get_rank() == 0:
            print(f"{label:28s} step {t[0].item():.3f} ms  host-issue {t[1].item():.3f} ms  leaf {t[2].item():.3f} ms",
                  flush=True)

    timed("default")
    peer.PEER_REDUCE = False
    timed("nccl write-back")
    peer.PEER_REDUCE = True
    rt.USE_BROADCAST = False
    timed("p2p fan-out (no bcast)")
    rt.USE_BROADCAST = True
    timed("default again")
    world.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
