"""GEMM -> reduce over peer memory vs NCCL write-back (torchrun, N GPUs).

    torchrun --nproc-per-node 2 tools/tuning/peer_bench.py [n]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from paper_2203_08069_b200 import peer  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = td.configure_distributed()
    size = dist.get_world_size()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else td.weak_gemm_n(size)
    cases = []
    if size == 2:
        cases = [("cosma 1x1x2", td.cosma_like((1, 1, 2), (1, 1, 1), dims=(n, n, n))),
                 ("summa 2x1", td.gemm_for_gpus(2, n))]
    elif size == 4:
        cases = [("cosma 2x1x2", td.cosma_like((2, 1, 2), (1, 1, 1), dims=(n, n, n))),
                 ("cannon 2x2", td.gemm_for_gpus(4, n))]
    for name, b in cases:
        cin, store = b.prepare(seed=0, world=world)
        out = b.statement.lhs.tensor.name
        for flag in (True, False):
            peer.PEER_REDUCE = flag

            def step():
                store.zero(out)
                td.execute(cin, store, record_requirements=False)
            for _ in range(3):
                step()
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps = 5
            s.record()
            for _ in range(steps):
                step()
            e.record()
            e.synchronize()
            dist.barrier(device_ids=[local])
            t = torch.tensor([s.elapsed_time(e) / steps], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
            if dist.get_rank() == 0:
                tf = 2.0 * n ** 3 / (ms / 1e3) / 1e12
                print(f"{name} n={n} peer={flag}: {ms:.2f} ms/step  {tf:.2f} TFLOP/s total, "
                      f"{tf / size:.2f} per GPU", flush=True)
        peer.PEER_REDUCE = True
        del store
        torch.cuda.empty_cache()
    world.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
