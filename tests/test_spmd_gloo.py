"""SPMD host logic at world_size 2 and 4 on CPU (gloo): every rank plans the
same launch in its own interpreter (fresh PYTHONHASHSEED) and the sends one
rank issues to a peer pair up, in order and size, with the receives that peer
issues -- the invariant NCCL needs for the GPU runs.  No GPU involved."""

import os
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bundles(td):
    return [td.summa(2, 1, dims=(64, 48, 80), chunk=16), td.cannon(2, 2, dims=(30, 26, 22)),
            td.cannon(3, 3, dims=(7, 7, 5)), td.pumma(3, 3, dims=(6, 6, 6)), td.johnson(2, 2, 2, dims=(9, 7, 5)),
            td.mttkrp(2, 2, dims=(6, 4, 5, 3)), td.solomonik(4, 4, 2, dims=(8, 8, 8)),
            td.innerprod(4, dims=(8, 6)), td.cosma_like((2, 2, 1), (1, 1, 2), dims=(5, 4, 7)),
            td.summa_hier(dims=(7, 6, 5), chunk=3), td.ttm2d(2, 2, dims=(5, 4, 6, 3))]


def _worker(rank, size, port, queue):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    import paper_2203_08069_b200 as td
    from paper_2203_08069_b200.planner import comm_schedule, plan_statement
    mine = []
    for b in _bundles(td):
        prog, trace = plan_statement(b.statement, b.machine, b.distributions, b.schedule)
        sched = comm_schedule(prog, b.machine, size)
        sends = [(b.name, ph, s, w, dst, n) for ph, s, w, src, dst, n in sched if src == rank]
        recvs = [(b.name, ph, s, w, src, n) for ph, s, w, src, dst, n in sched if dst == rank]
        mine.append((sends, recvs, len(trace.events)))
    allv = [None] * size
    dist.all_gather_object(allv, mine)
    ok = True
    for k in range(len(mine)):
        for a in range(size):
            for bb in range(size):
                if a == bb:
                    continue
                out = [x[:4] + (x[5],) for x in allv[a][k][0] if x[4] == bb]
                inn = [x[:4] + (x[5],) for x in allv[bb][k][1] if x[4] == a]
                ok &= out == inn
        ok &= len({allv[r][k][2] for r in range(size)}) == 1   # identical ledgers
    dist.destroy_process_group()
    queue.put((rank, ok))


@pytest.mark.parametrize("size", [2, 4, 8])
def test_spmd_send_recv_pairing(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + size
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(results[r] for r in range(size)), results
