"""Multi-GPU paths (skipped unless >= 2 GPUs are visible).

* single process driving several GPUs (`configure(devices)`, ncclCommInitAll,
  grouped NCCL calls from one thread, sub-communicator broadcasts);
* SPMD under torchrun (tests/mp_check.py) at 2 GPUs.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_single_process_multi_gpu():
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2203_08069_b200 as td
from oracle.contractions import seq_eval
n = min(4, __import__('torch').cuda.device_count())
td.configure(list(range(n)))
for b in (td.summa(4, 1, dims=(64, 48, 80), chunk=16), td.cannon(2, 2, dims=(40, 36, 44)),
          td.johnson(2, 2, 2, dims=(24, 20, 28)), td.mttkrp(2, 2, dims=(12, 8, 10, 9)),
          td.innerprod3(2, dims=(8, 6, 30)), td.cosma_like((1, 1, 2), (1, 1, 1), dims=(72, 56, 90))):
    res, ins = b.run(seed=2)
    want = seq_eval(td.format_statement(b.statement), b.statement.extents, {k: v.data for k, v in ins.items()})
    assert np.array_equal(res.output.data, np.asarray(want)), b.name
# pipelined first step, forced on at test sizes
from paper_2203_08069_b200 import runtime as rt
rt.SPLIT_MIN_BYTES = 0
for b in (td.cannon(2, 2, dims=(520, 392, 1000)), td.johnson(2, 2, 2, dims=(264, 200, 1040))):
    res, ins = b.run(seed=9)
    want = seq_eval(td.format_statement(b.statement), b.statement.extents, {k: v.data for k, v in ins.items()})
    assert np.array_equal(res.output.data, np.asarray(want)), "split " + b.name
rt.SPLIT_MIN_BYTES = 32 << 20
# peer-memory write-back (cosma k-split): same bits as the NCCL path, twice in a row
from paper_2203_08069_b200 import peer
from oracle.generator import generate
b = td.cosma_like((1, 1, 2), (1, 1, 1), dims=(200, 136, 264))
res = {}
for flag in (True, False):
    peer.PEER_REDUCE = flag
    cin, store = b.prepare(seed=4, mode=1, world=td.comm.world())
    outs = []
    for _ in range(2):
        store.zero("A")
        td.execute(cin, store)
        outs.append(store["A"].tensor.data.copy())
    res[flag] = outs
peer.PEER_REDUCE = True
assert all(np.array_equal(res[True][0], x) for x in res[True][1:] + res[False]), "peer vs nccl write-back"
assert any(s.inboxes for s in td.comm.world().inbox_sets.values()), "peer inbox path not taken"
print("single-process multi-gpu OK")
""" % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_spmd_torchrun_two_gpus():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tests", "mp_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "mp_check world=2: OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_nccl_watchdog_aborts_instead_of_hanging():
    """A receive with no sender: World.wait gives up after its timeout, aborts
    the communicators and raises CommError (tests/nccl_watchdog_check.py)."""
    cmd = ["timeout", "180", sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "tests", "nccl_watchdog_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0 and "nccl_watchdog_check: OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_abi_collectives_allgather_and_shift():
    """td_allgather / td_shift (§8(b) ABI) on a one-process clique of the visible GPUs."""
    code = r"""
import ctypes as C, sys, torch
sys.path.insert(0, %r)
from paper_2203_08069_b200 import _native as nat
lib = nat.load()
n = min(4, torch.cuda.device_count())
devs = (C.c_int * n)(*range(n))
assert lib.td_init(n, devs) == 0
comms = (C.c_void_p * n)()
nat.call("td_comm_init_all", comms, n, devs)
cnt = 1000
send = [torch.full((cnt,), float(r + 1), dtype=torch.float64, device=f"cuda:{r}") for r in range(n)]
gath = [torch.zeros(n * cnt, dtype=torch.float64, device=f"cuda:{r}") for r in range(n)]
shf = [torch.zeros(cnt, dtype=torch.float64, device=f"cuda:{r}") for r in range(n)]
sts = [torch.cuda.current_stream(r).cuda_stream for r in range(n)]
nat.call("td_group_start")
for r in range(n):
    nat.call("td_allgather", C.c_void_p(comms[r]), C.c_void_p(sts[r]), C.c_void_p(send[r].data_ptr()),
             C.c_void_p(gath[r].data_ptr()), cnt)
nat.call("td_group_end")
nat.call("td_group_start")
for r in range(n):
    nat.call("td_shift", C.c_void_p(comms[r]), C.c_void_p(sts[r]), C.c_void_p(send[r].data_ptr()),
             C.c_void_p(shf[r].data_ptr()), cnt, 1)
nat.call("td_group_end")
assert lib.td_finalize() == 0
for r in range(n):
    want = torch.cat([torch.full((cnt,), float(q + 1), dtype=torch.float64) for q in range(n)])
    assert torch.equal(gath[r].cpu(), want), r
    assert torch.equal(shf[r].cpu(), torch.full((cnt,), float((r - 1) %% n + 1), dtype=torch.float64)), r
for r in range(n):
    nat.call("td_comm_destroy", C.c_void_p(comms[r]))
print("abi collectives OK")
""" % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "abi collectives OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_reference_suite_under_spmd():
    """The reference's own unit tests with every launch spread over 2 GPUs (tests/ref_suite_spmd.py)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", "29543", os.path.join(ROOT, "tests", "ref_suite_spmd.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ref_suite_spmd world=2" in out.stdout and "OK" in out.stdout, \
        out.stdout[-3000:] + out.stderr[-3000:]
