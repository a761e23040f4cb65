"""Multi-GPU parity run (SPMD, one process per GPU over NCCL).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_check.py

Every rank runs the same bundles; processors map onto the N GPUs
(Machine.device_of) and all cross-GPU CommEvents travel over NCCL.  Each
result is compared on every rank with the golden reference output
(tests/golden/bundles.json, integer inputs => bit-exact) or with the CPU
oracle.  Exits non-zero on any mismatch.  Also exercises redistribute and
the single-process multi-GPU mode is covered by test_multigpu.py.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402
from _cases import build, case_id, load  # noqa: E402
from oracle.contractions import seq_eval  # noqa: E402
from oracle.generator import generate  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = td.configure_distributed()
    rank, size = dist.get_rank(), dist.get_world_size()
    failures = []

    for fix in load("bundles.json"):
        b = build(td, fix["case"])
        for policy in ("auto", "exact"):
            res, _ = b.run(seed=13, leaf_policy=policy)
            want = np.asarray(fix["output"], dtype=np.float64).reshape(fix["dims"])
            if not np.array_equal(res.output.data, want):
                failures.append(f"{case_id(fix['case'])} {policy}")
        # real-valued inputs: exact policy is bitwise the reference
        ins = {}
        for k, name in enumerate(b.input_names):
            dims = b.statement.tensors()[name].dims
            ins[name] = td.DenseTensor(dims, generate(dims, 13, k + 1, 1))
        res, _ = b.run(inputs=ins, leaf_policy="exact")
        want = np.array([float.fromhex(x) for x in fix["real_output_hex"]]).reshape(fix["dims"])
        if not np.array_equal(res.output.data, want):
            failures.append(f"{case_id(fix['case'])} real-exact")

    # larger shapes through the native leaves, checked against the oracle
    for b in (td.summa(2, 1, dims=(192, 160, 256), chunk=32), td.cannon(2, 2, dims=(200, 144, 176)),
              td.johnson(2, 2, 2, dims=(128, 96, 160)), td.mttkrp(2, 2, dims=(40, 32, 48, 36)),
              td.ttm2d(2, 2, dims=(16, 12, 40, 24)), td.innerprod3(4, dims=(24, 10, 70)),
              td.ttv(4, dims=(20, 12, 90)), td.solomonik(2, 2, 2, dims=(64, 48, 80)),
              td.summa(4, 1, dims=(96, 80, 128), chunk=16), td.summa(4, 2, dims=(64, 48, 96), chunk=8),
              td.cosma_like((4, 1, 1), (1, 1, 2), dims=(64, 40, 72))):
        res, ins = b.run(seed=3)  # same inputs on every rank (SPMD)
        want = seq_eval(td.format_statement(b.statement), b.statement.extents,
                        {n: t.data for n, t in ins.items()})
        if not np.array_equal(res.output.data, np.asarray(want)):
            failures.append(f"oracle {b.name} {b.machine}")

    # 8 logical processors on the job's GPUs (two per GPU at 4 GPUs, Machine.device_of): the
    # BASELINE p = 8 layouts -- Johnson 2x2x2, MTTKRP / TTM on 4x2, TTV / innerprod on 8
    for b in (td.johnson(2, 2, 2, dims=(256, 192, 320)), td.mttkrp(4, 2, dims=(64, 24, 48, 40)),
              td.ttm2d(4, 2, dims=(32, 24, 40, 16)), td.ttv(8, dims=(40, 12, 90)),
              td.innerprod3(8, dims=(48, 10, 70))):
        res, ins = b.run(seed=4)
        want = seq_eval(td.format_statement(b.statement), b.statement.extents,
                        {n: t.data for n, t in ins.items()})
        if not np.array_equal(res.output.data, np.asarray(want)):
            failures.append(f"8-proc {b.name} {b.machine}")

    # Johnson 2x2x2 with its depth pairs on different GPUs (cyclic placement at 4 GPUs, as at 8):
    # the depth partials travel through peer inboxes, eagerly and from replayed launch plans
    if size == 4:
        from paper_2203_08069_b200 import machine as mach
        mach.set_placement("cyclic")
        try:
            b = td.johnson(2, 2, 2, dims=(128, 96, 160))
            cin, store = b.prepare(seed=17, mode=0, world=world)
            ins = {n: generate(b.statement.tensors()[n].dims, 17, k + 1, 0) for k, n in enumerate(b.input_names)}
            want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
            for rep in range(4):
                store.zero("C")
                td.execute(cin, store)
                if not np.array_equal(store["C"].tensor.data, want):
                    failures.append(f"johnson cyclic run {rep}")
            used = sum(len(s.inboxes) for s in world.inbox_sets.values())
            if used == 0:
                failures.append("johnson cyclic: no peer inbox used")
            if rank == 0:
                print(f"peer johnson 2x2x2 (cyclic on {size} GPUs): inboxes in use {used}", flush=True)
        finally:
            mach.set_placement("block")

    # launch plans under SPMD: each rank records its own ops (NCCL groups, peer-inbox tokens and
    # credits, leaves) on the second execute and replays them from the third
    from paper_2203_08069_b200 import runtime as rt
    pcases = [td.summa(2, 1, dims=(200, 160, 512), chunk=64), td.cosma_like((1, 1, 2), (1, 1, 1), dims=(136, 120, 300)),
              td.mttkrp(2, 1, dims=(48, 16, 40, 36)), td.johnson(2, 2, 2, dims=(96, 80, 112))]
    if size >= 4:
        pcases += [td.cannon(2, 2, dims=(200, 144, 176)), td.cosma_like((2, 1, 2), (1, 1, 1), dims=(130, 96, 150)),
                   td.mttkrp(2, 2, dims=(40, 32, 48, 36))]
    for b in pcases:
        cin, store = b.prepare(seed=16, mode=0, world=world)
        out = b.statement.lhs.tensor.name
        ins = {n: generate(b.statement.tensors()[n].dims, 16, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
        for rep in range(5):
            store.zero(out)
            td.execute(cin, store)
            if not np.array_equal(store[out].tensor.data, want):
                failures.append(f"plan {b.name} {b.machine} run {rep}")
        if not any(isinstance(v, tuple) for v in store.__dict__.get("_launch_plans", {}).values()):
            failures.append(f"plan {b.name} {b.machine}: nothing recorded")

    # copy-engine shifts (peer.CE_SHIFTS): transfers after step 0 go by cudaMemcpy into a
    # persistent buffer on the receiver + 8-byte NCCL tokens / credits; forced on at test
    # sizes, eagerly and from replayed launch plans, bit-exact against the oracle
    from paper_2203_08069_b200 import peer as _peer
    saved_shift = _peer.SHIFT_MIN_BYTES
    _peer.SHIFT_MIN_BYTES = 0
    shifted = 0
    try:
        for b in (td.cannon(2, 2, dims=(200, 144, 176)), td.cannon(2, 2, dims=(130, 96, 150)),
                  td.summa(2, 1, dims=(192, 160, 256), chunk=32), td.pumma(2, 2, dims=(96, 80, 112)),
                  td.solomonik(2, 2, 2, dims=(64, 48, 80))):
            cin, store = b.prepare(seed=21, mode=0, world=world)
            out = b.statement.lhs.tensor.name
            ins = {n: generate(b.statement.tensors()[n].dims, 21, k + 1, 0) for k, n in enumerate(b.input_names)}
            want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
            for rep in range(5):
                store.zero(out)
                td.execute(cin, store)
                if not np.array_equal(store[out].tensor.data, want):
                    failures.append(f"ce-shift {b.name} {b.machine} run {rep}")
            shifted += sum(len(st.by_transfer()) for st in world.inbox_sets.values())
    finally:
        _peer.SHIFT_MIN_BYTES = saved_shift
    if shifted == 0 and size > 1 and _peer.CE_SHIFTS:
        failures.append("ce-shift: no copy-engine shift used")
    if rank == 0:
        print(f"copy-engine shifts in use: {shifted}", flush=True)

    # pipelined first step (k-pieces on the transfers and the GEMM leaves), forced on at test sizes
    saved = rt.SPLIT_MIN_BYTES
    rt.SPLIT_MIN_BYTES = 0
    for b in (td.cannon(2, 2, dims=(520, 392, 1000)), td.johnson(2, 2, 2, dims=(264, 200, 1040)),
              td.summa(2, 1, dims=(200, 160, 2048), chunk=512),
              td.cosma_like((1, 1, 2), (1, 1, 1), dims=(136, 120, 1200))):
        for seed in (9, 10):
            res, ins = b.run(seed=seed)
            want = seq_eval(td.format_statement(b.statement), b.statement.extents,
                            {n: t.data for n, t in ins.items()})
            if not np.array_equal(res.output.data, np.asarray(want)):
                failures.append(f"split {b.name} {b.machine} seed {seed}")
    # real-valued inputs: the k-pieces reassociate the k sum, so compare with the whole-step run
    # within the stated bound |got - want| <= 2 gamma_K (|A||B|)_ij, gamma_K = K u / (1 - K u)
    b = td.cannon(2, 2, dims=(520, 392, 1000))
    outs = {}
    for thr in (0, 1 << 62):
        rt.SPLIT_MIN_BYTES = thr
        cin, store = b.prepare(seed=15, mode=1, world=world)
        td.execute(cin, store)
        outs[thr] = store["C"].tensor.data.copy()
    rt.SPLIT_MIN_BYTES = 0
    a_abs = np.abs(generate(b.statement.tensors()["A"].dims, 15, 1, 1))
    b_abs = np.abs(generate(b.statement.tensors()["B"].dims, 15, 2, 1))
    kk = b.statement.extents["k"]
    u = 2.0 ** -53
    bound = 2 * (kk * u / (1 - kk * u)) * (a_abs @ b_abs)
    if not np.all(np.abs(outs[0] - outs[1 << 62]) <= bound):
        failures.append("split real-valued tolerance")

    if size >= 4:
        # split first step + peer inboxes together (Johnson 2x2x2 at 8 GPUs does both), twice in a row
        b = td.cosma_like((2, 1, 2), (1, 1, 1), dims=(130, 96, 1200))
        cin, store = b.prepare(seed=6, mode=0, world=world)
        ins = {n: generate(b.statement.tensors()[n].dims, 6, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
        for rep in range(2):
            store.zero("A")
            td.execute(cin, store)
            if not np.array_equal(store["A"].tensor.data, want):
                failures.append(f"split+peer {b.machine} rep {rep}")
    rt.SPLIT_MIN_BYTES = saved

    # e2e shape: inputs uploading in k-slabs from host pieces, pipelined first step in 8 slab-aligned
    # pieces, row-streamed output (bench.py bench_gemm_e2e), checked against the oracle
    from oracle.generator import generate_box
    rt.SPLIT_MIN_BYTES = 0
    b = td.cannon(2, 2, dims=(520, 392, 1024)) if size >= 4 else td.summa(2, 1, dims=(600, 160, 1024), chunk=512)
    cin = b.scheduled()
    st2 = td.RegionStore(b.machine, world)
    for k, name in enumerate(b.input_names):
        dd = b.distributions[name]
        pieces = {c: generate_box(dd.tensor_dims, box.lo, box.shape, 12, k + 1, 0) for c, box in st2.local_colors(dd)}
        st2.place_local(name, dd, pieces, defer=True)
        for c, _ in st2.local_colors(dd):
            st2.upload(name, c, slabs=8 if name == "A" else 4, axis=1 if name == "A" else 0, copy_stream=k)
    out = b.statement.lhs.tensor.name
    st2.place_zeros(out, b.distributions[out])
    st2.stream_rows, st2.first_step_pieces = 4, 8
    td.execute(cin, st2)
    ins = {n: generate(b.statement.tensors()[n].dims, 12, k + 1, 0) for k, n in enumerate(b.input_names)}
    want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
    if not np.array_equal(st2[out].tensor.data, want):
        failures.append(f"e2e-shape {b.name} {b.machine}")
    rt.SPLIT_MIN_BYTES = saved

    # output streaming: the last step's leaves in row pieces with per-piece events (e2e D2H overlap)
    for b in (td.cannon(2, 2, dims=(520, 392, 1000)), td.summa(2, 1, dims=(600, 160, 512), chunk=128)):
        cin, store = b.prepare(seed=8, mode=0, world=world)
        store.stream_rows = 4
        td.execute(cin, store)
        out = b.statement.lhs.tensor.name
        ins = {n: generate(b.statement.tensors()[n].dims, 8, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
        owns_task = rank < b.machine.size            # one processor per GPU here, in rank order
        if (owns_task and not store.row_done) or any(len(v) < 2 for v in store.row_done.values()):
            failures.append(f"stream rows {b.name}: no row pieces")
        if not np.array_equal(store[out].tensor.data, want):
            failures.append(f"stream rows {b.name} values")

    # peer-memory write-backs: the leaf stores its partial into the home GPU's
    # inbox (peer.py); bitwise equal to the NCCL write-back path, also when one
    # program runs twice (inbox reuse behind the credit token)
    from paper_2203_08069_b200 import peer
    peer_cases = [td.cosma_like((1, 1, 2), (1, 1, 1), dims=(136, 120, 200))]
    if size >= 4:
        peer_cases.append(td.cosma_like((2, 1, 2), (1, 1, 1), dims=(130, 96, 150)))
    if size >= 8:
        peer_cases.append(td.johnson(2, 2, 2, dims=(128, 96, 160)))
    for b in peer_cases:
        got = {}
        for flag in (True, False):
            peer.PEER_REDUCE = flag
            for mode in (0, 1):
                cin, store = b.prepare(seed=5, mode=mode, world=world)
                outs = []
                for _ in range(2):
                    store.zero(b.statement.lhs.tensor.name)
                    td.execute(cin, store)
                    outs.append(store[b.statement.lhs.tensor.name].tensor.data.copy())
                got[(flag, mode)] = outs
        peer.PEER_REDUCE = True
        used = sum(len(s.inboxes) for s in world.inbox_sets.values())
        for mode in (0, 1):
            a, bb = got[(True, mode)], got[(False, mode)]
            if not (np.array_equal(a[0], a[1]) and np.array_equal(a[0], bb[0]) and np.array_equal(bb[0], bb[1])):
                failures.append(f"peer {b.name} {b.machine} mode {mode}")
        ins = {n: generate(b.statement.tensors()[n].dims, 5, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = seq_eval(td.format_statement(b.statement), b.statement.extents, ins)
        if not np.array_equal(got[(True, 0)][0], np.asarray(want)):
            failures.append(f"peer oracle {b.name} {b.machine}")
        if rank == 0:
            print(f"peer {b.name} {b.machine}: inboxes in use {used}", flush=True)

    # placement-phase movement over NCCL
    machine = td.grid(2, 2)
    old = td.TensorDistribution((6, 8), machine, [(("x", "y"), ("x", 0))])
    new = td.TensorDistribution((6, 8), machine, [(("x", "y"), ("y", "x"))])
    store = td.RegionStore(machine, world)
    data = td.DenseTensor((6, 8), np.arange(48, dtype=float).reshape(6, 8))
    store.place("T", data, old)
    trace = td.ExecutionTrace(machine)
    td.redistribute(store, "T", new, trace)
    if not np.array_equal(store["T"].tensor.data, data.data):
        failures.append("redistribute")

    # multi-GPU CUDA graphs: one execute (NCCL groups, peer-inbox tokens, leaves) captured per rank and
    # replayed.  Last: after a capture NCCL synchronises eager work on the communicator with the graph's;
    # the graphs are destroyed before the communicators are
    from paper_2203_08069_b200.runtime import CapturedLaunch
    gcases = [td.summa(2, 1, dims=(200, 160, 512), chunk=64), td.cosma_like((1, 1, 2), (1, 1, 1), dims=(136, 120, 300))]
    if size >= 4:
        gcases += [td.cannon(2, 2, dims=(200, 144, 176)), td.mttkrp(2, 2, dims=(40, 32, 48, 36)),
                   td.summa(2, 2, dims=(256, 256, 256), chunk=32)]
    for b in gcases:
        cin, store = b.prepare(seed=14, mode=0, world=world)
        out = b.statement.lhs.tensor.name
        cap = CapturedLaunch(cin, store)
        ins = {n: generate(b.statement.tensors()[n].dims, 14, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
        for rep in range(3):
            cap.replay()
            if not np.array_equal(store[out].tensor.data, want):
                failures.append(f"graph {b.name} {b.machine} replay {rep}")
        td.execute(cin, store)    # eager again after replays (accumulates onto the last replay's output)
        store.zero(out)
        td.execute(cin, store)
        if not np.array_equal(store[out].tensor.data, want):
            failures.append(f"graph {b.name} {b.machine} eager after replays")
        del cap
    # a captured launch whose shifts go by copy engine (forced on at test size)
    from paper_2203_08069_b200 import peer as _peer
    saved_shift, _peer.SHIFT_MIN_BYTES = _peer.SHIFT_MIN_BYTES, 0
    try:
        b = td.cannon(2, 2, dims=(264, 200, 312))
        cin, store = b.prepare(seed=19, mode=0, world=world)
        cap = CapturedLaunch(cin, store)
        ins = {n: generate(b.statement.tensors()[n].dims, 19, k + 1, 0) for k, n in enumerate(b.input_names)}
        want = np.asarray(seq_eval(td.format_statement(b.statement), b.statement.extents, ins))
        for rep in range(3):
            cap.replay()
            if not np.array_equal(store["C"].tensor.data, want):
                failures.append(f"graph ce-shift cannon replay {rep}")
        if _peer.CE_SHIFTS and not any(st.by_transfer() for st in world.inbox_sets.values()):
            failures.append("graph ce-shift: no copy-engine shift used")
        del cap
    finally:
        _peer.SHIFT_MIN_BYTES = saved_shift
    import gc
    gc.collect()
    torch.cuda.synchronize()

    flag = torch.tensor([len(failures)], device="cuda")
    dist.all_reduce(flag)
    if rank == 0:
        print(f"mp_check world={size}: {'OK' if flag.item() == 0 else 'FAIL'}", flush=True)
    if failures:
        print(f"rank {rank} failures: {failures}", flush=True)
    dist.barrier(device_ids=[local])
    world.close()
    dist.destroy_process_group()
    sys.exit(1 if flag.item() else 0)


if __name__ == "__main__":
    main()
