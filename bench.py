#!/usr/bin/env python
"""Benchmark of the B200 DISTAL path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload all|gemm] [--cpu-baseline|--no-cpu-baseline]

Headline (`value`): fp64 GEMM, weak-scaled from 16384^3 with constant flop
per GPU (n = 16384 * p^(1/3) rounded up to 256): Cannon 1x1 at p=1, SUMMA
2x1 at p=2, Cannon 2x2 at p=4, Johnson 2x2x2 at p=8.
One step = one `execute` of the scheduled statement over inputs already
resident in HBM (output reset, every NCCL transfer, every leaf, every
commit); `value` = total GFLOP/s of the job (2 n^3 / max-over-ranks step
time).  Inputs (2-8 GiB per operand) are far larger than the 126 MB L2, so
no flush is needed between steps.

`e2e`: the same GEMM through the public API with host buffers: per step the
H2D copy of this rank's input pieces from pinned memory, `execute`, and the
D2H copy of this rank's output pieces into pinned memory.

`kernels` (workload "all"): the other BASELINE configs through the same
runtime on device-resident inputs -- TTV and 3-order innerprod on 2048^3 per
GPU (GB/s vs HBM), TTM 1024^3 x 64 and MTTKRP 1024^3 rank 32 per GPU
(GFLOP/s vs FP64 peak), weak-scaled over the GPUs.

Under torchrun (WORLD_SIZE > 1) every rank drives its GPU; times are
max-over-ranks of CUDA-event measurements bracketed by barriers.
`--impl reference` times the REFERENCE itself on rank 0: tendist (staged
in oracle/_ref) running the same GEMM bundle through its own
`run_statement`, with a numpy/OpenBLAS leaf substituted through its plugin
API (oracle/ref_bench.py), at the same n on all host cores; plus CPU-A, the
reference as shipped (per-point interpreter, one core) at a scaled shape.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 GEMM GFLOP/s/GPU at 1/2/4/8 B200; TTM/MTTKRP GFLOP/s, TTV GB/s vs roof"
FP64_PEAK_TFLOPS = 37.07      # DMMA/DFMA probe on this pool's B200 (profiles/peaks_r01.json)
DGEMM_CUBLAS_TFLOPS = 36.14   # cuBLAS DGEMM 16384^3 on the same pool (profiles/peaks_r01.json)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[3]) for r in self.rows if _num(r[3])), default=None)}


def _num(x):
    try:
        float(x)
        return True
    except ValueError:
        return False


# ------------------------------------------------------------------ helpers
class Job:
    def __init__(self, n_gpus, procs=0):
        import torch
        self.torch = torch
        self.size = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        if self.size > 1:
            import torch.distributed as dist
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist = dist
        else:
            self.dist = None
        import paper_2203_08069_b200 as td
        self.td = td
        self.world = td.configure_distributed() if self.size > 1 else td.comm.world()
        self.device = self.world.device(self.world.owned[0])
        self.n_gpus = max(n_gpus, self.size)
        # logical processors of the BASELINE layout (default one per GPU; e.g. 8 on 4 GPUs
        # runs the p = 8 programs two processors per GPU, Machine.device_of)
        self.procs = procs or self.n_gpus

    def close(self):
        # same teardown order as tests/mp_check.py: communicators, then the process group
        if self.dist is not None:
            self.torch.cuda.synchronize()
            self.barrier()
            self.world.close()
            self.dist.destroy_process_group()

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier(device_ids=[self.device.index])
        self.torch.cuda.synchronize(self.device)

    def max_over_ranks(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return float(t.item())

    def timed(self, fn, steps, warmup):
        """max-over-ranks device time (ms) of `steps` calls of fn after `warmup`."""
        torch = self.torch
        for _ in range(warmup):
            fn()
        self.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        e.synchronize()
        self.barrier()
        return self.max_over_ranks(s.elapsed_time(e))


def _leaf_timing(td, kind):
    """mean device time (ms) of the native `kind` launches recorded by leaves.TIMING."""
    from paper_2203_08069_b200 import leaves
    ts = [a.elapsed_time(b) for k, a, b in (leaves.TIMING or []) if k == kind]
    return (sum(ts) / len(ts), len(ts)) if ts else (None, 0)


def _profile_traffic(name):
    """DRAM bytes per launch of the kernel from the latest committed ncu capture."""
    import glob
    found = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")))
    if not found:
        return None
    path = found[-1]
    try:
        with open(path) as fh:
            return json.load(fh).get(name, {}).get("dram_bytes_per_launch")
    except OSError:
        return None


# ------------------------------------------------------------------ GEMM
def bench_gemm(job, steps, warmup, e2e_steps):
    td, torch = job.td, job.torch
    from paper_2203_08069_b200 import leaves, _native
    p = job.procs
    n = td.weak_gemm_n(p)
    bundle = td.gemm_for_gpus(p, n)
    cin, store = bundle.prepare(seed=0, mode=0, world=job.world)
    out = bundle.statement.lhs.tensor.name

    def step():
        store.zero(out)
        td.execute(cin, store, record_requirements=False)

    leaves.TIMING = None
    for _ in range(warmup):
        step()
    job.barrier()
    launches0 = _native.launch_count()
    gpu = job.world.owned[0]
    # the timed steps run as every repeated launch does: replaying the recorded
    # launch plan (td_execute_plan; its temporaries stay allocated)
    with Clocks(job.device.index) as clk:
        ms = job.timed(step, steps, 0)
    launches = _native.launch_count() - launches0
    # the DMMA launch durations for the roofline: the same steps again with a CUDA
    # event pair around every leaf on its stream (plans do not record leaf timing,
    # so this pass runs the Python step loop)
    leaves.TIMING = []
    job.timed(step, steps, 0)
    dgemm_ms, n_dgemm = _leaf_timing(td, "dgemm")
    leaves.TIMING = None
    flop = 2.0 * n ** 3
    value = flop * steps / (ms / 1e3) / 1e9
    # the same steps with communication serialised behind computation: the gap is the
    # overlap the side-stream NCCL groups buy (zero at p=1, where nothing moves)
    overlap = None
    if p > 1:
        from paper_2203_08069_b200 import runtime as rt
        rt.OVERLAP_COMM = False
        try:
            ms_serial = job.timed(step, steps, 1)
        finally:
            rt.OVERLAP_COMM = True
        overlap = {"ms_per_step_overlapped": ms / steps, "ms_per_step_serialised": ms_serial / steps,
                   "saved_ms_per_step": (ms_serial - ms) / steps}
    # parity spot check of the last step: exact on integer inputs (Freivalds-style row sample)
    check = _gemm_spot_check(job, store, bundle, n)

    # roofline of the dominant kernel on this rank: the rank's algorithmic GEMM flop
    # over the summed device time of its DMMA launches (the pipelined first step
    # runs its k-range as two launches, so launches differ in size)
    flop_per_launch = 2.0 * n ** 3 / job.n_gpus * steps / n_dgemm if n_dgemm else None
    achieved = flop_per_launch / (dgemm_ms / 1e3) / 1e12 if dgemm_ms else None

    # e2e through the public API with host buffers
    del store, step
    gc.collect()
    torch.cuda.empty_cache()
    e2e = bench_gemm_e2e(job, bundle, cin, e2e_steps)
    gc.collect()
    torch.cuda.empty_cache()
    return {
        "n": n, "bundle": bundle.name, "machine": str(bundle.machine), "ms_per_step": ms / steps,
        "value": value, "per_gpu": value / job.n_gpus, "gpu_launches": launches, "launches_per_step": launches / steps,
        "dgemm_launches_timed": n_dgemm, "dgemm_ms_per_launch": dgemm_ms, "check": check,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None,
                     "traffic": _profile_traffic("dgemm"),
                     "peak_source": "builder-measured FP64 DMMA probe (profiles/peaks_r01.json; MEASURED_PEAKS.json "
                                    "has no FP64 entry); cuBLAS DGEMM on the same GPUs: "
                                    f"{DGEMM_CUBLAS_TFLOPS} TFLOP/s",
                     "frac_of_cublas_dgemm": (achieved / DGEMM_CUBLAS_TFLOPS) if achieved else None,
                     "flop_per_launch": flop_per_launch,
                     "timing": "CUDA event pair around every DMMA leaf on its stream, over a second pass of the "
                               "same steps (the value's pass replays the launch plan, which records no leaf "
                               "timing)"},
        "clocks": clk.summary(), "e2e": e2e, "overlap": overlap,
    }


def _gemm_spot_check(job, store, bundle, n):
    """Rows of the distributed result vs A[rows] @ B from the generated inputs
    (integer-valued, so the comparison is exact)."""
    torch, td = job.torch, job.td
    from oracle.generator import generate_box
    rows = [0, n // 3, n - 1]
    ok = True
    for box, buf in store.local_pieces(bundle.statement.lhs.tensor.name):
        # the piece's first and last 64 columns of the sampled rows (bounded host work at any n)
        w = min(64, box.hi[1] - box.lo[1])
        blocks = [(box.lo[1], generate_box((n, n), (0, box.lo[1]), (n, w), 0, 2, 0)),
                  (box.hi[1] - w, generate_box((n, n), (0, box.hi[1] - w), (n, w), 0, 2, 0))]
        for r in rows:
            if not (box.lo[0] <= r < box.hi[0]):
                continue
            a_row = generate_box((n, n), (r, 0), (1, n), 0, 1, 0)
            got = buf[r - box.lo[0]].cpu().numpy()
            for c0, b_cols in blocks:
                want = (a_row @ b_cols).ravel()
                ok = ok and bool(np.array_equal(got[c0 - box.lo[1]:c0 - box.lo[1] + w], want))
    return {"rows_exact": ok}


def bench_gemm_e2e(job, bundle, cin, steps):
    """Host buffers -> H2D -> execute -> D2H, per step, through the public API.

    Inputs arrive in k-slabs on two copy streams (A and B concurrently,
    RegionStore.place_local(slabs=..)) so uploads overlap the DMMA leaves of
    earlier k-chunks, and each output piece is downloaded as soon as its last
    write is done (store.done events) while later tasks still compute.  At
    p=1 the GEMM runs as SUMMA on a 4x1 grid placed on the one GPU (row
    blocks of C finish one after another, task-major) with 8 k-chunks; p>1
    keeps the headline algorithm."""
    td, torch = job.td, job.torch
    from oracle.generator import generate_box
    if bundle.name == "cannon" and bundle.machine.size == 1:
        n = bundle.statement.extents["i"]
        bundle = td.summa(4, 1, dims=(n, n, n), chunk=-(-n // 8))
        cin = bundle.scheduled()
    slab_axis = {"A": 1, "B": 0}
    nslabs = {"A": 8, "B": 4}
    d2h_stream = torch.cuda.Stream(device=job.device)
    st = td.RegionStore(bundle.machine, job.world)
    host = {}
    h2d = 0
    for k, name in enumerate(bundle.input_names):
        dist = bundle.distributions[name]
        pieces = {}
        for color, box in st.local_colors(dist):
            t = torch.empty(box.shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = generate_box(dist.tensor_dims, box.lo, box.shape, 0, k + 1, 0)
            pieces[color] = t.numpy()
            h2d += t.numel() * 8
        host[name] = pieces
    out = bundle.statement.lhs.tensor.name
    out_dist = bundle.distributions[out]
    sink = {}
    d2h = 0
    for color, box in st.local_colors(out_dist):
        sink[color] = torch.empty(box.shape, dtype=torch.float64, pin_memory=True)

    def step():
        s2 = td.RegionStore(bundle.machine, job.world)
        for k, name in enumerate(bundle.input_names):
            s2.place_local(name, bundle.distributions[name], host[name], defer=True)
        if bundle.machine.flat_dims == (4, 1) and job.world.ngpus == 1:
            # task-major on one GPU: task 0 needs A0 and every B k-slab first,
            # in k order; the other A row blocks can follow.  The first k-chunk
            # arrives in 8 sub-slabs that task 0's first GEMM consumes piece by
            # piece (first_step_pieces), so compute starts after 1/64 of A0 and B
            for q in range(8):
                s2.upload("B", (0, 0), slabs=16, axis=0, only=[q])
                s2.upload("A", (0, 0), slabs=64, axis=1, only=[q])
            s2.upload("B", (0, 0), slabs=16, axis=0, only=range(8, 16))
            for s in range(1, 8):
                if s >= 2:
                    s2.upload("B", (s // 2, 0), slabs=2, axis=0, only=[s % 2])
                s2.upload("A", (0, 0), slabs=64, axis=1, only=range(8 * s, 8 * s + 8))
            for q in range(1, 4):
                s2.upload("A", (q, 0), slabs=8, axis=1)
        else:
            for k, name in enumerate(bundle.input_names):
                for color, _ in s2.local_colors(bundle.distributions[name]):
                    s2.upload(name, color, slabs=nslabs[name], axis=slab_axis[name], copy_stream=k)
        s2.place_zeros(out, out_dist)
        # the last step's leaves of each output piece run in row pieces and each piece's
        # rows download as soon as they are done (at p > 1 every output piece is final
        # only after the last step; at p = 1 this shortens the last row block's tail)
        s2.stream_rows = 8
        # the first step's GEMM runs in 8 k-pieces that wait only for their own slabs (p > 1:
        # the pipelined first step, in the A upload's 8 slabs; p = 1: task 0's first k-chunk)
        s2.first_step_pieces = 8
        td.execute(cin, s2, record_requirements=False)
        nbytes = 0
        for color, box, _ in out_dist.pieces():
            gpus = s2[out].gpus_of(color)
            if gpus and job.world.owns(gpus[0]):
                piece = s2[out].piece(gpus[0], color)
                rows = s2.row_done.get((out, gpus[0], color))
                if rows:
                    for lo, hi, ev in rows:
                        d2h_stream.wait_event(ev)
                        with torch.cuda.stream(d2h_stream):
                            sink[color][lo:hi].copy_(piece[lo:hi], non_blocking=True)
                    ev = s2.done.get((out, gpus[0], color))
                    if ev is not None:
                        d2h_stream.wait_event(ev)
                else:
                    ev = s2.done.get((out, gpus[0], color))
                    if ev is not None:
                        d2h_stream.wait_event(ev)
                    else:
                        d2h_stream.wait_stream(torch.cuda.current_stream(job.device))
                    with torch.cuda.stream(d2h_stream):
                        sink[color].copy_(piece, non_blocking=True)
                piece.record_stream(d2h_stream)
                nbytes += box.volume * 8
        d2h_stream.synchronize()
        torch.cuda.current_stream(job.device).synchronize()
        return nbytes

    d2h = step()  # warm-up (also sizes D2H)
    job.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    job.barrier()
    dt = job.max_over_ranks(time.perf_counter() - t0)
    # the downloaded output of the last e2e step: sampled rows exact (integer inputs)
    n = bundle.statement.extents["i"]
    ok = True
    for color, box, _ in out_dist.pieces():
        if color not in sink:
            continue
        w = min(64, box.hi[1] - box.lo[1])
        b_cols = generate_box((n, n), (0, box.lo[1]), (n, w), 0, 2, 0)
        for r in (box.lo[0], (box.lo[0] + box.hi[0]) // 2, box.hi[0] - 1):
            a_row = generate_box((n, n), (r, 0), (1, n), 0, 1, 0)
            ok = ok and bool(np.array_equal(sink[color][r - box.lo[0], :w].numpy(), (a_row @ b_cols).ravel()))
    ok = job.sum_over_ranks(0.0 if ok else 1.0) == 0.0
    flop = 2.0 * bundle.statement.extents["i"] * bundle.statement.extents["j"] * bundle.statement.extents["k"]
    return {"value": flop * steps / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(job.sum_over_ranks(h2d)),
            "d2h_bytes_per_step": int(job.sum_over_ranks(d2h)), "ms_per_step": dt * 1e3 / steps,
            "steps": steps, "algorithm": f"{bundle.name} {bundle.machine}", "rows_exact": ok,
            "algorithm_note": ("p = 1: the same 16384^3 GEMM as SUMMA on a 4x1 grid placed on the one GPU (4 row "
                               "blocks x 8 k-chunks), so the upload of later k-slabs and the download of finished "
                               "row blocks overlap the DMMA leaves; the device-resident `value` runs Cannon 1x1")
            if bundle.machine.size == 4 and job.world.ngpus == 1 else "the headline algorithm",
            "how": "pinned host pieces -> RegionStore.place_local (async H2D in k-slabs on two copy streams; "
                   "leaves and NCCL sends wait only for the slabs they touch: p=1 task-major k-chunks, p>1 "
                   "the pipelined first step in the A upload's 8 k-slabs) -> execute -> D2H of output rows as "
                   "soon as their row piece of the last step is done (RegionStore.stream_rows / row_done); "
                   "host wall clock, max over ranks"}


def _spot_check(job, bundle, store, per_piece=4):
    """Result check of a timed config on every rank: sampled points of this
    rank's output pieces against the exact integer value recomputed on the
    host from the generated input slices (oracle/spot.py; integer inputs, so
    the comparison is bit-exact).  Scalar outputs (innerprod) are checked in
    tests/test_fullsize_gpu.py instead (the host total takes minutes)."""
    from oracle.spot import points
    stmt = bundle.statement
    out = stmt.lhs.tensor.name
    if not stmt.lhs.var_names:
        return {"points": 0, "exact": None, "note": "scalar output: tests/test_fullsize_gpu.py"}
    rng = np.random.default_rng(job.rank)
    coords, got = [], []
    for box, buf in store.local_pieces(out):
        for k in range(per_piece):
            c = tuple(int(lo if k == 0 else hi - 1 if k == 1 else rng.integers(lo, hi))
                      for lo, hi in zip(box.lo, box.hi))
            coords.append(c)
            got.append(float(buf[tuple(x - lo for x, lo in zip(c, box.lo))].item()))
    bad = sum(1 for g, (e, _, _) in zip(got, points(stmt, coords, seed=0, mode=0)) if g != e)
    npts = job.sum_over_ranks(float(len(coords)))
    nbad = job.sum_over_ranks(float(bad))
    return {"points": int(npts), "exact": nbad == 0}


# ------------------------------------------------------------------ other configs
def bench_kernels(job, steps, warmup):
    td, torch = job.td, job.torch
    from paper_2203_08069_b200 import leaves
    p = job.procs
    hbm = _peaks().get("hbm_gbs", 6544.3)
    results = {}

    def run(name, bundle, work, unit, roof, kind):
        cin, store = bundle.prepare(seed=0, mode=0, world=job.world)
        out = bundle.statement.lhs.tensor.name

        def step():
            store.zero(out)
            td.execute(cin, store, record_requirements=False)

        for _ in range(warmup):
            step()
        # short steps (2-20 ms): time enough of them (>= ~100 ms) that the host's issue
        # latency before the first step does not count against the device rate.  The
        # step rate is measured with launch plans replaying (runtime._launch); the kernel
        # rate in a second pass with per-leaf CUDA events (which runs the eager loop)
        est = job.timed(step, 1, 0)
        nsteps = max(steps, min(50, int(100.0 / max(est, 1e-3)) + 1))
        ms = job.timed(step, nsteps, 0)
        leaves.TIMING = []
        ms_eager = job.timed(step, nsteps, 0)
        kms, nk = _leaf_timing(td, kind)
        leaves.TIMING = None
        check = _spot_check(job, bundle, store)
        per_task_work = work / p          # one leaf launch per task per step
        rate = work * nsteps / (ms / 1e3) / 1e9
        kern = per_task_work / (kms / 1e3) / 1e9 if kms else None
        results[name] = {
            "config": bundle.name + " " + str(bundle.machine) + " dims " + str(
                tuple(bundle.statement.extents[v] for v in bundle.statement.var_order)),
            "value": rate, "unit": unit, "per_gpu": rate / job.n_gpus, "ms_per_step": ms / nsteps, "steps": nsteps,
            "ms_per_step_eager_timed": ms_eager / nsteps,
            "kernel": kind, "kernel_ms": kms, "kernel_rate_per_gpu": kern,
            "frac_of_roof": (kern / roof) if kern else None, "roof": roof, "check": check,
        }
        del store, step
        gc.collect()
        torch.cuda.empty_cache()

    n = 2048
    run("ttv_2048", td.ttv(p, dims=(n * p, n, n)), 8.0 * (n ** 3 + n + n * n) * p, "GB/s", hbm, "ttv")
    if p <= job.n_gpus:     # 2 x 2048^3 per processor: two processors per GPU would exceed HBM
        run("innerprod3_2048", td.innerprod3(p, dims=(n * p, n, n)), 16.0 * n ** 3 * p, "GB/s", hbm, "innerprod")
    g1, g2 = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}[p]
    m = 1024
    run("ttm_1024_64", td.ttm2d(g1, g2, dims=(m * g1, m * g2, m, 64)), 2.0 * m ** 3 * 64 * p, "GFLOP/s",
        FP64_PEAK_TFLOPS * 1e3, "ttm")
    run("mttkrp_1024_r32", td.mttkrp(g1, g2, dims=(m * g1, 32, m * g2, m)),
        (2.0 * m ** 3 * 32 + 2.0 * m * m * 32) * p, "GFLOP/s", FP64_PEAK_TFLOPS * 1e3, "mttkrp")
    # G1: SUMMA 1024^3 on a 2x2 grid, chunk 128 (the reference's results-oracle config;
    # fixed size, latency-bound: 4 tasks x 8 steps of 512x512x128 DMMA leaves).  Last:
    # once a communicator has NCCL work captured in a graph, NCCL synchronises its later
    # eager work with the graph's, which would slow the configs above
    g1 = td.summa(2, 2, dims=(1024, 1024, 1024), chunk=128)
    cin, store = g1.prepare(seed=0, mode=0, world=job.world)

    def g1_step():
        store.zero("C")
        td.execute(cin, store, record_requirements=False)

    from paper_2203_08069_b200 import runtime as rt
    ms = job.timed(g1_step, 50, 5)               # launch plans replaying (td_execute_plan)
    rt.PLANS = False
    try:
        ms_eager = job.timed(g1_step, 20, 3)     # the Python step loop every time
    finally:
        rt.PLANS = True
    results["summa_1024_2x2"] = {"config": "summa 2x2 dims (1024, 1024, 1024) chunk 128", "value":
                                 2.0 * 1024 ** 3 * 50 / (ms / 1e3) / 1e9, "unit": "GFLOP/s",
                                 "ms_per_step": ms / 50, "ms_per_step_python_loop": ms_eager / 20,
                                 "check": _spot_check(job, g1, store), "scaling": "strong (fixed size)"}
    if job.world.ngpus == 1 or job.world.nprocs == job.world.ngpus:   # captured once as a CUDA graph, replayed
        from paper_2203_08069_b200.runtime import CapturedLaunch
        cap = CapturedLaunch(cin, store)
        gms = job.timed(cap.replay, 50, 5)
        results["summa_1024_2x2"].update({"graph_ms_per_step": gms / 50,
                                          "graph_value": 2.0 * 1024 ** 3 * 50 / (gms / 1e3) / 1e9})
        del cap
    del store, g1_step
    gc.collect()
    return results


# ------------------------------------------------------------------ CPU side
def _ints(n, seed):
    """n x n integer-valued fp64 in [-4, 4] (numpy's fast generator: the
    reference arm's inputs only need the right shape and value range)."""
    rng = np.random.default_rng(seed)
    return rng.integers(-4, 5, size=(n, n), dtype=np.int8).astype(np.float64)


def _host_ram_fits(n, tasks) -> bool:
    """Can tendist's run_statement hold n^2 GEMM operands in host RAM?  It
    keeps the caller's inputs, its placed copies (simulator.py:303), one
    full-size zeroed output per task alive at once (cin.py:441-446) and the
    canonical output."""
    import psutil
    need = 8.0 * n * n * (4 + tasks + 1)
    return need < 0.85 * psutil.virtual_memory().available


REFERENCE_BUDGET_S = 240.0


def reference_gemm(p, steps, n=None, budget_s=REFERENCE_BUDGET_S):
    """The REFERENCE (tendist from oracle/_ref) on the headline GEMM of p GPUs:
    its own run_statement with the numpy/BLAS leaf substituted through its
    plugin API (oracle/ref_bench.py), at the full headline n when host RAM
    allows (else the largest multiple of 256 that fits, stated).  Up to
    `steps` runs, stopping once `budget_s` of CPU time is spent (p = 8 at
    32768^3 is ~2 minutes per run on 16 cores); the runs made are reported."""
    import paper_2203_08069_b200 as td
    from oracle.ref_bench import blas_threads, run_reference
    full = td.weak_gemm_n(p)
    bundle = td.gemm_for_gpus(p, full)
    tasks = bundle.machine.size
    n = n or full
    while not _host_ram_fits(n, tasks) and n > 1024:
        n -= 256 * max(1, n // 4096)
    bundle = td.gemm_for_gpus(p, n)
    a, b = _ints(n, 1), _ints(n, 2)
    ins = {"A": td.DenseTensor((n, n), a), "B": td.DenseTensor((n, n), b)}
    times = []
    out = None
    for _ in range(max(1, steps)):
        out, secs, _ = run_reference(bundle, ins)
        times.append(secs)
        if sum(times) + secs > budget_s:
            break
    rows = [0, n // 2, n - 1]
    ok = bool(np.array_equal(out[rows], a[rows] @ b))
    secs = statistics.median(times)
    del out, ins, a, b
    gc.collect()
    return {"value": 2.0 * n ** 3 / secs / 1e9, "secs": secs, "n": n, "same_shape": n == full,
            "cores": blas_threads(), "rows_exact": ok,
            "sample": f"tendist run_statement ({bundle.name} on {bundle.machine}, n={n}"
                      f"{'' if n == full else f'; the headline n={full} does not fit host RAM'}) with a numpy/"
                      f"OpenBLAS leaf substituted through its own plugin API (register_leaf_kernel + "
                      f"substitute_leaf; oracle/ref_bench.py), {blas_threads()} BLAS threads, median of "
                      f"{len(times)} run(s), inputs placed by run_statement inside the timing",
            "runs": len(times)}


def reference_interpreter_rate(p):
    """CPU-A: the reference AS SHIPPED (its per-point Python interpreter leaf,
    workers=1 -> one core) on the headline algorithm at a scaled shape."""
    import paper_2203_08069_b200 as td
    from oracle.ref_bench import run_reference
    n = 32
    bundle = td.gemm_for_gpus(p, n)
    _, secs, _ = run_reference(bundle, leaf="interpreter")
    pts = float(n) ** 3
    return {"value": 2.0 * pts / secs / 1e6, "unit": "MFLOP/s", "kpoints_per_s": pts / secs / 1e3, "cores": 1,
            "sample": f"tendist run_statement as shipped (per-point interpreter) {bundle.name} on {bundle.machine}, "
                      f"n={n}", "full_shape_hours": 2.0 * td.weak_gemm_n(p) ** 3 / (2.0 * pts / secs) / 3600}


def reference_kernels():
    """cpu_baseline of the other BASELINE configs: the reference + numpy leaf
    at scaled shapes (the full ones exceed host RAM / minutes of CPU)."""
    import paper_2203_08069_b200 as td
    from oracle.ref_bench import blas_threads, run_reference
    out = {}
    m = 512
    cases = [("ttv_2048", td.ttv(1, dims=(m, m, m)), 8.0 * (m ** 3 + m + m * m), "GB/s"),
             ("innerprod3_2048", td.innerprod3(1, dims=(m, m, m)), 16.0 * m ** 3, "GB/s"),
             ("ttm_1024_64", td.ttm2d(1, 1, dims=(m, m, m, 64)), 2.0 * m ** 3 * 64, "GFLOP/s"),
             ("mttkrp_1024_r32", td.mttkrp(1, 1, dims=(m, 32, m, m)), 2.0 * m ** 3 * 32 + 2.0 * m * m * 32,
              "GFLOP/s")]
    for name, bundle, work, unit in cases:
        run_reference(bundle)   # warm
        _, secs, _ = run_reference(bundle)
        out[name] = {"value": work / secs / 1e9, "unit": unit, "cores": blas_threads(), "kind": "reference",
                     "sample": f"tendist run_statement + numpy leaf, {bundle.name} on {bundle.machine} at "
                               f"{m}^3 ({secs:.2f} s)"}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2203_08069_b200 as td
    p = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    # warm-up: the same code path at a small shape (BLAS threads, imports)
    for _ in range(max(0, args.warmup)):
        reference_gemm(p, steps=1, n=1024)
    t0 = time.perf_counter()
    r = reference_gemm(p, steps=args.steps)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "GFLOP/s", "n_gpus": p,
        "steps": r["runs"], "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": r["secs"] * 1e3,
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": gemm_config(td, p) if r["same_shape"] else {**gemm_config(td, p), "cpu_n": r["n"]},
        "cpu_baseline": {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
                         "sample": r["sample"], "rows_exact": r["rows_exact"]},
        "e2e": {"value": r["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_a": reference_interpreter_rate(p),
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="all", choices=["all", "gemm"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="e2e steps (default: --steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--procs", type=int, default=0,
                    help="logical processors of the BASELINE layout (default: one per GPU)")
    ap.add_argument("--placement", default="block", choices=("block", "cyclic"),
                    help="processor -> GPU mapping when --procs exceeds the GPUs (Machine.device_of)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    from paper_2203_08069_b200 import machine as _machine
    _machine.set_placement(args.placement)
    job = Job(args.gpus, args.procs)
    gemm = bench_gemm(job, args.steps, args.warmup, args.e2e_steps or args.steps)
    kernels = bench_kernels(job, max(2, args.steps // 2), max(3, args.warmup)) if args.workload == "all" else None
    if job.rank == 0:
        report(args, job, gemm, kernels)
    job.close()


def gemm_config(td, p, gpus=None):
    """The headline workload's `config` -- identical in both arms."""
    n = td.weak_gemm_n(p)
    b = td.gemm_for_gpus(p, n)
    gpus = gpus or p
    if gpus == p:
        par = f"{p} GPU(s), one task per GPU"
    else:
        from paper_2203_08069_b200.machine import placement
        par = f"{p} processors on {gpus} GPUs ({placement()} placement)"
    return {"workload": f"fp64 GEMM {n}^3 weak-scaled from 16384^3 ({b.name} on {b.machine})", "n": n,
            "algorithm": b.name, "grid": str(b.machine), "parallelism": par,
            "l2": "inputs (>= 2 GiB per operand) exceed the 126 MB L2; no flush needed",
            "inputs": "integer-valued fp64 in [-4,4]"}


def report(args, job, gemm, kernels):
    cpu = None
    if job.n_gpus == 1 and not args.no_cpu_baseline:
        # the reference itself on the headline workload (16384^3, ~10 s on the box's cores), one run
        r = reference_gemm(1, steps=1)
        cpu = {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
               "sample": r["sample"], "rows_exact": r["rows_exact"]}
        if kernels:
            for name, cb in reference_kernels().items():
                if name in kernels:
                    kernels[name]["cpu_baseline"] = cb
    p = job.n_gpus
    line = {
        "metric": METRIC, "value": gemm["value"], "unit": "GFLOP/s", "n_gpus": p, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": gemm["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": gemm_config(job.td, job.procs, job.n_gpus),
        "per_gpu": gemm["per_gpu"], "check": gemm["check"], "roofline": gemm["roofline"],
        "cpu_baseline": cpu, "e2e": gemm["e2e"], "gpu_launches": gemm["gpu_launches"],
        "gpu_launches_per_step": gemm["launches_per_step"], "clocks": gemm["clocks"],
        "comm_overlap": gemm["overlap"],
        "kernels": kernels,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
