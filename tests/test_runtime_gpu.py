"""Runtime behaviours of the reference's simulator tests, on the B200
(reference pkg/tests/test_simulator.py, test_cin.py, test_algorithms.py)."""

import numpy as np
import pytest

import paper_2203_08069_b200 as td
from paper_2203_08069_b200.cin import LeafKernel, LeafRuntime, with_relations
from paper_2203_08069_b200.errors import (ExtentMismatch, GridMismatch, MissingDistribution,
                                          MissingInput, OverlappingWrites, TendistError, VerifyFail,
                                          WriteToReplica)

pytestmark = pytest.mark.gpu


def _block(dims, machine):
    names = ("x", "y", "z")[: len(dims)]
    return td.TensorDistribution(dims, machine, [(names, names)])


def _gemm_setup(n=4):
    stmt = td.parse_statement("C(i, j) = A(i, k) * B(k, j)", {"i": n, "j": n, "k": n})
    machine = td.grid(2, 2)
    dists = {name: _block((n, n), machine) for name in ("A", "B", "C")}
    sched = (td.schedule().divide("i", "io", "ii", 2).divide("j", "jo", "ji", 2)
             .reorder("io", "jo", "ii", "ji").distribute("io").distribute("jo")
             .split("k", "ko", "ki", 2).reorder("ko", "ii", "ji")
             .communicate("A", "jo").communicate(("B", "C"), "ko"))
    rng = np.random.default_rng(7)
    inputs = {name: td.DenseTensor((n, n), rng.integers(-3, 4, (n, n)).astype(float)) for name in ("A", "B")}
    return stmt, machine, dists, inputs, sched


def test_broadcast_run_matches_reference_and_anchor():
    stmt, machine, dists, inputs, sched = _gemm_setup()
    res = td.run_statement(stmt, machine, dists, inputs, sched)
    td.verify_result(stmt, inputs, res)
    assert np.array_equal(res.output.data, inputs["A"].data @ inputs["B"].data)
    assert (res.trace.total_messages, res.trace.total_elements, res.trace.high_water) == (8, 32, 24)


def test_verify_catches_tampering():
    stmt, machine, dists, inputs, sched = _gemm_setup()
    res = td.run_statement(stmt, machine, dists, inputs, sched)
    res.output.data[0, 0] += 1.0
    with pytest.raises(VerifyFail):
        td.verify_result(stmt, inputs, res)


def test_reduce_into_replica():
    stmt, machine, dists, inputs, sched = _gemm_setup()
    dists["C"] = td.TensorDistribution((4, 4), machine, [(("x", "y"), ("x", "*"))])
    res = td.run_statement(stmt, machine, dists, inputs, sched)
    td.verify_result(stmt, inputs, res)
    homes = res.store["C"].residency
    assert homes[(0, 1)] == [] and homes[(1, 1)] == []


def test_runtime_rejections():
    stmt, machine, dists, inputs, sched = _gemm_setup()
    with pytest.raises(MissingDistribution):
        td.run_statement(stmt, machine, {"A": dists["A"]}, inputs, sched)
    with pytest.raises(MissingInput):
        td.run_statement(stmt, machine, dists, {"A": inputs["A"]}, sched)
    bad = dict(inputs)
    bad["B"] = td.DenseTensor((2, 2))
    with pytest.raises(ExtentMismatch):
        td.run_statement(stmt, machine, dists, bad, sched)
    add = td.parse_statement("D(i, j) = A(i, j) + B(i, j)", {"i": 4, "j": 4})
    repl = td.TensorDistribution((4, 4), machine, [(("x", "y"), ("x", "*"))])
    s2 = (td.schedule().divide("i", "io", "ii", 2).divide("j", "jo", "ji", 2)
          .reorder("io", "jo", "ii", "ji").distribute("io").distribute("jo"))
    with pytest.raises(WriteToReplica):
        td.run_statement(add, machine, {"A": dists["A"], "B": dists["A"], "D": repl}, inputs, s2)
    s3 = td.schedule().divide("i", "io", "ii", 2).reorder("io", "ii").distribute("io")
    with pytest.raises(GridMismatch):
        td.run_statement(stmt, machine, dists, inputs, s3)


def test_overlapping_copy_writes_rejected():
    D, A = td.TensorVar("D", (4, 4)), td.TensorVar("A", (4, 4))
    leaf = td.Assign(D("i", "ji"), A("i", "ji"))
    body = td.Forall("io", 0, 2, td.Forall("jo", 0, 2, td.Forall("ii", 0, 2, td.Forall("ji", 0, 2, leaf))))
    cin = with_relations(body, (td.Divide("i", "io", "ii", 2, 4), td.Divide("j", "jo", "ji", 2, 4),
                                td.Distribute("io"), td.Distribute("jo")))
    machine = td.grid(2, 2)
    block = _block((4, 4), machine)
    with pytest.raises(OverlappingWrites):
        td.run_statement(cin, machine, {"A": block, "D": block}, {"A": td.DenseTensor((4, 4))})


def test_single_processor_matvec_and_assign_statement():
    stmt = td.parse_statement("b(i) = A(i, j) * c(j)", {"i": 3, "j": 3})
    machine = td.grid(1)
    one = td.TensorDistribution((3, 3), machine, [(("x", "y"), ("x",))])
    vec = td.TensorDistribution((3,), machine, [(("x",), ("x",))])
    sched = td.schedule().divide("i", "io", "ii", 1).distribute("io")
    inputs = {"A": td.DenseTensor((3, 3), np.arange(9, dtype=float).reshape(3, 3)),
              "c": td.DenseTensor((3,), [1.0, 0.0, 2.0])}
    res = td.run_statement(stmt, machine, {"A": one, "c": vec, "b": vec}, inputs, sched)
    td.verify_result(stmt, inputs, res)
    assert res.trace.total_messages == 0
    add = td.parse_statement("D(i, j) = A(i, j) + B(i, j) * 2", {"i": 5, "j": 3})
    m2 = td.grid(2)
    d2 = td.TensorDistribution((5, 3), m2, [(("x", "y"), ("x",))])
    s2 = td.schedule().divide("i", "io", "ii", 2).distribute("io").communicate(("A", "B"), "io")
    ins = {"A": td.DenseTensor((5, 3), np.arange(15.0).reshape(5, 3)),
           "B": td.DenseTensor((5, 3), np.ones((5, 3)))}
    res = td.run_statement(add, m2, {"A": d2, "B": d2, "D": d2}, ins, s2)
    assert np.array_equal(res.output.data, ins["A"].data + 2)


def test_redistribute_moves_pieces():
    machine = td.grid(2, 2)
    old = td.TensorDistribution((4, 4), machine, [(("x", "y"), ("x", 0))])
    new = td.TensorDistribution((4, 4), machine, [(("x", "y"), ("x", "y"))])
    store = td.RegionStore(machine)
    data = td.DenseTensor((4, 4), np.arange(16, dtype=float).reshape(4, 4))
    store.place("T", data, old)
    trace = td.ExecutionTrace(machine)
    td.redistribute(store, "T", new, trace)
    assert [(e.src, e.dst, e.elements) for e in trace.events] == [((0, 0), (0, 1), 4), ((1, 0), (1, 1), 4)]
    assert store["T"].dist is new
    assert np.array_equal(store["T"].tensor.data, data.data)
    assert trace.memory[(0, 0)] == 8 and trace.memory[(0, 1)] == 4


def test_execute_twice_accumulates_like_the_reference():
    """A second execute on the same store adds into the canonical output
    (reference commit: canon[rect] += partial, simulator.py:631-632) and the
    trace accumulates both launches."""
    for b in (td.summa(2, 2, dims=(24, 20, 28), chunk=8), td.johnson(2, 2, 2, dims=(16, 12, 20))):
        cin, store = b.prepare(seed=6)
        trace = td.ExecutionTrace(b.machine)
        td.execute(cin, store, trace=trace)
        once = store.gather("C").data.copy()
        td.execute(cin, store, trace=trace)
        assert np.array_equal(store.gather("C").data, 2 * once)
        assert len(trace.launches) == 2 and trace.total_messages % 2 == 0


def test_captured_launch_replays():
    """CUDA-graph capture of a whole multi-step, multi-task launch."""
    from paper_2203_08069_b200.runtime import CapturedLaunch
    torch = pytest.importorskip("torch")
    for b in (td.summa(2, 2, dims=(64, 48, 80), chunk=16), td.mttkrp(2, 2, dims=(12, 8, 10, 9)),
              td.innerprod3(2, dims=(8, 6, 30))):
        cin, store = b.prepare(seed=4)
        cap = CapturedLaunch(cin, store)
        out = b.statement.lhs.tensor.name
        first = store.gather(out).data.copy()
        for _ in range(3):
            cap.replay()
        torch.cuda.synchronize()
        assert np.array_equal(store.gather(out).data, first)
        ins = {n: store.gather(n) for n in b.input_names}
        want = td.sequential_evaluate(b.statement, ins)
        assert np.array_equal(first, want.data), b.name


def test_binary_tensor_io_into_sharded_hbm(tmp_path):
    """Reference binary format (tensors.py:72-92) loaded piecewise into HBM,
    executed, and saved back."""
    b = td.summa(2, 2, dims=(12, 10, 14), chunk=4)
    ins = td.random_inputs(b.statement, seed=9)
    for name, t in ins.items():
        td.save_tensor(t, tmp_path / f"{name}.bin")
    store = td.RegionStore(b.machine)
    for name in ins:
        store.place_file(name, tmp_path / f"{name}.bin", b.distributions[name])
        assert store[name].tensor == ins[name]
    store.place_zeros("C", b.distributions["C"])
    td.execute(b.scheduled(), store)
    store.save_file("C", tmp_path / "C.bin")
    assert np.array_equal(td.load_tensor(tmp_path / "C.bin").data, ins["A"].data @ ins["B"].data)


def test_python_leaf_plugin_and_interpreter_leaf():
    calls = []

    def doubler(rt: LeafRuntime):
        calls.append([v for v, _, _ in rt.loops])
        for x in range(rt.loops[0][1], rt.loops[0][2]):
            rt.execute_point({**rt.env, rt.loops[0][0]: x})

    td.register_leaf_kernel("doubler", doubler)
    stmt = td.parse_statement("D(x) = A(x) * 2", {"x": 4})
    cin = with_relations(td.lower_to_cin(stmt), (LeafKernel(("x",), "doubler"),))
    out = td.interpret(cin, {"A": td.DenseTensor((4,), [1.0, 2.0, 3.0, 4.0])})
    assert out["D"].data.tolist() == [2.0, 4.0, 6.0, 8.0]
    assert calls == [["x"]]
    cin2 = with_relations(td.lower_to_cin(stmt), (LeafKernel(("x",), "missing-kernel"),))
    with pytest.raises(TendistError):
        td.interpret(cin2, {"A": td.DenseTensor((4,))})


def test_substitute_native_dgemm_leaf():
    """The paper's .substitute({ii, ji, ki}, GeMM) with the native DMMA leaf."""
    b = td.summa(2, 2, dims=(64, 48, 80), chunk=16)
    sched = b.schedule.substitute_leaf(("ii", "ji", "ki"), "dgemm")
    ins = td.random_inputs(b.statement, seed=4)
    from paper_2203_08069_b200 import leaves
    leaves.reset_stats()
    res = td.run_statement(b.statement, b.machine, b.distributions, ins, sched)
    assert leaves.STATS["dgemm"] == 4 * 5 and leaves.STATS["nest"] == 0
    assert np.array_equal(res.output.data, ins["A"].data @ ins["B"].data)
    ref = td.run_statement(b.statement, b.machine, b.distributions, ins,
                           b.schedule.substitute_leaf(("ii", "ji", "ki"), "interpreter"))
    assert np.array_equal(ref.output.data, res.output.data)


def test_native_leaves_are_used_for_bundles():
    from paper_2203_08069_b200 import leaves
    for b, kind in [(td.cannon(2, 2, dims=(32, 32, 32)), "dgemm"), (td.ttv(2, dims=(8, 6, 40)), "ttv"),
                    (td.ttm(2, dims=(6, 5, 16, 8)), "ttm"), (td.mttkrp(2, 2, dims=(8, 6, 10, 12)), "mttkrp"),
                    (td.innerprod3(2, dims=(6, 5, 64)), "innerprod"), (td.johnson(2, 2, 2, dims=(16, 16, 16)), "dgemm")]:
        leaves.reset_stats()
        res, ins = b.run(seed=1)
        assert leaves.STATS[kind] > 0 and leaves.STATS["nest"] == 0, (b.name, leaves.STATS)
        td.verify_result(b.statement, ins, res)


def test_timed_launch_fills_measured_stats(tmp_path):
    """execute(timed=True): trace.timings gets the launch's device time and
    algorithmic work; stats() reports it under "measured" beside the
    reference schema (which is otherwise unchanged)."""
    b = td.cannon(1, 1, dims=(1024, 1024, 1024))
    res, _ = b.run(seed=1, timed=True)
    st = res.trace.stats({"algorithm": "cannon"})
    m = st["measured"]
    (row,) = m["launches"]
    assert row["flops"] == 2.0 * 1024 ** 3 and row["bound"] == "tensor" and row["device_ms"] > 0
    assert row["rate_unit"] == "GFLOP/s" and 0 < row["frac_of_peak"] < 1.2
    t = td.ttv(1, dims=(256, 256, 256))
    res, _ = t.run(seed=1, timed=True)
    (row,) = res.trace.stats()["measured"]["launches"]
    assert row["bound"] == "hbm" and row["rate_unit"] == "GB/s"
    untimed, _ = b.run(seed=1)
    assert "measured" not in untimed.trace.stats()


def test_cli_timing_and_stats(tmp_path, capsys):
    from paper_2203_08069_b200 import cli
    path = tmp_path / "s.json"
    assert cli.main(["--algorithm", "summa", "--dims", "512x512x512", "--chunk", "64", "--timing", "--verify",
                     "--stats", str(path)]) == 0
    out = capsys.readouterr().out
    assert "verify: OK" in out and "% of the tensor roof" in out
    import json
    stats = json.loads(path.read_text())
    assert stats["measured"]["launches"][0]["device_ms"] > 0


def test_place_file_rejects_wrong_payload_size(tmp_path):
    """A file whose payload disagrees with its header dims fails with
    ExtentMismatch, as the reference's from_bytes does (tensors.py:84-92)."""
    from paper_2203_08069_b200.errors import ExtentMismatch
    t = td.DenseTensor((4, 6), np.arange(24, dtype=float).reshape(4, 6))
    good = tmp_path / "t.bin"
    td.save_tensor(t, good)
    raw = good.read_bytes()
    b = td.summa(2, 2, dims=(4, 6, 6))
    store = td.RegionStore(b.machine)
    for bad in (raw[:-8], raw + b"\0" * 8):
        p = tmp_path / "bad.bin"
        p.write_bytes(bad)
        with pytest.raises(ExtentMismatch):
            store.place_file("A", p, b.distributions["A"])
    store.place_file("A", good, b.distributions["A"])
    assert store["A"].tensor == t


def test_nvtx_ranges_do_not_change_results():
    from paper_2203_08069_b200 import runtime
    b = td.cannon(2, 2, dims=(40, 36, 44))
    runtime.NVTX = True
    try:
        res, ins = b.run(seed=2)
    finally:
        runtime.NVTX = False
    assert np.array_equal(res.output.data, ins["A"].data @ ins["B"].data)


def test_lazy_zero_reads_and_launches():
    """RegionStore.zero only marks the pieces (the next launch's first leaf
    overwrites them): reads before any launch (gather, local_pieces) still
    see +0.0, and zero -> execute equals a fresh run, eagerly and from
    replayed launch plans, on every bundle shape."""
    for b in (td.summa(2, 2, dims=(24, 20, 28), chunk=8), td.johnson(2, 2, 2, dims=(16, 12, 20)),
              td.mttkrp(2, 2, dims=(12, 8, 10, 9)), td.ttv(2, dims=(6, 5, 7)),
              td.innerprod3(2, dims=(8, 6, 30))):
        cin, store = b.prepare(seed=9)
        out = b.statement.lhs.tensor.name
        td.execute(cin, store, record_requirements=False)
        want = store.gather(out).data.copy()
        store.zero(out)
        assert not store.gather(out).data.any(), b.name          # materialised on read
        store.zero(out)
        for _ in range(3):                                          # eager, then plan replays
            store.zero(out)
            td.execute(cin, store, record_requirements=False)
            assert np.array_equal(store.gather(out).data, want), b.name
        store.zero(out)
        for _, piece in store.local_pieces(out):
            assert not piece.any(), b.name
