"""Command-line front end (reference `pkg/src/tendist/cli.py:29-251`).

Same flags, outputs and exit codes as the reference's `tendist` command:

  * registry mode  -- ``--algorithm summa [--machine 2x2] [--n 64 | --dims ..] [--chunk c]``
  * custom mode    -- ``--kernel gemm | --expr "C(i, j) = A(i, k) * B(k, j)"``
                      with ``--machine``, one ``--dist 'A: xy -> xy'`` per tensor
                      and a ``--schedule`` (file, or inline commands split on ';')
  * ``--explain``  -- print the statement, placements and the statement after
                      each schedule command instead of running

Every run writes the stats JSON (``--stats``, the reference schema), can dump
the ledger (``--dump-trace``) and the per-edge CSV (``--edges-csv``), and
``--verify`` compares with the single-memory evaluation.  Exit codes: 0 ok,
1 verification failure, 2 configuration error.

B200 additions: the launch runs on the GPUs; ``--timing`` launches it once
more after the run (which serves as the warm-up) with CUDA events and adds the "measured" section (device ms, GFLOP/s or GB/s,
fraction of the FP64 / HBM roof) to the stats; ``--leaf-policy exact``
forces the exact-order nest kernel.  Without a GPU or the native library
the run raises DeviceUnavailable (there is no CPU fallback).

    python -m paper_2203_08069_b200.cli --algorithm cannon --n 4096 --timing --verify
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import re
import sys

from .algorithms import ALGORITHMS, bundle_from_config, random_inputs
from .cin import lower_to_cin, pretty
from .distribution import TensorDistribution, lower_placement, parse_distribution
from .errors import ConfigError, DeviceUnavailable, TendistError, VerifyFail
from .ir import format_statement, parse_statement
from .machine import parse_machine
from .runtime import run_statement, verify_result
from .scheduling import parse_schedule
from .trace import write_edge_csv

#: named statement shapes of --kernel
KERNELS = {
    "gemm": "C(i, j) = A(i, k) * B(k, j)",
    "ttv": "A(i, j) = B(i, j, k) * c(k)",
    "ttm": "Y(i, j, l) = B(i, j, k) * C(k, l)",
    "innerprod": "a = A(i, j) * B(i, j)",
    "mttkrp": "A(i, j) = B(i, k, l) * C(k, j) * D(l, j)",
}

#: tensor order of each registry algorithm when only --n is given
_ALGO_ORDER = {"ttv": 3, "ttm": 4, "mttkrp": 4, "innerprod": 2}

# (flags, keyword arguments) of every option, grouped as in --help
_OPTIONS = {
    "what to run": [
        (("--algorithm",), dict(choices=ALGORITHMS, help="one of the bundled algorithm recipes")),
        (("--kernel",), dict(choices=sorted(KERNELS), help="a named statement (gemm, ttv, ttm, innerprod, mttkrp)")),
        (("--expr",), dict(help="any statement in index notation, e.g. 'C(i, j) = A(i, k) * B(k, j)'")),
    ],
    "problem shape": [
        (("--n",), dict(type=int, help="the same extent N for every index")),
        (("--dims",), dict(help="extents per index, e.g. 8x4x6 (indices in order of appearance)")),
        (("--chunk",), dict(type=int, default=1, help="chunk / round factor of the sequential loop (default 1)")),
        (("--seed",), dict(type=int, default=0, help="seed of the integer-valued inputs")),
    ],
    "placement and schedule": [
        (("--machine",), dict(help="processor grid, e.g. 3x3 or the two-level 2x2/4")),
        (("--dist",), dict(action="append", default=[], metavar="SPEC",
                           help="placement of one tensor, e.g. 'A: xy -> xy*'; give one per tensor")),
        (("--schedule",), dict(help="schedule: a script file, or commands inline with ';' between them")),
    ],
    "outputs": [
        (("--verify",), dict(action="store_true", help="check the result against the single-memory evaluation")),
        (("--stats",), dict(default="stats.json", help="where to write the stats JSON (default stats.json)")),
        (("--dump-trace",), dict(action="store_true", help="print the ledger, one transfer per line")),
        (("--edges-csv",), dict(metavar="PATH", help="write per-edge message/element totals as CSV")),
        (("--explain",), dict(action="store_true",
                              help="show the statement, placements and each schedule stage; do not run")),
        (("--timing",), dict(action="store_true",
                             help="measure the launch on the GPUs (stats section 'measured')")),
    ],
    "execution": [
        (("--workers",), dict(type=int, default=None,
                              help="accepted for compatibility (default: TENDIST_WORKERS or 1)")),
        (("--leaf-policy",), dict(default="auto", choices=("auto", "exact"),
                                  help="native contractions (auto) or the exact-order nest kernel")),
    ],
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="tendist-b200",
        description="compile and run distributed dense tensor statements on B200 GPUs")
    for title, options in _OPTIONS.items():
        group = parser.add_argument_group(title)
        for flags, kw in options:
            group.add_argument(*flags, **kw)
    return parser


def _workers(args) -> int:
    chosen = args.workers if args.workers is not None else int(os.environ.get("TENDIST_WORKERS", "1"))
    return max(1, chosen)


def _statement_source(args) -> str:
    for text in (args.expr, KERNELS.get(args.kernel or "")):
        if text:
            return text
    raise ConfigError("give --algorithm, --kernel or --expr")


def _extents(args, text: str) -> dict:
    """Index extents: --dims in first-appearance order of the indices, else --n (default 8)."""
    names = list(dict.fromkeys(v.strip() for grp in re.findall(r"\(([^)]*)\)", text)
                               for v in grp.split(",") if v.strip()))
    if not args.dims:
        return dict.fromkeys(names, 8 if args.n is None else args.n)
    sizes = [int(d) for d in args.dims.split("x")]
    if len(sizes) != len(names):
        raise ConfigError(f"--dims has {len(sizes)} extents but the statement indexes {names}")
    return dict(zip(names, sizes))


def _schedule(spec: str):
    if os.path.exists(spec):
        with open(spec) as fh:
            return parse_schedule(fh.read())
    return parse_schedule(spec.replace(";", "\n"))


def _distributions(args, stmt, machine) -> dict:
    tensors = stmt.tensors()
    dists = {}
    for spec in args.dist:
        name, levels = parse_distribution(spec)
        if name not in tensors:
            raise ConfigError(f"--dist for {name}: the statement has tensors {sorted(tensors)}")
        dists[name] = TensorDistribution(tensors[name].dims, machine, levels)
    missing = sorted(set(tensors) - set(dists))
    if missing:
        raise ConfigError(f"no --dist given for {', '.join(missing)}")
    return dists


def explain(args) -> int:
    text = _statement_source(args)
    stmt = parse_statement(text, _extents(args, text))
    cin = lower_to_cin(stmt)
    lines = [f"statement: {format_statement(stmt)}", f"loops:     {pretty(cin)}"]
    if args.machine and args.dist:
        dists = _distributions(args, stmt, parse_machine(args.machine))
        tensors = stmt.tensors()
        for name in sorted(dists):
            lines += [f"placement {name}: {dists[name].describe()}",
                      f"  {pretty(lower_placement(tensors[name], dists[name]))}"]
    if args.schedule:
        for desc, staged in _schedule(args.schedule).steps(cin):
            lines += [f"after {desc}:", f"  {pretty(staged)}"]
    print("\n".join(lines))
    return 0


def _report(args, result, stmt, inputs, config) -> int:
    trace = result.trace
    if args.dump_trace:
        for e in trace.events:
            print(f"step {e.timestep} {e.phase} {e.kind} {e.tensor} {e.rect}: "
                  f"{e.src} -> {e.dst} ({e.elements} elements)")
    stats = trace.stats(config)
    stats["generated_at"] = datetime.datetime.now(datetime.timezone.utc).isoformat()
    if args.stats:
        with open(args.stats, "w") as fh:
            json.dump(stats, fh, indent=2, sort_keys=True)
    if args.edges_csv:
        write_edge_csv(trace, args.edges_csv)
    totals = stats["totals"]
    print(f"machine {stats['machine']}: {totals['messages']} messages, {totals['elements']} elements moved, "
          f"{stats['num_steps']} steps, memory high-water {stats['memory_high_water']['overall']}")
    measured = stats.get("measured")
    if measured:
        for row in measured["launches"]:
            frac = f", {100 * row['frac_of_peak']:.1f} % of the {row['bound']} roof" if row["frac_of_peak"] else ""
            print(f"launch {row['label']}: {row['device_ms']:.3f} ms on the GPU(s), "
                  f"{row['rate']:.1f} {row['rate_unit']}{frac}")
    if args.verify:
        verify_result(stmt, inputs, result)
        print("verify: OK")
    return 0


def _timed_rerun(result, cin, label, policy) -> None:
    """--timing: the run above was the warm-up (kernel loading, tensor maps,
    planning); launch once more on the same store with CUDA events and keep
    its record in the run's trace.  Same inputs, same output bits."""
    from .runtime import execute
    from .trace import ExecutionTrace
    result.store.zero(result.output_name)
    scratch = ExecutionTrace(result.store.machine)
    execute(cin, result.store, trace=scratch, label=label, record_requirements=False, leaf_policy=policy,
            timed=True)
    result.trace.timings.extend(scratch.timings)


def run_algorithm(args) -> int:
    machine = parse_machine(args.machine) if args.machine else None
    if args.dims:
        dims = tuple(int(d) for d in args.dims.split("x"))
    elif args.n is not None:
        dims = (args.n,) * _ALGO_ORDER.get(args.algorithm, 3)
    else:
        dims = None
    bundle = bundle_from_config(args.algorithm, machine, dims, args.chunk)
    inputs = random_inputs(bundle.statement, args.seed)
    result, _ = bundle.run(inputs=inputs, workers=_workers(args), leaf_policy=args.leaf_policy)
    if args.timing:
        _timed_rerun(result, bundle.scheduled(), bundle.name, args.leaf_policy)
    config = {"algorithm": bundle.name, "machine": str(bundle.machine),
              "statement": format_statement(bundle.statement), "extents": dict(bundle.statement.extents),
              "chunk": args.chunk, "seed": args.seed}
    return _report(args, result, bundle.statement, inputs, config)


def run_custom(args) -> int:
    text = _statement_source(args)
    stmt = parse_statement(text, _extents(args, text))
    if not args.machine:
        raise ConfigError("a --kernel/--expr run needs --machine")
    if not args.schedule:
        raise ConfigError("a --kernel/--expr run needs a --schedule that distributes its loops")
    machine = parse_machine(args.machine)
    dists = _distributions(args, stmt, machine)
    inputs = random_inputs(stmt, args.seed)
    sched = _schedule(args.schedule)
    result = run_statement(stmt, machine, dists, inputs, sched, workers=_workers(args),
                           leaf_policy=args.leaf_policy)
    if args.timing:
        _timed_rerun(result, sched.apply(lower_to_cin(stmt)), None, args.leaf_policy)
    config = {"machine": str(machine), "statement": format_statement(stmt), "extents": dict(stmt.extents),
              "seed": args.seed, "distributions": {n: d.describe() for n, d in sorted(dists.items())}}
    return _report(args, result, stmt, inputs, config)


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.explain:
            if args.algorithm:
                raise ConfigError("--explain works with --kernel/--expr runs")
            return explain(args)
        return run_algorithm(args) if args.algorithm else run_custom(args)
    except VerifyFail as exc:
        print(f"verify: FAIL ({exc})", file=sys.stderr)
        return 1
    except DeviceUnavailable:
        raise          # no GPU / library: not a configuration error of the run
    except TendistError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
