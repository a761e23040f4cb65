"""The reference's own unit tests under SPMD (one process per GPU over NCCL).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/ref_suite_spmd.py

Every rank runs every reference test (staged in oracle/_ref/tests) with
`tendist` aliased to this package, so each run_statement / interpret /
sequential_evaluate inside them spreads its processors over the N GPUs and
moves data with NCCL -- the tests' own assertions then check the values.
Tests needing pytest fixtures other than tmp_path are skipped (capsys,
monkeypatch: CLI output capture).  Exits non-zero if any rank saw a failure.
"""

import inspect
import os
import sys
import tempfile
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_08069_b200 as td  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = td.configure_distributed()
    rank, size = dist.get_rank(), dist.get_world_size()
    import test_reference_suite as suite
    ran = skipped = 0
    failures = []
    for fname, name, fn, kwargs in suite.CASES:
        kwargs = dict(kwargs)
        params = inspect.signature(fn).parameters
        if any(p not in kwargs and p != "tmp_path" for p in params):
            skipped += 1
            continue
        saved = suite._alias()
        try:
            with tempfile.TemporaryDirectory() as tmp:
                if "tmp_path" in params:
                    import pathlib
                    kwargs["tmp_path"] = pathlib.Path(tmp)
                fn(**kwargs)
            ran += 1
        except Exception as exc:   # noqa: BLE001 -- report every failing reference test
            failures.append(f"{fname}::{name}: {type(exc).__name__}: {exc}")
            if rank == 0:
                traceback.print_exc()
        finally:
            suite._restore(saved)
    bad = torch.tensor([len(failures)], device="cuda")
    dist.all_reduce(bad)
    if rank == 0:
        print(f"ref_suite_spmd world={size}: ran {ran}, skipped {skipped} (fixtures), "
              f"{'OK' if bad.item() == 0 else 'FAIL'}", flush=True)
    if failures:
        print(f"rank {rank} failures: {failures[:10]}", flush=True)
    dist.barrier(device_ids=[local])
    world.close()
    dist.destroy_process_group()
    sys.exit(1 if bad.item() else 0)


if __name__ == "__main__":
    main()
