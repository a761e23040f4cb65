"""A non-Python host on the C ABI alone: examples/plan_demo.c builds a
three-op launch plan (fill, two k-half DMMA GEMMs) and issues it with one
td_execute_plan call, then checks the product on the host (exact integers)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "examples", "plan_demo")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(DEMO), reason="examples/plan_demo not built (make examples)")
def test_c_host_runs_a_launch_plan():
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "plan_demo OK" in out.stdout, out.stdout + out.stderr
