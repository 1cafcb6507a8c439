"""-m gpu: the C ABI from plain C (examples/c_abi_demo.c): plan, layout,
shard, all-gather and reduce-scatter(avg) over three simulated ranks, checked
bit-exactly inside the program; no Python on the data path."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_c_abi_demo():
    from paper_2411_00284_b200.build import build_examples
    exe = build_examples()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all-gather: bit-exact on every rank" in r.stdout
    assert "reduce-scatter(avg): bit-exact on every rank" in r.stdout
    assert "scheduled step with a C compute hook: hook ran per phase, re-gather bit-exact" in r.stdout
    assert r.stdout.strip().endswith("OK")
