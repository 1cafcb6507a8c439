"""CPU check of bench.py's contract on the path that runs without a GPU: the
reference arm (the oracle on the host cores) prints one JSON line with the
keys the driver reads, and nothing in bench.py or __graft_entry__ reads
/root/reference at run time."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "impl", "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_no_runtime_reads_of_reference():
    for f in ("bench.py", "__graft_entry__.py"):
        src = open(os.path.join(ROOT, f)).read()
        assert "/root/reference" not in src, f
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2411_00284_b200")):
        for f in files:
            if f.endswith((".py", ".cc", ".cu", ".h")):
                assert "/root/reference" not in open(os.path.join(dirpath, f), errors="ignore").read(), f


def test_product_never_imports_oracle():
    # the product path (package + csrc) shares no code with the oracle
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2411_00284_b200")):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
    import re
    pat = re.compile(r"^\s*(import|from)\s+(paper_2411_00284_b200|torch|ctypes)", re.M)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "oracle")):
        for f in files:
            if f.endswith(".py"):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_reference_arm_multi_gpu_unit():
    """--impl reference at N > 1 states its value in the multi-GPU headline's
    unit (bus bytes), at N = 1 in HBM bytes -- the same definitions as ours."""
    for gpus, kind in (("2", "bus"), ("1", "hbm")):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", gpus,
                            "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
        assert d["value_kind"] == kind and d["value"] > 0 and d["config"]["world"] == (8 if gpus == "1" else 2)
