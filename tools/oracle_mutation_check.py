#!/usr/bin/env python
"""Does every plausible slip in the oracle fail one of its pins?  (test
infrastructure for the oracle, CPU only)

Applies one mutation at a time to a COPY of the repository's oracle/ (the
working tree is never edited), runs the `-m "not gpu"` oracle pins against it
(tests/test_oracle_*.py with PYTHONPATH pointing at the copy), and records
whether at least one pin failed.  Each mutation is a dropped term, a wrong
index, a wrong sign or rounding, a transposed reading -- the mistakes a pin
must catch (task brief ③).  Writes one JSON object.

    python tools/oracle_mutation_check.py [--out profiles/r02_oracle_mutations.json]
"""
import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file under oracle/, exact text, replacement)
MUTATIONS = [
    ("M_i default without the world factor N (G13)", "planner.py",
     "mem_bytes = [world * (-(-d // world)) * r * param_bytes", "mem_bytes = [(-(-d // world)) * r * param_bytes"),
    ("T_AG with n = seg instead of N seg (G8)", "planner.py",
     "return comm_time(self.world * seg, *self.ag)", "return comm_time(seg, *self.ag)"),
    ("T_RS with n = seg instead of N seg (G8)", "planner.py",
     "return comm_time(self.world * seg, *self.rs)", "return comm_time(seg, *self.rs)"),
    ("T_c of the open bucket instead of the closed one (G14)", "planner.py",
     "            t_c = pi.t_c(closed[-1])", "            t_c = pi.t_c(closed[-1] + [i])"),
    ("T^RS of b_{j-1} instead of b_{j-2} (G11)", "planner.py",
     "pi.t_rs(closed[-2]) if (pi.phase == BWD and len(closed) >= 2)",
     "pi.t_rs(closed[-1]) if (pi.phase == BWD and len(closed) >= 2)"),
    ("strict < instead of <= (G15)", "planner.py",
     "time_ok = (t_lhs <= t_rhs)", "time_ok = (t_lhs < t_rhs)"),
    ("memory test dropped", "planner.py", "mem_ok = m_lhs <= m_rhs", "mem_ok = True"),
    ("RS without the 1/N average (G6)", "collectives.py",
     "    inv = inv_world_f32(world)\n", "    inv = np.float32(1.0)\n"),
    ("tail rank loses a row (G1)", "shard.py",
     "    v = max(0, min(d - rank * c, c))",
     "    v = max(0, min(d - rank * c, c - 1 if rank == world - 1 and c > 1 else c))"),
    ("floor instead of ceil chunk (G1)", "shard.py", "    c = -(-d // world)", "    c = max(1, d // world)"),
    ("no alignment between members (G4)", "layout.py",
     "        cur = align_up(cur + c * r * elem_bytes, align)", "        cur = cur + c * r * elem_bytes"),
    ("cost model floor instead of ceil (G9)", "cost.py",
     "return alpha_ns + -(-(nbytes * beta_fs_per_byte) // 10**6)",
     "return alpha_ns + (nbytes * beta_fs_per_byte) // 10**6"),
    ("prefetch placed after the wait under BEFORE (Table 6)", "schedule.py",
     "        s += (pre + wait) if placement == BEFORE else (wait + pre)\n        s.append(_e(0, COMPUTE_F, b))",
     "        s += (wait + pre)\n        s.append(_e(0, COMPUTE_F, b))"),
    ("Wr(j-1) after RS(j) (P:191)", "schedule.py",
     """        if b >= 1:
            s += [_e(1, WAIT_RS, b - 1), _e(1, COPYOUT_RS, b - 1)]
        s.append(_e(1, RS, b))""",
     """        s.append(_e(1, RS, b))
        if b >= 1:
            s += [_e(1, WAIT_RS, b - 1), _e(1, COPYOUT_RS, b - 1)]"""),
    ("a wait does not block the compute stream (S:303)", "sim.py",
     "            if c > t_cmp:", "            if False:"),
    ("bf16 narrow truncates instead of RNE (O1)", "bf16.py",
     "    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)",
     "    r = (u >> np.uint64(16)).astype(np.uint16)"),
]


def run_pins(oracle_parent):
    env = dict(os.environ, PYTHONPATH=oracle_parent + os.pathsep + os.environ.get("PYTHONPATH", ""))
    tests = sorted(os.path.join("tests", f) for f in os.listdir(os.path.join(ROOT, "tests"))
                   if f.startswith("test_oracle_"))
    # the copy's oracle/ shadows the repo's: conftest puts ROOT on sys.path
    # first, so run pytest from the copy's directory with the tests linked in
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "not gpu"] + tests,
                       cwd=oracle_parent, env=env, capture_output=True, text=True, timeout=1800)
    return r.returncode, (r.stdout.strip().splitlines() or [""])[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    results = []
    with tempfile.TemporaryDirectory() as tmp:
        shutil.copytree(os.path.join(ROOT, "tests"), os.path.join(tmp, "tests"))
        shutil.copytree(os.path.join(ROOT, "workloads"), os.path.join(tmp, "workloads"))
        base_rc, base_tail = None, None
        for name, f, a, b in [("(none)", None, None, None)] + MUTATIONS:
            od = os.path.join(tmp, "oracle")
            if os.path.exists(od):
                shutil.rmtree(od)
            shutil.copytree(os.path.join(ROOT, "oracle"), od)
            if f:
                p = os.path.join(od, f)
                s = open(p).read()
                assert a in s, (name, a)
                open(p, "w").write(s.replace(a, b, 1))
            rc, tail = run_pins(tmp)
            if f is None:
                base_rc, base_tail = rc, tail
                continue
            results.append({"mutation": name, "file": "oracle/" + f, "caught": rc != 0, "pytest": tail})
    out = {"unmutated": {"rc": base_rc, "pytest": base_tail}, "mutations": results,
           "all_caught": base_rc == 0 and all(r["caught"] for r in results)}
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
    return 0 if out["all_caught"] else 1


if __name__ == "__main__":
    sys.exit(main())
