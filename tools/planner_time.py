#!/usr/bin/env python
"""Planner time, the analog of the paper's Table 4 "Bucket" column (P:531-546:
0.71 s manual / 3.87 s auto for Llama 3.1 8B inside TorchInductor).  Times
fsdp_plan_buckets (C++, both phases) for the Llama 8B / 70B / 405B parameter
lists, MANUAL and GREEDY, and the NumPy oracle planner beside it.  Host-only.

    python tools/planner_time.py [--out F]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def best_of(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def raw_calls(descs, world, tf, tb, link, mem, mode):
    """The two fsdp_plan_buckets calls with their arguments marshalled up front
    (so only the C++ planner is timed)."""
    import ctypes as C
    from paper_2411_00284_b200 import _lib as L
    calls = []
    P = len(descs)
    for phase, t in ((L.PHASE_FWD, tf), (L.PHASE_BWD, tb)):
        pin = L.PlanIn()
        keep = [L.descs(descs), L.i64_array(t)]
        pin.params, pin.t_compute_ns, pin.mem_bytes = keep[0], keep[1], None
        pin.ag = L.Link(*link)
        pin.rs = L.Link(*link)
        pin.mem_max_bytes = mem
        pin.n_params, pin.world, pin.align_bytes = P, world, 16
        pin.mode, pin.phase, pin.param_dtype, pin.reduce_bytes, pin.reserved = mode, phase, L.BF16, 4, 0
        bb = (C.c_int32 * (P + 1))()
        nb = C.c_int32()

        def call(pin=pin, bb=bb, nb=nb, keep=keep):
            L.check(L.lib.fsdp_plan_buckets(C.byref(pin), bb, C.byref(nb), None))
        calls.append(call)
    return calls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--tokens", type=int, default=1024)
    a = ap.parse_args()
    from oracle.planner import BWD, FWD, GREEDY, MANUAL, PlanInput, plan
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    world, link, mem = 8, (20000, 1215), 2 * 10 ** 9
    rows = {}
    for model in ("8b", "70b", "405b"):
        specs = llama(model)
        tf, tb = per_param_compute_ns(specs, a.tokens)
        descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
        r = {"params": len(specs)}
        for name, mode, omode in (("manual", L.PLAN_MANUAL, MANUAL), ("greedy", L.PLAN_GREEDY, GREEDY)):
            lib_s = best_of(lambda: H.plans_for(specs, world, mode, tf, tb, link, link, mem), 20)
            calls = raw_calls(descs, world, tf, tb, link, mem, mode)
            raw_s = best_of(lambda: [c() for c in calls], 200)

            def oracle_both():
                for ph, t in ((FWD, tf), (BWD, tb)):
                    plan(PlanInput(descs, world, t, link, link, mem, omode, ph, param_bytes=2, reduce_bytes=4,
                                   align=16))
            orc_s = best_of(oracle_both, 3)
            r[name] = {"library_call_us": round(raw_s * 1e6, 1), "with_python_marshalling_us": round(lib_s * 1e6, 1),
                       "oracle_ms": round(orc_s * 1e3, 2)}
        rows["llama3-" + model] = r
    out = {"what": "fsdp_plan_buckets for both phases (forward + backward plan), best of 200 for the C++ calls alone (best of 20 and through "
                   "the Python binding); the NumPy "
                   "oracle planner (test infrastructure) beside it, best of 3; N = 8, T = %d" % a.tokens,
           "paper_table4_s": {"manual": 0.71, "auto": 3.87, "note": "Inductor bucket pass, Llama 3.1 8B, H100 "
                                                                     "host (P:531-546)"},
           "results": rows}
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
