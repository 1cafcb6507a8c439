#!/usr/bin/env python
"""Simulator-guided bucket plans (beyond the paper): local search over
contiguous partitions of each phase, scored by the library's two-stream
timeline (fsdp_simulate_schedule) instead of Algorithm 1's greedy rule.

The paper's auto-wrap merges a parameter while its all-gather still fits the
previous bucket's compute window and concedes that it can lose to
manual wrapping when that local estimate misleads.  Here every
candidate plan is scored by the whole phase's predicted time -- the same
two-stream model the bench uses for its N-rank prediction: collectives
alpha + beta n on a FIFO comm stream, copy kernels (K3 copy-out, K4 gradient
pack) at their measured HBM rates, per-parameter compute T_c -- under the
memory cap M(bucket) <= M_max.  Moves: merge two neighbours, split a bucket,
shift a boundary by one; first-improvement hill climbing from the manual,
greedy and per-parameter plans, best result kept.  The search itself is the
library's fsdp_plan_search (C++); this file holds the Python reference of the
same moves and model (`--python`; tests/test_plan_search_host.py checks that
both give the same plan).  Host-only; the plans are
then timed on the B200 with measured op durations
(tools/plan_search_validate.sh, GPU; bench.py --plan-file).

    python tools/plan_search.py [--tokens T] [--world N] [--out plans.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# copy-kernel model (profiles/r01_bench_default_final2.json): K3 6.47 TB/s,
# K4 6.68 TB/s, ~6 us of launch + ramp + tail per copy launch; a bucket's
# compute is charged 16 us on top of its T_c (the median overhead the compute
# proxy measured over 582 per-parameter ops at T = 2048 before its affine
# calibration; now 2-8 us, so the charge is conservative: it keeps the search
# from plans of hundreds of buckets whose launch costs a real model pays)
K3_BPUS, K4_BPUS, LAUNCH_NS, COMPUTE_NS = 6470000, 6680000, 6000, 16000   # rates in bytes per microsecond


class PhaseModel:
    def __init__(self, specs, world, phase, t_c, link, mem_max):
        import paper_2411_00284_b200 as F
        from paper_2411_00284_b200 import _lib as L
        self.F, self.L = F, L
        self.specs, self.N, self.phase, self.link, self.mem_max = specs, world, phase, link, mem_max
        P = len(specs)
        self.order = list(range(P)) if phase == 0 else list(range(P - 1, -1, -1))
        self.t_c = t_c
        self.cache = {}
        self.seq_cache = {}

    def bucket(self, a, b):
        """Durations of bucket = phase positions [a, b): (unpack, compute, pack_rs, ag, rs, mem)."""
        key = (a, b)
        if key in self.cache:
            return self.cache[key]
        F, N = self.F, self.N
        m = sorted(self.order[a:b])
        d = [(self.specs[j].dim0, self.specs[j].row_numel, self.specs[j].module_id) for j in m]
        ag_seg = F.layout(d, N, 2, 16)[1]
        rs_seg = F.layout(d, N, 4, 16)[1]
        full = sum(2 * x[0] * x[1] for x in d)
        direct = len(d) == 1 and d[0][0] % N == 0 and ag_seg == d[0][0] // N * d[0][1] * 2
        # integer ns, the same formulas as fsdp_plan_search (include/fsdp.h)
        unpack = 0 if direct else 2 * full * 1000 // K3_BPUS + LAUNCH_NS
        pack_rs = (full // 2) * 6 * 1000 // K4_BPUS + LAUNCH_NS if self.phase == 1 else 0
        comp = sum(self.t_c[j] for j in m) + COMPUTE_NS
        ag = F.comm_time_ns(N * ag_seg, self.link)
        rs = F.comm_time_ns(N * rs_seg, self.link) if self.phase == 1 else 0
        mem = sum(N * (-(-x[0] // N)) * x[1] * 2 for x in d)     # M_j = padded gathered bytes (G13)
        r = (unpack, comp, pack_rs, ag, rs, mem)
        self.cache[key] = r
        return r

    def feasible(self, cuts):
        return all(self.bucket(a, b)[5] <= self.mem_max or b - a == 1 for a, b in zip(cuts, cuts[1:]))

    def seq(self, k, flags):
        key = (k, flags)
        if key not in self.seq_cache:
            L = self.L
            rep = self.F.run_schedule(None, None, None, n_fwd=k if self.phase == 0 else 0,
                                      n_bwd=k if self.phase == 1 else 0, flags=flags | L.SCHED_DRY_RUN)
            self.seq_cache[key] = rep["log"]
        return self.seq_cache[key]

    def time(self, cuts, flags):
        L = self.L
        bs = [self.bucket(a, b) for a, b in zip(cuts, cuts[1:])]
        seq = self.seq(len(bs), flags)
        dur = []
        for ph, op, b, _s, _n, _t in seq:
            u, c, prs, ag, rs, _m = bs[b]
            dur.append({L.OP_UNPACK: u, L.OP_COMPUTE_F: c, L.OP_COMPUTE_B: c, L.OP_PACK_RS: prs, L.OP_AG: ag,
                        L.OP_RS: rs}.get(op, 0))
        tot, exp, _, _ = self.F.simulate_schedule(seq, dur)
        return tot, exp


def cuts_of(plan, P, phase):
    """Plan (buckets of forward indices in execution order) -> phase-position cuts."""
    cuts, pos = [0], 0
    for b in plan:
        pos += len(b)
        cuts.append(pos)
    assert cuts[-1] == P
    return cuts


def plan_of(cuts, model):
    return [[model.order[i] for i in range(a, b)] for a, b in zip(cuts, cuts[1:])]


def library_cost(flags):
    """The same model as fsdp_search_cost for fsdp_plan_search."""
    return dict(unpack_bytes_per_us=K3_BPUS, pack_rs_bytes_per_us=K4_BPUS, copy_launch_ns=LAUNCH_NS,
                compute_overhead_ns=COMPUTE_NS, sched_flags=flags, max_moves=0)


def search(model, start, flags, budget_s=60.0):
    best = list(start)
    best_t = model.time(best, flags)[0]
    t0 = time.perf_counter()
    improved = True
    while improved and time.perf_counter() - t0 < budget_s:
        improved = False
        cands = []
        for i in range(1, len(best) - 1):
            cands.append(best[:i] + best[i + 1:])                               # merge
            for dlt in (-1, 1):                                                 # shift
                c = best[i] + dlt
                if best[i - 1] < c < best[i + 1]:
                    cands.append(best[:i] + [c] + best[i + 1:])
        for i in range(len(best) - 1):                                          # split
            a, b = best[i], best[i + 1]
            for c in sorted({a + (b - a) // 2, a + 1, b - 1}):
                if a < c < b:
                    cands.append(best[:i + 1] + [c] + best[i + 1:])
        for c in cands:
            if not model.feasible(c):
                continue
            t = model.time(c, flags)[0]
            if t < best_t:
                best, best_t, improved = c, t, True
                break
    return best, best_t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--mem-limit", type=float, default=2e9)
    ap.add_argument("--model", default="8b")
    ap.add_argument("--f-eff", type=float, default=1.0e15,
                    help="achieved dense bf16 FLOP/s of the compute model (1.33e15 = the cuBLASLt GEMMs measured)")
    ap.add_argument("--budget-s", type=float, default=90.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--python", action="store_true", help="use the Python reference search instead of the library")
    a = ap.parse_args()
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    specs = llama(a.model)
    P = len(specs)
    tf, tb = per_param_compute_ns(specs, a.tokens, f_eff=a.f_eff)
    link = (20000, round((a.world - 1) / a.world / 720e9 * 1e15))
    flags = {0: L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, 1: L.SCHED_REORDER}
    starts = {}
    for name, mode in (("manual", L.PLAN_MANUAL), ("greedy", L.PLAN_GREEDY), ("per_param", L.PLAN_PER_PARAM)):
        starts[name] = H.plans_for(specs, a.world, mode, tf, tb, link, link, int(a.mem_limit))
    out = {"model": "llama3-" + a.model, "world": a.world, "tokens_per_gpu": a.tokens, "link": link, "mem_max": a.mem_limit,
           "copy_model": {"K3_bytes_per_us": K3_BPUS, "K4_bytes_per_us": K4_BPUS, "launch_ns": LAUNCH_NS,
                          "compute_overhead_ns": COMPUTE_NS}, "phases": {}, "plans": {}}
    for phase, t_c in ((0, tf), (1, tb)):
        model = PhaseModel(specs, a.world, phase, t_c, link, a.mem_limit)
        rows = {}
        best = None
        for name, (fp, bp) in starts.items():
            cuts = cuts_of(fp if phase == 0 else bp, P, phase)
            t0, e0 = model.time(cuts, flags[phase])
            rows[name] = {"buckets": len(cuts) - 1, "total_ms": round(t0 / 1e6, 3), "exposed_ms": round(e0 / 1e6, 3)}
            if a.python:   # the reference implementation (time-bounded)
                c, t = search(model, cuts, flags[phase], a.budget_s / 3)
            else:          # fsdp_plan_search: the same moves and model, in C++, to convergence
                descs = [(x.dim0, x.row_numel, x.module_id) for x in specs]
                plan, t = F.plan_search(descs, a.world, t_c, link, link, int(a.mem_limit), phase,
                                        fp if phase == 0 else bp, library_cost(flags[phase]))
                c = cuts_of(plan, P, phase)
            e = model.time(c, flags[phase])[1]
            rows["search from " + name] = {"buckets": len(c) - 1, "total_ms": round(t / 1e6, 3),
                                           "exposed_ms": round(e / 1e6, 3)}
            if best is None or t < best[1]:
                best = (c, t)
        rows["best"] = {"buckets": len(best[0]) - 1, "total_ms": round(best[1] / 1e6, 3)}
        out["phases"]["fwd" if phase == 0 else "bwd"] = rows
        out["plans"]["fwd" if phase == 0 else "bwd"] = plan_of(best[0], model)
        print(("forward" if phase == 0 else "backward"), json.dumps(rows), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
