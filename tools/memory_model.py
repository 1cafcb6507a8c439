#!/usr/bin/env python
"""Peak FSDP-buffer memory of the Table 5 / Table 6 variants (the paper's
memory column) under the G40 allocate-on-produce /
free-after-last-use model (fsdp_simulate_memory), Llama-3-8B at N = 8.
Host-only: plans (fsdp_plan_buckets), segment sizes (fsdp_layout) and op
sequences (fsdp_run_schedule dry run) all come from the library without a GPU.

    python tools/memory_model.py [--tokens T] [--world N] [--out F]

The greedy plan takes the per-op compute model's T_c at T tokens and the
modelled NVLink link (alpha 20 us, 720 GB/s bus), M_max 2 GB.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bucket_sizes(specs, world, plan):
    import paper_2411_00284_b200 as F
    ag, full, grad, rs = [], [], [], []
    for b in plan:
        m = sorted(b)
        d = [(specs[j].dim0, specs[j].row_numel, specs[j].module_id) for j in m]
        ag.append(world * F.layout(d, world, 2, 16)[1])
        rs.append(world * F.layout(d, world, 4, 16)[1])
        n = sum(specs[j].dim0 * specs[j].row_numel for j in m)
        full.append(2 * n)
        grad.append(2 * n)
    return ag, full, grad, rs


def variant(specs, world, mode, flags, tf, tb, link, mem_max):
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    fplan, bplan = H.plans_for(specs, world, mode, tf, tb, link, link, mem_max)
    agf, fuf, _, _ = bucket_sizes(specs, world, fplan)
    agb, fub, grb, rsb = bucket_sizes(specs, world, bplan)
    rep = F.run_schedule(None, None, None, n_fwd=len(fplan), n_bwd=len(bplan), flags=flags | L.SCHED_DRY_RUN)
    peak, live = F.simulate_memory(rep["log"], agf, fuf, agb, fub, grb, rsb)
    return {"buckets_fwd": len(fplan), "buckets_bwd": len(bplan), "peak_GiB": round(peak / 2 ** 30, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--model", default="8b")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2411_00284_b200 import _lib as L
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    link = (20000, round((a.world - 1) / a.world / 720e9 * 1e15))
    R, FB, BB = L.SCHED_REORDER, L.SCHED_FWD_AG_BEFORE_WAIT, L.SCHED_BWD_AG_BEFORE_WAIT
    out = {"model": "llama3-%s" % a.model, "world": a.world, "tokens_per_gpu": a.tokens,
           "model_def": "G40: FSDP buffers (flat AG, full params, full grads, flat RS input) allocated on "
                        "produce, freed after last use, in the library's enqueue order; shards, gradient "
                        "shards and activations excluded"}
    # whole model (the 1 GB embedding / output buckets set the peak) and the
    # transformer blocks alone (where per-block bucketing and prefetch differ)
    for key, emb in (("whole_model", True), ("blocks_only", False)):
        specs = llama(a.model, with_embeddings=emb)
        tf, tb = per_param_compute_ns(specs, a.tokens)
        rows = {}
        for name, mode, flags in (("vanilla", L.PLAN_PER_PARAM, 0), ("+reorder", L.PLAN_PER_PARAM, R | FB),
                                  ("+bucket", L.PLAN_MANUAL, 0), ("+reorder & bucket", L.PLAN_MANUAL, R | FB),
                                  ("greedy + reorder", L.PLAN_GREEDY, R | FB),
                                  ("Table 6: fwd before / bwd before", L.PLAN_MANUAL, R | FB | BB),
                                  ("Table 6: fwd before / bwd after", L.PLAN_MANUAL, R | FB),
                                  ("Table 6: fwd after / bwd before", L.PLAN_MANUAL, R | BB),
                                  ("Table 6: fwd after / bwd after", L.PLAN_MANUAL, R)):
            rows[name] = variant(specs, a.world, mode, flags, tf, tb, link, 2 * 10 ** 9)
        out[key] = rows
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
