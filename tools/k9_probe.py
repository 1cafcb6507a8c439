#!/usr/bin/env python
"""K9 (fused peer-memory reduce-scatter) in the scheduled step vs alone
(measurement tool, not the product path).

Rank 0 of a simulated 8-way Llama-3-8B job with the 7 peers' gradient slots
in local HBM (harness.setup_p2p_simulated), per-block plan:
  * in_step: a FSDP_SCHED_P2P step with FSDP_SCHED_TIMING -- per backward
    bucket, the event-timed K9 (the RS op on the comm stream) and its
    algorithmic bytes (fsdp_bucket_query p2p_bytes);
  * alone:   fsdp_p2p_reduce_scatter_bucket on the same buckets (no epoch
    handshake), single launches between event pairs and back to back.
Prints one JSON object.
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_00284_b200 as F  # noqa: E402
from paper_2411_00284_b200 import _lib as L  # noqa: E402
from paper_2411_00284_b200 import harness as H  # noqa: E402
from workloads import llama  # noqa: E402


def main():
    world = 8
    specs = llama("8b", n_layers=int(os.environ.get("K9_LAYERS", "8")))
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=3)
    st.setup_p2p_simulated(seed=4)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT | L.SCHED_P2P
    for _ in range(3):
        st.step(flags, cs.cuda_stream, ms.cuda_stream)
    reps = [st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, want_log=True) for _ in range(5)]
    torch.cuda.synchronize()
    st.check_p2p()
    out = {"world": world, "buckets": []}
    k9b = [b.query()["p2p_bytes"][1] for b in st.bwd]
    for j, b in enumerate(st.bwd):
        ts = [e[4] for r in reps for e in r["log"] if e[0] == 1 and e[1] == L.OP_RS and e[2] == j]
        t_in = statistics.median(ts)
        # alone: single launches between event pairs, then 10 back to back
        single = []
        for _ in range(5):
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ms)
            F.p2p_reduce_scatter_bucket(ctx, b, st.rs_peers[j], ms.cuda_stream)
            c.record(ms)
            c.synchronize()
            single.append(a.elapsed_time(c) * 1e6)
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ms)
        for _ in range(10):
            F.p2p_reduce_scatter_bucket(ctx, b, st.rs_peers[j], ms.cuda_stream)
        c.record(ms)
        c.synchronize()
        b2b = a.elapsed_time(c) * 1e6 / 10
        out["buckets"].append({"bucket": j, "members": len(b.members), "bytes": k9b[j],
                               "in_step_us": round(t_in / 1e3, 1), "in_step_GBps": round(k9b[j] / t_in, 1),
                               "alone_single_us": round(statistics.median(single) / 1e3, 1),
                               "alone_b2b_us": round(b2b / 1e3, 1), "alone_b2b_GBps": round(k9b[j] / b2b, 1)})
    tot_in = sum(x["in_step_us"] for x in out["buckets"])
    tot_b = sum(x["bytes"] for x in out["buckets"])
    out["in_step_GBps_total"] = round(tot_b / (tot_in * 1e3), 1)
    out["alone_b2b_GBps_total"] = round(tot_b / (sum(x["alone_b2b_us"] for x in out["buckets"]) * 1e3), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
