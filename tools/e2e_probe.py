#!/usr/bin/env python
"""e2e A/B (measurement tool): the bench's end-to-end step -- shards H2D from
pinned host memory, fp32 gradient shards D2H, through fsdp_run_schedule --
with the step ending after its own D2H (sync) or letting the next step overlap
it (fsdp_host_io.async_d2h), K steps per repetition, repetitions interleaved.
Rank 0 of a simulated 8-way Llama-3-8B job, per-block plan, reorder.  Prints
one JSON object (ms per step per repetition)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_00284_b200 as F  # noqa: E402
from paper_2411_00284_b200 import _lib as L  # noqa: E402
from paper_2411_00284_b200 import harness as H  # noqa: E402
from workloads import llama  # noqa: E402


def main(K=10, reps=3):
    world = 8
    specs = llama("8b")
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=1)
    h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8, pin_memory=True)
    h_gs = torch.empty(st.gshard_buf.numel(), dtype=torch.uint8, pin_memory=True)
    h_sh.copy_(st.shard_buf)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    out = {"K": K, "sync": [], "async": []}
    for _ in range(reps):
        for mode in ("sync", "async"):
            io = st.host_io(h_sh, h_gs, h2d.cuda_stream, d2h.cuda_stream, async_d2h=mode == "async")
            st.step(flags, cs.cuda_stream, ms.cuda_stream, io=io)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event()
            a.record(cs)
            for _ in range(K):
                st.step(flags, cs.cuda_stream, ms.cuda_stream, io=io)
            e.record(cs)
            d2h.wait_event(e)
            b.record(d2h)
            b.synchronize()
            out[mode].append(round(a.elapsed_time(b) / K, 2))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
