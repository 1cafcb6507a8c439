#!/usr/bin/env python
"""Collective bandwidth sweep and alpha/beta fit (the cost model of P:222,
a11 in SURVEY §8(a); the planner's inputs).

    torchrun --nproc-per-node N tools/busbw_sweep.py [--collective nccl|p2p] [--out F]

For every full-bucket size n (2^13 .. 2^31 bytes, plus the Llama-3 bucket
sizes) one bucket holding one [d, 1024] bf16 parameter runs a forward AG and a
backward AG + RS through fsdp_run_schedule with FSDP_SCHED_TIMING; the AG / RS
entries of the log are CUDA events around the collective alone on the comm
stream.  Median of --reps, max over ranks.  Reports algbw = n / t and busbw =
(N - 1) / N * n / t, and fits alpha = median t at the smallest size, beta =
least-squares slope over n >= 64 MiB, rounded to integer ns / fs per byte
(fsdp_plan_in.ag / .rs).  At N = 1 it runs (1-rank communicator) but measures
local copies only.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--collective", default="nccl", choices=["nccl", "p2p"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=31)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads.shapes import ParamSpec

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    p2p = args.collective == "p2p"
    if world > 1:
        dist.init_process_group("gloo" if p2p else "nccl", **({} if p2p else {"device_id": torch.device("cuda", local)}))
    if p2p:
        ctx = F.Ctx(world, rank, local)
    else:
        uid = [F.nccl_get_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        ctx = F.Ctx(world, rank, local, nccl_uid=uid[0])
    R = 1024
    sizes = [2 ** k for k in range(13, args.max_log2 + 1)]
    sizes += [436224000, 1050673152]          # 8B block / embedding bucket (bf16 gathered bytes)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    rows = []

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if p2p else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for n in sorted(set(sizes)):
        d = max(world, (n // (2 * R)) // world * world)
        spec = [ParamSpec("x", d, R, 0)]
        plan = [[0]]
        st = H.RankState(spec, world, rank, plan, plan, ctx, ipc=p2p and world > 1)
        if p2p:
            if world > 1:
                def exchange(obj):
                    out = [None] * world
                    dist.all_gather_object(out, obj)
                    return out
                st.setup_p2p_ipc(exchange)
            else:
                st.setup_p2p_simulated()
        flags = L.SCHED_REORDER | L.SCHED_TIMING | (L.SCHED_P2P if p2p else 0)
        ag, rs = [], []
        for i in range(args.reps + 2):
            rep = st.step(flags, cs.cuda_stream, ms.cuda_stream, want_log=True)
            if i < 2:
                continue
            ag += [e[4] for e in rep["log"] if e[1] == L.OP_AG]
            rs += [e[4] for e in rep["log"] if e[1] == L.OP_RS]
        full_ag = world * st.fwd[0].ag_seg
        full_rs = world * st.bwd[0].rs_seg
        t_ag = max_over_ranks(float(np.median(ag)))
        t_rs = max_over_ranks(float(np.median(rs)))
        rows.append(dict(ag_bytes=full_ag, rs_bytes=full_rs, ag_ns=t_ag, rs_ns=t_rs,
                         ag_busbw=(world - 1) / world * full_ag / t_ag if world > 1 else None,
                         rs_busbw=(world - 1) / world * full_rs / t_rs if world > 1 else None,
                         ag_algbw=full_ag / t_ag, rs_algbw=full_rs / t_rs))
        if p2p:
            st.close_ipc()
        del st
        torch.cuda.empty_cache()

    def fit(key_b, key_t):
        small = min(rows, key=lambda r: r[key_b])
        big = [r for r in rows if r[key_b] >= 64 * 2 ** 20]
        x = np.array([r[key_b] for r in big], dtype=np.float64)
        y = np.array([r[key_t] for r in big], dtype=np.float64)
        beta = float(np.polyfit(x, y, 1)[0]) if len(big) >= 2 else 0.0
        return dict(alpha_ns=int(round(small[key_t])), beta_fs_per_byte=int(round(beta * 1e6)))

    res = dict(world=world, collective=args.collective, rows=rows,
               fit=dict(ag=fit("ag_bytes", "ag_ns"), rs=fit("rs_bytes", "rs_ns")))
    if rank == 0:
        print(json.dumps(res), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
