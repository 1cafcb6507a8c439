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

    import torch
    import torch.distributed as dist
    import paper_2411_00284_b200 as F
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

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    for n in sorted(set(sizes)):
        d = max(world, (n // (2 * R)) // world * world)
        r = H.time_bucket_collectives([ParamSpec("x", d, R, 0)], world, rank, ctx, cs.cuda_stream, ms.cuda_stream,
                                      reps=args.reps, warmup=2, p2p=p2p, exchange=exchange,
                                      max_over_ranks=max_over_ranks)
        r.update(ag_busbw=(world - 1) / world * r["ag_bytes"] / r["ag_ns"] if world > 1 else None,
                 rs_busbw=(world - 1) / world * r["rs_bytes"] / r["rs_ns"] if world > 1 else None,
                 ag_algbw=r["ag_bytes"] / r["ag_ns"], rs_algbw=r["rs_bytes"] / r["rs_ns"])
        rows.append(r)

    res = dict(world=world, collective=args.collective, rows=rows,
               fit={op: dict(zip(("alpha_ns", "beta_fs_per_byte"), H.fit_link(rows, op + "_bytes", op + "_ns")))
                    for op in ("ag", "rs")})
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
