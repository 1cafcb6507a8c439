#!/usr/bin/env python
"""Bandwidth probe of single launches (not part of the product path).

Times, with CUDA events on the launching stream (median of R launches, 4
rotating buffer sets so nothing is L2-resident), on the Llama-3-8B embedding
shard at N = 8 (16032 x 4096 bf16 = 131 MB) and one 8B block at N = 8:
  k1_direct   K1 of a direct-gather bucket (own rows -> the full parameter)
  k1_pack     K1 of a two-member bucket (own rows -> staging)
  k1_master   K1 rounding fp32 master shards to bf16 (FSDP_BUCKET_FP32_MASTER)
  k3_unpack   K3 of the two-member bucket
  k6_copy     K6 copy-out of the block's RS segment
  k6_accum    K6 in gradient-accumulation mode (shard += segment)
  k6_bf16     K6 rounding into bf16 gradient shards (FSDP_BUCKET_BF16_GRAD_SHARDS)
  torch_copy  torch copy_ of the same bytes (reference point)
Prints one JSON object; GB/s are algorithmic bytes (read + write) / time.
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
from workloads import llama  # noqa: E402

R = 20
SETS = 4


def timed(fn, nbytes, stream):
    ts = []
    for i in range(R + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn(i % SETS)
        b.record(stream)
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    return {"ms": round(ms, 4), "GB/s": round(nbytes / ms / 1e6, 1)}


def main():
    torch.cuda.init()
    s = torch.cuda.current_stream()
    cs = s.cuda_stream
    world, rank = 8, 0
    ctx = F.Ctx(world, rank)
    out = {}
    d, Rn = 128256, 4096
    c = -(-d // world)
    shard_b = c * Rn * 2
    # direct gather: one unpadded member, shards in segment layout
    full = [torch.empty(d * Rn, dtype=torch.int16, device="cuda") for _ in range(SETS)]
    shards = [torch.randint(-2**15, 2**15, (c * Rn,), dtype=torch.int16, device="cuda") for _ in range(SETS)]
    stag = [torch.empty(world * shard_b + (1 << 20), dtype=torch.uint8, device="cuda") for _ in range(SETS)]
    bd = [F.Bucket(ctx, [(d, Rn, 0)], shards=[shards[i].data_ptr()], fulls=[full[i].data_ptr()],
                   flags=L.BUCKET_SEGMENT_SHARDS) for i in range(SETS)]
    assert bd[0].query()["ag_direct"]
    out["k1_direct"] = timed(lambda i: F.allgather_bucket(ctx, bd[i], stag[i].data_ptr(), cs, 0, L.ISSUE),
                             2 * shard_b, s)
    # two-member bucket: the same shard plus a 1-D norm -> K1 pack into staging, K3 unpack
    norm = [torch.zeros(4096 // world, dtype=torch.int16, device="cuda") for _ in range(SETS)]
    nfull = [torch.empty(4096, dtype=torch.int16, device="cuda") for _ in range(SETS)]
    b2 = [F.Bucket(ctx, [(d, Rn, 0), (4096, 1, 1)], shards=[shards[i].data_ptr(), norm[i].data_ptr()],
                   fulls=[full[i].data_ptr(), nfull[i].data_ptr()]) for i in range(SETS)]
    out["k1_pack"] = timed(lambda i: F.allgather_bucket(ctx, b2[i], stag[i].data_ptr(), cs, 0, L.ISSUE),
                           2 * shard_b, s)
    out["k3_unpack"] = timed(lambda i: F.allgather_bucket(ctx, b2[i], stag[i].data_ptr(), cs, 0, L.WAIT),
                             2 * d * Rn * 2, s)
    out["torch_copy_131MB"] = timed(lambda i: full[i][:c * Rn].copy_(shards[i]), 2 * shard_b, s)
    del b2, bd
    # fp32 master shards -> bf16 (4 B read + 2 B written per element)
    masters = [torch.randn(c * Rn, dtype=torch.float32, device="cuda") for _ in range(SETS)]
    bm = [F.Bucket(ctx, [(d, Rn, 0), (4096, 1, 1)], shards=[masters[i].data_ptr(), norm[i].data_ptr()],
                   fulls=[full[i].data_ptr(), nfull[i].data_ptr()], flags=L.BUCKET_FP32_MASTER)
          for i in range(SETS)]
    out["k1_master"] = timed(lambda i: F.allgather_bucket(ctx, bm[i], stag[i].data_ptr(), cs, 0, L.ISSUE),
                             6 * c * Rn, s)
    del bm, masters, full, shards, stag
    torch.cuda.empty_cache()
    # K6 copy-out vs accumulation on one 8B block's RS segment
    specs = llama("8b", n_layers=1, with_embeddings=False)
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    _, rseg = F.layout(descs, world, 4, 16)
    gsh = [[torch.zeros(-(-dd // world) * rr, dtype=torch.float32, device="cuda") for dd, rr, _ in descs]
           for _ in range(SETS)]
    rst = [torch.zeros(world * rseg // 4, dtype=torch.float32, device="cuda") for _ in range(SETS)]
    bb = [F.Bucket(ctx, descs, grad_shards=[g.data_ptr() for g in gsh[i]]) for i in range(SETS)]
    out["k6_copy"] = timed(lambda i: F.reduce_scatter_bucket(ctx, bb[i], rst[i].data_ptr(), cs, 0, L.WAIT),
                           2 * rseg, s)
    # accumulation mode is latched at ISSUE: bind full gradients, ISSUE once, then time WAIT
    gfull = [[torch.zeros(dd * rr, dtype=torch.int16, device="cuda") for dd, rr, _ in descs] for _ in range(2)]
    del bb
    ba = [F.Bucket(ctx, descs, full_grads=[g.data_ptr() for g in gfull[i % 2]],
                   grad_shards=[g.data_ptr() for g in gsh[i]]) for i in range(SETS)]
    for i, b in enumerate(ba):
        b.set_grad_accumulation(True)
        F.reduce_scatter_bucket(ctx, b, rst[i].data_ptr(), cs, 0, L.ISSUE)   # latch the mode
    out["k6_accum"] = timed(lambda i: F.reduce_scatter_bucket(ctx, ba[i], rst[i].data_ptr(), cs, 0, L.WAIT),
                            3 * rseg, s)
    del ba
    # K6 rounding into bf16 gradient shards (FSDP_BUCKET_BF16_GRAD_SHARDS, G41): 4 B read + 2 B written
    gsh16 = [[torch.zeros(-(-dd // world) * rr, dtype=torch.int16, device="cuda") for dd, rr, _ in descs]
             for _ in range(SETS)]
    b16 = [F.Bucket(ctx, descs, grad_shards=[g.data_ptr() for g in gsh16[i]], flags=L.BUCKET_BF16_GRAD_SHARDS)
           for i in range(SETS)]
    out["k6_bf16"] = timed(lambda i: F.reduce_scatter_bucket(ctx, b16[i], rst[i].data_ptr(), cs, 0, L.WAIT),
                           rseg + rseg // 2, s)
    torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
