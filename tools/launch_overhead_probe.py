#!/usr/bin/env python
"""Where does a copy launch's time go?  (measurement tool, not the product path)

For K3 (one 8B block's copy-out, 872 MB algorithmic), K6 (one 8B block's RS
read-out, 218 MB), K1 (the embedding's own rows of a direct-gather bucket, 262
MB) and torch copy_ of the same bytes, at N = 8 layout (rank 0, layout-only
ctx), with SETS rotating buffer sets so nothing is L2-resident:

  single      one launch between a CUDA event pair (how the bench's per-op
              TIMING pass sees it), median of R
  batch       R launches back to back, one event pair around the batch
  graph       the same R launches captured in a CUDA graph, one event pair
  empty       an event pair around nothing / around an empty kernel

Prints one JSON object: ms per launch and algorithmic GB/s per mode, so the
fixed per-launch overhead (single - graph) can be read off.
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


def single(fn, s):
    ts = []
    for i in range(R + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(i % SETS)
        b.record(s)
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def batch(fn, s):
    for i in range(SETS):
        fn(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(R):
        fn(i % SETS)
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / R


def graph(fn, s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                fn(i % SETS)
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            g.replay()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) / R)
    return statistics.median(ts)


def probe(name, fn_for_stream, nbytes, s, out):
    row = {}
    for mode, f in (("single", single), ("batch", batch), ("graph", graph)):
        ms = f(fn_for_stream(s), s)
        row[mode] = {"ms": round(ms, 4), "GB/s": round(nbytes / ms / 1e6, 1)}
    row["bytes"] = nbytes
    row["overhead_us_single_minus_graph"] = round(1e3 * (row["single"]["ms"] - row["graph"]["ms"]), 2)
    out[name] = row


def main():
    torch.cuda.init()
    s = torch.cuda.Stream()
    world = 8
    ctx = F.Ctx(world, 0)
    out = {"gpu": torch.cuda.get_device_name(), "R": R, "sets": SETS}

    # empty event pair
    ts = []
    for i in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    out["empty_event_pair_us"] = round(1e3 * statistics.median(ts), 2)
    x = torch.zeros(1, device="cuda")
    ts = []
    for i in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            x.add_(1)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    out["tiny_kernel_event_pair_us"] = round(1e3 * statistics.median(ts), 2)

    # K3: one 8B block, copy-out of the gathered bucket
    specs = llama("8b", n_layers=1, with_embeddings=False)
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    _, aseg = F.layout(descs, world, 2, 16)
    _, rseg = F.layout(descs, world, 4, 16)
    fulls = [[torch.empty(d * r, dtype=torch.int16, device="cuda") for d, r, _ in descs] for _ in range(SETS)]
    agst = [torch.zeros(world * aseg, dtype=torch.uint8, device="cuda") for _ in range(SETS)]
    b3 = [F.Bucket(ctx, descs, fulls=[t.data_ptr() for t in fulls[i]]) for i in range(SETS)]
    valid = 2 * sum(d * r for d, r, _ in descs)
    probe("k3_unpack_8b_block", lambda st: (lambda i: F.allgather_bucket(ctx, b3[i], agst[i].data_ptr(),
                                                                          st.cuda_stream, 0, L.WAIT)),
          2 * valid, s, out)
    flat_src = [agst[i][:valid] for i in range(SETS)]
    flat_dst = [torch.empty(valid, dtype=torch.uint8, device="cuda") for _ in range(SETS)]

    def tcopy(st):
        def f(i):
            with torch.cuda.stream(st):
                flat_dst[i].copy_(flat_src[i])
        return f
    probe("torch_copy_872MB", tcopy, 2 * valid, s, out)
    del b3, fulls, agst, flat_src, flat_dst
    torch.cuda.empty_cache()

    # K6: one 8B block's RS read-out (this rank's fp32 segment -> grad shards)
    gsh = [[torch.zeros(-(-d // world) * r, dtype=torch.float32, device="cuda") for d, r, _ in descs]
           for _ in range(SETS)]
    rst = [torch.zeros(world * rseg // 4, dtype=torch.float32, device="cuda") for _ in range(SETS)]
    b6 = [F.Bucket(ctx, descs, grad_shards=[g.data_ptr() for g in gsh[i]]) for i in range(SETS)]
    probe("k6_copyout_8b_block", lambda st: (lambda i: F.reduce_scatter_bucket(ctx, b6[i], rst[i].data_ptr(),
                                                                               st.cuda_stream, 0, L.WAIT)),
          2 * rseg, s, out)
    src6 = [rst[i][:rseg // 4] for i in range(SETS)]
    dst6 = [torch.empty(rseg // 4, dtype=torch.float32, device="cuda") for _ in range(SETS)]

    def tcopy6(st):
        def f(i):
            with torch.cuda.stream(st):
                dst6[i].copy_(src6[i])
        return f
    probe("torch_copy_218MB", tcopy6, 2 * rseg, s, out)
    del b6, gsh, rst, src6, dst6
    torch.cuda.empty_cache()

    # K1: direct-gather embedding bucket, own rows -> full parameter
    d, Rn = 128256, 4096
    c = -(-d // world)
    shard_b = c * Rn * 2
    full = [torch.empty(d * Rn, dtype=torch.int16, device="cuda") for _ in range(SETS)]
    shards = [torch.randint(-2 ** 15, 2 ** 15, (c * Rn,), dtype=torch.int16, device="cuda") for _ in range(SETS)]
    stag = [torch.empty(world * shard_b + (1 << 20), dtype=torch.uint8, device="cuda") for _ in range(SETS)]
    bd = [F.Bucket(ctx, [(d, Rn, 0)], shards=[shards[i].data_ptr()], fulls=[full[i].data_ptr()],
                   flags=L.BUCKET_SEGMENT_SHARDS) for i in range(SETS)]
    probe("k1_direct_emb", lambda st: (lambda i: F.allgather_bucket(ctx, bd[i], stag[i].data_ptr(), st.cuda_stream,
                                                                    0, L.ISSUE)),
          2 * shard_b, s, out)
    torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
