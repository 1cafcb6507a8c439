#!/usr/bin/env python
"""Tuning sweep of the data-kernel engines (not part of the product path).

    python tools/kernel_sweep.py --build            # here: compile the variants (CPU)
    python tools/kernel_sweep.py --run [--out F]    # on the B200: time every variant

Each variant is libfsdp_b200.so built with different FSDP_* macros
(kernels.cu), loaded in its own process through FSDP_B200_LIB, and timed on
the BASELINE configs[1] per-rank workload: four distinct Llama-3-8B blocks at
N = 8 (rank 0), each kernel launched through the public ABI (layout-only ctx:
AG ISSUE = K1, AG WAIT = K3, RS ISSUE = K4, RS WAIT = K6), CUDA events on the
launching stream, blocks rotated so nothing is L2-resident (436 MB > 126 MB).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SWEEP2 = {
    "c16": ["FSDP_CTAS_PER_SM=16"],
    "c32": ["FSDP_CTAS_PER_SM=32"],
    "c1k": ["FSDP_CTAS_PER_SM=1024"],
    "c16_k16": ["FSDP_CTAS_PER_SM=16", "FSDP_CHUNK_KB=16"],
    "c32_k16": ["FSDP_CTAS_PER_SM=32", "FSDP_CHUNK_KB=16"],
    "c1k_k16": ["FSDP_CTAS_PER_SM=1024", "FSDP_CHUNK_KB=16"],
    "c32_k64": ["FSDP_CTAS_PER_SM=32", "FSDP_CHUNK_KB=64"],
    "c32_u4": ["FSDP_CTAS_PER_SM=32", "FSDP_UNROLL=4"],
    "c32_st": ["FSDP_CTAS_PER_SM=32", "FSDP_ST_HINT=1"],
    "c32_t128": ["FSDP_CTAS_PER_SM=32", "FSDP_THREADS=128", "FSDP_MIN_BLOCKS=8"],
    "bulk_4x3_k16_all": ["FSDP_BULK=2", "FSDP_BULK_STAGES=3", "FSDP_CHUNK_KB=16", "FSDP_BULK_CTAS_PER_SM=4",
                         "FSDP_BULK_GRID_PER_SM=1024"],
    "bulk_2x3_all": ["FSDP_BULK=2", "FSDP_BULK_STAGES=3", "FSDP_BULK_CTAS_PER_SM=2", "FSDP_BULK_GRID_PER_SM=1024"],
    "bulk_4x2_k16_c32": ["FSDP_BULK=2", "FSDP_BULK_STAGES=2", "FSDP_CHUNK_KB=16", "FSDP_BULK_CTAS_PER_SM=4",
                         "FSDP_BULK_GRID_PER_SM=32", "FSDP_CTAS_PER_SM=32"],
}

SWEEP3 = {
    "d1_c1k": ["FSDP_CTAS_PER_SM=1024"],
    "d2_c1k_u4": ["FSDP_CTAS_PER_SM=1024", "FSDP_UNROLL=4"],
    "d3_c32": ["FSDP_CTAS_PER_SM=32"],
    "d4_c32_u4": ["FSDP_CTAS_PER_SM=32", "FSDP_UNROLL=4"],
    "d5_c1k_u4_nov8": ["FSDP_CTAS_PER_SM=1024", "FSDP_UNROLL=4", "FSDP_WIDEN_V8=0"],
    "d6_c1k_k64": ["FSDP_CTAS_PER_SM=1024", "FSDP_CHUNK_KB=64"],
    "d7_c1k_u4_mb8": ["FSDP_CTAS_PER_SM=1024", "FSDP_UNROLL=4", "FSDP_MIN_BLOCKS=8"],
    "d8_c1k_t128_u4": ["FSDP_CTAS_PER_SM=1024", "FSDP_THREADS=128", "FSDP_UNROLL=4", "FSDP_MIN_BLOCKS=16"],
}

SWEEP4 = {
    "e0_default": [],
    "e1_k9tpl": ["FSDP_K9_TEMPLATED=1"],
    "e2_k9tpl_mb2": ["FSDP_K9_TEMPLATED=1", "FSDP_K9_MIN_BLOCKS=2"],
    "e3_k9_mb2": ["FSDP_K9_MIN_BLOCKS=2"],
    "e4_k9tpl_k16": ["FSDP_K9_TEMPLATED=1", "FSDP_CHUNK_KB=16"],
}

SWEEP5 = {
    "f1_bulk_s8_l2_k16_c1": ["FSDP_BULK=2", "FSDP_BULK_STAGES=8", "FSDP_BULK_LAG=2", "FSDP_CHUNK_KB=16",
                             "FSDP_BULK_CTAS_PER_SM=1", "FSDP_BULK_GRID_PER_SM=1"],
    "f2_bulk_s6_l2_k32_c1": ["FSDP_BULK=2", "FSDP_BULK_STAGES=6", "FSDP_BULK_LAG=2",
                             "FSDP_BULK_CTAS_PER_SM=1", "FSDP_BULK_GRID_PER_SM=1"],
    "f3_bulk_s4_l1_k16_c2": ["FSDP_BULK=2", "FSDP_BULK_STAGES=6", "FSDP_BULK_LAG=1", "FSDP_CHUNK_KB=16",
                             "FSDP_BULK_CTAS_PER_SM=2", "FSDP_BULK_GRID_PER_SM=2"],
    "f4_bulk_s8_l3_k16_c1": ["FSDP_BULK=2", "FSDP_BULK_STAGES=12", "FSDP_BULK_LAG=3", "FSDP_CHUNK_KB=16",
                             "FSDP_BULK_CTAS_PER_SM=1", "FSDP_BULK_GRID_PER_SM=1"],
    "f5_bulk_s4_l1_k16_c3": ["FSDP_BULK=2", "FSDP_BULK_STAGES=4", "FSDP_BULK_LAG=1", "FSDP_CHUNK_KB=16",
                             "FSDP_BULK_CTAS_PER_SM=3", "FSDP_BULK_GRID_PER_SM=3"],
}

VARIANTS = {
    **SWEEP5,
    **SWEEP4,
    **SWEEP3,
    **SWEEP2,
    "base": [],
    "u16": ["FSDP_UNROLL=16", "FSDP_MIN_BLOCKS=2"],
    "u4": ["FSDP_UNROLL=4"],
    "ctas4": ["FSDP_CTAS_PER_SM=4"],
    "ctas16": ["FSDP_CTAS_PER_SM=16"],
    "chunk64": ["FSDP_CHUNK_KB=64"],
    "chunk16": ["FSDP_CHUNK_KB=16"],
    "sthint": ["FSDP_ST_HINT=1"],
    "ldcs": ["FSDP_LD_HINT=1"],
    "t512": ["FSDP_THREADS=512", "FSDP_MIN_BLOCKS=2"],
    "bulk2": ["FSDP_BULK=2"],
    "bulk2_s3x2": ["FSDP_BULK=2", "FSDP_BULK_STAGES=3", "FSDP_BULK_CTAS_PER_SM=2"],
    "bulk2_s4_c16": ["FSDP_BULK=2", "FSDP_BULK_STAGES=12", "FSDP_CHUNK_KB=16"],
}


def lib_path(name):
    return os.path.join(ROOT, "paper_2411_00284_b200", "_build", "variants", name, "libfsdp_b200.so")


def build_all(names):
    from paper_2411_00284_b200.build import build
    for n in names:
        print(n, build(defines=VARIANTS[n], variant=n), flush=True)


def measure(reps=5, nblocks=4):
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from workloads import llama

    world = 8
    specs = llama("8b", n_layers=1, with_embeddings=False)
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    full = [p.dim0 * p.row_numel for p in specs]
    shard = [-(-p.dim0 // world) * p.row_numel for p in specs]
    ctx = F.Ctx(world, 0)
    blocks = []
    for b in range(nblocks):
        sh = [torch.randn(n, device="cuda").to(torch.bfloat16) for n in shard]
        fu = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for n in full]
        gr = [torch.randn(n, device="cuda").to(torch.bfloat16) for n in full]
        gs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in shard]
        bk = F.Bucket(ctx, descs, shards=[x.data_ptr() for x in sh], fulls=[x.data_ptr() for x in fu],
                      full_grads=[x.data_ptr() for x in gr], grad_shards=[x.data_ptr() for x in gs])
        ag = torch.empty(world * bk.ag_seg, dtype=torch.uint8, device="cuda")
        rs = torch.empty(world * bk.rs_seg, dtype=torch.uint8, device="cuda")
        blocks.append((bk, ag, rs, sh, fu, gr, gs))
    s = torch.cuda.Stream()
    ops = {
        "K1_ag_pack": (lambda b: F.allgather_bucket(ctx, b[0], b[1].data_ptr(), s.cuda_stream, 0, L.ISSUE),
                       2 * 2 * sum(shard)),
        "K3_ag_unpack": (lambda b: F.allgather_bucket(ctx, b[0], b[1].data_ptr(), s.cuda_stream, 0, L.WAIT),
                         2 * 2 * sum(full)),
        "K4_rs_pack": (lambda b: F.reduce_scatter_bucket(ctx, b[0], b[2].data_ptr(), s.cuda_stream, 0, L.ISSUE),
                       6 * sum(full)),
        "K6_rs_copyout": (lambda b: F.reduce_scatter_bucket(ctx, b[0], b[2].data_ptr(), s.cuda_stream, 0, L.WAIT),
                          8 * sum(shard)),
    }
    # peer-memory kernels: rank 0 of 8, the 7 peers' buffers simulated in local HBM
    goffs, gtot = [], 0
    for n in full:
        goffs.append(gtot)
        gtot += -(-2 * n // 256) * 256
    soffs, sseg = F.layout(descs, world, 2, 16)
    pblocks = []
    for b in range(nblocks):
        stor = [torch.randn(sseg // 2, device="cuda").to(torch.bfloat16) for _ in range(world)]
        greg = [torch.randn(gtot // 2, device="cuda").to(torch.bfloat16) for _ in range(world)]
        fu = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for n in full]
        gs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in shard]
        bk = F.Bucket(ctx, descs, shards=[stor[0].data_ptr() + o for o in soffs], fulls=[x.data_ptr() for x in fu],
                      full_grads=[greg[0].data_ptr() + o for o in goffs], grad_shards=[x.data_ptr() for x in gs],
                      flags=L.BUCKET_SEGMENT_SHARDS)
        pblocks.append((bk, [x.data_ptr() for x in stor], [x.data_ptr() for x in greg], stor, greg, fu, gs))
    q0 = pblocks[0][0].query()["p2p_bytes"]
    pops = {
        "K8_p2p_ag": (lambda b: F.p2p_allgather_bucket(ctx, b[0], b[1], s.cuda_stream), q0[0]),
        "K9_p2p_rs": (lambda b: F.p2p_reduce_scatter_bucket(ctx, b[0], b[2], s.cuda_stream), q0[1]),
    }
    out = {}
    for name, (fn, nbytes) in pops.items():
        for b in pblocks:
            fn(b)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            for b in pblocks:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn(b)
                e1.record(s)
                times.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in times)
        med = ms[len(ms) // 2]
        out[name] = {"GB/s": round(nbytes / (med * 1e-3) / 1e9, 1), "ms": round(med, 4), "bytes": nbytes}
    del pblocks
    torch.cuda.empty_cache()
    for name, (fn, nbytes) in ops.items():
        for b in blocks:       # warm-up
            fn(b)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            for b in blocks:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn(b)
                e1.record(s)
                times.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in times)
        med = ms[len(ms) // 2]
        out[name] = {"GB/s": round(nbytes / (med * 1e-3) / 1e9, 1), "ms": round(med, 4), "bytes": nbytes}
    # reference copy: torch copy_ of 1 Gi bf16 elements (the MEASURED_PEAKS method)
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    c = torch.empty_like(a)
    c.copy_(a)
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["torch_copy_1Gi_bf16"] = {"GB/s": round(4 * 2 ** 30 / (best * 1e-3) / 1e9, 1)}
    return out


def main():
    names = [a for a in sys.argv[1:] if a in VARIANTS] or list(VARIANTS)
    if "--build" in sys.argv:
        build_all(names)
        return
    if "--measure" in sys.argv:
        print("RESULT " + json.dumps(measure()), flush=True)
        return
    if "--run" in sys.argv:
        res = {}
        for n in names:
            env = dict(os.environ, FSDP_B200_LIB=lib_path(n))
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--measure"], env=env,
                               capture_output=True, text=True, timeout=600)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            res[n] = json.loads(line[0][7:]) if line else {"error": (r.stderr or r.stdout)[-2000:]}
            print(n, json.dumps(res[n]), flush=True)
        out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
        if out:
            with open(out, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
