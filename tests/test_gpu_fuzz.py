"""-m gpu randomized parity sweep over the storage / alignment / world-size
combinations the library supports, every result bit-exact against the oracle:

  * plain pointers vs segment-layout storage (FSDP_BUCKET_SEGMENT_SHARDS) vs
    direct gather (one unpadded parameter), A in {1, 2, 4, 16, 256}, N up to 16;
  * bf16 and fp32 parameters / gradients, shapes with d < N (zero-row ranks),
    odd row lengths (unaligned runs), chunk-boundary-crossing sizes;
  * the NCCL-path kernels through simulated ranks and the peer-memory kernels.
"""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from oracle.layout import bucket_layout
from oracle.shard import shard
from workloads.data import grad_tensor, param_tensor
from workloads.shapes import ParamSpec

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.Generator(np.random.Philox(9000 + seed))
    world = int(rng.choice([1, 2, 3, 5, 8, 11, 16]))
    k = int(rng.integers(1, 7))
    big = seed % 5 == 0    # cross 32 KiB chunk boundaries
    dims = [(int(rng.integers(1, 3 * world + 40)), int(rng.integers(1, 9000 if big else 70))) for _ in range(k)]
    align = int(rng.choice([1, 2, 4, 16, 256]))
    dt = L.BF16 if rng.integers(0, 2) else L.FP32
    return world, dims, align, dt


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_allgather_reduce_scatter(seed):
    world, dims, align, dt = _case(seed)
    s = "bf16" if dt == L.BF16 else "f32"
    e = 2 if dt == L.BF16 else 4
    specs = [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]
    params = [param_tensor(p, s, seed * 13 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, s, seed, q) for p in specs] for q in range(world)]
    descs = [(d, r, 0) for d, r in dims]
    offs, seg = bucket_layout(dims, world, e, align)
    roffs, rseg = bucket_layout(dims, world, 4, align)
    g_ref, _ = OC.bucketed_all_gather(params, world, align)
    ins_ref, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, align)
    segment = seed % 2 == 1
    # segment storage needs 16-B aligned member offsets only through its base;
    # shards then live at base + off_j
    stor, bks, ctxs, outs = [], [], [], []
    staging = DevArray(nbytes=world * seg, fill=0xCD)
    for r in range(world):
        ctx = F.Ctx(world, r)
        if segment:
            buf = np.zeros(seg, dtype=np.uint8)
            for p, o in zip(params, offs):
                b = shard(p, world, r).reshape(-1).view(np.uint8)
                buf[o:o + b.size] = b
            sa = DevArray(buf)
            shard_ptrs, flags = [sa.ptr + o for o in offs], L.BUCKET_SEGMENT_SHARDS
            stor.append(sa)
        else:
            sas = [DevArray(shard(p, world, r)) for p in params]
            shard_ptrs, flags = [a.ptr for a in sas], 0
            stor.append(sas)
        out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
        gd = [DevArray(g) for g in grads[r]]
        gs = [DevArray(nbytes=-(-d // world) * R * 4, fill=0x77, dtype=np.float32) for d, R in dims]
        b = F.Bucket(ctx, descs, shards=shard_ptrs, fulls=[o.ptr for o in out], full_grads=[g.ptr for g in gd],
                     grad_shards=[g.ptr for g in gs], param_dtype=dt, grad_dtype=dt, align=align, flags=flags)
        bks.append((b, gd, gs))
        ctxs.append(ctx)
        outs.append(out)
        F.allgather_bucket(ctx, b, staging.ptr, flags=L.ISSUE)
    direct = bks[0][0].query()["ag_direct"]
    host = staging.get()
    for r in range(world):
        if direct:
            host[r * seg:(r + 1) * seg] = outs[r][0].get().reshape(-1).view(np.uint8)[r * seg:(r + 1) * seg]
        elif segment:
            host[r * seg:(r + 1) * seg] = stor[r].get()
    assert np.array_equal(host, g_ref)
    if direct:
        for r in range(world):
            o = outs[r][0]
            o.t[o.off:o.off + o.nbytes].copy_(torch.from_numpy(host))
    else:
        staging.t[staging.off:staging.off + staging.nbytes].copy_(torch.from_numpy(host))
    for r in range(world):
        F.allgather_bucket(ctxs[r], bks[r][0], staging.ptr, flags=L.WAIT)
        for o, p in zip(outs[r], params):
            assert np.array_equal(bits(o.get()), bits(p))
    # reduce-scatter through simulated ranks
    rst = [DevArray(nbytes=world * rseg, fill=0xEF, dtype=np.float32) for _ in range(world)]
    for r in range(world):
        F.reduce_scatter_bucket(ctxs[r], bks[r][0], rst[r].ptr, flags=L.ISSUE)
    packed = [x.get() for x in rst]
    for r in range(world):
        assert np.array_equal(bits(packed[r]), bits(ins_ref[r]))
    outs_rs = OC.reduce_scatter(packed, world)
    for q in range(world):
        h = packed[q].copy()
        h[q * rseg // 4:(q + 1) * rseg // 4] = outs_rs[q]
        rst[q].t[rst[q].off:rst[q].off + rst[q].nbytes].copy_(torch.from_numpy(h.view(np.uint8)))
        F.reduce_scatter_bucket(ctxs[q], bks[q][0], rst[q].ptr, flags=L.WAIT)
        for j, g in enumerate(bks[q][2]):
            assert np.array_equal(bits(g.get()), bits(shards_ref[q][j].reshape(-1)))


@pytest.mark.parametrize("seed", range(20))
def test_fuzz_peer_memory(seed):
    world, dims, align, dt = _case(100 + seed)
    world = min(world, 16)
    s = "bf16" if dt == L.BF16 else "f32"
    e = 2 if dt == L.BF16 else 4
    specs = [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]
    params = [param_tensor(p, s, seed * 17 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, s, seed + 50, q) for p in specs] for q in range(world)]
    descs = [(d, r, 0) for d, r in dims]
    offs, seg = bucket_layout(dims, world, e, align)
    _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, align)
    stor, regs = [], []
    for q in range(world):
        buf = np.zeros(-(-seg // 16) * 16 + 16, dtype=np.uint8)
        for p, o in zip(params, offs):
            b = shard(p, world, q).reshape(-1).view(np.uint8)
            buf[o:o + b.size] = b
        stor.append(DevArray(buf))
        goffs, cur = [], 0
        for g in grads[q]:
            goffs.append(cur)
            cur += -(-g.nbytes // 16) * 16
        gb = np.zeros(cur, dtype=np.uint8)
        for g, o in zip(grads[q], goffs):
            gb[o:o + g.nbytes] = g.reshape(-1).view(np.uint8)
        regs.append((DevArray(gb), goffs))
    for r in sorted({0, world - 1}):
        ctx = F.Ctx(world, r)
        out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
        gs = [DevArray(nbytes=-(-d // world) * R * 4, fill=0x77, dtype=np.float32) for d, R in dims]
        b = F.Bucket(ctx, descs, shards=[stor[r].ptr + o for o in offs], fulls=[o.ptr for o in out],
                     full_grads=[regs[r][0].ptr + o for o in regs[r][1]], grad_shards=[g.ptr for g in gs],
                     param_dtype=dt, grad_dtype=dt, align=align, flags=L.BUCKET_SEGMENT_SHARDS)
        F.p2p_allgather_bucket(ctx, b, [x.ptr for x in stor])
        F.p2p_reduce_scatter_bucket(ctx, b, [x[0].ptr for x in regs])
        torch.cuda.synchronize()
        for o, p in zip(out, params):
            assert np.array_equal(bits(o.get()), bits(p))
        for j, g in enumerate(gs):
            assert np.array_equal(bits(g.get()), bits(shards_ref[r][j].reshape(-1)))


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_master_weights_and_accumulation(seed):
    """fp32 master shards (K1 rounds to bf16) and gradient accumulation over
    two micro-batches, random shapes / alignments / world sizes."""
    from .test_gpu_mixed_precision import sim_master_allgather
    world, dims, align, dt = _case(300 + seed)
    rng = np.random.Generator(np.random.Philox(77 + seed))
    masters = [rng.standard_normal(d, dtype=np.float32) for d in dims]
    assert sim_master_allgather(masters, world, align)
    s = "bf16" if dt == L.BF16 else "f32"
    specs = [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]
    descs = [(d, r, 0) for d, r in dims]
    _, rseg = bucket_layout(dims, world, 4, align)
    held = [[rng.standard_normal((-(-d // world), r), dtype=np.float32) for d, r in dims] for _ in range(world)]
    want = [list(h) for h in held]
    ctxs = [F.Ctx(world, r) for r in range(world)]
    gds = [[DevArray(nbytes=d * r * (2 if dt == L.BF16 else 4), fill=0) for d, r in dims] for _ in range(world)]
    gss = [[DevArray(h) for h in held[q]] for q in range(world)]
    bks = [F.Bucket(ctxs[q], descs, full_grads=[g.ptr for g in gds[q]], grad_shards=[g.ptr for g in gss[q]],
                    param_dtype=dt, grad_dtype=dt, align=align) for q in range(world)]
    rst = [DevArray(nbytes=world * rseg, fill=0xEF, dtype=np.float32) for _ in range(world)]
    for m in range(2):
        grads = [[grad_tensor(p, s, 400 + 10 * seed + m, q) for p in specs] for q in range(world)]
        for q in range(world):
            bks[q].set_grad_accumulation(True)
            for dv, g in zip(gds[q], grads[q]):
                dv.t[dv.off:dv.off + dv.nbytes].copy_(torch.from_numpy(g.reshape(-1).view(np.uint8)))
            F.reduce_scatter_bucket(ctxs[q], bks[q], rst[q].ptr, flags=L.ISSUE)
        packed = [x.get() for x in rst]
        outs = OC.reduce_scatter(packed, world)
        _, _, ref = OC.bucketed_reduce_scatter(grads, world, align)
        for q in range(world):
            h = packed[q].copy()
            h[q * rseg // 4:(q + 1) * rseg // 4] = outs[q]
            rst[q].t[rst[q].off:rst[q].off + rst[q].nbytes].copy_(torch.from_numpy(h.view(np.uint8)))
            F.reduce_scatter_bucket(ctxs[q], bks[q], rst[q].ptr, flags=L.WAIT)
            want[q] = OC.accumulate_grad_shards(want[q], ref[q])
    for q in range(world):
        for j, g in enumerate(gss[q]):
            assert np.array_equal(bits(g.get()), bits(want[q][j])), (q, j)
