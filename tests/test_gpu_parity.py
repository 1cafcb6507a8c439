"""-m gpu parity: the CUDA path (through the C ABI) against the oracle,
element by element on the same seeded inputs.

1-GPU simulated ranks: one layout-only ctx per simulated rank;
every rank's K1 pack writes its own segment of one shared staging buffer,
which is then exactly the buffer an all-gather would leave on every rank, so
K3 on it is checked bit-exactly against the oracle.  For the reduce-scatter,
each rank's K4 output is checked bit-exactly, the collective's sum is taken by
the oracle's rank-order reduce_scatter (standing in for NCCL), written into
each rank's own segment, and K6 is checked bit-exactly.
"""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from oracle import schedule as OS
from oracle.layout import bucket_layout
from oracle.shard import shard, shard_rows
from workloads import llama, toy_mlp
from workloads.data import EDGE_BF16_BITS, EDGE_F32_BITS, grad_tensor, param_tensor
from workloads.shapes import ParamSpec

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"
    torch.cuda.init()


def _np(dt):
    return np.uint16 if dt == L.BF16 else np.float32


def _esize(dt):
    return 2 if dt == L.BF16 else 4


def _specs_from_dims(dims):
    return [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]


def _shard_on_device(full_devs, params, world, rank, dt):
    out = []
    for p, fd in zip(params, full_devs):
        d, r = p.shape
        c, _, _ = shard_rows(d, world, rank)
        sd = DevArray(nbytes=c * r * _esize(dt), fill=0xAB, dtype=_np(dt), shape=(c, r))
        info = F.shard(world, rank, (d, r, 0), dt, fd.ptr, sd.ptr)
        assert info["shard_rows"] == c
        out.append(sd)
    return out


def sim_allgather(params, world, dt, align=16, check_all_ranks=True):
    """Shard (K0) -> pack (K1) per simulated rank -> unpack (K3); compare."""
    dims = [p.shape for p in params]
    descs = [(d, r, 0) for d, r in dims]
    full_devs = [DevArray(p) for p in params]
    ctxs = [F.Ctx(world, r) for r in range(world)]
    shards = [_shard_on_device(full_devs, params, world, r, dt) for r in range(world)]
    for r in (range(world) if check_all_ranks else [0, world - 1]):
        for p, s in zip(params, shards[r]):
            assert np.array_equal(bits(s.get()), bits(shard(p, world, r)))
    _, seg = bucket_layout(dims, world, _esize(dt), align)
    # a one-parameter bucket with no padding gathers straight into the full
    # parameter (direct gather): every rank then needs its own full buffer
    direct = len(params) == 1 and dims[0][0] % world == 0 and seg == dims[0][0] // world * dims[0][1] * _esize(dt)
    out_ranks = range(world) if direct else {0, world - 1}
    outs = {r: [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
            for r in out_ranks}
    buckets = [F.Bucket(ctxs[r], descs, shards=[s.ptr for s in shards[r]],
                        fulls=[o.ptr for o in outs[r]] if r in outs else None,
                        param_dtype=dt, grad_dtype=dt, align=align) for r in range(world)]
    assert buckets[0].ag_seg == seg
    assert buckets[0].query()["ag_direct"] == direct
    staging = DevArray(nbytes=world * seg, fill=0xCD)
    for r in range(world):
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.ISSUE)
    g_ref, fulls_ref = OC.bucketed_all_gather(params, world, align)
    if direct:
        # ISSUE wrote each rank's own rows into its full parameter; the
        # all-gather (NCCL on real GPUs) gives every rank every rank's rows
        assert np.all(staging.get() == 0xCD)                 # staging untouched
        own = [outs[r][0].get().reshape(-1).view(np.uint8)[r * seg:(r + 1) * seg].copy() for r in range(world)]
        assert np.array_equal(np.concatenate(own), g_ref)
        for r in outs:
            o = outs[r][0]
            o.t[o.off:o.off + o.nbytes].copy_(torch.from_numpy(np.concatenate(own)))
    for r in outs:
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.WAIT)
    if not direct:
        assert np.array_equal(staging.get(), g_ref)       # raw buffer incl. zero pads
    for r in outs:
        for o, p in zip(outs[r], params):
            assert np.array_equal(bits(o.get()), bits(p))  # all_gather(shard(p)) == p
    return True


def sim_reduce_scatter(grads_per_rank, world, gdt, align=16):
    """K4 per simulated rank (bit-exact), oracle sum in rank order, K6 (bit-exact)."""
    dims = [g.shape for g in grads_per_rank[0]]
    descs = [(d, r, 0) for d, r in dims]
    _, seg = bucket_layout(dims, world, 4, align)
    ctxs = [F.Ctx(world, r) for r in range(world)]
    gdev = [[DevArray(g) for g in gs] for gs in grads_per_rank]
    gsh = [[DevArray(nbytes=-(-d // world) * r * 4, fill=0x77, dtype=np.float32, shape=(-(-d // world), r))
            for d, r in dims] for _ in range(world)]
    buckets = [F.Bucket(ctxs[r], descs, full_grads=[g.ptr for g in gdev[r]], grad_shards=[g.ptr for g in gsh[r]],
                        param_dtype=gdt, grad_dtype=gdt, align=align) for r in range(world)]
    assert buckets[0].rs_seg == seg
    stag = [DevArray(nbytes=world * seg, fill=0xEF, dtype=np.float32) for _ in range(world)]
    for r in range(world):
        F.reduce_scatter_bucket(ctxs[r], buckets[r], stag[r].ptr, flags=L.ISSUE)
    ins_ref, outs_ref, shards_ref = OC.bucketed_reduce_scatter(grads_per_rank, world, align)
    packed = [s.get() for s in stag]
    for r in range(world):
        assert np.array_equal(bits(packed[r]), bits(ins_ref[r]))
    # the collective (NCCL on real GPUs): rank-order fp32 sum of the device-packed inputs
    outs = OC.reduce_scatter(packed, world)
    for q in range(world):
        host = stag[q].get()
        host[q * seg // 4:(q + 1) * seg // 4] = outs[q]
        stag[q].t[stag[q].off:stag[q].off + stag[q].nbytes].copy_(torch.from_numpy(host.view(np.uint8).copy()))
        F.reduce_scatter_bucket(ctxs[q], buckets[q], stag[q].ptr, flags=L.WAIT)
    for q in range(world):
        for j in range(len(dims)):
            assert np.array_equal(bits(gsh[q][j].get()), bits(shards_ref[q][j]))
    return True


# ---------------------------------------------------------------- all-gather
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dt", [L.FP32, L.BF16])
def test_toy_mlp_allgather(world, dt):
    params = [param_tensor(p, "f32" if dt == L.FP32 else "bf16", 100 + i) for i, p in enumerate(toy_mlp())]
    assert sim_allgather(params, world, dt)


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_allgather(seed):
    rng = np.random.Generator(np.random.Philox(seed))
    world = int(rng.integers(2, 9))
    k = int(rng.integers(1, 13))
    dims = [(int(rng.integers(1, 300)), int(rng.integers(1, 70))) for _ in range(k)]
    dt = L.BF16 if seed % 2 else L.FP32
    align = 1 if seed % 3 == 0 else 16
    params = [param_tensor(s, "bf16" if dt == L.BF16 else "f32", seed * 31 + i)
              for i, s in enumerate(_specs_from_dims(dims))]
    assert sim_allgather(params, world, dt, align)


def test_edge_values_allgather():
    p = [np.tile(EDGE_BF16_BITS, 7).reshape(-1, 1), np.tile(EDGE_F32_BITS, 3).view(np.uint16).reshape(-1, 4)]
    assert sim_allgather(p, 3, L.BF16)


def test_llama8b_block_allgather_full_size():
    # BASELINE configs[1] bucket: one 8B transformer block, bf16, N = 8 (436.2 MB gathered)
    specs = llama("8b", n_layers=1, with_embeddings=False)
    params = [param_tensor(s, "bf16", 7 + i) for i, s in enumerate(specs)]
    assert sim_allgather(params, 8, L.BF16, check_all_ranks=False)


# ------------------------------------------------------------ reduce-scatter
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("gdt", [L.FP32, L.BF16])
def test_toy_mlp_reduce_scatter(world, gdt):
    specs = toy_mlp()
    g = [[grad_tensor(s, "f32" if gdt == L.FP32 else "bf16", 3, r) for s in specs] for r in range(world)]
    assert sim_reduce_scatter(g, world, gdt)


@pytest.mark.parametrize("seed", range(8))
def test_random_shapes_reduce_scatter(seed):
    rng = np.random.Generator(np.random.Philox(1000 + seed))
    world = int(rng.integers(2, 9))
    dims = [(int(rng.integers(1, 200)), int(rng.integers(1, 50))) for _ in range(int(rng.integers(1, 9)))]
    kind = "exact" if seed % 2 else "normal"
    g = [[grad_tensor(s, "bf16", seed, r, kind) for s in _specs_from_dims(dims)] for r in range(world)]
    assert sim_reduce_scatter(g, world, L.BF16, align=1 if seed % 3 == 0 else 16)


def test_edge_values_reduce_scatter():
    # +-0, subnormals, +-inf, NaN: widen + scale on device vs oracle; NaN by class
    g = [[np.tile(EDGE_BF16_BITS, 5).reshape(-1, 3)] for _ in range(2)]
    dims = [g[0][0].shape]
    _, seg = bucket_layout(dims, 2, 4, 16)
    ctx = F.Ctx(2, 0)
    gd = DevArray(g[0][0])
    b = F.Bucket(ctx, [(dims[0][0], dims[0][1], 0)], full_grads=[gd.ptr],
                 grad_shards=[DevArray(nbytes=4 * 3 * 10).ptr], param_dtype=L.BF16, grad_dtype=L.BF16)
    st = DevArray(nbytes=2 * seg, fill=0xEF, dtype=np.float32)
    F.reduce_scatter_bucket(ctx, b, st.ptr, flags=L.ISSUE)
    got = st.get()
    ref = OC.rs_pack(g[0], 2, 16)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(bits(got[~nan]), bits(ref[~nan]))


def test_llama8b_block_rs_pack_full_size():
    # K4 on the full 8B block at N = 8 for two ranks, bit-exact; copy-out checked on rank 0
    specs = llama("8b", n_layers=1, with_embeddings=False)
    world = 8
    dims = [(s.dim0, s.row_numel) for s in specs]
    _, seg = bucket_layout(dims, world, 4, 16)
    for r in (0, 5):
        g = [grad_tensor(s, "bf16", 11, r) for s in specs]
        ctx = F.Ctx(world, r)
        gd = [DevArray(x) for x in g]
        gs = [DevArray(nbytes=-(-d // world) * R * 4, dtype=np.float32, shape=(-(-d // world), R)) for d, R in dims]
        b = F.Bucket(ctx, [(d, R, 0) for d, R in dims], full_grads=[x.ptr for x in gd],
                     grad_shards=[x.ptr for x in gs], param_dtype=L.BF16, grad_dtype=L.BF16)
        st = DevArray(nbytes=world * seg, fill=0xEF, dtype=np.float32)
        F.reduce_scatter_bucket(ctx, b, st.ptr, flags=L.ISSUE | L.WAIT)  # layout-only: pack then copy-out
        packed = st.get()
        assert np.array_equal(bits(packed), bits(OC.rs_pack(g, world, 16)))
        # with no collective the own segment holds this rank's pre-scaled chunk
        own = packed[r * seg // 4:(r + 1) * seg // 4]
        for j, sh in enumerate(OC.rs_copyout(own, dims, world, 16)):
            assert np.array_equal(bits(gs[j].get()), bits(sh))
        del gd, gs, st, b, ctx
        torch.cuda.empty_cache()


def test_405b_layer_allgather_64bit_offsets():
    # BASELINE configs[4]: one 405B layer as one bucket at N = 8 (6.38 GB gathered,
    # byte offsets beyond 2^32).  Filled on device; checked by the property
    # all_gather(shard(p)) == p at full size plus oracle-computed sampled bytes.
    specs = llama("405b", n_layers=1, with_embeddings=False)
    world = 8
    dims = [(s.dim0, s.row_numel) for s in specs]
    descs = [(d, R, 0) for d, R in dims]
    offs, seg = bucket_layout(dims, world, 2, 16)
    assert world * seg > 2 ** 32
    gen = torch.Generator(device="cuda").manual_seed(405)
    fulls_src = [torch.randint(-32768, 32767, (d, R), dtype=torch.int16, device="cuda", generator=gen) for d, R in dims]
    ctxs = [F.Ctx(world, r) for r in range(world)]
    staging = torch.full((world * seg,), 0xCD, dtype=torch.uint8, device="cuda")
    out = [torch.empty_like(x) for x in fulls_src]
    buckets = []
    for r in range(world):
        sh = []
        for (d, R), src in zip(dims, fulls_src):
            c = -(-d // world)
            s = torch.empty((c, R), dtype=torch.int16, device="cuda")
            F.shard(world, r, (d, R, 0), L.BF16, src.data_ptr(), s.data_ptr())
            sh.append(s)
        b = F.Bucket(ctxs[r], descs, shards=[s.data_ptr() for s in sh],
                     fulls=[o.data_ptr() for o in out], param_dtype=L.BF16)
        F.allgather_bucket(ctxs[r], b, staging.data_ptr(), flags=L.ISSUE)
        buckets.append((b, sh))
    F.allgather_bucket(ctxs[0], buckets[0][0], staging.data_ptr(), flags=L.WAIT)
    torch.cuda.synchronize()
    for o, s in zip(out, fulls_src):
        assert torch.equal(o, s)
    # sampled staging bytes, located one by one with the oracle's layout
    rng = np.random.Generator(np.random.Philox(9))
    st16 = staging.view(torch.int16)
    for _ in range(200):
        q = int(rng.integers(0, world))
        j = int(rng.integers(0, len(dims)))
        d, R = dims[j]
        c, begin, v = shard_rows(d, world, q)
        row = int(rng.integers(0, c))
        col = int(rng.integers(0, R))
        pos = (q * seg + offs[j]) // 2 + row * R + col
        want = int(fulls_src[j][begin + row, col]) if row < v else 0
        assert int(st16[pos]) == want


# ------------------------------------------------- segment-layout storage
def _segment_storage(params, world, rank, dt, align, elem):
    """One buffer holding this rank's shards at the library's segment offsets
    (garbage in the gaps, which fsdp_bucket_create must zero)."""
    descs = [(p.shape[0], p.shape[1], 0) for p in params]
    offs, seg = F.layout(descs, world, elem, align)
    buf = np.full(seg, 0xEE, dtype=np.uint8)
    for p, o in zip(params, offs):
        b = shard(p, world, rank).reshape(-1).view(np.uint8)
        buf[o:o + b.size] = b
    return DevArray(buf), offs, seg


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("dt", [L.FP32, L.BF16])
def test_zero_copy_allgather_simulated(world, dt):
    specs = toy_mlp()
    params = [param_tensor(p, "f32" if dt == L.FP32 else "bf16", 300 + i) for i, p in enumerate(specs)]
    descs = [(p.shape[0], p.shape[1], 0) for p in params]
    stor, buckets, ctxs, outs = [], [], [], []
    for r in range(world):
        sbuf, offs, seg = _segment_storage(params, world, r, dt, 16, _esize(dt))
        ctx = F.Ctx(world, r)
        out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
        b = F.Bucket(ctx, descs, shards=[sbuf.ptr + o for o in offs], fulls=[o.ptr for o in out],
                     param_dtype=dt, grad_dtype=dt, flags=L.BUCKET_SEGMENT_SHARDS)
        assert b.query()["ag_zero_copy"] and b.query()["kernel_bytes"][0] == 0
        stor.append(sbuf)
        buckets.append(b)
        ctxs.append(ctx)
        outs.append(out)
    g_ref, _ = OC.bucketed_all_gather(params, world, 16)
    staging = DevArray(nbytes=world * seg, fill=0xCD)
    for r in range(world):
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.ISSUE)   # no pack: nothing written
        seg_r = stor[r].get()
        assert np.array_equal(seg_r, g_ref[r * seg:(r + 1) * seg])           # storage == packed segment, gaps zeroed
    # the all-gather (NCCL on real GPUs): every rank's storage segment into the staging
    host = staging.get()
    for r in range(world):
        host[r * seg:(r + 1) * seg] = stor[r].get()
    staging.t[staging.off:staging.off + staging.nbytes].copy_(torch.from_numpy(host))
    for r in range(world):
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.WAIT)
        for o, p in zip(outs[r], params):
            assert np.array_equal(bits(o.get()), bits(p))


def test_zero_copy_with_nccl_world1():
    # out-of-place AG from the storage and RS straight into gradient-shard storage
    specs = toy_mlp()
    params = [param_tensor(p, "bf16", 400 + i) for i, p in enumerate(specs)]
    grads = [grad_tensor(p, "bf16", 401, 0) for p in specs]
    descs = [(p.shape[0], p.shape[1], 0) for p in params]
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    sbuf, offs, seg = _segment_storage(params, 1, 0, L.BF16, 16, 2)
    roffs, rseg = F.layout(descs, 1, 4, 16)
    gstor = DevArray(nbytes=rseg, fill=0x33, dtype=np.float32)
    out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
    gd = [DevArray(g) for g in grads]
    b = F.Bucket(ctx, descs, shards=[sbuf.ptr + o for o in offs], fulls=[o.ptr for o in out],
                 full_grads=[g.ptr for g in gd], grad_shards=[gstor.ptr + o for o in roffs],
                 flags=L.BUCKET_SEGMENT_SHARDS | L.BUCKET_SEGMENT_GRAD_SHARDS)
    q = b.query()
    assert q["ag_zero_copy"] and q["rs_zero_copy"] and q["kernel_bytes"][0] == 0 and q["kernel_bytes"][3] == 0
    ag = DevArray(nbytes=seg, fill=0xCD)
    rs = DevArray(nbytes=rseg, fill=0xCD)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    F.allgather_bucket(ctx, b, ag.ptr, cs.cuda_stream, ms.cuda_stream)
    F.reduce_scatter_bucket(ctx, b, rs.ptr, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    g_ref, _ = OC.bucketed_all_gather(params, 1, 16)
    assert np.array_equal(ag.get(), g_ref)            # NCCL copied the storage segment
    for o, p in zip(out, params):
        assert np.array_equal(o.get(), p)
    _, _, shards_ref = OC.bucketed_reduce_scatter([grads], 1, 16)
    got = gstor.get()
    for j, o in enumerate(roffs):
        n = shards_ref[0][j].size
        assert np.array_equal(got[o // 4:o // 4 + n].view(np.uint32), shards_ref[0][j].reshape(-1).view(np.uint32))
    ctx.close()


# ------------------------------------------------------------------ schedule
def _schedule_case(world_comm):
    specs = toy_mlp()
    params = [param_tensor(p, "bf16", 50 + i) for i, p in enumerate(specs)]
    grads = [grad_tensor(p, "bf16", 51, 0) for p in specs]
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    if world_comm:
        ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    else:
        ctx = F.Ctx(1, 0)
    fb, _ = F.plan_buckets(descs, 1, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_FWD)
    bb, _ = F.plan_buckets(descs, 1, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_BWD)
    shards = [DevArray(p) for p in params]            # world 1: shard == param
    fulls = [DevArray(nbytes=p.nbytes, fill=0x11, dtype=np.uint16, shape=p.shape) for p in params]
    gd = [DevArray(g) for g in grads]
    gs = [DevArray(nbytes=g.size * 4, fill=0x22, dtype=np.float32, shape=g.shape) for g in grads]

    def mk(members):
        m = sorted(members)
        return F.Bucket(ctx, [descs[j] for j in m], shards=[shards[j].ptr for j in m],
                        fulls=[fulls[j].ptr for j in m], full_grads=[gd[j].ptr for j in m],
                        grad_shards=[gs[j].ptr for j in m])
    fwd = [mk(b) for b in fb]
    bwd = [mk(b) for b in bb]
    big_ag = max(b.ag_seg for b in fwd + bwd)
    big_rs = max(b.rs_seg for b in bwd)
    ag = [DevArray(nbytes=big_ag) for _ in range(2)]
    rs = [DevArray(nbytes=big_rs) for _ in range(2)]
    return ctx, params, grads, fulls, gs, fwd, bwd, ag, rs


@pytest.mark.parametrize("world_comm", [False, True])
@pytest.mark.parametrize("flags", [0, L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT,
                                   L.SCHED_REORDER | L.SCHED_BWD_AG_BEFORE_WAIT, L.SCHED_REORDER])
def test_schedule_executes_and_logs(world_comm, flags):
    ctx, params, grads, fulls, gs, fwd, bwd, ag, rs = _schedule_case(world_comm)
    s = torch.cuda.Stream()
    c = torch.cuda.Stream(priority=-1)
    rep = F.run_schedule(ctx, fwd, bwd, ag_staging=(ag[0].ptr, ag[1].ptr), rs_staging=(rs[0].ptr, rs[1].ptr),
                         compute=s.cuda_stream, comm=c.cuda_stream, flags=flags | L.SCHED_TIMING,
                         proxy_iters_fwd=[1000] * len(fwd), proxy_iters_bwd=[2000] * len(bwd))
    torch.cuda.synchronize()
    want = OS.step_sequence(len(fwd), len(bwd), bool(flags & L.SCHED_REORDER),
                            OS.BEFORE if flags & L.SCHED_FWD_AG_BEFORE_WAIT else OS.AFTER,
                            OS.BEFORE if flags & L.SCHED_BWD_AG_BEFORE_WAIT else OS.AFTER)
    assert [e[:4] for e in rep["log"]] == want
    assert rep["step_ns"] > 0
    assert rep["collectives"] == (len(fwd) + 2 * len(bwd) if world_comm else 0)
    for f, p in zip(fulls, params):
        assert np.array_equal(f.get(), p)
    for g_out, g in zip(gs, grads):
        assert np.array_equal(bits(g_out.get()), bits(OC.bf16.widen(g)))
    ctx.close()


def test_proxy_calibration_scales():
    ctx = F.Ctx(1, 0)
    t1 = F.proxy_calibrate(ctx, 20000)
    t2 = F.proxy_calibrate(ctx, 40000)
    assert t1 > 0 and 1.6 < t2 / t1 < 2.4


def test_segment_flag_validated():
    ctx = F.Ctx(2, 0)
    p = DevArray(np.zeros((64, 4), np.uint16))
    with pytest.raises(F.FsdpError):   # second member not at its segment offset
        F.Bucket(ctx, [(8, 4, 0), (8, 4, 0)], shards=[p.ptr, p.ptr + 1024], fulls=[p.ptr, p.ptr],
                 flags=L.BUCKET_SEGMENT_SHARDS)
    b = F.Bucket(ctx, [(8, 4, 0), (8, 4, 0)], shards=[p.ptr, p.ptr + 32], fulls=[p.ptr, p.ptr],
                 flags=L.BUCKET_SEGMENT_SHARDS)
    assert b.query()["ag_zero_copy"]


def test_abi_rejects_misaligned_staging_and_foreign_bucket():
    ctx, ctx2 = F.Ctx(2, 0), F.Ctx(2, 1)
    p = DevArray(np.zeros((4, 4), np.uint16))
    b = F.Bucket(ctx, [(8, 4, 0)], shards=[p.ptr], fulls=[p.ptr])
    st = DevArray(nbytes=1024)
    with pytest.raises(F.FsdpError):
        F.allgather_bucket(ctx, b, st.ptr + 2)
    with pytest.raises(F.FsdpError):
        F.allgather_bucket(ctx2, b, st.ptr)
    with pytest.raises(F.FsdpError):
        F.reduce_scatter_bucket(ctx, b, st.ptr)  # created without gradient pointers


def test_degenerate_steps_and_zero_row_ranks():
    """Edge cases the method has: an empty step (no buckets), a forward-only
    step, and ranks that own zero rows of every member (d < N)."""
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    rep = F.run_schedule(ctx, [], [], flags=L.SCHED_REORDER)
    assert rep["log_len"] == 0 and rep["kernel_launches"] == 0 and rep["collectives"] == 0
    ctx.close()
    # world 8, members with d in {1, 3, 7}: ranks 1..7 own zero rows of d = 1, ranks 3..7 of d = 3
    params = [param_tensor(s, "bf16", 90 + i) for i, s in enumerate(_specs_from_dims([(1, 24), (3, 8), (7, 1)]))]
    assert sim_allgather(params, 8, L.BF16)
    grads = [[grad_tensor(s, "bf16", 91, r) for s in _specs_from_dims([(1, 24), (3, 8), (7, 1)])] for r in range(8)]
    assert sim_reduce_scatter(grads, 8, L.BF16)
    # forward-only step on a layout-only ctx
    lay = F.Ctx(2, 1)
    p = param_tensor(ParamSpec("w", 10, 16, 0), "bf16", 5)
    sh = DevArray(shard(p, 2, 1))
    out = DevArray(nbytes=p.nbytes, fill=0, dtype=p.dtype, shape=p.shape)
    b = F.Bucket(lay, [(10, 16, 0)], shards=[sh.ptr], fulls=[out.ptr])
    ag = [DevArray(nbytes=2 * b.ag_seg, fill=0) for _ in range(2)]
    rep = F.run_schedule(lay, [b], [], ag_staging=(ag[0].ptr, ag[1].ptr), flags=L.SCHED_REORDER)
    torch.cuda.synchronize()
    assert rep["op_count"][L.OP_PACK_AG] == 1 and rep["op_count"][L.OP_RS] == 0
    # rank 1's own rows [5, 10) are in place; rank 0's rows come from a peer (none here)
    assert np.array_equal(out.get()[5:], p[5:])


def test_bulk_copy_engine_variant_parity():
    """The TMA bulk-copy engine build (FSDP_BULK=2: cp.async.bulk global ->
    shared -> global for the 16-B-aligned copy chunks of K0 / K1 / K3 / K6;
    measured slower than the LSU engine on B200 and off by default, DESIGN.md
    §6) moves the same bytes: the all-gather and reduce-scatter parity tests
    pass against it."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2411_00284_b200 import build as B
    lib = os.path.join(B.BUILD, "variants", "bulk", "libfsdp_b200.so")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(B.LIB):   # stale vs the main build
        lib = B.build(defines=["FSDP_BULK=2"], variant="bulk")
    env = dict(os.environ, FSDP_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "allgather or reduce_scatter or zero_copy", os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
