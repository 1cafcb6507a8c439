"""-m gpu parity of gradient accumulation (fsdp_bucket_set_grad_accumulation,
SURVEY §8(f) NEXT #2): later reduce-scatters add their averaged shards to the
shards already held -- one fp32 addition per element, checked bit-exactly
against oracle.collectives.accumulate_grad_shards on every RS path: the
NCCL path's K6 (simulated ranks, the oracle's rank-order sum standing in for
NCCL), NCCL at world 1 with segment-layout gradient storage, the peer-memory
K9, and a scheduled step."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from workloads import toy_mlp
from workloads.data import grad_tensor
from workloads.shapes import ParamSpec

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"
    torch.cuda.init()


def _put(dev, host):
    dev.t[dev.off:dev.off + dev.nbytes].copy_(torch.from_numpy(np.ascontiguousarray(host).reshape(-1).view(np.uint8)))


def _existing(dims, world, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    return [rng.standard_normal((-(-d // world), r), dtype=np.float32) for d, r in dims]


@pytest.mark.parametrize("world,gdt,align", [(1, L.BF16, 16), (2, L.BF16, 16), (3, L.FP32, 16), (8, L.BF16, 16),
                                             (5, L.BF16, 1)])
def test_sim_reduce_scatter_accumulates(world, gdt, align):
    specs = toy_mlp() + [ParamSpec("odd", 37, 3, 9)]
    s = "bf16" if gdt == L.BF16 else "f32"
    dims = [(p.dim0, p.row_numel) for p in specs]
    descs = [(d, r, 0) for d, r in dims]
    ctxs = [F.Ctx(world, r) for r in range(world)]
    held = [_existing(dims, world, 70 + q) for q in range(world)]
    gsh = [[DevArray(h) for h in held[q]] for q in range(world)]
    micro = 3
    grads = [[[grad_tensor(p, s, 80 + m, r) for p in specs] for r in range(world)] for m in range(micro)]
    gdev = [[DevArray(g) for g in grads[0][r]] for r in range(world)]
    buckets = [F.Bucket(ctxs[r], descs, full_grads=[g.ptr for g in gdev[r]], grad_shards=[g.ptr for g in gsh[r]],
                        param_dtype=gdt, grad_dtype=gdt, align=align) for r in range(world)]
    for b in buckets:
        b.set_grad_accumulation(True)
    seg = buckets[0].rs_seg
    stag = [DevArray(nbytes=world * seg, fill=0xEF, dtype=np.float32) for _ in range(world)]
    want = [list(h) for h in held]
    for m in range(micro):
        for r in range(world):
            for g, dv in zip(grads[m][r], gdev[r]):
                _put(dv, g)
            F.reduce_scatter_bucket(ctxs[r], buckets[r], stag[r].ptr, flags=L.ISSUE)
        packed = [st.get() for st in stag]
        outs = OC.reduce_scatter(packed, world)          # stands in for NCCL
        _, _, shards_ref = OC.bucketed_reduce_scatter(grads[m], world, align)
        for q in range(world):
            host = stag[q].get()
            host[q * seg // 4:(q + 1) * seg // 4] = outs[q]
            _put(stag[q], host)
            F.reduce_scatter_bucket(ctxs[q], buckets[q], stag[q].ptr, flags=L.WAIT)
            want[q] = OC.accumulate_grad_shards(want[q], shards_ref[q])
        for q in range(world):
            for j in range(len(dims)):
                assert np.array_equal(bits(gsh[q][j].get()), bits(want[q][j])), (m, q, j)


def test_accumulation_toggle_overwrites_again():
    dims = [(64, 32), (7, 5)]
    descs = [(d, r, 0) for d, r in dims]
    ctx = F.Ctx(1, 0)
    g = [grad_tensor(ParamSpec("a", d, r, 0), "bf16", 3, 0) for d, r in dims]
    gd = [DevArray(x) for x in g]
    gs = [DevArray(h) for h in _existing(dims, 1, 5)]
    b = F.Bucket(ctx, descs, full_grads=[x.ptr for x in gd], grad_shards=[x.ptr for x in gs])
    st = DevArray(nbytes=b.rs_seg, fill=0)
    _, _, ref = OC.bucketed_reduce_scatter([g], 1)
    b.set_grad_accumulation(True)
    F.reduce_scatter_bucket(ctx, b, st.ptr)
    F.reduce_scatter_bucket(ctx, b, st.ptr)
    b.set_grad_accumulation(False)
    F.reduce_scatter_bucket(ctx, b, st.ptr)   # overwrite: exactly this RS's shards
    torch.cuda.synchronize()
    for x, r in zip(gs, ref[0]):
        assert np.array_equal(bits(x.get()), bits(r))
    assert L.lib.fsdp_bucket_set_grad_accumulation(b.h, 2) == L.FSDP_ERR_INVALID_ARG


def test_nccl_world1_segment_grad_storage_accumulates():
    specs = toy_mlp()
    dims = [(p.dim0, p.row_numel) for p in specs]
    descs = [(d, r, 0) for d, r in dims]
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    roffs, rseg = F.layout(descs, 1, 4, 16)
    held = _existing(dims, 1, 8)
    stor = np.zeros(rseg // 4, dtype=np.float32)
    for h, o in zip(held, roffs):
        stor[o // 4:o // 4 + h.size] = h.reshape(-1)
    gstor = DevArray(stor)
    gd = [DevArray(grad_tensor(p, "bf16", 90, 0)) for p in specs]
    b = F.Bucket(ctx, descs, full_grads=[x.ptr for x in gd], grad_shards=[gstor.ptr + o for o in roffs],
                 flags=L.BUCKET_SEGMENT_GRAD_SHARDS)
    assert b.query()["rs_zero_copy"]
    rs = DevArray(nbytes=rseg, fill=0xCD)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    want = list(held)
    for m in range(3):
        g = [grad_tensor(p, "bf16", 91 + m, 0) for p in specs]
        for x, h in zip(gd, g):
            _put(x, h)
        b.set_grad_accumulation(m > 0)    # first micro-batch overwrites
        torch.cuda.synchronize()
        F.reduce_scatter_bucket(ctx, b, rs.ptr, cs.cuda_stream, ms.cuda_stream)
        torch.cuda.synchronize()
        _, _, ref = OC.bucketed_reduce_scatter([g], 1, 16)
        want = ref[0] if m == 0 else OC.accumulate_grad_shards(want, ref[0])
        got = gstor.get()
        for j, o in enumerate(roffs):
            n = want[j].size
            assert np.array_equal(got[o // 4:o // 4 + n].view(np.uint32), want[j].reshape(-1).view(np.uint32))
    ctx.close()


@pytest.mark.parametrize("world", [1, 3, 8])
def test_p2p_reduce_scatter_accumulates(world):
    from .test_gpu_p2p import _grad_region
    specs = toy_mlp() + [ParamSpec("odd", 29, 3, 9)]
    dims = [(p.dim0, p.row_numel) for p in specs]
    descs = [(d, r, 0) for d, r in dims]
    grads = [[[grad_tensor(p, "bf16", 300 + m, r) for p in specs] for r in range(world)] for m in range(2)]
    for r in range(world):
        regions = [[_grad_region(grads[m][q]) for q in range(world)] for m in range(2)]
        ctx = F.Ctx(world, r)
        held = _existing(dims, world, 400 + r)
        gs = [DevArray(h) for h in held]
        b = F.Bucket(ctx, descs, full_grads=[regions[0][r][0].ptr + o for o in regions[0][r][1]],
                     grad_shards=[x.ptr for x in gs])
        b.set_grad_accumulation(True)
        want = held
        for m in range(2):
            F.p2p_reduce_scatter_bucket(ctx, b, [regions[m][q][0].ptr for q in range(world)])
            torch.cuda.synchronize()
            _, _, ref = OC.bucketed_reduce_scatter(grads[m], world, 16)
            want = OC.accumulate_grad_shards(want, ref[r])
            for x, w in zip(gs, want):
                assert np.array_equal(bits(x.get()), bits(w)), (r, m)


def test_schedule_accumulates_over_micro_batches():
    from .test_gpu_parity import _schedule_case
    ctx, params, grads, fulls, gs, fwd, bwd, ag, rs = _schedule_case(True)
    for b in bwd:
        b.set_grad_accumulation(True)
    sh = [g.get().copy() for g in gs]          # 0x22 fill as fp32: the "held" gradients
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        F.run_schedule(ctx, fwd, bwd, ag_staging=(ag[0].ptr, ag[1].ptr), rs_staging=(rs[0].ptr, rs[1].ptr),
                       compute=cs.cuda_stream, comm=ms.cuda_stream, flags=L.SCHED_REORDER)
    torch.cuda.synchronize()
    _, _, ref = OC.bucketed_reduce_scatter([[g for g in grads]], 1, 16)
    for g, h, r in zip(gs, sh, ref[0]):
        want = OC.accumulate_grad_shards(OC.accumulate_grad_shards([h], [r]), [r])[0]
        assert np.array_equal(bits(g.get()), bits(want))
    ctx.close()
