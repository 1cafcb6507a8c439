"""-m gpu: bf16 gradient shards (FSDP_BUCKET_BF16_GRAD_SHARDS, reading G41):
the reduce-scatter still sums in fp32 (reduce_dtype) and K6 rounds this
rank's fp32 segment to bf16 once (RNE) while copying it out.

* simulated ranks (the oracle's rank-order fp32 sum standing in for NCCL):
  bit-exact against oracle rs_copyout_bf16, toy / random / Llama-block shapes;
* a real NCCL communicator at world 1: bf16 gradients widened, x 1, summed
  over one rank and rounded back are the gradients' own bits (and within the
  north star's 1 bf16 ulp, which is what N > 2 NCCL sums are held to);
* the combinations that would write fp32 into bf16 storage are rejected."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from oracle.layout import bucket_layout
from workloads import llama, toy_mlp
from workloads.data import grad_tensor

from .gpu_util import DevArray, bf16_ulp_distance, bits
from .test_gpu_parity import _specs_from_dims

pytestmark = pytest.mark.gpu


def sim_rs_bf16(grads_per_rank, world, gdt, align=16, ranks=None):
    dims = [g.shape for g in grads_per_rank[0]]
    descs = [(d, r, 0) for d, r in dims]
    _, seg = bucket_layout(dims, world, 4, align)
    ctxs = [F.Ctx(world, r) for r in range(world)]
    gdev = [[DevArray(g) for g in gs] for gs in grads_per_rank]
    gsh = [[DevArray(nbytes=-(-d // world) * r * 2, fill=0x77, dtype=np.uint16, shape=(-(-d // world), r))
            for d, r in dims] for _ in range(world)]
    buckets = [F.Bucket(ctxs[r], descs, full_grads=[g.ptr for g in gdev[r]], grad_shards=[g.ptr for g in gsh[r]],
                        param_dtype=gdt, grad_dtype=gdt, align=align, flags=L.BUCKET_BF16_GRAD_SHARDS)
               for r in range(world)]
    n_shard = sum(-(-d // world) * r for d, r in dims)
    assert buckets[0].query()["kernel_bytes"][3] == 6 * n_shard     # K6: 4 B read + 2 B written per element
    stag = [DevArray(nbytes=world * seg, fill=0xEF, dtype=np.float32) for _ in range(world)]
    for r in range(world):
        F.reduce_scatter_bucket(ctxs[r], buckets[r], stag[r].ptr, flags=L.ISSUE)
    packed = [s.get() for s in stag]
    outs = OC.reduce_scatter(packed, world)           # the collective: rank-order fp32 sum
    for q in (ranks if ranks is not None else range(world)):
        host = stag[q].get()
        host[q * seg // 4:(q + 1) * seg // 4] = outs[q]
        stag[q].t[stag[q].off:stag[q].off + stag[q].nbytes].copy_(torch.from_numpy(host.view(np.uint8).copy()))
        F.reduce_scatter_bucket(ctxs[q], buckets[q], stag[q].ptr, flags=L.WAIT)
        want = OC.rs_copyout_bf16(outs[q], dims, world, align)
        for j in range(len(dims)):
            got = gsh[q][j].get()
            nan = np.isnan(OC.bf16.widen(want[j]))
            assert np.array_equal(nan, np.isnan(OC.bf16.widen(got)))
            assert np.array_equal(bits(got)[~nan], bits(want[j])[~nan])
    return True


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("gdt", [L.FP32, L.BF16])
def test_toy_mlp_bf16_shards(world, gdt):
    specs = toy_mlp()
    g = [[grad_tensor(s, "f32" if gdt == L.FP32 else "bf16", 5, r) for s in specs] for r in range(world)]
    assert sim_rs_bf16(g, world, gdt)


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_bf16_shards(seed):
    rng = np.random.Generator(np.random.Philox(2000 + seed))
    world = int(rng.integers(2, 9))
    dims = [(int(rng.integers(1, 200)), int(rng.integers(1, 50))) for _ in range(int(rng.integers(1, 9)))]
    kind = "exact" if seed % 2 else "normal"
    g = [[grad_tensor(s, "bf16", seed, r, kind) for s in _specs_from_dims(dims)] for r in range(world)]
    assert sim_rs_bf16(g, world, L.BF16, align=1 if seed % 3 == 0 else 16)


def test_llama8b_block_bf16_shards():
    specs = llama("8b", n_layers=1, with_embeddings=False)
    world = 4
    g = [[grad_tensor(s, "bf16", 13, r) for s in specs] for r in range(world)]
    assert sim_rs_bf16(g, world, L.BF16, ranks=[0, 3])
    torch.cuda.empty_cache()


def test_nccl_world1_bf16_shards_roundtrip():
    specs = toy_mlp()
    dims = [(s.dim0, s.row_numel) for s in specs]
    g = [grad_tensor(s, "bf16", 17, 0) for s in specs]
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    gd = [DevArray(x) for x in g]
    gs = [DevArray(nbytes=d * r * 2, fill=0x77, dtype=np.uint16, shape=(d, r)) for d, r in dims]
    b = F.Bucket(ctx, [(d, r, 0) for d, r in dims], full_grads=[x.ptr for x in gd], grad_shards=[x.ptr for x in gs],
                 param_dtype=L.BF16, grad_dtype=L.BF16, flags=L.BUCKET_BF16_GRAD_SHARDS)
    _, seg = bucket_layout(dims, 1, 4, 16)
    st = DevArray(nbytes=seg, fill=0xEF, dtype=np.float32)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    F.reduce_scatter_bucket(ctx, b, st.ptr, cs.cuda_stream, ms.cuda_stream, flags=L.ISSUE | L.WAIT)
    torch.cuda.synchronize()
    for x, y in zip(gs, g):
        assert np.array_equal(bits(x.get()), bits(y))              # widen, x 1, one-rank sum, RNE: identity
        assert bf16_ulp_distance(x.get(), y).max() <= 1
    del b
    ctx.close()


def test_bf16_shards_rejections():
    dims = [(16, 8)]
    ctx = F.Ctx(2, 0)
    gd = DevArray(nbytes=16 * 8 * 2)
    gs = DevArray(nbytes=8 * 8 * 2)
    with pytest.raises(L.FsdpError):   # the fp32 RS cannot land in bf16 segment storage
        F.Bucket(ctx, [(16, 8, 0)], full_grads=[gd.ptr], grad_shards=[gs.ptr], param_dtype=L.BF16,
                 grad_dtype=L.BF16, flags=L.BUCKET_BF16_GRAD_SHARDS | L.BUCKET_SEGMENT_GRAD_SHARDS)
    b = F.Bucket(ctx, [(16, 8, 0)], full_grads=[gd.ptr], grad_shards=[gs.ptr], param_dtype=L.BF16,
                 grad_dtype=L.BF16, flags=L.BUCKET_BF16_GRAD_SHARDS)
    with pytest.raises(L.FsdpError):   # accumulation is an fp32 add
        b.set_grad_accumulation(True)
    b.set_grad_accumulation(False)
    with pytest.raises(L.FsdpError):   # K9 writes fp32 shards
        F.p2p_reduce_scatter_bucket(ctx, b, [gd.ptr, gd.ptr])
    del b
    ctx.close()
    assert dims
