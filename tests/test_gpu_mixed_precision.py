"""-m gpu parity of the mixed-precision all-gather (FSDP_BUCKET_FP32_MASTER,
P:302 "parameters are cast to param_dtype"): fp32 master shards, rounded to
bf16 by the pack kernel K1, gathered and copied out in bf16 -- bit-exact
against oracle.collectives.mixed_precision_all_gather (NaN by class, G27).

1-GPU simulated ranks as in test_gpu_parity: every rank's K1 writes its own
segment of one shared staging buffer, which is then exactly what the
all-gather leaves on every rank.
"""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle.collectives import mixed_precision_all_gather
from oracle.layout import bucket_layout
from oracle.shard import shard, shard_rows
from workloads import llama, toy_mlp
from workloads.data import EDGE_F32_BITS, param_tensor

from .gpu_util import DevArray

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"
    torch.cuda.init()


def _same_bf16(a, b):
    """bit-exact, except that NaNs compare by class (payload unspecified, G27)."""
    a = np.asarray(a, dtype=np.uint16)
    b = np.asarray(b, dtype=np.uint16)
    na = ((a & 0x7F80) == 0x7F80) & ((a & 0x7F) != 0)
    nb = ((b & 0x7F80) == 0x7F80) & ((b & 0x7F) != 0)
    return np.array_equal(na, nb) and np.array_equal(a[~na], b[~nb])


def sim_master_allgather(masters, world, align=16, ranks_out=None):
    dims = [m.shape for m in masters]
    descs = [(d, r, 0) for d, r in dims]
    g_ref, fulls_ref = mixed_precision_all_gather(masters, world, align)
    _, seg = bucket_layout(dims, world, 2, align)
    direct = len(dims) == 1 and dims[0][0] % world == 0 and seg == dims[0][0] // world * dims[0][1] * 2
    ctxs = [F.Ctx(world, r) for r in range(world)]
    # fp32 master shards, cut on the device by K0 and checked against the oracle
    mdev = [DevArray(m) for m in masters]
    shards = []
    for r in range(world):
        row = []
        for m, md in zip(masters, mdev):
            d, R = m.shape
            c, _, _ = shard_rows(d, world, r)
            sd = DevArray(nbytes=c * R * 4, fill=0xAB, dtype=np.float32, shape=(c, R))
            F.shard(world, r, (d, R, 0), L.FP32, md.ptr, sd.ptr)
            assert np.array_equal(sd.get().view(np.uint32), shard(m, world, r).view(np.uint32))
            row.append(sd)
        shards.append(row)
    out_ranks = list(range(world)) if direct else sorted(ranks_out or {0, world - 1})
    outs = {r: [DevArray(nbytes=d * R * 2, fill=0x5A, dtype=np.uint16, shape=(d, R)) for d, R in dims]
            for r in out_ranks}
    buckets = [F.Bucket(ctxs[r], descs, shards=[s.ptr for s in shards[r]],
                        fulls=[o.ptr for o in outs[r]] if r in outs else None,
                        param_dtype=L.BF16, grad_dtype=L.BF16, align=align, flags=L.BUCKET_FP32_MASTER)
               for r in range(world)]
    assert buckets[0].ag_seg == seg and buckets[0].query()["ag_direct"] == direct
    staging = DevArray(nbytes=world * seg, fill=0xCD)
    for r in range(world):
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.ISSUE)
    if direct:
        own = [outs[r][0].get().reshape(-1)[r * (seg // 2):(r + 1) * (seg // 2)].copy() for r in range(world)]
        gathered = np.concatenate(own)
        assert _same_bf16(gathered, g_ref.view(np.uint16))
        for r in outs:   # the all-gather NCCL would do
            o = outs[r][0]
            o.t[o.off:o.off + o.nbytes].copy_(torch.from_numpy(gathered.view(np.uint8)))
    else:
        assert _same_bf16(staging.get().view(np.uint16), g_ref.view(np.uint16))
        raw = staging.get()
        nan_free = not np.isnan(np.concatenate([m.reshape(-1) for m in masters])).any()
        if nan_free:
            assert np.array_equal(raw, g_ref)   # every byte, pads and gaps included
    for r in outs:
        F.allgather_bucket(ctxs[r], buckets[r], staging.ptr, flags=L.WAIT)
        for o, f in zip(outs[r], fulls_ref):
            assert _same_bf16(o.get(), f)
    return True


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_toy_mlp_master_allgather(world):
    masters = [param_tensor(p, "f32", 40 + i) for i, p in enumerate(toy_mlp())]
    assert sim_master_allgather(masters, world)


@pytest.mark.parametrize("seed", range(8))
def test_random_shapes_master_allgather(seed):
    rng = np.random.Generator(np.random.Philox(1000 + seed))
    world = int(rng.integers(1, 9))
    k = int(rng.integers(1, 10))
    dims = [(int(rng.integers(1, 300)), int(rng.integers(1, 70))) for _ in range(k)]
    masters = [rng.standard_normal(d, dtype=np.float32) for d in dims]
    assert sim_master_allgather(masters, world, 1 if seed % 3 == 0 else 16)


def test_direct_gather_master():
    # one unpadded parameter: K1 rounds the own rows straight into the full param
    m = np.random.Generator(np.random.Philox(9)).standard_normal((64, 256), dtype=np.float32)
    assert sim_master_allgather([m], 4)


def test_device_rounding_all_tie_boundaries():
    """The device cast (cvt.rn.bf16x2.f32) against the oracle's RNE on every
    bf16 upper half with the low halves that decide rounding (exact, just
    below / at / just above the tie, maximal), plus the fp32 edge set:
    infinities, NaNs, subnormals, +-0, overflow to inf at the top."""
    hi = np.arange(65536, dtype=np.uint32) << 16
    lows = np.array([0x0000, 0x0001, 0x7FFF, 0x8000, 0x8001, 0xFFFF], dtype=np.uint32)
    pat = (hi[:, None] | lows[None, :]).reshape(-1)
    pat = np.concatenate([pat, EDGE_F32_BITS.astype(np.uint32)])
    pat = np.concatenate([pat, np.zeros((-pat.size) % 96, dtype=np.uint32)])
    m = pat.view(np.float32).reshape(-1, 96)
    assert sim_master_allgather([m, m[:37, :5].copy()], 3, ranks_out=[0, 1, 2])
    # and the scalar (unit-4) tail path: odd row lengths, unaligned segments
    assert sim_master_allgather([m[:, :7].copy(), m[:50, :3].copy()], 2, align=1, ranks_out=[0, 1])


def test_llama8b_block_master_allgather_full_size():
    specs = llama("8b", n_layers=1, with_embeddings=False)
    masters = [param_tensor(s, "f32", 70 + i) for i, s in enumerate(specs)]
    assert sim_master_allgather(masters, 8)


def test_master_flag_validated():
    ctx = F.Ctx(2, 0)
    a = DevArray(nbytes=4096, fill=0)
    with pytest.raises(Exception):
        F.Bucket(ctx, [(8, 8, 0)], shards=[a.ptr], param_dtype=L.FP32, grad_dtype=L.FP32,
                 flags=L.BUCKET_FP32_MASTER)
    with pytest.raises(Exception):
        F.Bucket(ctx, [(8, 8, 0)], shards=[a.ptr], param_dtype=L.BF16, grad_dtype=L.BF16,
                 flags=L.BUCKET_FP32_MASTER | L.BUCKET_SEGMENT_SHARDS)
