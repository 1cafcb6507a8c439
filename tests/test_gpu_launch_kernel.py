"""-m gpu: fsdp_bucket_launch_kernel (the bench's back-to-back kernel timing)
launches each data kernel exactly as the step does -- same bytes as the
oracle's pack / copy-out, and nothing where the step skips the kernel."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from oracle.shard import shard
from workloads import toy_mlp
from workloads.data import grad_tensor, param_tensor

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


def test_launch_kernel_matches_the_oracle_and_the_step_skips():
    world, rank = 3, 1
    specs = toy_mlp()
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    params = [param_tensor(p, "bf16", 40 + i) for i, p in enumerate(specs)]
    grads = [grad_tensor(p, "bf16", 41, rank) for p in specs]
    ctx = F.Ctx(world, rank)
    full_src = [DevArray(p) for p in params]
    shards = []
    for (d, r, _), fs in zip(descs, full_src):
        c = -(-d // world)
        sd = DevArray(nbytes=c * r * 2, fill=0, dtype=np.uint16, shape=(c, r))
        F.shard(world, rank, (d, r, 0), L.BF16, fs.ptr, sd.ptr)
        shards.append(sd)
    fulls = [DevArray(nbytes=p.nbytes, fill=0xEE, dtype=np.uint16, shape=p.shape) for p in params]
    gfull = [DevArray(g) for g in grads]
    gsh = [DevArray(nbytes=-(-d // world) * r * 4, fill=0xCD, dtype=np.float32, shape=(-(-d // world), r))
           for d, r, _ in descs]
    b = F.Bucket(ctx, descs, shards=[x.ptr for x in shards], fulls=[x.ptr for x in fulls],
                 full_grads=[x.ptr for x in gfull], grad_shards=[x.ptr for x in gsh])
    s = torch.cuda.Stream()
    # K1: this rank's segment of the staging, zero pads (oracle ag_pack)
    ag_st = DevArray(nbytes=world * b.ag_seg, fill=0, dtype=np.uint8)
    assert F.bucket_launch_kernel(ctx, b, L.OP_PACK_AG, ag_st.ptr, s.cuda_stream) == 1
    s.synchronize()
    want = OC.ag_pack([shard(p, world, rank) for p in params], world, rank)
    got = ag_st.get()[rank * b.ag_seg:(rank + 1) * b.ag_seg]
    assert np.array_equal(got, want)
    # K3: from the oracle's gathered buffer into the full parameters
    segs = [OC.ag_pack([shard(p, world, q) for p in params], world, q) for q in range(world)]
    g = OC.all_gather(segs)
    ag_full = DevArray(g)
    assert F.bucket_launch_kernel(ctx, b, L.OP_UNPACK, ag_full.ptr, s.cuda_stream) == 1
    s.synchronize()
    for x, p in zip(fulls, params):
        assert np.array_equal(bits(x.get()), bits(p))
    # K4 into the RS staging (oracle rs_pack), then K6 out of this rank's segment
    rs_st = DevArray(nbytes=world * b.rs_seg, fill=0x77, dtype=np.float32)
    assert F.bucket_launch_kernel(ctx, b, L.OP_PACK_RS, rs_st.ptr, s.cuda_stream) == 1
    s.synchronize()
    packed = OC.rs_pack(grads, world)
    assert np.array_equal(bits(rs_st.get()), bits(packed))
    assert F.bucket_launch_kernel(ctx, b, L.OP_COPYOUT_RS, rs_st.ptr, s.cuda_stream) == 1
    s.synchronize()
    seg = packed[rank * b.rs_seg // 4:(rank + 1) * b.rs_seg // 4]
    for x, w in zip(gsh, OC.rs_copyout(seg, [p.shape for p in params], world)):
        assert np.array_equal(bits(x.get()), bits(w))
    with pytest.raises(L.FsdpError):
        F.bucket_launch_kernel(ctx, b, L.OP_AG, ag_st.ptr, s.cuda_stream)
    b.close()
    # segment-layout shard storage: the step runs no pack, so neither does this
    seg_store = DevArray(nbytes=b.ag_seg, fill=0, dtype=np.uint8)
    offs, _ = F.layout(descs, world, 2, 16)
    b2 = F.Bucket(ctx, descs, shards=[seg_store.ptr + o for o in offs], fulls=[x.ptr for x in fulls],
                  flags=L.BUCKET_SEGMENT_SHARDS)
    assert F.bucket_launch_kernel(ctx, b2, L.OP_PACK_AG, ag_st.ptr, s.cuda_stream) == 0
    b2.close()
    ctx.close()
