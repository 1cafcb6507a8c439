"""-m gpu: FSDP_BUCKET_GROUPED_AG -- the bucket's all-gather as one NCCL group
of per-member all-gathers straight into the full parameters (no staging, no
copy-in / copy-out).  Simulated ranks: each rank's ISSUE writes exactly its own
rows; world 1 with a real communicator: whole scheduled steps give the same
bytes as the flat bucketing, with no K3 launched."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from oracle.shard import shard
from workloads import llama
from workloads.data import param_tensor
from workloads.shapes import ParamSpec

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_grouped_issue_writes_own_rows(world):
    dims = [(8 * world, 24), (2 * world, 1), (world, 4096)]
    specs = [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]
    params = [param_tensor(s, "bf16", 40 + i) for i, s in enumerate(specs)]
    descs = [(d, r, 0) for d, r in dims]
    for r in range(world):
        ctx = F.Ctx(world, r)
        sh = [DevArray(shard(p, world, r)) for p in params]
        out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
        b = F.Bucket(ctx, descs, shards=[x.ptr for x in sh], fulls=[o.ptr for o in out], flags=L.BUCKET_GROUPED_AG)
        q = b.query()
        assert q["ag_grouped"] and q["kernel_bytes"][1] == 0          # no K3 copy-out
        st = DevArray(nbytes=world * b.ag_seg, fill=0xCD)
        F.allgather_bucket(ctx, b, st.ptr)
        torch.cuda.synchronize()
        assert np.all(st.get() == 0xCD)                                  # staging untouched
        for p, o in zip(params, out):
            c = p.shape[0] // world
            got = o.get()
            assert np.array_equal(bits(got[r * c:(r + 1) * c]), bits(p[r * c:(r + 1) * c]))
            mask = np.ones(p.shape[0], bool)
            mask[r * c:(r + 1) * c] = False
            assert np.all(got[mask].view(np.uint8) == 0x5A)                # nothing else written
        b.close()
        ctx.close()


def test_grouped_rejects_padded_members():
    ctx = F.Ctx(4, 0)
    a = DevArray(nbytes=1 << 16, fill=0)
    with pytest.raises(L.FsdpError):
        F.Bucket(ctx, [(10, 8, 0)], shards=[a.ptr], fulls=[a.ptr], flags=L.BUCKET_GROUPED_AG)   # 4 does not divide 10
    with pytest.raises(L.FsdpError):
        F.Bucket(ctx, [(8, 8, 0)], shards=[a.ptr], fulls=[a.ptr], flags=L.BUCKET_GROUPED_AG | L.BUCKET_FP32_MASTER)


def test_grouped_step_matches_flat_world1():
    specs = llama("8b", n_layers=1)
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    res = {}
    for mode in ("flat", "grouped"):
        ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
        fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
        st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=5, ag_grouped=mode == "grouped")
        cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
        rep = st.step(flags, cs.cuda_stream, ms.cuda_stream)
        torch.cuda.synchronize()
        res[mode] = ([t.cpu() for t in st.full_slots], st.gshard_buf.cpu(), rep, st.kernel_bytes())
        del st
        ctx.close()
    (f0, g0, r0, k0), (f1, g1, r1, k1) = res["flat"], res["grouped"]
    assert all(torch.equal(a, b) for a, b in zip(f0, f1)) and torch.equal(g0, g1)
    assert k1[L.OP_UNPACK] == 0 and k0[L.OP_UNPACK] > 0                 # no K3 in the grouped step
    assert r1["kernel_launches"] < r0["kernel_launches"]
