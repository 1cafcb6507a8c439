"""-m gpu: the NVLS (NVLink SHARP multicast) reduce-scatter read-out K10.

One GPU = a team of one device: the multicast object, the binding of this
GPU's physical staging, both mappings and the multimem.ld_reduce kernel run
for real, and the switch's "sum over the team" is the single member, so
grad_shards == the packed own segment == the oracle's world-1 reduce-scatter,
bit-exact (and with accumulation, held + that).  Skipped only where the
device reports no multicast / fabric-handle support."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from workloads import llama, toy_mlp
from workloads.data import grad_tensor

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


def _nvls(ctx, nbytes):
    try:
        m = F.Nvls(ctx, nbytes)
    except L.FsdpError as e:
        if getattr(e, "status", None) == L.FSDP_ERR_UNSUPPORTED:
            pytest.skip("NVLS multicast unavailable on this platform: %s" % e)
        raise
    return m


@pytest.mark.parametrize("specs_name", ["toy", "llama_block"])
@pytest.mark.parametrize("accumulate", [False, True])
def test_nvls_reduce_scatter_world1(specs_name, accumulate):
    specs = toy_mlp() if specs_name == "toy" else llama("8b", n_layers=1, with_embeddings=False)
    gdt = L.BF16
    ctx = F.Ctx(1, 0)
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    grads = [grad_tensor(p, "bf16", 33, 0) for p in specs]
    gd = [DevArray(g) for g in grads]
    rng = np.random.Generator(np.random.Philox(4))
    held = [rng.standard_normal((p.dim0, p.row_numel), dtype=np.float32) for p in specs]
    gs = [DevArray(h) for h in held]
    b = F.Bucket(ctx, descs, full_grads=[x.ptr for x in gd], grad_shards=[x.ptr for x in gs],
                 param_dtype=gdt, grad_dtype=gdt)
    b.set_grad_accumulation(accumulate)
    m = _nvls(ctx, b.rs_seg)
    uc, mc, n = m.bind()
    assert n >= b.rs_seg and uc % 16 == 0 and mc % 16 == 0
    F.reduce_scatter_bucket(ctx, b, uc, flags=L.ISSUE | L.NO_COLLECTIVE)   # K4 pack into the bound staging
    torch.cuda.synchronize()
    F.nvls_reduce_scatter_bucket(ctx, b, mc)                                   # K10 through the multicast mapping
    torch.cuda.synchronize()
    _, _, ref = OC.bucketed_reduce_scatter([grads], 1, 16)
    want = OC.accumulate_grad_shards(held, ref[0]) if accumulate else ref[0]
    for x, w in zip(gs, want):
        assert np.array_equal(bits(x.get()), bits(w))
    b.close()
    m.close()
    ctx.close()


def test_no_collective_flag_rules():
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    g = DevArray(nbytes=64 * 4, fill=0)
    gs = DevArray(nbytes=64 * 4, fill=0)
    b = F.Bucket(ctx, [(64, 1, 0)], full_grads=[g.ptr], grad_shards=[gs.ptr])
    st = DevArray(nbytes=b.rs_seg, fill=0)
    with pytest.raises(L.FsdpError):
        F.reduce_scatter_bucket(ctx, b, st.ptr, flags=L.WAIT | L.NO_COLLECTIVE)
    F.reduce_scatter_bucket(ctx, b, st.ptr, flags=L.ISSUE | L.NO_COLLECTIVE)   # pack only, no NCCL call
    torch.cuda.synchronize()
    b.close()
    ctx.close()
