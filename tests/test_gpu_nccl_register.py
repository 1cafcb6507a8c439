"""-m gpu: NCCL buffer registration (fsdp_mem_alloc / fsdp_register_buffer).
Registration changes how NCCL moves bytes, never the bytes: a scheduled step
over ncclMemAlloc'd, registered buffers (local and symmetric-window) leaves
exactly the same full parameters and gradient shards as the same step over
plain torch allocations, at world 1 with a real communicator."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

pytestmark = pytest.mark.gpu


def _run(mode):
    specs = llama("8b", n_layers=1)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=7, nccl_register=mode)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        rep = st.step(L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    out = (st.gshard_buf[: st.gshard_buf.numel()].cpu().clone(),
           [t.cpu().clone() for t in st.full_slots], rep["collectives"])
    st.close_nccl_mem()
    del st
    ctx.close()
    return out


@pytest.mark.parametrize("mode", ["local", "symmetric"])
def test_registered_buffers_same_results(mode):
    g0, f0, c0 = _run(None)
    g1, f1, c1 = _run(mode)
    assert c0 == c1 and c0 > 0
    n = min(g0.numel(), g1.numel())
    assert torch.equal(g0[:n], g1[:n])
    for a, b in zip(f0, f1):
        m = min(a.numel(), b.numel())
        assert torch.equal(a[:m], b[:m])


def test_register_errors():
    lay = F.Ctx(2, 0)                    # layout-only: no communicator
    with pytest.raises(RuntimeError):
        F.mem_alloc(lay, 1 << 20)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    p = F.mem_alloc(ctx, 1 << 20)
    assert p % 4096 == 0
    with pytest.raises(RuntimeError):
        F.register_buffer(ctx, p + 16, 4096, L.REG_SYMMETRIC)   # unaligned window
    with pytest.raises(RuntimeError):
        F.register_buffer(ctx, p, 4096, 7)                       # unknown mode
    F.register_buffer(ctx, p, 1 << 20, L.REG_LOCAL)
    F.mem_free(ctx, p)                                           # deregisters first
    ctx.close()
