"""-m gpu: NCCL communicator settings (fsdp_ctx_create_config: min / max /
NVLS CTAs, CTA policy -- SURVEY §5, bounding NCCL's SM footprint against the
overlapped compute) and NCCL's own collective time estimate
(fsdp_nccl_estimate_ns, ncclGroupSimulateEnd), at world 1 with a real
communicator: a configured ctx runs a Llama-3-8B block step to the same
bytes as a default one; bad arguments are rejected before NCCL is touched."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

pytestmark = pytest.mark.gpu


def _step_bytes(ctx):
    specs = llama("8b", n_layers=1, with_embeddings=False)
    fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=21)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    rep = st.step(L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    # the gathered parameters of the (single) backward bucket, slot 0; the
    # rest of the slots is uninitialised memory
    used = H._carve([st.full_numel[j] * 2 for j in st.bwd[0].members])[1]
    out = (st.gshard_buf.clone(), [st.full_slots[0][:used].clone()])
    assert rep["collectives"] == len(st.fwd) + 2 * len(st.bwd)
    del st
    return out


def test_configured_comm_runs_the_same_step():
    ctx_d = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    want_g, want_f = _step_bytes(ctx_d)
    ctx_d.close()
    ctx_c = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id(),
                  nccl_config=dict(min_ctas=1, max_ctas=8, nvls_ctas=4, cta_policy=-1))
    got_g, got_f = _step_bytes(ctx_c)
    ctx_c.close()
    if not torch.equal(got_g, want_g):
        d = (got_g != want_g).nonzero().flatten()
        raise AssertionError("grad shards differ at %d bytes, first %s, of %d" % (d.numel(), d[:8].tolist(),
                                                                                 got_g.numel()))
    assert all(torch.equal(a, b) for a, b in zip(got_f, want_f))


def test_config_rejections():
    with pytest.raises(L.FsdpError):
        F.Ctx(1, 0, 0, nccl_config=dict(max_ctas=4))                     # no nccl_uid
    with pytest.raises(L.FsdpError):
        F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id(), nccl_config=dict(min_ctas=8, max_ctas=4))


def test_nccl_estimate():
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    block = 436224000    # one Llama-3-8B block, bf16 gathered bytes
    for op, n in ((L.OP_AG, block), (L.OP_RS, 2 * block)):
        try:
            assert ctx.nccl_estimate_ns(op, n) >= 0
        except L.FsdpError as e:       # NCCL models no time for a 1-rank communicator
            assert e.status == L.FSDP_ERR_UNSUPPORTED, e
    with pytest.raises(L.FsdpError):
        ctx.nccl_estimate_ns(L.OP_PACK_AG, block)       # not a collective
    with pytest.raises(L.FsdpError):
        ctx.nccl_estimate_ns(L.OP_RS, 6)                # not a multiple of world x 4 B
    ctx.close()
    lay = F.Ctx(1, 0, 0)
    with pytest.raises(L.FsdpError):
        lay.nccl_estimate_ns(L.OP_AG, block)            # layout-only ctx: no communicator
    lay.close()
