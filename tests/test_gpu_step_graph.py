"""-m gpu: one step captured into a CUDA graph (fsdp_step_graph_*) replays to
exactly the bytes the eager fsdp_run_schedule produces -- layout-only and with
a real NCCL communicator (world 1), toy and one Llama-3-8B block -- and the
capture rejects what cannot be baked in."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

from .test_gpu_parity import _schedule_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world_comm", [False, True])
@pytest.mark.parametrize("flags", [0, L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT])
def test_graph_replay_matches_eager_toy(world_comm, flags):
    ctx, params, grads, fulls, gs, fwd, bwd, ag, rs = _schedule_case(world_comm)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    kw = dict(ag_staging=(ag[0].ptr, ag[1].ptr), rs_staging=(rs[0].ptr, rs[1].ptr), compute=cs.cuda_stream,
              comm=ms.cuda_stream, flags=flags)
    rep = F.run_schedule(ctx, fwd, bwd, **kw)
    torch.cuda.synchronize()
    want_f = [f.get().copy() for f in fulls]
    want_g = [g.get().copy() for g in gs]
    for x in fulls + gs:   # scrub the outputs, then replay
        x.t[x.off:x.off + x.nbytes].fill_(0x6B)
    torch.cuda.synchronize()   # the scrub (default stream) before the replay (cs)
    g = F.StepGraph(ctx, fwd, bwd, **kw)
    assert g.kernel_launches == rep["kernel_launches"] and g.collectives == rep["collectives"]
    for _ in range(3):
        g.launch(cs.cuda_stream)
    torch.cuda.synchronize()
    for a, b in zip(fulls, want_f):
        assert np.array_equal(a.get(), b)
    for a, b in zip(gs, want_g):
        assert np.array_equal(a.get(), b)
    g.close()
    ctx.close()


def test_graph_replay_matches_eager_llama_block():
    specs = llama("8b", n_layers=1)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=3)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    st.step(flags, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    want = st.gshard_buf.clone()
    wantf = [t.clone() for t in st.full_slots]
    st.gshard_buf.fill_(0x11)
    torch.cuda.synchronize()   # the scrub (default stream) before the replay (cs)
    g = st.capture(flags, cs.cuda_stream, ms.cuda_stream)
    g.launch(cs.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(st.gshard_buf, want)
    assert all(torch.equal(a, b) for a, b in zip(st.full_slots, wantf))
    g.close()
    del st
    ctx.close()


def test_graph_rejections():
    ctx, params, grads, fulls, gs, fwd, bwd, ag, rs = _schedule_case(False)
    cs = torch.cuda.Stream()
    kw = dict(ag_staging=(ag[0].ptr, ag[1].ptr), rs_staging=(rs[0].ptr, rs[1].ptr))
    with pytest.raises(L.FsdpError):
        F.StepGraph(ctx, fwd, bwd, compute=0, **kw)                                  # default stream
    with pytest.raises(L.FsdpError):
        F.StepGraph(ctx, fwd, bwd, compute=cs.cuda_stream, flags=L.SCHED_TIMING, **kw)
    with pytest.raises(L.FsdpError):
        F.StepGraph(ctx, fwd, bwd, compute=cs.cuda_stream, flags=L.SCHED_P2P, **kw)
    ctx.close()
