"""-m gpu: the compute hook (fsdp_compute_hook) drives real Llama-3 compute
(paper_2411_00284_b200/llama_compute.py) inside fsdp_run_schedule.  The
gradient shards the step leaves behind -- gathered parameters -> forward ->
re-gathered parameters -> backward -> full gradients -> K4 widen x 1/N ->
reduce-scatter -> copy-out -- equal plain torch autograd of the same model on
the full parameters (world 1: the shards are the parameters, 1/N = 1), for
the per-block plan and the greedy plan, layout-only and with a real NCCL
communicator; and an exception in the hook aborts the step and surfaces."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from paper_2411_00284_b200 import llama_compute as LC
from workloads import llama
from workloads.compute_model import per_param_compute_ns

pytestmark = pytest.mark.gpu

T = 256


def _state(plan, comm, layers=2):
    specs = llama("8b", n_layers=layers)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id()) if comm else F.Ctx(1, 0, 0)
    tf, tb = per_param_compute_ns(specs, T)
    link = (20000, 1500)
    fplan, bplan = H.plans_for(specs, 1, plan, tf, tb, link, link, int(2e9))
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=5)
    return specs, ctx, st


@pytest.mark.parametrize("plan,comm", [(L.PLAN_MANUAL, False), (L.PLAN_GREEDY, False), (L.PLAN_MANUAL, True)])
def test_hooked_llama_step_matches_autograd(plan, comm):
    specs, ctx, st = _state(plan, comm)
    lc = LC.LlamaCompute(st, T, seed=9)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    st.gshard_buf.fill_(0x5A)
    torch.cuda.synchronize()   # setup fills ran on torch's default stream; the step runs on cs
    rep = st.step(flags, cs.cuda_stream, ms.cuda_stream, hook=lc.hook)
    torch.cuda.synchronize()
    assert rep["op_count"][L.OP_COMPUTE_F] == len(st.fwd) and rep["op_count"][L.OP_COMPUTE_B] == len(st.bwd)
    loss = lc.state[0].item()
    # reference: the full parameters are this rank's shards (world 1)
    params = [st.shard_buf[st.shard_offs[j]:st.shard_offs[j] + 2 * n].view(torch.bfloat16).view(
        s.dim0, s.row_numel) if s.row_numel > 1 else
        st.shard_buf[st.shard_offs[j]:st.shard_offs[j] + 2 * n].view(torch.bfloat16)
        for j, (s, n) in enumerate(zip(specs, st.full_numel))]
    ref_loss, ref = LC.reference_grads(specs, params, lc.ops.tokens, lc.ops.targets)
    assert abs(loss - ref_loss.item()) <= 1e-3 * abs(ref_loss.item())
    for j, s in enumerate(specs):
        n = st.full_numel[j]
        g = st.gshard_buf[st.gs_offs[j]:st.gs_offs[j] + 4 * n].view(torch.float32)
        r = ref[j].float().reshape(-1)
        assert torch.isfinite(g).all(), s.name
        err = ((g - r).norm() / r.norm().clamp_min(1e-30)).item()
        assert err < 2e-2, (s.name, err)
    del lc, st
    ctx.close()


def test_hook_exception_aborts_step():
    specs, ctx, st = _state(L.PLAN_MANUAL, False, layers=1)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    calls = []

    def bad(phase, bucket, stream):
        calls.append((phase, bucket, stream))
        raise RuntimeError("model failed")
    with pytest.raises(RuntimeError, match="model failed"):
        st.step(0, cs.cuda_stream, ms.cuda_stream, hook=bad)
    torch.cuda.synchronize()
    assert calls == [(0, 0, cs.cuda_stream)]
    del st
    ctx.close()


def test_hook_called_in_schedule_order():
    specs, ctx, st = _state(L.PLAN_MANUAL, False, layers=1)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    calls = []
    rep = st.step(L.SCHED_REORDER, cs.cuda_stream, ms.cuda_stream, want_log=True,
                  hook=lambda p, b, s: calls.append((p, b)))
    torch.cuda.synchronize()
    want = [(ph, b) for ph, op, b, _s, _n, _t in rep["log"] if op in (L.OP_COMPUTE_F, L.OP_COMPUTE_B)]
    assert calls == want and len(calls) == len(st.fwd) + len(st.bwd)
    del st
    ctx.close()


def test_hooked_step_as_one_torch_graph():
    """The whole step -- gathers, Llama layers (torch ops through the hook),
    gradient pack, reduce-scatter, read-out -- captured into one CUDA graph
    (RankState.capture_with_torch) and replayed: same loss, same gradient
    shards as the eager step (within autograd's nondeterministic attention
    backward)."""
    specs, ctx, st = _state(L.PLAN_MANUAL, True)
    lc = LC.LlamaCompute(st, T, seed=9)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    for _ in range(2):     # warm-up (cuBLAS handles, allocator)
        st.step(flags, cs.cuda_stream, ms.cuda_stream, hook=lc.hook)
    torch.cuda.synchronize()
    want_loss = lc.state[0].clone()
    want = st.gshard_buf.clone()
    g = st.capture_with_torch(flags, cs, ms.cuda_stream, hook=lc.hook)
    st.gshard_buf.fill_(0x11)
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(lc.state[0], want_loss)
    got, ref = st.gshard_buf.view(torch.float32), want.view(torch.float32)
    assert torch.isfinite(got).all()
    assert ((got - ref).norm() / ref.norm()).item() < 1e-2
    del g, lc, st
    ctx.close()
