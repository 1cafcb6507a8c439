"""-m gpu: emulated collectives (fsdp_comm_emulation, kernel K11) -- the
measurement device behind bench.py's `emulated` exposure: on a layout-only
ctx of a simulated 8-way job every AG / RS becomes a comm-stream kernel that
lasts at least alpha + beta n; the step enqueues the collectives a real
communicator would; the zero-copy skips of the NCCL path apply; it captures
into a step graph; it is rejected where it cannot stand in."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

pytestmark = pytest.mark.gpu

LINK = (20000, 1215)
EM = dict(ag=LINK, rs=LINK, ctas=64)   # K11 now also writes the own slot of out-of-place gathers


def _state(world=8):
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=4)
    return ctx, st


def test_emulated_collectives_take_their_modelled_time():
    ctx, st = _state()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    want_ag = sum(F.comm_time_ns(st.world * b.ag_seg, LINK) for b in st.fwd + st.bwd)
    want_rs = sum(F.comm_time_ns(st.world * b.rs_seg, LINK) for b in st.bwd)
    # vanilla order: every collective runs alone (the compute stream waits on
    # it), so it lasts its modelled time
    st.step(0, cs.cuda_stream, ms.cuda_stream, emulate=EM)               # warm-up
    rep = st.step(L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, emulate=EM)
    torch.cuda.synchronize()
    assert rep["collectives"] == len(st.fwd) + 2 * len(st.bwd)
    got_ag, got_rs = rep["op_ns"][L.OP_AG], rep["op_ns"][L.OP_RS]
    assert want_ag <= got_ag <= 1.15 * want_ag + 100000, (got_ag, want_ag)
    assert want_rs <= got_rs <= 1.15 * want_rs + 100000, (got_rs, want_rs)
    # reordered: collectives overlap the copy kernels and never run shorter
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, emulate=EM)
    torch.cuda.synchronize()
    assert rep["op_ns"][L.OP_AG] >= want_ag and rep["op_ns"][L.OP_RS] >= want_rs
    # as with a communicator: segment-layout storage needs no RS read-out
    assert rep["op_ns"][L.OP_COPYOUT_RS] < rep["op_ns"][L.OP_PACK_RS] / 10
    # without emulation the layout-only step issues nothing
    rep0 = st.step(flags, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    assert rep0["collectives"] == 0
    del st
    ctx.close()


def test_emulated_step_captures_into_a_graph():
    ctx, st = _state()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    g = F.StepGraph(ctx, st.fwd, st.bwd, ag_staging=(st.ag_st[0].data_ptr(), st.ag_st[1].data_ptr()),
                    rs_staging=(st.rs_st[0].data_ptr(), st.rs_st[1].data_ptr()), compute=cs.cuda_stream,
                    comm=ms.cuda_stream, flags=flags, emulate=EM)
    assert g.collectives == len(st.fwd) + 2 * len(st.bwd)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.launch(cs.cuda_stream)
    a.record(cs)
    g.launch(cs.cuda_stream)
    b.record(cs)
    torch.cuda.synchronize()
    floor = sum(F.comm_time_ns(st.world * x.ag_seg, LINK) for x in st.fwd) / 1e6   # forward AGs are serial
    assert a.elapsed_time(b) >= floor
    g.close()
    del st
    ctx.close()


def test_emulated_gather_writes_this_ranks_rows():
    """An out-of-place gather (segment-layout shard storage) writes this rank's
    own slot too, as NCCL's does: after an emulated step the direct-gather
    buckets' full parameters (embedding, output) hold this rank's shard rows
    -- no stale rows under the compute."""
    ctx, st = _state()
    for t in st.full_slots:
        t.fill_(0xEE)
    torch.cuda.synchronize()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    st.step(0, cs.cuda_stream, ms.cuda_stream, emulate=EM)
    torch.cuda.synchronize()
    checked = 0
    for b in st.bwd[-2:]:
        if not b.query()["ag_direct"]:
            continue
        slot = st.full_slots[b.full_slot]
        for j, o in zip(b.members, b.full_offs):
            n = st.shard_numel[j] * 2
            assert torch.equal(slot[o:o + n], st.shard_buf[st.shard_offs[j]:st.shard_offs[j] + n])
            checked += 1
    assert checked >= 1
    del st
    ctx.close()


def test_emulation_rejections():
    specs = llama("8b", n_layers=1)
    fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=4)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    with pytest.raises(L.FsdpError):        # a real communicator is present
        st.step(0, cs.cuda_stream, ms.cuda_stream, emulate=EM)
    del st
    ctx.close()
    ctx2, st2 = _state()
    with pytest.raises(L.FsdpError):        # bad CTA count
        st2.step(0, cs.cuda_stream, ms.cuda_stream, emulate=dict(EM, ctas=0))
    del st2
    ctx2.close()


def test_paced_peer_kernels_keep_their_results_and_take_the_link_time():
    """FSDP_SCHED_P2P with fsdp_comm_emulation: K8 / K9 run on a grid of
    `ctas` CTAs held to alpha + beta n -- same bytes as without pacing, and
    every collective op lasts at least its modelled time."""
    specs = llama("8b", n_layers=1)
    world = 8
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=6)
    st.setup_p2p_simulated(seed=7)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_P2P
    st.step(flags, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    want_g = st.gshard_buf.clone()
    want_f = [t.clone() for t in st.full_slots]
    st.gshard_buf.fill_(0x33)
    torch.cuda.synchronize()
    rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, emulate=EM)
    torch.cuda.synchronize()
    assert int(st.p2p_err.item()) == 0
    assert torch.equal(st.gshard_buf, want_g)
    assert all(torch.equal(a, b) for a, b in zip(st.full_slots, want_f))
    ag = sum(F.comm_time_ns(world * b.ag_seg, LINK) for b in st.fwd + st.bwd)
    rs = sum(F.comm_time_ns(world * b.rs_seg // 2, LINK) for b in st.bwd)     # bf16 gradients on the wire
    assert rep["op_ns"][L.OP_AG] >= ag and rep["op_ns"][L.OP_RS] >= rs
    del st
    ctx.close()


def test_p2p_grid_cap_same_bytes():
    """fsdp_p2p_schedule.max_ctas (the N > 1 grid cap of K8 / K9) changes
    no result; a negative cap is rejected."""
    specs = llama("8b", n_layers=1)
    world = 8
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=8)
    st.setup_p2p_simulated(seed=9)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_P2P
    st.step(flags, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    want_g, want_f = st.gshard_buf.clone(), [t.clone() for t in st.full_slots]
    st.gshard_buf.fill_(0x21)
    torch.cuda.synchronize()
    st.p2p_max_ctas = H.emulation_ctas_p2p(world)
    st.step(flags, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    assert int(st.p2p_err.item()) == 0
    assert torch.equal(st.gshard_buf, want_g) and all(torch.equal(a, b) for a, b in zip(st.full_slots, want_f))
    st.p2p_max_ctas = -1
    with pytest.raises(L.FsdpError):
        st.step(flags, cs.cuda_stream, ms.cuda_stream)
    st.p2p_max_ctas = 0
    del st
    ctx.close()
