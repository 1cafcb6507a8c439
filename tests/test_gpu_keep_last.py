"""-m gpu: FSDP_SCHED_KEEP_LAST_GATHERED (reading G42; FSDP2's reshard-after-
forward off for the boundary module): the first backward bucket reuses the
last forward bucket's gathered parameters -- the step's results are the same
bytes as with the re-gather, with one collective and four logged ops fewer;
on a layout-only ctx, with a real NCCL communicator (world 1) and on the
peer-memory path; a backward bucket that does not bind the same parameters is
rejected."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

pytestmark = pytest.mark.gpu


def _run(st, flags):
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    st.gshard_buf.fill_(0x3C)
    torch.cuda.synchronize()
    rep = st.step(flags, cs.cuda_stream, ms.cuda_stream, want_log=True)
    torch.cuda.synchronize()
    if getattr(st, "p2p_err", None) is not None:
        assert int(st.p2p_err.item()) == 0
    return rep, st.gshard_buf.clone(), [t.clone() for t in st.full_slots]


@pytest.mark.parametrize("mode", ["layout", "nccl", "p2p"])
def test_keep_last_same_bytes(mode):
    world = 1 if mode == "nccl" else 8
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0, 0, nccl_uid=F.nccl_get_unique_id()) if mode == "nccl" else F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=12)
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    if mode == "p2p":
        st.setup_p2p_simulated(seed=13)
        flags |= L.SCHED_P2P
    rep0, g0, f0 = _run(st, flags)
    rep1, g1, f1 = _run(st, flags | L.SCHED_KEEP_LAST_GATHERED)
    assert torch.equal(g0, g1)
    assert all(torch.equal(a, b) for a, b in zip(f0, f1))
    assert rep1["log_len"] == rep0["log_len"] - 4
    if mode != "layout":
        assert rep1["collectives"] == rep0["collectives"] - 1
    del st
    ctx.close()


def test_keep_last_rejects_a_different_bucket():
    specs = llama("8b", n_layers=1)
    P = len(specs)
    ctx = F.Ctx(8, 0)
    fplan = [[j] for j in range(P - 2)] + [[P - 2, P - 1]]    # last forward bucket: final norm + output
    bplan = [[P - 1], [P - 2]] + [[j] for j in range(P - 3, -1, -1)]
    st = H.RankState(specs, 8, 0, fplan, bplan, ctx, seed=3)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    with pytest.raises(L.FsdpError):
        st.step(L.SCHED_REORDER | L.SCHED_KEEP_LAST_GATHERED, cs.cuda_stream, ms.cuda_stream)
    del st
    ctx.close()
