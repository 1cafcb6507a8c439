"""-m gpu: FSDP_SCHED_COPY_STREAM (pack / copy-out kernels on a third stream,
ordered by events) leaves exactly the bytes of the one-compute-stream step:
full parameters, full gradients and gradient shards bit-identical, with the
calibrated proxy and with real linear-layer GEMMs (which read the gathered
parameters and write the gradients the RS averages), eager and as a CUDA
graph, layout-only and with an NCCL world-1 communicator; the op log is the
same sequence with the copy ops on stream 2; a plan whose adjacent buckets
share full-parameter memory under prefetch is rejected."""
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama
from workloads.compute_model import per_param_compute_ns

pytestmark = pytest.mark.gpu

RF = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT


def _run(world, comm, compute, flags, graph=False, seed=21, tokens=256, mode=L.PLAN_MANUAL):
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0, 0, nccl_uid=F.nccl_get_unique_id()) if comm else F.Ctx(world, 0)
    tf, tb = per_param_compute_ns(specs, tokens)
    fplan, bplan = H.plans_for(specs, world, mode, tf, tb, (20000, 1215), (20000, 1215), 2 * 10 ** 9)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=seed)
    for t in st.full_slots:      # rows no kernel writes (peers' rows of direct-gather
        t.zero_()                # buckets on a layout-only rank) compare equal
    torch.cuda.synchronize()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    gemm = pf = pb = None
    if compute == "gemm":
        gemm = st.setup_gemm(tokens)
    else:
        nspi = H.calibrate_proxy(ctx, cs.cuda_stream)
        pf = H.proxy_iters(H.bucket_times(fplan, tf), nspi)
        pb = H.proxy_iters(H.bucket_times(bplan, tb), nspi)
    if graph:
        g = st.capture(flags, cs.cuda_stream, ms.cuda_stream, pf, pb, gemm=gemm)
        g.launch(cs.cuda_stream)
        g.close()
    else:
        rep = st.step(flags, cs.cuda_stream, ms.cuda_stream, pf, pb, gemm=gemm, want_log=True)
    torch.cuda.synchronize()
    out = ([t.clone() for t in st.full_slots], [t.clone() for t in st.grad_slots], st.gshard_buf.clone(),
           None if graph else rep["log"])
    del st
    ctx.close()
    return out


@pytest.mark.parametrize("compute", ["proxy", "gemm"])
@pytest.mark.parametrize("comm", [False, True])
@pytest.mark.parametrize("graph", [False, True])
def test_copy_stream_step_is_bit_identical(compute, comm, graph):
    world = 1 if comm else 8
    a = _run(world, comm, compute, RF, graph)
    b = _run(world, comm, compute, RF | L.SCHED_COPY_STREAM, graph)
    for x, y in zip(a[0], b[0]):
        assert torch.equal(x, y)
    for x, y in zip(a[1], b[1]):
        assert torch.equal(x, y)
    assert torch.equal(a[2], b[2])
    if not graph:
        la, lb = a[3], b[3]
        assert [e[:3] for e in la] == [e[:3] for e in lb]
        copy_ops = {L.OP_PACK_AG, L.OP_WAIT_AG, L.OP_UNPACK, L.OP_PACK_RS, L.OP_WAIT_RS, L.OP_COPYOUT_RS}
        for e in lb:
            assert e[3] == (1 if e[1] in (L.OP_AG, L.OP_RS) else 2 if e[1] in copy_ops else 0)


def test_copy_stream_vanilla_and_after_placement():
    for flags in (0, L.SCHED_REORDER, L.SCHED_REORDER | L.SCHED_BWD_AG_BEFORE_WAIT):
        a = _run(8, False, "gemm", flags)
        b = _run(8, False, "gemm", flags | L.SCHED_COPY_STREAM)
        assert torch.equal(a[2], b[2]) and all(torch.equal(x, y) for x, y in zip(a[1], b[1]))


def test_copy_stream_rejects_shared_adjacent_slots():
    world = 8
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=3)
    # rebind every bucket's full parameters into ONE slot: with prefetch the
    # next bucket's gather would overwrite what the current one computes on
    one = []
    for b in st.fwd + st.bwd:
        one.append(F.Bucket(ctx, [st.descs[j] for j in b.members],
                            shards=[st.shard_buf.data_ptr() + st.shard_offs[j] for j in b.members],
                            fulls=[st.full_slots[0].data_ptr() + o for o in b.full_offs],
                            full_grads=[st.grad_slots[0].data_ptr() + o for o in b.grad_offs],
                            grad_shards=[st.gshard_buf.data_ptr() + st.gs_offs[j] for j in b.members],
                            flags=L.BUCKET_SEGMENT_SHARDS | L.BUCKET_SEGMENT_GRAD_SHARDS))
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    kw = dict(ag_staging=(st.ag_st[0].data_ptr(), st.ag_st[1].data_ptr()),
              rs_staging=(st.rs_st[0].data_ptr(), st.rs_st[1].data_ptr()), compute=cs.cuda_stream,
              comm=ms.cuda_stream)
    nf = len(st.fwd)
    with pytest.raises(L.FsdpError):
        F.run_schedule(ctx, one[:nf], one[nf:], flags=RF | L.SCHED_COPY_STREAM, **kw)
    # vanilla (no prefetch) may share one slot
    F.run_schedule(ctx, one[:nf], one[nf:], flags=L.SCHED_COPY_STREAM, **kw)
    torch.cuda.synchronize()
    for b in one:
        b.close()
    del st
    ctx.close()


def test_copy_stream_with_host_io():
    """fsdp_host_io with the copy stream: the H2D'd shards feed the gathers
    and the gradient D2H follows the copy-outs, same host bytes as without."""
    world = 2
    specs = llama("8b", n_layers=2)
    outs = []
    for flags in (RF, RF | L.SCHED_COPY_STREAM):
        ctx = F.Ctx(world, 0)
        fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
        st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=12)
        h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8).pin_memory()
        h_sh.copy_(torch.randint(0, 256, (h_sh.numel(),), dtype=torch.uint8,
                                 generator=torch.Generator().manual_seed(4)))
        gaps = torch.ones(st.shard_buf.numel(), dtype=torch.bool)
        for j, o in enumerate(st.shard_offs):
            gaps[o:o + st.shard_numel[j] * 2] = False
        h_sh[gaps] = 0
        h_gs = torch.zeros(st.gshard_buf.numel(), dtype=torch.uint8).pin_memory()
        cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
        for t in st.full_slots:
            t.zero_()
        st.shard_buf[gaps.cuda()] = 0
        torch.cuda.synchronize()
        for _ in range(2):
            st.step(flags, cs.cuda_stream, ms.cuda_stream, io=st.host_io(h_sh, h_gs))
        cs.synchronize()
        outs.append((h_gs.clone(), [t.cpu() for t in st.full_slots]))
        assert torch.equal(st.shard_buf.cpu(), h_sh)
        del st
        ctx.close()
    assert torch.equal(outs[0][0], outs[1][0])
    for x, y in zip(outs[0][1], outs[1][1]):
        assert torch.equal(x, y)


@pytest.mark.parametrize("mode", [L.PLAN_PER_PARAM, L.PLAN_GREEDY])
def test_copy_stream_other_plans(mode):
    """Per-parameter buckets (many small copies) and Algorithm 1's greedy
    buckets (different forward / backward groupings): same bytes."""
    a = _run(8, False, "gemm", RF, mode=mode)
    b = _run(8, False, "gemm", RF | L.SCHED_COPY_STREAM, mode=mode)
    for x, y in zip(a[0], b[0]):
        assert torch.equal(x, y)
    assert torch.equal(a[2], b[2]) and all(torch.equal(x, y) for x, y in zip(a[1], b[1]))
