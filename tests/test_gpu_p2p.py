"""-m gpu parity of the peer-memory ("fused") collectives K8 / K9.

One process, N simulated ranks on one GPU: every rank's segment-layout shard
storage and full-gradient region is a real device buffer, and rank r's kernel
reads the others' buffers exactly as it would read NVLink-mapped peer memory.
K8 must reproduce all_gather(shard(p)) == p bit-exactly; K9 sums in rank order
in fp32 like the oracle, so it is bit-exact at EVERY world size (the NCCL path
is bit-exact only where the summation order cannot matter).
"""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import collectives as OC
from oracle.shard import shard
from workloads import llama, toy_mlp
from workloads.data import grad_tensor, param_tensor
from workloads.shapes import ParamSpec

from .gpu_util import DevArray, bits

pytestmark = pytest.mark.gpu


def _esize(dt):
    return 2 if dt == L.BF16 else 4


def _storage(params, world, rank, elem):
    descs = [(p.shape[0], p.shape[1], 0) for p in params]
    offs, seg = F.layout(descs, world, elem, 16)
    buf = np.full(seg, 0xEE, dtype=np.uint8)
    for p, o in zip(params, offs):
        b = shard(p, world, rank).reshape(-1).view(np.uint8)
        buf[o:o + b.size] = b
    return DevArray(buf), offs


def _grad_region(grads):
    """One rank's full gradients back to back at 256-B aligned offsets (the
    same offsets on every rank: a symmetric layout)."""
    offs, cur = [], 0
    for g in grads:
        offs.append(cur)
        cur += -(-g.nbytes // 256) * 256
    buf = np.zeros(cur, dtype=np.uint8)
    for g, o in zip(grads, offs):
        buf[o:o + g.nbytes] = g.reshape(-1).view(np.uint8)
    return DevArray(buf), offs


def run_p2p(params, grads_per_rank, world, dt, gdt):
    descs = [(p.shape[0], p.shape[1], 0) for p in params]
    stor = [_storage(params, world, r, _esize(dt)) for r in range(world)]
    regions = [_grad_region(grads_per_rank[r]) for r in range(world)]
    _, _, shards_ref = OC.bucketed_reduce_scatter(grads_per_rank, world, 16)
    for r in range(world):
        ctx = F.Ctx(world, r)
        out = [DevArray(nbytes=p.nbytes, fill=0x5A, dtype=p.dtype, shape=p.shape) for p in params]
        gs = [DevArray(nbytes=-(-d // world) * R * 4, fill=0x77, dtype=np.float32, shape=(-(-d // world), R))
              for d, R, _ in descs]
        sbuf, soffs = stor[r]
        gbuf, goffs = regions[r]
        b = F.Bucket(ctx, descs, shards=[sbuf.ptr + o for o in soffs], fulls=[o.ptr for o in out],
                     full_grads=[gbuf.ptr + o for o in goffs], grad_shards=[g.ptr for g in gs],
                     param_dtype=dt, grad_dtype=gdt, flags=L.BUCKET_SEGMENT_SHARDS)
        F.p2p_allgather_bucket(ctx, b, [stor[q][0].ptr for q in range(world)])
        F.p2p_reduce_scatter_bucket(ctx, b, [regions[q][0].ptr for q in range(world)])
        torch.cuda.synchronize()
        for o, p in zip(out, params):
            assert np.array_equal(bits(o.get()), bits(p))
        for j, g in enumerate(gs):
            assert np.array_equal(bits(g.get()), bits(shards_ref[r][j])), (r, j)
    return True


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("dt", [L.FP32, L.BF16])
def test_toy_p2p_bit_exact_any_world(world, dt):
    specs = toy_mlp()
    s = "f32" if dt == L.FP32 else "bf16"
    params = [param_tensor(p, s, 500 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, s, 501, r) for p in specs] for r in range(world)]
    assert run_p2p(params, grads, world, dt, dt)


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_p2p(seed):
    rng = np.random.Generator(np.random.Philox(2000 + seed))
    world = int(rng.integers(2, 9))
    dims = [(int(rng.integers(1, 200)), int(rng.integers(1, 40))) for _ in range(int(rng.integers(1, 9)))]
    specs = [ParamSpec("p%d" % i, d, r, 0) for i, (d, r) in enumerate(dims)]
    params = [param_tensor(p, "bf16", seed * 7 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, "bf16", seed, r) for p in specs] for r in range(world)]
    assert run_p2p(params, grads, world, L.BF16, L.BF16)


def test_llama8b_block_p2p_full_size():
    # BASELINE configs[1] bucket at N = 8: two of the eight ranks checked
    specs = llama("8b", n_layers=1, with_embeddings=False)
    world = 8
    params = [param_tensor(p, "bf16", 600 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, "bf16", 601, r) for p in specs] for r in range(world)]
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    stor = [_storage(params, world, r, 2) for r in range(world)]
    regions = [_grad_region(grads[r]) for r in range(world)]
    _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
    for r in (0, 5):
        ctx = F.Ctx(world, r)
        out = [torch.empty(p.size, dtype=torch.int16, device="cuda") for p in params]
        gs = [torch.empty(-(-d // world) * R, dtype=torch.float32, device="cuda") for d, R, _ in descs]
        b = F.Bucket(ctx, descs, shards=[stor[r][0].ptr + o for o in stor[r][1]], fulls=[o.data_ptr() for o in out],
                     full_grads=[regions[r][0].ptr + o for o in regions[r][1]], grad_shards=[g.data_ptr() for g in gs],
                     flags=L.BUCKET_SEGMENT_SHARDS)
        F.p2p_allgather_bucket(ctx, b, [s[0].ptr for s in stor])
        F.p2p_reduce_scatter_bucket(ctx, b, [g[0].ptr for g in regions])
        torch.cuda.synchronize()
        for o, p in zip(out, params):
            assert np.array_equal(o.cpu().numpy().view(np.uint16), p.reshape(-1))
        for j, g in enumerate(gs):
            assert np.array_equal(g.cpu().numpy().view(np.uint32), shards_ref[r][j].reshape(-1).view(np.uint32))


def test_signal_wait_and_timeout():
    world = 4
    ctxs = [F.Ctx(world, r) for r in range(world)]
    flags = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    # every rank q writes epoch 3 into slot q of every rank's flag array
    for q in range(world):
        F.p2p_signal(ctxs[q], [flags[r].data_ptr() + 8 * q for r in range(world)], 3, s.cuda_stream)
    for r in range(world):
        F.p2p_wait(ctxs[r], flags[r].data_ptr(), 3, 10**9, err.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert all(torch.equal(f, torch.full((world,), 3, dtype=torch.int64, device="cuda")) for f in flags)
    # an epoch nobody signals: the wait gives up after the timeout and flags the error
    F.p2p_wait(ctxs[0], flags[0].data_ptr(), 4, 2 * 10**6, err.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    assert int(err.item()) == 1


@pytest.mark.parametrize("flags", [L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, 0,
                                   L.SCHED_REORDER | L.SCHED_BWD_AG_BEFORE_WAIT])
def test_p2p_schedule_step_bit_exact(flags):
    """A whole step through fsdp_run_schedule with FSDP_SCHED_P2P for rank 1 of
    4 simulated ranks (peers' buffers hold the peers' real data): every full
    parameter gathered, every gradient shard equal to the oracle's RS."""
    world, rank = 4, 1
    specs = toy_mlp()
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    params = [param_tensor(p, "bf16", 800 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, "bf16", 801, q) for p in specs] for q in range(world)]
    fplan, _ = F.plan_buckets(descs, world, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_FWD)
    bplan, _ = F.plan_buckets(descs, world, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_BWD)
    ctx = F.Ctx(world, rank)
    # segment storage of every rank for every (forward) bucket; backward buckets have the same members
    seg_of = {}
    keep = []
    for members in fplan:
        m = tuple(sorted(members))
        bufs = []
        for q in range(world):
            sbuf, offs = _storage([params[j] for j in m], world, q, 2)
            bufs.append((sbuf, offs))
            keep.append(sbuf)
        seg_of[m] = bufs
    fulls = {}

    def bucket(members, phase, i):
        m = tuple(sorted(members))
        sbuf, offs = seg_of[m][rank]
        out = [DevArray(nbytes=params[j].nbytes, fill=0x5A, dtype=np.uint16, shape=params[j].shape) for j in m]
        fulls[(phase, i)] = (m, out)
        kw = {}
        if phase == 1:
            regions = [_grad_region([grads[q][j] for j in m]) for q in range(world)]
            gs = [DevArray(nbytes=-(-params[j].shape[0] // world) * params[j].shape[1] * 4, fill=0x77,
                           dtype=np.float32) for j in m]
            keep.extend(r[0] for r in regions)
            kw = dict(full_grads=[regions[rank][0].ptr + o for o in regions[rank][1]], grad_shards=[g.ptr for g in gs])
            fulls[(phase, i)] = (m, out, gs, [r[0].ptr for r in regions])
        return F.Bucket(ctx, [descs[j] for j in m], shards=[sbuf.ptr + o for o in offs], fulls=[o.ptr for o in out],
                        flags=L.BUCKET_SEGMENT_SHARDS, **kw)
    fwd = [bucket(m, 0, i) for i, m in enumerate(fplan)]
    bwd = [bucket(m, 1, i) for i, m in enumerate(bplan)]
    ag_peers = [[seg_of[tuple(sorted(m))][q][0].ptr for q in range(world)] for m in list(fplan) + list(bplan)]
    rs_peers = [fulls[(1, i)][3] for i in range(len(bplan))]
    ready = torch.full((world,), 2 ** 62, dtype=torch.int64, device="cuda")
    done = torch.full((world,), 2 ** 62, dtype=torch.int64, device="cuda")
    ready[rank] = 0
    done[rank] = 0
    sink = torch.zeros(2 * world, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    p2p = dict(ag_peers=ag_peers, rs_peers=rs_peers,
               ready_slots=[ready.data_ptr() + 8 * rank if q == rank else sink.data_ptr() + 8 * q for q in range(world)],
               done_slots=[done.data_ptr() + 8 * rank if q == rank else sink.data_ptr() + 8 * (world + q)
                           for q in range(world)],
               ready_flags=ready.data_ptr(), done_flags=done.data_ptr(), epoch_base=0, timeout_ns=5 * 10**9,
               error_flag=err.data_ptr())
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    rep = F.run_schedule(ctx, fwd, bwd, compute=cs.cuda_stream, comm=ms.cuda_stream,
                         flags=flags | L.SCHED_P2P | L.SCHED_TIMING, p2p=p2p)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert rep["collectives"] == len(fwd) + 2 * len(bwd)
    assert int(ready[rank].item()) == len(bwd) + 2 and int(done[rank].item()) == len(bwd) + 1
    _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
    for (phase, i), v in fulls.items():
        for j, o in zip(v[0], v[1]):
            assert np.array_equal(o.get(), params[j]), (phase, i, j)
        if phase == 1:
            for j, g in zip(v[0], v[2]):
                assert np.array_equal(g.get().view(np.uint32), shards_ref[rank][j].reshape(-1).view(np.uint32))


@pytest.mark.parametrize("mode", ["eager", "graph"])
@pytest.mark.parametrize("world", [2, 4])
def test_p2p_schedule_all_ranks_concurrently(world, mode):
    """Every rank of a `world`-way job runs its whole FSDP_SCHED_P2P step at the
    same time on one GPU (own streams per rank), reading the other ranks' real
    buffers and synchronising through the real epoch flags (no pre-set slots):
    two consecutive steps, every rank's full parameters and gradient shards
    bit-exact against the oracle, no wait times out.  mode "graph": every rank's
    step captured once (fsdp_step_graph) with a device epoch counter, and the
    two steps are graph replays whose epochs advance on the device."""
    specs = toy_mlp()
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    params = [param_tensor(p, "bf16", 900 + i) for i, p in enumerate(specs)]
    grads = [[grad_tensor(p, "bf16", 901, q) for p in specs] for q in range(world)]
    fplan, _ = F.plan_buckets(descs, world, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_FWD)
    bplan, _ = F.plan_buckets(descs, world, [0] * 8, (0, 0), (0, 0), 0, L.PLAN_MANUAL, L.PHASE_BWD)
    keep = []
    stor = {}      # (bucket members, rank) -> (DevArray, offsets)
    for members in fplan:
        m = tuple(sorted(members))
        for q in range(world):
            stor[(m, q)] = _storage([params[j] for j in m], world, q, 2)
    gregion = {}   # (bucket members, rank) -> (DevArray, offsets)  own region per backward bucket
    for members in bplan:
        m = tuple(sorted(members))
        for q in range(world):
            gregion[(m, q)] = _grad_region([grads[q][j] for j in m])
    ready = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
    done = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ranks = []
    for r in range(world):
        ctx = F.Ctx(world, r)
        outs, gss = {}, {}

        def bucket(members, phase, i):
            m = tuple(sorted(members))
            sbuf, offs = stor[(m, r)]
            out = [DevArray(nbytes=params[j].nbytes, fill=0x5A, dtype=np.uint16) for j in m]
            outs[(phase, i)] = (m, out)
            kw = {}
            if phase == 1:
                gbuf, goffs = gregion[(m, r)]
                gs = [DevArray(nbytes=-(-params[j].shape[0] // world) * params[j].shape[1] * 4, fill=0x77,
                               dtype=np.float32) for j in m]
                gss[i] = (m, gs)
                kw = dict(full_grads=[gbuf.ptr + o for o in goffs], grad_shards=[g.ptr for g in gs])
            return F.Bucket(ctx, [descs[j] for j in m], shards=[sbuf.ptr + o for o in offs],
                            fulls=[o.ptr for o in out], flags=L.BUCKET_SEGMENT_SHARDS, **kw)
        fwd = [bucket(m, 0, i) for i, m in enumerate(fplan)]
        bwd = [bucket(m, 1, i) for i, m in enumerate(bplan)]
        p2p = dict(ag_peers=[[stor[(tuple(sorted(m)), q)][0].ptr for q in range(world)] for m in list(fplan) + list(bplan)],
                   rs_peers=[[gregion[(tuple(sorted(m)), q)][0].ptr for q in range(world)] for m in bplan],
                   ready_slots=[ready[q].data_ptr() + 8 * r for q in range(world)],
                   done_slots=[done[q].data_ptr() + 8 * r for q in range(world)],
                   ready_flags=ready[r].data_ptr(), done_flags=done[r].data_ptr(), timeout_ns=20 * 10**9,
                   error_flag=err.data_ptr())
        ranks.append(dict(ctx=ctx, fwd=fwd, bwd=bwd, p2p=p2p, outs=outs, gss=gss,
                          cs=torch.cuda.Stream(), ms=torch.cuda.Stream(priority=-1)))
    torch.cuda.synchronize()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT | L.SCHED_P2P
    if mode == "graph":
        for rk in ranks:
            rk["ctr"] = torch.zeros(1, dtype=torch.int64, device="cuda")
            p = dict(rk["p2p"], epoch_base=0, epoch_counter=rk["ctr"].data_ptr())
            rk["graph"] = F.StepGraph(rk["ctx"], rk["fwd"], rk["bwd"], compute=rk["cs"].cuda_stream,
                                      comm=rk["ms"].cuda_stream, flags=flags, p2p=p)
    epoch = 0
    for _ in range(2):                       # two steps: epochs keep increasing
        for rk in ranks:                     # enqueue every rank; they run concurrently
            if mode == "graph":
                rk["graph"].launch(rk["cs"].cuda_stream)
            else:
                p = dict(rk["p2p"], epoch_base=epoch)
                F.run_schedule(rk["ctx"], rk["fwd"], rk["bwd"], compute=rk["cs"].cuda_stream,
                               comm=rk["ms"].cuda_stream, flags=flags, p2p=p, want_log=False)
        epoch += len(bplan) + 2
        torch.cuda.synchronize()
        assert int(err.item()) == 0, "an epoch wait timed out"
    if mode == "graph":
        assert all(int(rk["ctr"].item()) == 2 * (len(bplan) + 2) for rk in ranks)
        for rk in ranks:
            rk["graph"].close()
    _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
    for r, rk in enumerate(ranks):
        for (phase, i), (m, out) in rk["outs"].items():
            for j, o in zip(m, out):
                assert np.array_equal(o.get().reshape(-1), params[j].reshape(-1)), (r, phase, i, j)
        for i, (m, gs) in rk["gss"].items():
            for j, g in zip(m, gs):
                assert np.array_equal(g.get().view(np.uint32), shards_ref[r][j].reshape(-1).view(np.uint32)), (r, j)
    assert all(int(f[q].item()) == 2 * (len(bplan) + 2) for f in ready for q in range(world))
    del keep


def test_p2p_rejects_plain_storage():
    ctx = F.Ctx(2, 0)
    p = DevArray(np.zeros((64, 4), np.uint16))
    b = F.Bucket(ctx, [(8, 4, 0)], shards=[p.ptr], fulls=[p.ptr])
    with pytest.raises(F.FsdpError):
        F.p2p_allgather_bucket(ctx, b, [p.ptr, p.ptr])


def test_fused_sync_variant_schedule():
    """The FSDP_P2P_FUSED_SYNC=1 build (epoch wait + signal inside K9) runs the
    scheduled p2p steps bit-exactly too, including all ranks concurrently."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2411_00284_b200 import build as B
    lib = os.path.join(B.BUILD, "variants", "fusedsync", "libfsdp_b200.so")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(B.LIB):   # stale vs the main build
        lib = B.build(defines=["FSDP_P2P_FUSED_SYNC=1"], variant="fusedsync")
    env = dict(os.environ, FSDP_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "p2p_schedule and not graph",
                        os.path.join(root, "tests", "test_gpu_p2p.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_timed_out_epoch_wait_fails_the_step():
    """A peer that never signals: the epoch waits time out, the timed step
    returns an error instead of results computed without the peer (ADVICE
    round 1), and the harness's check raises."""
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    specs = llama("8b", n_layers=1, with_embeddings=False)
    world = 4
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=5)
    st.setup_p2p_simulated(seed=6)
    st.ready[2] = 0                      # simulated peer 2 never reports ready
    st.p2p_timeout_ns = 2_000_000        # 2 ms per wait
    torch.cuda.synchronize()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_P2P | L.SCHED_TIMING
    with pytest.raises(L.FsdpError):
        st.step(flags, cs.cuda_stream, ms.cuda_stream)
    with pytest.raises(RuntimeError):
        st.check_p2p()
    del st
    ctx.close()
