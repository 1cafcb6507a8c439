"""-m gpu: parity of the bench configuration itself (BASELINE configs[1] at
the launch configuration bench.py times): the full Llama-3-8B rank state at
layout world 8, one reordered step through fsdp_run_schedule, then checks on
sampled outputs the oracle computes one element at a time, and on properties
that hold at any size.

With a layout-only ctx (rank 0, no peers) the step's observable results are:
  * every gradient shard = this rank's own chunk, widened and times fl32(1/8)
    (the reduce-scatter has no other contributor), element-exact;
  * the full-parameter slots of the last two backward buckets hold this rank's
    shard in rows [0, c) and the (never written, zero-initialised) peer
    segments in rows [c, d).
"""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from oracle import bf16
from oracle.collectives import inv_world_f32
from workloads import llama

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nproc", [2, 3])
def test_bench_p2p_two_processes_one_gpu(nproc):
    """bench.py's multi-rank peer-memory path (IPC handle exchange over
    torch.distributed, epoch flags across processes) end to end with 2 ranks
    on one GPU (--same-device, time-sliced: the timings mean nothing)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", str(nproc), "--collective", "p2p", "--same-device", "--steps", "2", "--warmup", "1",
           "--layers", "1", "--no-e2e", "--exposure-tokens", "256"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == nproc and line["p2p_wait_timeouts"] == 0
    assert line["kernels"]["fsdp_p2p_allgather_kernel"]["launches_per_step"] == 2 * line["config"]["buckets_fwd"]
    # the N > 1 self-checks of the line: K8 / K9 across the two processes' IPC
    # mappings against the oracle (bit-exact), the isolated-block busbw, the
    # alpha / beta fit and the measured exposure variants all ran
    par = line["parity"]
    assert par["ok"] and par["ag"]["bit_exact"] and par["rs"]["bit_exact"], par
    assert par["ag"]["elements"] > 0 and par["rs"]["elements"] > 0
    if nproc == 3:      # 4096 / 14336 / 128256 rows split 3 ways: padded shards, pad rows +0.0
        assert par["rs"]["pad_rows"] > 0 and par["rs"]["pad_nonzero"] == 0
    assert line["value_kind"] == "bus" and line["busbw_block"]["ag_GBps"] > 0
    assert line["alpha_beta"]["source"].startswith("measured") and len(line["alpha_beta"]["rows"]) == 10
    assert len(line["exposure"]["variants"]) == 3
    for v in line["exposure"]["variants"].values():
        assert v["step_ms"] > 0 and v["compute_only_ms"] > 0
    nv = line["nvls_block"]     # K10 leg: measured and oracle-checked, or the platform's refusal
    assert "unavailable" in nv or nv["parity"]["ok"], nv


@pytest.mark.parametrize("collective", ["nccl", "p2p"])
def test_bench_distributed_path_world1(collective):
    """The N > 1 code path of bench.py (torchrun, process group, NCCL unique-id
    broadcast / IPC exchange, barriers, max over ranks, real collectives) at
    world 1 with a real communicator: what the driver's --gpus 2/4/8 runs use."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", "1", "--dist", "--collective", collective, "--steps", "3", "--warmup", "3",
           "--n-rank-legs-at-world1", "--exposure-tokens", "256"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["config"]["layout_world"] == 1 and line["value"] > 0
    assert line["value_kind"] == "hbm"       # world 1: no bus
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["parity"]["ok"], line["parity"]
    # the N > 1 legs' code with a real communicator (world 1: bus fractions are 0)
    assert line["busbw_block"]["ag_ms"] > 0 and line["alpha_beta"]["source"].startswith("measured")
    assert len(line["alpha_beta"]["rows"]) == 10 and len(line["exposure"]["variants"]) == 3
    nv = line["nvls_block"]
    assert "unavailable" in nv or nv["parity"]["ok"], nv
    if collective == "nccl":
        assert line["collectives"]["ag_ms_per_step"] > 0
        assert line["nccl_info"] is not None and any("NCCL" in x for x in line["nccl_info"]["lines"])
    else:
        assert line["p2p_wait_timeouts"] == 0


def test_gemm_compute_feeds_real_gradients():
    """fsdp_gemm_compute: the backward GEMM dW = dY^T X of every linear member
    writes the full gradient the reduce-scatter then averages; dW matches an
    fp32 torch reference within bf16 output rounding, and the gradient shards
    equal widen(dW rows of this rank) * fl32(1/N) bit-exactly."""
    world, T = 2, 256
    specs = llama("8b", n_layers=1, with_embeddings=False)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=9)
    gemm = st.setup_gemm(T)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    rep = st.step(L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream,
                  gemm=gemm)
    torch.cuda.synchronize()
    assert rep["op_ns"][L.OP_COMPUTE_B] > 0
    bk = st.bwd[0]
    goffs, _ = H._carve([st.full_numel[j] * 2 for j in bk.members])
    X = st.g_x.float().cpu()
    dY = st.g_dy.float().cpu()
    for j, go in zip(bk.members, goffs):
        p = specs[j]
        if p.row_numel == 1:
            continue
        out, inn = p.dim0, p.row_numel
        dW = st.grad_slots[0][go:go + 2 * out * inn].view(torch.bfloat16).view(out, inn)
        ref = dY[:T * out].view(T, out).t() @ X[:T * inn].view(T, inn)
        assert torch.allclose(dW.float().cpu(), ref, rtol=2e-2, atol=2e-2 * float(ref.abs().max())), p.name
        c = -(-out // world)
        gs = st.gshard_buf[st.gs_offs[j]:st.gs_offs[j] + 4 * c * inn].view(torch.float32).view(c, inn)
        want = (dW[:c].float() * 0.5).cpu()
        assert torch.equal(gs.cpu().view(torch.int32), want.view(torch.int32)), p.name


def test_host_io_step():
    """fsdp_host_io: the step loads every forward bucket's shards from pinned
    host memory before its all-gather and stores every backward bucket's
    gradient shards to host memory before the step ends."""
    from workloads import toy_mlp
    world = 2
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=5)
    h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8, pin_memory=True)
    g = torch.Generator().manual_seed(3)
    h_sh.copy_(torch.randint(0, 256, (h_sh.numel(),), dtype=torch.uint8, generator=g))
    # the gap bytes of the segment storage are zero by contract
    dev_before = st.shard_buf.cpu()
    gaps = torch.ones(st.shard_buf.numel(), dtype=torch.bool)
    for j, o in enumerate(st.shard_offs):
        gaps[o:o + st.shard_numel[j] * 2] = False
    h_sh[gaps] = dev_before[gaps]
    h_gs = torch.full((st.gshard_buf.numel(),), 0xAB, dtype=torch.uint8).pin_memory()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    io = st.host_io(h_sh, h_gs)
    assert all(io["fwd_host_shards"]) and all(io["bwd_host_grads"])
    st.step(L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, cs.cuda_stream, ms.cuda_stream, io=io)
    cs.synchronize()   # the step's compute stream waits for the D2H copies
    assert torch.equal(st.shard_buf.cpu(), h_sh)
    seg_bytes = torch.zeros(st.gshard_buf.numel(), dtype=torch.bool)
    for b in st.bwd:
        base = st.gs_offs[b.members[0]]
        seg_bytes[base:base + b.rs_seg] = True
    assert torch.equal(h_gs[seg_bytes], st.gshard_buf.cpu()[seg_bytes])
    del toy_mlp


def test_host_io_next_step_loads_after_last_reader():
    """Two host-I/O steps back to back with different host shards: the second
    step's H2D (which overlaps the first step's gradient D2H) must not land
    before the first step's last reader of the shard storage -- the first
    step's backward re-gathers see the first host buffer, the second step's
    the second."""
    world = 2
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=6)
    dev0 = st.shard_buf.cpu()
    gaps = torch.ones(st.shard_buf.numel(), dtype=torch.bool)
    for j, o in enumerate(st.shard_offs):
        gaps[o:o + st.shard_numel[j] * 2] = False
    hosts = []
    for seed in (11, 12):
        h = torch.randint(0, 256, (st.shard_buf.numel(),), dtype=torch.uint8,
                          generator=torch.Generator().manual_seed(seed))
        h[gaps] = dev0[gaps]
        hosts.append(h.pin_memory())
    h_gs = torch.zeros(st.gshard_buf.numel(), dtype=torch.uint8).pin_memory()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    st.step(flags, cs.cuda_stream, ms.cuda_stream, io=st.host_io(hosts[1], h_gs))   # a released event exists
    snaps = []
    for h in hosts:
        st.step(flags, cs.cuda_stream, ms.cuda_stream, io=st.host_io(h, h_gs))
        with torch.cuda.stream(cs):     # stream-ordered after this step, before the next one
            snaps.append([t.clone() for t in st.full_slots])
    cs.synchronize()
    # the last two backward buckets' gathered parameters: this rank's rows come
    # from the shards the step loaded
    for h, snap in zip(hosts, snaps):
        for b in st.bwd[-2:]:
            slot = snap[b.full_slot]
            for j, foff in zip(b.members, b.full_offs):
                sp = st.specs[j]
                c = -(-sp.dim0 // world)
                n = min(c, sp.dim0) * sp.row_numel * 2
                assert torch.equal(slot[foff:foff + n].cpu(), h[st.shard_offs[j]:st.shard_offs[j] + n])


def test_host_io_async_d2h_orders_the_next_gradient_writer():
    """fsdp_host_io.async_d2h: the step does not wait for its gradient D2H;
    the next step's gradient-shard writers do, bucket by bucket.  Two steps
    with different gradients, each D2H into its own host buffer: each buffer
    holds its own step's averaged shards (layout-only rank 0 at N = 2: this
    rank's rows widened x fl32(1/2))."""
    world = 2
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=8)
    h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8).pin_memory()
    h_sh.copy_(st.shard_buf.cpu())
    hosts = [torch.zeros(st.gshard_buf.numel(), dtype=torch.uint8).pin_memory() for _ in range(2)]
    cs, ms, d2h = torch.cuda.Stream(), torch.cuda.Stream(priority=-1), torch.cuda.Stream()
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    grads = []
    for k, h in enumerate(hosts):
        with torch.cuda.stream(cs):      # new gradients, stream-ordered between the steps
            if k:
                for t in st.grad_slots:
                    t.copy_(torch.roll(t, 2))   # whole bf16 values move: new gradients
            grads.append([t.clone() for t in st.grad_slots])
        st.step(flags, cs.cuda_stream, ms.cuda_stream,
                io=st.host_io(h_sh, h, d2h=d2h.cuda_stream, async_d2h=True))
    torch.cuda.synchronize()
    inv = inv_world_f32(world)
    for k, h in enumerate(hosts):
        for bk in st.bwd:
            slot = grads[k][bk.grad_slot]
            for j, goff in zip(bk.members, bk.grad_offs):
                n = st.shard_numel[j]
                c = n // st.specs[j].row_numel
                v = min(c, st.specs[j].dim0)
                g = slot[goff:goff + 2 * v * st.specs[j].row_numel].view(torch.int16).cpu().numpy().view(np.uint16)
                want = (bf16.widen(g) * inv).astype(np.float32)
                got = h[st.gs_offs[j]:st.gs_offs[j] + 4 * want.size].numpy().view(np.float32)
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (k, st.specs[j].name)
    del st
    ctx.close()


@pytest.mark.parametrize("graph", [False, True])
def test_llama8b_bench_step_sampled_parity(graph):
    """graph=True: the step as bench.py times it -- captured once into a CUDA
    graph (fsdp_step_graph) and replayed."""
    world = 8
    specs = llama("8b")
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=77)
    st.gshard_buf.fill_(0xAB)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    rep = st.step(flags, cs.cuda_stream, ms.cuda_stream, want_log=True)
    torch.cuda.synchronize()
    if graph:   # scrub the outputs, then replay the captured step
        sg = st.capture(flags, cs.cuda_stream, ms.cuda_stream)
        st.gshard_buf.fill_(0xCD)
        for t in st.full_slots:
            t.fill_(0xEE)
        torch.cuda.synchronize()
        sg.launch(cs.cuda_stream)
        torch.cuda.synchronize()
        sg.close()
    # 35 buckets per phase; shards live in segment layout, so no pack (K1):
    # forward unpack, backward unpack + grad pack + copy-out (no peers: K6 runs)
    assert st.zero_copy()["ag_buckets"] == 70
    assert rep["kernel_launches"] == 4 * 35, rep["kernel_launches"]
    assert rep["log_len"] == 5 * 35 + 9 * 35, rep["log_len"]

    _sampled_step_checks(st, specs, world)


def _sampled_step_checks(st, specs, world):
    """Rank 0 of a layout-only `world`-way job after one step: every gradient
    shard = this rank's chunk of its full gradient widened x fl32(1/N) (no
    other contributor; sampled elements, oracle O1 widen / O5 scale); the last
    two backward buckets' gathered parameters hold this rank's shard rows."""
    inv = inv_world_f32(world)
    rng = np.random.Generator(np.random.Philox(5))
    gs_u8 = st.gshard_buf
    for b, bk in enumerate(st.bwd):
        slot = st.grad_slots[b % st.n_grad_slots]
        offs, _ = H._carve([st.full_numel[j] * 2 for j in bk.members])
        for j, goff in zip(bk.members, offs):
            n = st.shard_numel[j]               # rank 0 owns rows [0, c): the first n elements
            idx = rng.integers(0, n, size=64)
            g = slot[goff:goff + 2 * st.full_numel[j]].view(torch.int16)[torch.from_numpy(idx).cuda()]
            want = bf16.widen(g.cpu().numpy().view(np.uint16)) * inv
            got = gs_u8[st.gs_offs[j]:st.gs_offs[j] + 4 * n].view(torch.float32)[torch.from_numpy(idx).cuda()]
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want.astype(np.float32).view(np.uint32)), \
                specs[j].name

    for b in (len(st.bwd) - 1, len(st.bwd) - 2):
        bk = st.bwd[b]
        offs, _ = H._carve([st.full_numel[j] * 2 for j in bk.members])
        slot = st.full_slots[st.full_slot_index(1, b)]
        for j, o in zip(bk.members, offs):
            full = slot[o:o + 2 * st.full_numel[j]]
            n = st.shard_numel[j]
            sh = st.shard_buf[st.shard_offs[j]:st.shard_offs[j] + 2 * n]
            assert torch.equal(full[:2 * n], sh), specs[j].name
            if not bk.query()["ag_direct"]:
                # peer rows come from the never-written (zero) staging segments; a
                # direct-gather bucket (emb / output / final norm) has no staging:
                # without a collective its peer rows are simply not written
                assert int(torch.count_nonzero(full[2 * n:])) == 0, specs[j].name


@pytest.mark.parametrize("cfg", ["70b_sizecap500MB", "405b_layer"])
def test_large_config_step_sampled_parity(cfg):
    """BASELINE configs[3] (Llama-3-70B shards at N = 8, a 500 MB size-cap
    plan: 17.6 GB of bf16 shards on this rank) and configs[4] (one Llama-3-405B
    layer as one 6.4 GB bucket, N = 8), one reordered step on rank 0 of a
    layout-only job, checked like the 8B bench step on sampled elements."""
    world = 8
    if cfg.startswith("70b"):
        specs = llama("70b")
        fplan, bplan = H.plans_for(specs, world, L.PLAN_SIZE_CAP, mem_max=500 * 10 ** 6)
    else:
        specs = llama("405b", n_layers=1)
        fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    ctx = F.Ctx(world, 0)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=78)
    st.gshard_buf.fill_(0xAB)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    st.step(L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    _sampled_step_checks(st, specs, world)
    del st
    torch.cuda.empty_cache()
    ctx.close()
