"""World-size 2 and 3 CPU tests (gloo) of the N > 1 host logic.

Every rank (a separate process) asks the library for its shard rows
(fsdp_shard metadata), the bucket layout (fsdp_layout) and the plan
(fsdp_plan_buckets); the test then moves bytes exactly where those say --
segment `rank` of an N-segment buffer for the all-gather, segment q for chunk q
of the reduce-scatter -- and runs a REAL collective (gloo
all_gather_into_tensor / reduce_scatter_tensor(sum)) with the same in-place
offsets the library hands to NCCL.  Results must equal the oracle.  This pins
the cross-process contract of the N > 1 path (layout, offsets, plan
agreement) without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2411_00284_b200 as F
        from paper_2411_00284_b200 import _lib as L
        from oracle import collectives as OC
        from workloads import toy_mlp, llama
        from workloads.compute_model import per_param_compute_ns
        from workloads.data import grad_tensor, param_tensor

        specs = toy_mlp()
        descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
        params = [param_tensor(p, "f32", 10 + i) for i, p in enumerate(specs)]

        # ---- all-gather: pack own segment at the library's offsets, gloo AG, unpack
        offs, seg = F.layout(descs, world, 4, 16)
        mine = np.zeros(seg, dtype=np.uint8)
        for (d, r, _), o, p in zip(descs, offs, params):
            info = F.shard(world, rank, (d, r, 0), L.FP32)
            rows = p[info["row_begin"]:info["row_begin"] + info["valid_rows"]]
            b = np.ascontiguousarray(rows).reshape(-1).view(np.uint8)
            mine[o:o + b.size] = b            # pad rows / gaps stay zero
        out = torch.empty(world * seg, dtype=torch.uint8)
        dist.all_gather_into_tensor(out, torch.from_numpy(mine))
        g = out.numpy()
        g_ref, _ = OC.bucketed_all_gather(params, world, 16)
        assert np.array_equal(g, g_ref), "gathered buffer differs from the oracle"
        for (d, r, _), o, p in zip(descs, offs, params):
            full = np.zeros((d, r), dtype=np.float32)
            for q in range(world):
                info = F.shard(world, q, (d, r, 0), L.FP32)
                v = info["valid_rows"]
                full[info["row_begin"]:info["row_begin"] + v] = \
                    g[q * seg + o:q * seg + o + v * r * 4].view(np.float32).reshape(v, r)
            assert np.array_equal(full.view(np.uint32), p.view(np.uint32))

        # ---- reduce-scatter: chunk q of every member into segment q, gloo RS(sum)
        grads = [[grad_tensor(p, "f32", 20, q) for p in specs] for q in range(world)]
        roffs, rseg = F.layout(descs, world, 4, 16)
        inv = np.float32(1.0) / np.float32(world)
        buf = np.zeros(world * rseg // 4, dtype=np.float32)
        for (d, r, _), o, gj in zip(descs, roffs, grads[rank]):
            for q in range(world):
                info = F.shard(world, q, (d, r, 0), L.FP32)
                v = info["valid_rows"]
                lo = (q * rseg + o) // 4
                buf[lo:lo + v * r] = (gj[info["row_begin"]:info["row_begin"] + v].reshape(-1) * inv)
        ins_ref, outs_ref, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
        assert np.array_equal(buf.view(np.uint32), ins_ref[rank].view(np.uint32))
        res = torch.empty(rseg // 4, dtype=torch.float32)
        dist.reduce_scatter_tensor(res, torch.from_numpy(buf))
        # gloo's summation order is its own: within the G7 bound of the oracle
        ref = outs_ref[rank].astype(np.float64)
        scale = sum(np.abs(b_.astype(np.float64)[rank * rseg // 4:(rank + 1) * rseg // 4]) for b_ in ins_ref)
        assert np.all(np.abs(res.numpy().astype(np.float64) - ref) <= 1.01 * world * 2.0 ** -24 * scale + 1e-45)

        # ---- every rank computes the same plans (greedy, both phases)
        ls = llama("8b", n_layers=2)
        f, b_ = per_param_compute_ns(ls, 1024)
        ld = [(p.dim0, p.row_numel, p.module_id) for p in ls]
        plans = [F.plan_buckets(ld, world, t, (20000, 1500), (20000, 1500), 10**9, L.PLAN_GREEDY, ph,
                                want_trace=True) for ph, t in ((L.PHASE_FWD, f), (L.PHASE_BWD, b_))]
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        assert all(p == allp[0] for p in allp)
        # ... and the same searched plans (fsdp_plan_search, via harness.plans_search)
        from paper_2411_00284_b200 import harness as H
        searched = H.plans_search(ls, world, f, b_, (20000, 1500), (20000, 1500), 10**9)
        alls = [None] * world
        dist.all_gather_object(alls, searched)
        assert all(x == alls[0] for x in alls)
        # ... and the same dry-run step sequence, with the boundary bucket kept (G42)
        seq = F.run_schedule(None, None, None, n_fwd=len(searched[0]), n_bwd=len(searched[1]),
                             flags=L.SCHED_DRY_RUN | L.SCHED_REORDER | L.SCHED_KEEP_LAST_GATHERED)["log"]
        allq = [None] * world
        dist.all_gather_object(allq, seq)
        assert all(x == allq[0] for x in allq)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        errq.put("rank %d: %s\n%s" % (rank, e, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_n_rank_contract_over_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
