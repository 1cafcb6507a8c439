"""-m gpu: the peer-memory collectives across PROCESSES (world 2 and 3 on one
GPU, CUDA IPC mappings instead of NVLink peers).

Each rank process allocates its segment-layout shard storage, its
full-gradient region and its flag array with fsdp_ipc_alloc, fills them with
the library's K0 copy, publishes the IPC handles, opens its peers', then runs
the release/acquire epoch protocol: signal "ready" (epoch 1) into every peer's
flag slot, wait for all peers, K8 + K9 straight from peer memory, signal
"done" (epoch 2) and wait before freeing.  Results are bit-exact against the
oracle (K9's rank-order fp32 sum matches the oracle's at any world size).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _worker(rank, world, q_out, q_in, q_res):
    sys.path.insert(0, ROOT)
    try:
        import numpy as np
        import torch
        import paper_2411_00284_b200 as F
        from paper_2411_00284_b200 import _lib as L
        from oracle import collectives as OC
        from workloads import toy_mlp
        from workloads.data import grad_tensor, param_tensor

        torch.cuda.set_device(0)
        specs = toy_mlp()
        descs = [(p.dim0, p.row_numel, 0) for p in specs]
        params = [param_tensor(p, "bf16", 700 + i) for i, p in enumerate(specs)]
        grads = [[grad_tensor(p, "bf16", 701, r) for p in specs] for r in range(world)]
        ctx = F.Ctx(world, rank)
        s = torch.cuda.Stream()

        def dcopy(dst_ptr, t):  # device copy through the library's K0 (world 1 = whole tensor)
            n = t.numel() * t.element_size()
            F.shard(1, 0, (n // 2, 1, 0), L.BF16, t.data_ptr(), dst_ptr)

        offs, seg = F.layout(descs, world, 2, 16)
        stor, stor_h = F.ipc_alloc(seg)
        for d, p, o in zip(descs, params, offs):
            full = torch.from_numpy(p.view(np.int16).copy()).cuda()
            F.shard(world, rank, d, L.BF16, full.data_ptr(), stor + o)
        goffs, cur = [], 0
        for g in grads[rank]:
            goffs.append(cur)
            cur += -(-g.nbytes // 256) * 256
        greg, greg_h = F.ipc_alloc(cur)
        for g, o in zip(grads[rank], goffs):
            dcopy(greg + o, torch.from_numpy(g.view(np.int16).copy()).cuda())
        flags, flags_h = F.ipc_alloc(256)
        dcopy(flags, torch.zeros(64, dtype=torch.int16, device="cuda"))
        torch.cuda.synchronize()

        q_out.put((rank, stor_h, greg_h, flags_h))
        handles = q_in.get(timeout=120)           # [(rank, stor_h, greg_h, flags_h)] for all ranks
        peers = {}
        opened = []
        for r, sh, gh, fh in handles:
            if r == rank:
                peers[r] = (stor, greg, flags)
            else:
                t = (F.ipc_open(sh), F.ipc_open(gh), F.ipc_open(fh))
                opened += list(t)
                peers[r] = t
        out = [torch.empty(p.size, dtype=torch.int16, device="cuda") for p in params]
        gs = [torch.empty(-(-d // world) * R, dtype=torch.float32, device="cuda") for d, R, _ in descs]
        b = F.Bucket(ctx, descs, shards=[stor + o for o in offs], fulls=[o.data_ptr() for o in out],
                     full_grads=[greg + o for o in goffs], grad_shards=[g.data_ptr() for g in gs],
                     flags=L.BUCKET_SEGMENT_SHARDS)
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        slots = [peers[q][2] + 8 * rank for q in range(world)]
        F.p2p_signal(ctx, slots, 1, s.cuda_stream)                       # my data is ready
        F.p2p_wait(ctx, flags, 1, 30 * 10**9, err.data_ptr(), s.cuda_stream)
        F.p2p_allgather_bucket(ctx, b, [peers[q][0] for q in range(world)], s.cuda_stream)
        F.p2p_reduce_scatter_bucket(ctx, b, [peers[q][1] for q in range(world)], s.cuda_stream)
        F.p2p_signal(ctx, slots, 2, s.cuda_stream)                       # done reading peers
        F.p2p_wait(ctx, flags, 2, 30 * 10**9, err.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        assert int(err.item()) == 0, "epoch wait timed out"
        ok_ag = all(np.array_equal(o.cpu().numpy().view(np.uint16), p.reshape(-1)) for o, p in zip(out, params))
        _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
        ok_rs = all(np.array_equal(g.cpu().numpy().view(np.uint32), r.reshape(-1).view(np.uint32))
                    for g, r in zip(gs, shards_ref[rank]))
        b.close()
        for p in opened:
            F.ipc_close(p)
        for p in (stor, greg, flags):
            F.ipc_free(p)
        q_res.put((rank, "ok" if ok_ag and ok_rs else "mismatch ag=%s rs=%s" % (ok_ag, ok_rs)))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q_res.put((rank, "error: %s\n%s" % (e, traceback.format_exc()[-2000:])))


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_collectives_across_processes(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_out, q_res = ctx.Queue(), ctx.Queue()
    q_in = [ctx.Queue() for _ in range(world)]
    ps = [ctx.Process(target=_worker, args=(r, world, q_out, q_in[r], q_res)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        handles = sorted(q_out.get(timeout=240) for _ in range(world))
        for q in q_in:
            q.put(handles)
        res = dict(q_res.get(timeout=240) for _ in range(world))
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(v == "ok" for v in res.values()), res
