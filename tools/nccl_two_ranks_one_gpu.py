#!/usr/bin/env python
"""Probe: can two NCCL ranks share one GPU here?  (exploration tool)

Spawns 2 processes on cuda:0, builds an owned NCCL communicator through the
library, runs one bucketed all-gather and one reduce-scatter of the toy MLP
and compares with the oracle.  Prints PASS / FAIL / REFUSED.
"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, uid, q):
    try:
        import numpy as np
        import torch
        import paper_2411_00284_b200 as F
        from paper_2411_00284_b200 import _lib as L
        from oracle import collectives as OC
        from oracle.shard import shard
        from workloads import toy_mlp
        from workloads.data import grad_tensor, param_tensor
        torch.cuda.set_device(0)
        specs = toy_mlp()
        descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
        params = [param_tensor(p, "f32", 10 + i) for i, p in enumerate(specs)]
        grads = [[grad_tensor(p, "f32", 20, r) for p in specs] for r in range(world)]
        ctx = F.Ctx(world, rank, 0, nccl_uid=uid)
        sh = [torch.from_numpy(shard(p, world, rank)).cuda() for p in params]
        fu = [torch.empty(p.shape, device="cuda") for p in params]
        gd = [torch.from_numpy(g).cuda() for g in grads[rank]]
        gs = [torch.empty(s.shape, device="cuda") for s in sh]
        b = F.Bucket(ctx, descs, [x.data_ptr() for x in sh], [x.data_ptr() for x in fu],
                     [x.data_ptr() for x in gd], [x.data_ptr() for x in gs], L.FP32, L.FP32)
        ag = torch.zeros(world * b.ag_seg, dtype=torch.uint8, device="cuda")
        rs = torch.zeros(world * b.rs_seg, dtype=torch.uint8, device="cuda")
        cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
        F.allgather_bucket(ctx, b, ag.data_ptr(), cs.cuda_stream, ms.cuda_stream)
        F.reduce_scatter_bucket(ctx, b, rs.data_ptr(), cs.cuda_stream, ms.cuda_stream)
        torch.cuda.synchronize()
        ok = all(np.array_equal(f.cpu().numpy(), p) for f, p in zip(fu, params))
        _, _, shards_ref = OC.bucketed_reduce_scatter(grads, world, 16)
        ok_rs = all(np.array_equal(g.cpu().numpy().view(np.uint32), r.view(np.uint32))
                    for g, r in zip(gs, shards_ref[rank]))
        q.put((rank, "PASS" if ok and ok_rs else "FAIL ag=%s rs=%s" % (ok, ok_rs)))
        ctx.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "REFUSED/ERROR: %s\n%s" % (e, traceback.format_exc()[-1500:])))


def main():
    import multiprocessing as mp
    sys.path.insert(0, ROOT)
    import paper_2411_00284_b200 as F
    world = 2
    uid = F.nccl_get_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, uid, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for r in sorted(res):
        print("rank %d: %s" % r)


if __name__ == "__main__":
    main()
