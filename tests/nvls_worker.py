"""torchrun worker of tests/test_gpu_multi.py: K10 (NVLS multimem.ld_reduce
reduce-scatter read-out) across N real GPUs, checked against the oracle.

Every rank packs its bf16 gradients (K4: widen x fl32(1/N)) into its unicast
mapping of one multicast object spanning the N GPUs; after a barrier K10 reads
this rank's segment through the multicast mapping, the NVSwitch summing the N
copies, into the fp32 gradient shards.  Expected: oracle O5 (rank-order sum)
within G7's bound, bit-exact at N <= 2.  Exit 3 (test skips) if the platform
refuses multicast objects; prints "NVLS OK" on rank 0 when every rank passed.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from oracle import bf16 as OB
    from oracle import collectives as OC
    from workloads import toy_mlp
    from workloads.data import grad_tensor
    from workloads.shapes import ParamSpec

    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    specs = toy_mlp() + [ParamSpec("w", 4096, 1024, 9), ParamSpec("n", 4099, 1, 10)]
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    grads = [[grad_tensor(p, "bf16", 33, r) for p in specs] for r in range(world)]
    gd = [torch.from_numpy(g.view(np.int16)).cuda() for g in grads[rank]]
    gs = [torch.zeros(-(-p.dim0 // world) * p.row_numel, dtype=torch.float32, device="cuda") for p in specs]
    ctx = F.Ctx(world, rank, local)
    b = F.Bucket(ctx, descs, full_grads=[x.data_ptr() for x in gd], grad_shards=[x.data_ptr() for x in gs],
                 param_dtype=L.BF16, grad_dtype=L.BF16)
    status = [None]
    m = None
    try:
        if rank == 0:
            m = F.Nvls(ctx, b.rs_seg)
            status[0] = m.handle
    except L.FsdpError as e:
        status[0] = ("unsupported" if getattr(e, "status", None) == L.FSDP_ERR_UNSUPPORTED else "error") + ": %s" % e
    dist.broadcast_object_list(status, src=0)
    if isinstance(status[0], str):
        if rank == 0:
            print(status[0], flush=True)
        dist.destroy_process_group()
        sys.exit(3 if status[0].startswith("unsupported") else 1)
    if rank != 0:
        m = F.Nvls(ctx, b.rs_seg, handle=status[0])
    dist.barrier()                       # every GPU added before any binding
    uc, mc, n = m.bind()
    dist.barrier()
    F.reduce_scatter_bucket(ctx, b, uc, flags=L.ISSUE | L.NO_COLLECTIVE)   # K4 into this GPU's unicast mapping
    torch.cuda.synchronize()
    dist.barrier()                       # every rank packed
    F.nvls_reduce_scatter_bucket(ctx, b, mc)                               # K10 through the multicast mapping
    torch.cuda.synchronize()
    dist.barrier()                       # every rank done reading before teardown
    _, _, ref = OC.bucketed_reduce_scatter(grads, world, 16)
    inv = float(OC.inv_world_f32(world))
    ok, worst = True, 0.0
    for j, p in enumerate(specs):
        c = -(-p.dim0 // world)
        got = gs[j].cpu().numpy().reshape(c, p.row_numel)
        want = ref[rank][j]
        scale = np.zeros(want.shape, dtype=np.float64)
        lo = rank * c
        for q in range(world):
            rows = OB.widen(grads[q][j][lo:lo + c]).astype(np.float64)
            scale[:rows.shape[0]] += np.abs(rows) * inv
        tol = 1.01 * world * 2.0 ** -24 * scale
        err = np.abs(got.astype(np.float64) - want.astype(np.float64))
        worst = max(worst, float(np.max(err / np.maximum(tol, 1e-300))))
        if world <= 2:
            ok &= bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))
    ok &= worst <= 1.0
    oks = [None] * world
    dist.all_gather_object(oks, (ok, worst))
    m.close()
    b.close()
    ctx.close()
    if rank == 0:
        print("NVLS %s worlds=%d worst_err_over_bound=%.3g" % ("OK" if all(o[0] for o in oks) else "FAIL", world,
                                                                max(o[1] for o in oks)), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all(o[0] for o in oks) else 1)


if __name__ == "__main__":
    main()
