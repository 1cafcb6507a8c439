"""Workload harness: device memory (torch, plumbing only) for an FSDP rank and
the ABI calls that run its steps.

A ``RankState`` holds what one rank of an N-way FSDP job keeps in HBM
(layout):

  shards      param_dtype, every parameter's padded dim-0 shard, 256-B aligned
              sub-buffers of one allocation (resident: FSDP keeps only shards);
  fulls[2]    two slots of gathered full parameters, bucket b of a phase uses
              slot b % 2 (gathered parameters are released after use);
  grads[2]    two slots of full gradients (bf16, as backward produces them);
  gshards     fp32 gradient shards (reduce_dtype), resident;
  ag_st[2]    all-gather staging, N x the largest AG segment each;
  rs_st[2]    reduce-scatter staging, N x the largest RS segment each.

The plan, layout, schedule and every byte moved come from libfsdp_b200.so.
"""
import numpy as np
import torch

from . import fsdp as F
from . import _lib as L

ALIGN = 256


def _carve(sizes, align=ALIGN):
    offs, cur = [], 0
    for s in sizes:
        offs.append(cur)
        cur += (int(s) + align - 1) // align * align
    return offs, max(cur, align)


class RankState:
    def __init__(self, specs, world, rank, fwd_plan, bwd_plan, ctx, param_dtype=L.BF16,
                 device="cuda", seed=0, fill=True):
        self.specs, self.world, self.rank, self.ctx = specs, world, rank, ctx
        self.descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
        self.param_dtype = param_dtype
        ep = 2 if param_dtype == L.BF16 else 4
        self.ep = ep
        P = len(specs)
        c = [-(-p.dim0 // world) for p in specs]
        self.shard_numel = [c[j] * specs[j].row_numel for j in range(P)]
        self.full_numel = [p.dim0 * p.row_numel for p in specs]
        self.shard_offs, tot = _carve([n * ep for n in self.shard_numel])
        self.shard_buf = torch.empty(tot, dtype=torch.uint8, device=device)
        self.gs_offs, tot_g = _carve([n * 4 for n in self.shard_numel])
        self.gshard_buf = torch.zeros(tot_g, dtype=torch.uint8, device=device)
        # slots sized to the largest bucket of either phase
        buckets = list(fwd_plan) + list(bwd_plan)
        self.slot_bytes = max(_carve([self.full_numel[j] * ep for j in sorted(b)])[1] for b in buckets)
        self.gslot_bytes = max(_carve([self.full_numel[j] * 2 for j in sorted(b)])[1] for b in buckets)
        self.full_slots = [torch.empty(self.slot_bytes, dtype=torch.uint8, device=device) for _ in range(2)]
        self.grad_slots = [torch.empty(self.gslot_bytes, dtype=torch.uint8, device=device) for _ in range(2)]
        if fill:
            g = torch.Generator(device=device).manual_seed(seed)
            # N(0, 0.02) bf16 parameters and N(0, 1e-3) bf16 gradients (DESIGN.md input recipe)
            self._fill_normal(self.shard_buf, 0.02, g, param_dtype)
            for t in self.grad_slots:
                self._fill_normal(t, 1e-3, g, L.BF16)
        sp = self.shard_buf.data_ptr()
        gp = self.gshard_buf.data_ptr()
        self.fwd, self.bwd = [], []
        max_ag = max_rs = 0
        for phase, plan, out in ((0, fwd_plan, self.fwd), (1, bwd_plan, self.bwd)):
            for b, members in enumerate(plan):
                m = sorted(members)
                offs, _ = _carve([self.full_numel[j] * ep for j in m])
                goffs, _ = _carve([self.full_numel[j] * 2 for j in m])
                fbase = self.full_slots[b % 2].data_ptr()
                gbase = self.grad_slots[b % 2].data_ptr()
                bk = F.Bucket(ctx, [self.descs[j] for j in m],
                              shards=[sp + self.shard_offs[j] for j in m],
                              fulls=[fbase + o for o in offs],
                              full_grads=[gbase + o for o in goffs] if phase == 1 else None,
                              grad_shards=[gp + self.gs_offs[j] for j in m] if phase == 1 else None,
                              param_dtype=param_dtype, grad_dtype=L.BF16)
                bk.members = m
                out.append(bk)
                max_ag = max(max_ag, bk.ag_seg)
                max_rs = max(max_rs, bk.rs_seg)
        self.ag_st = [torch.zeros(world * max_ag + ALIGN, dtype=torch.uint8, device=device) for _ in range(2)]
        self.rs_st = [torch.zeros(world * max(max_rs, 16) + ALIGN, dtype=torch.uint8, device=device)
                      for _ in range(2)]

    @staticmethod
    def _fill_normal(buf, std, gen, dtype):
        if dtype == L.BF16:
            v = buf[: buf.numel() // 2 * 2].view(torch.bfloat16)
        else:
            v = buf[: buf.numel() // 4 * 4].view(torch.float32)
        v.normal_(0.0, std, generator=gen)

    def step(self, flags, compute, comm, proxy_fwd=None, proxy_bwd=None, ctas_per_sm=1, smem=0,
             want_log=False):
        return F.run_schedule(self.ctx, self.fwd, self.bwd,
                              ag_staging=(self.ag_st[0].data_ptr(), self.ag_st[1].data_ptr()),
                              rs_staging=(self.rs_st[0].data_ptr(), self.rs_st[1].data_ptr()),
                              compute=compute, comm=comm, flags=flags, proxy_iters_fwd=proxy_fwd,
                              proxy_iters_bwd=proxy_bwd, proxy_ctas_per_sm=ctas_per_sm,
                              proxy_smem_bytes=smem, want_log=want_log)

    # -------------------------------------------------------------- accounting
    def step_bytes(self):
        """Full (gathered / reduced) bucket bytes one step moves through its
        collectives, per rank: forward AG + backward AG in param dtype, RS in fp32."""
        ag = sum(self.world * b.ag_seg for b in self.fwd) + sum(self.world * b.ag_seg for b in self.bwd)
        rs = sum(self.world * b.rs_seg for b in self.bwd)
        return ag, rs

    def kernel_bytes(self):
        """Algorithmic HBM bytes per step of each data kernel:
        K1 read+write of the rank's shard, K3 read+write of the valid rows,
        K4 2 B read + 4 B write per gradient element, K6 4 + 4 B per shard element."""
        ep = self.ep
        k1 = k3 = k4 = k6 = 0
        for b in self.fwd + self.bwd:
            k1 += sum(2 * self.shard_numel[j] * ep for j in b.members)
            k3 += sum(2 * self.full_numel[j] * ep for j in b.members)
        for b in self.bwd:
            k4 += sum(6 * self.full_numel[j] for j in b.members)
            k6 += sum(8 * self.shard_numel[j] for j in b.members)
        return {L.OP_PACK_AG: k1, L.OP_UNPACK: k3, L.OP_PACK_RS: k4, L.OP_COPYOUT_RS: k6}


def plans_for(specs, world, mode, t_fwd=None, t_bwd=None, ag=(0, 0), rs=(0, 0), mem_max=0,
              param_dtype=L.BF16):
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    z = [0] * len(specs)
    fb, _ = F.plan_buckets(descs, world, t_fwd or z, ag, rs, mem_max, mode, L.PHASE_FWD, param_dtype)
    bb, _ = F.plan_buckets(descs, world, t_bwd or z, ag, rs, mem_max, mode, L.PHASE_BWD, param_dtype)
    return fb, bb


def calibrate_proxy(ctx, stream, ctas_per_sm=1, smem=0, probe_iters=200000):
    """ns per proxy iteration on this device, now (clocks vary): median of 5."""
    ns = F.proxy_calibrate(ctx, probe_iters, ctas_per_sm, smem, 5, stream)
    return ns / probe_iters


def proxy_iters(t_ns_per_bucket, ns_per_iter):
    return [int(round(t / ns_per_iter)) if t > 0 else 0 for t in t_ns_per_bucket]


def bucket_times(plan, t_per_param):
    return [sum(t_per_param[j] for j in b) for b in plan]


def np_dtype(dt):
    return np.uint16 if dt == L.BF16 else np.float32
