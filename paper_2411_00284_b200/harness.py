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
                 device="cuda", seed=0, fill=True, segment_storage=True, ipc=False, nccl_register=None,
                 ag_grouped=False, grad_slots=2, windows=False):
        # ipc=True: the buffers peers read in the peer-memory path (shard
        # storage, gradient slots) come from fsdp_ipc_alloc so that other
        # processes can map them (setup_p2p_ipc).
        # nccl_register="local" / "symmetric": every buffer an NCCL collective
        # sends from or receives into (shard storage, full-parameter slots, AG /
        # RS staging, gradient-shard storage) comes from fsdp_mem_alloc and is
        # registered with the ctx's communicator (fsdp_register_buffer).
        # windows=True: those buffers instead come from fsdp_mem_alloc and are
        # registered as NCCL symmetric windows (a collective, same sizes and
        # order on every rank); setup_p2p_windows then takes the peer tables
        # from NCCL (fsdp_window_peer_pointers) -- no IPC handles.
        self.ipc_handles = {}
        self._ipc_ptrs = []
        self._nccl_ptrs = []
        self.win_bases = {}
        self.windows = windows
        reg_mode = {None: None, "none": None, "local": L.REG_LOCAL, "symmetric": L.REG_SYMMETRIC}[nccl_register]
        dev_index = torch.device(device).index or torch.cuda.current_device()

        def nccl_buf(nbytes, zero=False, mode=None):
            from .dlpack_view import uint8_view
            nbytes = max(int(nbytes), 4096)
            ptr = F.mem_alloc(ctx, nbytes)
            self._nccl_ptrs.append(ptr)
            F.register_buffer(ctx, ptr, nbytes, reg_mode if mode is None else mode)
            t = uint8_view(ptr, nbytes, dev_index)
            if zero:
                t.zero_()
            return t

        def alloc(name, nbytes, zero=False, collective=False, peer=False):
            # collective: an NCCL send / receive buffer; peer: read by peers (K8 / K9)
            if windows and peer:
                t = nccl_buf(nbytes, zero, L.REG_SYMMETRIC)
                self.win_bases[name] = t.data_ptr()
                return t
            if collective and reg_mode is not None:
                return nccl_buf(nbytes, zero)
            if not (ipc and peer):
                return (torch.zeros if zero else torch.empty)(nbytes, dtype=torch.uint8, device=device)
            from .dlpack_view import uint8_view
            ptr, handle = F.ipc_alloc(nbytes)
            self._ipc_ptrs.append(ptr)
            self.ipc_handles[name] = handle
            t = uint8_view(ptr, nbytes, torch.device(device).index or torch.cuda.current_device())
            if zero:
                t.zero_()
            return t
        self.specs, self.world, self.rank, self.ctx = specs, world, rank, ctx
        self.descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
        self.param_dtype = param_dtype
        ep = 2 if param_dtype == L.BF16 else 4
        self.ep = ep
        # shard rows / valid rows from the library (fsdp_shard metadata, G1)
        info = [F.shard(world, rank, d, param_dtype) for d in self.descs]
        c = [x["shard_rows"] for x in info]
        self.valid_rows = [x["valid_rows"] for x in info]
        self.shard_numel = [x["shard_numel"] for x in info]
        self.full_numel = [p.dim0 * p.row_numel for p in specs]
        if segment_storage:
            # shards stored in the forward plan's AG segment layout, gradient
            # shards in the backward plan's RS segment layout: the library
            # detects it (fsdp_bucket_create) and drops the pack (K1) and,
            # with a communicator, the copy-out (K6)
            self.shard_offs, tot = self._segment_offsets(fwd_plan, ep)
            self.gs_offs, tot_g = self._segment_offsets(bwd_plan, 4)
        else:
            self.shard_offs, tot = _carve([n * ep for n in self.shard_numel])
            self.gs_offs, tot_g = _carve([n * 4 for n in self.shard_numel])
        self.shard_buf = alloc("shards", tot, zero=True, collective=True, peer=True)
        self.gshard_buf = alloc("gshards", tot_g, zero=True, collective=True)
        # slots sized to the largest bucket of either phase
        buckets = list(fwd_plan) + list(bwd_plan)
        self.slot_bytes = max(_carve([self.full_numel[j] * ep for j in sorted(b)])[1] for b in buckets)
        self.gslot_bytes = max(_carve([self.full_numel[j] * 2 for j in sorted(b)])[1] for b in buckets)
        self.full_slots = [alloc("fulls%d" % i, self.slot_bytes, collective=True) for i in range(2)]
        # backward bucket b produces its full gradients in slot b % n_grad_slots
        self.n_grad_slots = int(grad_slots)
        self.grad_slots = [alloc("grads%d" % i, self.gslot_bytes, peer=True) for i in range(self.n_grad_slots)]
        if fill:
            g = torch.Generator(device=device).manual_seed(seed)
            # N(0, 0.02) bf16 parameters and N(0, 1e-3) bf16 gradients (DESIGN.md input recipe)
            self._fill_normal(self.shard_buf, 0.02, g, param_dtype)
            for t in self.grad_slots:
                self._fill_normal(t, 1e-3, g, L.BF16)
            # shard padding rows hold +0 (fsdp_shard contract)
            for j, p in enumerate(specs):
                v = self.valid_rows[j]
                if v < c[j]:
                    o = self.shard_offs[j] + v * p.row_numel * ep
                    self.shard_buf[o:self.shard_offs[j] + self.shard_numel[j] * ep].zero_()
        sp = self.shard_buf.data_ptr()
        gp = self.gshard_buf.data_ptr()
        self.fwd, self.bwd = [], []
        # backward bucket b gathers into full-parameter slot (b + off) % 2 with off
        # chosen so that backward bucket 0 uses the last forward bucket's slot:
        # with FSDP_SCHED_KEEP_LAST_GATHERED (G42) it reuses those parameters
        self._bwd_slot_off = (len(fwd_plan) - 1) % 2 if len(fwd_plan) else 0
        max_ag = max_rs = 0
        for phase, plan, out in ((0, fwd_plan, self.fwd), (1, bwd_plan, self.bwd)):
            for b, members in enumerate(plan):
                m = sorted(members)
                offs, _ = _carve([self.full_numel[j] * ep for j in m])
                goffs, _ = _carve([self.full_numel[j] * 2 for j in m])
                flags = 0
                if self._follows_segment(m, self.shard_offs, ep):
                    flags |= L.BUCKET_SEGMENT_SHARDS
                if phase == 1 and self._follows_segment(m, self.gs_offs, 4):
                    flags |= L.BUCKET_SEGMENT_GRAD_SHARDS
                if ag_grouped and all(specs[j].dim0 % world == 0 for j in m):
                    flags |= L.BUCKET_GROUPED_AG    # per-member AGs in one NCCL group, no copies
                fbase = self.full_slots[self.full_slot_index(phase, b)].data_ptr()
                gbase = self.grad_slots[b % self.n_grad_slots].data_ptr()
                bk = F.Bucket(ctx, [self.descs[j] for j in m],
                              shards=[sp + self.shard_offs[j] for j in m],
                              fulls=[fbase + o for o in offs],
                              full_grads=[gbase + o for o in goffs] if phase == 1 else None,
                              grad_shards=[gp + self.gs_offs[j] for j in m] if phase == 1 else None,
                              param_dtype=param_dtype, grad_dtype=L.BF16, flags=flags)
                bk.members = m
                bk.full_offs = offs          # member byte offsets in its full-parameter slot
                bk.grad_offs = goffs         # member byte offsets in its full-gradient slot
                bk.full_slot = self.full_slot_index(phase, b)
                bk.grad_slot = b % self.n_grad_slots if phase == 1 else None
                out.append(bk)
                max_ag = max(max_ag, bk.ag_seg)
                max_rs = max(max_rs, bk.rs_seg)
        self.ag_st = [alloc("ag_st%d" % i, world * max_ag + ALIGN, zero=True, collective=True) for i in range(2)]
        self.rs_st = [alloc("rs_st%d" % i, world * max(max_rs, 16) + ALIGN, zero=True, collective=True)
                      for i in range(2)]
        if torch.device(device).type == "cuda":
            # fills / zeroing ran on torch's current stream; steps run on the caller's streams
            torch.cuda.synchronize(device)

    def full_slot_index(self, phase, b):
        """Full-parameter slot of bucket b of a phase (forward b % 2; backward
        shifted so that its bucket 0 shares the last forward bucket's slot)."""
        return b % 2 if phase == 0 else (b + self._bwd_slot_off) % 2

    def _segment_offsets(self, plan, elem_bytes):
        """Per-parameter byte offsets placing each bucket's members at the
        library's segment offsets (fsdp_layout), buckets 256-B aligned."""
        offs = [None] * len(self.specs)
        cur = 0
        for members in plan:
            m = sorted(members)
            moffs, seg = F.layout([self.descs[j] for j in m], self.world, elem_bytes, 16)
            for j, o in zip(m, moffs):
                offs[j] = cur + o
            cur += (seg + ALIGN - 1) // ALIGN * ALIGN
        return offs, max(cur, ALIGN)

    def _follows_segment(self, members, offs, elem_bytes):
        moffs, _ = F.layout([self.descs[j] for j in members], self.world, elem_bytes, 16)
        return all(offs[j] - offs[members[0]] == o for j, o in zip(members, moffs)) and offs[members[0]] % 16 == 0

    @staticmethod
    def _fill_normal(buf, std, gen, dtype):
        if dtype == L.BF16:
            v = buf[: buf.numel() // 2 * 2].view(torch.bfloat16)
        else:
            v = buf[: buf.numel() // 4 * 4].view(torch.float32)
        v.normal_(0.0, std, generator=gen)

    # ------------------------------------------------------ peer-memory path
    def setup_p2p_simulated(self, seed=1, fill=True):
        """Peer-memory (FSDP_SCHED_P2P) state for this rank with the other
        world - 1 ranks SIMULATED on the same GPU: their shard storage and
        gradient slots are separate device buffers (same layout as ours, as on
        real peers), read by K8 / K9 exactly as NVLink-mapped peer memory would
        be; their flag slots are pre-set far ahead so the epoch waits only
        track this rank's own signals."""
        W, r = self.world, self.rank
        g = torch.Generator(device=self.shard_buf.device).manual_seed(seed)
        self.peer_shards, self.peer_grads = [], []
        for q in range(W):
            if q == r:
                self.peer_shards.append(self.shard_buf)
                self.peer_grads.append(self.grad_slots)
                continue
            sb = torch.zeros_like(self.shard_buf)
            gs = [torch.empty_like(t) for t in self.grad_slots]
            if fill:
                self._fill_normal(sb, 0.02, g, self.param_dtype)
                for t in gs:
                    self._fill_normal(t, 1e-3, g, L.BF16)
            self.peer_shards.append(sb)
            self.peer_grads.append(gs)
        dev = self.shard_buf.device
        self.ready = torch.full((W,), 2 ** 62, dtype=torch.int64, device=dev)
        self.done = torch.full((W,), 2 ** 62, dtype=torch.int64, device=dev)
        self.ready[r] = 0
        self.done[r] = 0
        self.sink = torch.zeros(2 * W, dtype=torch.int64, device=dev)   # simulated peers' slots
        self.p2p_err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ready_slots = [self.ready.data_ptr() + 8 * r if q == r else self.sink.data_ptr() + 8 * q
                            for q in range(W)]
        self.done_slots = [self.done.data_ptr() + 8 * r if q == r else self.sink.data_ptr() + 8 * (W + q)
                           for q in range(W)]
        self._p2p_tables([t.data_ptr() for t in self.peer_shards],
                         [[t.data_ptr() for t in gs] for gs in self.peer_grads])

    def setup_p2p_ipc(self, exchange):
        """Peer-memory state across processes: ``exchange(obj)`` returns the
        list of every rank's obj (e.g. torch.distributed.all_gather_object).
        Requires RankState(..., ipc=True).  Shards, gradient slots and the flag
        arrays of every peer are mapped with fsdp_ipc_open."""
        W, r = self.world, self.rank
        flags_ptr, flags_h = F.ipc_alloc(16 * W)
        self._ipc_ptrs.append(flags_ptr)
        from .dlpack_view import uint8_view
        fl = uint8_view(flags_ptr, 16 * W, torch.cuda.current_device())
        fl.zero_()
        torch.cuda.synchronize()
        self.ready = fl[:8 * W].view(torch.int64)
        self.done = fl[8 * W:].view(torch.int64)
        self.p2p_err = torch.zeros(1, dtype=torch.int32, device=self.shard_buf.device)
        mine = dict(rank=r, shards=self.ipc_handles["shards"], flags=flags_h,
                    grads=[self.ipc_handles["grads%d" % i] for i in range(self.n_grad_slots)])
        allh = sorted(exchange(mine), key=lambda d: d["rank"])
        self._opened = []
        shard_base, grad_base, flag_base = [], [], []
        for q, h in enumerate(allh):
            if q == r:
                shard_base.append(self.shard_buf.data_ptr())
                grad_base.append([t.data_ptr() for t in self.grad_slots])
                flag_base.append(flags_ptr)
                continue
            ptrs = [F.ipc_open(h["shards"]), F.ipc_open(h["flags"])] + [F.ipc_open(g) for g in h["grads"]]
            self._opened += ptrs
            shard_base.append(ptrs[0])
            flag_base.append(ptrs[1])
            grad_base.append(ptrs[2:])
        self.ready_slots = [flag_base[q] + 8 * r for q in range(W)]
        self.done_slots = [flag_base[q] + 8 * W + 8 * r for q in range(W)]
        self._p2p_tables(shard_base, grad_base)

    def setup_p2p_windows(self):
        """Peer-memory state from NCCL symmetric windows (RankState(...,
        windows=True); the ctx has a communicator): peers' shard storage,
        gradient slots and flag arrays through fsdp_window_peer_pointers.  The
        flag array is registered here -- a collective: every rank calls this."""
        from .dlpack_view import uint8_view
        W, r = self.world, self.rank
        nb = max(16 * W, 4096)
        fptr = F.mem_alloc(self.ctx, nb)
        self._nccl_ptrs.append(fptr)
        F.register_buffer(self.ctx, fptr, nb, L.REG_SYMMETRIC)
        fl = uint8_view(fptr, nb, torch.cuda.current_device())
        fl.zero_()
        torch.cuda.synchronize()
        self.ready = fl[:8 * W].view(torch.int64)
        self.done = fl[8 * W:16 * W].view(torch.int64)
        self.p2p_err = torch.zeros(1, dtype=torch.int32, device=self.shard_buf.device)
        shard_base = F.window_peer_pointers(self.ctx, self.win_bases["shards"])
        flag_base = F.window_peer_pointers(self.ctx, fptr)
        gslots = [F.window_peer_pointers(self.ctx, self.win_bases["grads%d" % i]) for i in range(self.n_grad_slots)]
        grad_base = [[gslots[i][q] for i in range(self.n_grad_slots)] for q in range(W)]
        # (NCCL maps every rank's window, this rank's too, into one flat VA
        # range: peer_ptrs[rank] aliases the buffer at a different address)
        self.ready_slots = [flag_base[q] + 8 * r for q in range(W)]
        self.done_slots = [flag_base[q] + 8 * W + 8 * r for q in range(W)]
        self._p2p_tables(shard_base, grad_base)

    def close_nccl_mem(self):
        """Releases the fsdp_mem_alloc buffers (and their registrations); call
        before the ctx is destroyed.  The torch views must not be used after."""
        for p in self._nccl_ptrs:
            F.mem_free(self.ctx, p)
        self._nccl_ptrs = []

    def close_ipc(self):
        """Closes this rank's mappings of the peers' buffers.  Its own exported
        buffers stay until free_ipc -- call that only after EVERY rank has
        closed its mappings (a barrier between the two)."""
        for p in getattr(self, "_opened", []):
            F.ipc_close(p)
        self._opened = []

    def free_ipc(self):
        """Frees this rank's IPC-exported buffers (shard storage, gradient
        slots, flags); their torch views must not be used afterwards."""
        for p in self._ipc_ptrs:
            F.ipc_free(p)
        self._ipc_ptrs = []

    def _p2p_tables(self, shard_base, grad_base):
        W = self.world
        self.ag_peers = [[shard_base[q] + self.shard_offs[b.members[0]] for q in range(W)] for b in self.fwd + self.bwd]
        self.rs_peers = [[grad_base[q][i % self.n_grad_slots] for q in range(W)] for i, b in enumerate(self.bwd)]
        self.epoch = 0   # fixed epoch_base: the epochs advance on the device (epoch_counter)
        self.epoch_ctr = torch.zeros(1, dtype=torch.int64, device=self.shard_buf.device)

    def p2p_schedule(self, timeout_ns=None):
        if timeout_ns is None:
            timeout_ns = getattr(self, "p2p_timeout_ns", 10 ** 10)
        return dict(ag_peers=self.ag_peers, rs_peers=self.rs_peers, ready_slots=self.ready_slots,
                    done_slots=self.done_slots, ready_flags=self.ready.data_ptr(), done_flags=self.done.data_ptr(),
                    epoch_base=self.epoch, timeout_ns=timeout_ns, error_flag=self.p2p_err.data_ptr(),
                    epoch_counter=self.epoch_ctr.data_ptr(), max_ctas=getattr(self, "p2p_max_ctas", 0),
                    grad_slots=self.n_grad_slots)

    def check_p2p(self):
        """Raise if a peer-memory epoch wait timed out since setup: a kernel then
        went ahead without its peers and the step's results are invalid
        (include/fsdp.h, fsdp_p2p_schedule.error_flag).  Synchronises."""
        err = getattr(self, "p2p_err", None)
        if err is not None and int(err.item()) != 0:
            raise RuntimeError("peer-memory epoch wait timed out: the step's results are invalid")

    def p2p_bytes(self):
        """Algorithmic bytes per step of K8 (peer AG, both phases) and K9 (peer RS)."""
        k8 = sum(b.query()["p2p_bytes"][0] for b in self.fwd + self.bwd)
        k9 = sum(b.query()["p2p_bytes"][1] for b in self.bwd)
        return k8, k9

    def host_io(self, host_shards, host_gshards, h2d=0, d2h=0, async_d2h=False):
        """fsdp_host_io for pinned host mirrors laid out like shard_buf /
        gshard_buf: forward bucket k streams in from host_shards at its segment
        offset, backward bucket j streams its gradient shards out to host_gshards."""
        hs, hg = host_shards.data_ptr(), host_gshards.data_ptr()
        fwd = [hs + self.shard_offs[b.members[0]] if b.query()["ag_zero_copy"] else 0 for b in self.fwd]
        bwd = [hg + self.gs_offs[b.members[0]] if b.query()["rs_zero_copy"] else 0 for b in self.bwd]
        return dict(fwd_host_shards=fwd, bwd_host_grads=bwd, h2d=h2d, d2h=d2h, async_d2h=async_d2h)

    def setup_gemm(self, tokens, seed=7, workspace_bytes=64 << 20):
        """Linear-layer compute (fsdp_gemm_compute) at `tokens` tokens: bf16
        activations X [T, max in] ~ N(0, 1) and upstream gradients dY [T, max
        out] ~ N(0, 1e-2), a [T, max(in, out)] scratch, a cuBLASLt workspace."""
        lin = [p for p in self.specs if p.row_numel > 1]
        max_in = max(p.row_numel for p in lin)
        max_out = max(p.dim0 for p in lin)
        dev = self.shard_buf.device
        g = torch.Generator(device=dev).manual_seed(seed)
        self.g_x = torch.empty(tokens * max_in, dtype=torch.bfloat16, device=dev).normal_(0, 1, generator=g)
        self.g_dy = torch.empty(tokens * max_out, dtype=torch.bfloat16, device=dev).normal_(0, 1e-2, generator=g)
        self.g_y = torch.empty(tokens * max(max_in, max_out), dtype=torch.bfloat16, device=dev)
        self.g_ws = torch.empty(workspace_bytes, dtype=torch.uint8, device=dev)
        self.gemm = dict(tokens=tokens, x=self.g_x.data_ptr(), dy=self.g_dy.data_ptr(), y=self.g_y.data_ptr(),
                         workspace=self.g_ws.data_ptr(), workspace_bytes=workspace_bytes)
        # FLOPs per step: 2 T out in forward, 4 T out in backward, per linear member of every bucket
        self.gemm_flops = sum(2 * tokens * self.specs[j].dim0 * self.specs[j].row_numel
                              for b in self.fwd for j in b.members if self.specs[j].row_numel > 1)
        self.gemm_flops += sum(4 * tokens * self.specs[j].dim0 * self.specs[j].row_numel
                               for b in self.bwd for j in b.members if self.specs[j].row_numel > 1)
        return self.gemm

    def step(self, flags, compute, comm, proxy_fwd=None, proxy_bwd=None, ctas_per_sm=1, smem=0,
             want_log=False, io=None, gemm=None, hook=None, emulate=None):
        p2p = None
        if flags & L.SCHED_P2P:
            p2p = self.p2p_schedule()   # the device epoch counter advances inside the step
        return F.run_schedule(self.ctx, self.fwd, self.bwd,
                              ag_staging=(self.ag_st[0].data_ptr(), self.ag_st[1].data_ptr()),
                              rs_staging=(self.rs_st[0].data_ptr(), self.rs_st[1].data_ptr()),
                              compute=compute, comm=comm, flags=flags, proxy_iters_fwd=proxy_fwd,
                              proxy_iters_bwd=proxy_bwd, proxy_ctas_per_sm=ctas_per_sm,
                              proxy_smem_bytes=smem, want_log=want_log, p2p=p2p, io=io, gemm=gemm, hook=hook,
                              emulate=emulate)

    def capture(self, flags, compute, comm, proxy_fwd=None, proxy_bwd=None, ctas_per_sm=1, smem=0, gemm=None):
        """The same step captured into a CUDA graph (fsdp_step_graph_create)."""
        p2p = self.p2p_schedule() if flags & L.SCHED_P2P else None
        return F.StepGraph(self.ctx, self.fwd, self.bwd, p2p=p2p,
                           ag_staging=(self.ag_st[0].data_ptr(), self.ag_st[1].data_ptr()),
                           rs_staging=(self.rs_st[0].data_ptr(), self.rs_st[1].data_ptr()),
                           compute=compute, comm=comm, flags=flags, proxy_iters_fwd=proxy_fwd,
                           proxy_iters_bwd=proxy_bwd, proxy_ctas_per_sm=ctas_per_sm, proxy_smem_bytes=smem,
                           gemm=gemm)

    def capture_with_torch(self, flags, compute_stream, comm, proxy_fwd=None, proxy_bwd=None, ctas_per_sm=1,
                           smem=0, gemm=None, hook=None):
        """The step -- library kernels and collectives AND a PyTorch compute
        hook's ops -- captured into one CUDA graph by torch (torch.cuda.graph
        on `compute_stream`, a torch.cuda.Stream, with torch's private memory
        pool for the hook's tensors; the comm stream joins through the
        library's events).  fsdp_step_graph cannot hold a hook that allocates
        through torch; this can.  Returns the torch.cuda.CUDAGraph (replay()
        on any stream)."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=compute_stream, capture_error_mode="thread_local"):
            self.step(flags, compute_stream.cuda_stream, comm, proxy_fwd, proxy_bwd, ctas_per_sm, smem,
                      gemm=gemm, hook=hook)
        return g

    # -------------------------------------------------------------- accounting
    def step_bytes(self):
        """Full (gathered / reduced) bucket bytes one step moves through its
        collectives, per rank: forward AG + backward AG in param dtype, RS in fp32."""
        ag = sum(self.world * b.ag_seg for b in self.fwd) + sum(self.world * b.ag_seg for b in self.bwd)
        rs = sum(self.world * b.rs_seg for b in self.bwd)
        return ag, rs

    def kernel_bytes(self):
        """Algorithmic HBM bytes per step of each data kernel, as the library's
        run tables define them (fsdp_bucket_query): K1 2 x shard
        bytes, K3 2 x valid full bytes, K4 6 B per gradient element, K6 8 B per
        shard element (+ the few pad bytes zeroed).  A kernel that does not run
        (zero-copy storage) counts 0."""
        tot = {L.OP_PACK_AG: 0, L.OP_UNPACK: 0, L.OP_PACK_RS: 0, L.OP_COPYOUT_RS: 0}
        for phase, bs in ((0, self.fwd), (1, self.bwd)):
            for b in bs:
                kb = b.query()["kernel_bytes"]
                tot[L.OP_PACK_AG] += kb[0]
                tot[L.OP_UNPACK] += kb[1]
                if phase == 1:
                    tot[L.OP_PACK_RS] += kb[2]
                    tot[L.OP_COPYOUT_RS] += kb[3]
        return tot

    def kernel_launches(self):
        """Launches per step of each data kernel (buckets whose table is non-empty)."""
        n = {L.OP_PACK_AG: 0, L.OP_UNPACK: 0, L.OP_PACK_RS: 0, L.OP_COPYOUT_RS: 0}
        for phase, bs in ((0, self.fwd), (1, self.bwd)):
            for b in bs:
                kb = b.query()["kernel_bytes"]
                n[L.OP_PACK_AG] += kb[0] > 0
                n[L.OP_UNPACK] += kb[1] > 0
                if phase == 1:
                    n[L.OP_PACK_RS] += kb[2] > 0
                    n[L.OP_COPYOUT_RS] += kb[3] > 0
        return n

    def zero_copy(self):
        q = [b.query() for b in self.fwd + self.bwd]
        return {"ag_buckets": sum(x["ag_zero_copy"] for x in q), "rs_buckets": sum(x["rs_zero_copy"] for x in q[len(self.fwd):]),
                "buckets": len(q)}


OP_NAMES = ["PACK_AG", "AG", "WAIT_AG", "UNPACK", "COMPUTE_F", "COMPUTE_B", "PACK_RS", "RS", "WAIT_RS",
            "COPYOUT_RS"]


def chrome_trace(log, path, pid=0):
    """Chrome-trace JSON of a FSDP_SCHED_TIMING step log (entries with
    start_ns / ns >= 0): one complete ("X") event per op, tid 0 compute /
    1 comm, microseconds."""
    import json
    ev = []
    for ph, op, b, stream, ns, start in log:
        if ns is None or ns < 0 or start is None or start < 0:
            continue
        ev.append({"name": "%s %s[%d]" % (OP_NAMES[op], "fwd" if ph == 0 else "bwd", b), "ph": "X",
                   "ts": start / 1e3, "dur": ns / 1e3, "pid": pid, "tid": stream,
                   "args": {"phase": ph, "op": OP_NAMES[op], "bucket": b}})
    with open(path, "w") as f:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ms"}, f)
    return len(ev)


def plans_for(specs, world, mode, t_fwd=None, t_bwd=None, ag=(0, 0), rs=(0, 0), mem_max=0,
              param_dtype=L.BF16):
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    z = [0] * len(specs)
    fb, _ = F.plan_buckets(descs, world, t_fwd or z, ag, rs, mem_max, mode, L.PHASE_FWD, param_dtype)
    bb, _ = F.plan_buckets(descs, world, t_bwd or z, ag, rs, mem_max, mode, L.PHASE_BWD, param_dtype)
    return fb, bb


def mirror_plan(fwd_plan):
    """The backward plan that re-gathers the forward plan's buckets in reverse
    (SPEC's mirrored reading).  The peer-memory path needs it when the
    two phases' plans differ: peers read this rank's shards in one segment
    layout, so both phases must bucket the same members together."""
    return [sorted(b, reverse=True) for b in reversed(fwd_plan)]


def same_buckets(fwd_plan, bwd_plan):
    return sorted(tuple(sorted(b)) for b in fwd_plan) == sorted(tuple(sorted(b)) for b in bwd_plan)


# fsdp_plan_search cost model (tools/plan_search.py documents the numbers)
SEARCH_COST = dict(unpack_bytes_per_us=6470000, pack_rs_bytes_per_us=6680000, copy_launch_ns=6000,
                   compute_overhead_ns=16000, max_moves=0)


def plans_search(specs, world, t_fwd, t_bwd, ag=(0, 0), rs=(0, 0), mem_max=0, flags=None, param_dtype=L.BF16):
    """Per phase, fsdp_plan_search from the manual and the greedy plan; the
    plan with the lower predicted phase time is kept."""
    if flags is None:
        flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    descs = [(p.dim0, p.row_numel, p.module_id) for p in specs]
    starts = [plans_for(specs, world, m, t_fwd, t_bwd, ag, rs, mem_max, param_dtype)
              for m in (L.PLAN_MANUAL, L.PLAN_GREEDY)]
    out = []
    for phase, t, ph_flags in ((L.PHASE_FWD, t_fwd, flags & ~L.SCHED_BWD_AG_BEFORE_WAIT),
                               (L.PHASE_BWD, t_bwd, flags & ~L.SCHED_FWD_AG_BEFORE_WAIT)):
        best = None
        for st in starts:
            cost = dict(SEARCH_COST, sched_flags=ph_flags)
            plan, ns = F.plan_search(descs, world, t, ag, rs, mem_max, phase, st[phase], cost,
                                     param_dtype=param_dtype)
            if best is None or ns < best[1]:
                best = (plan, ns)
        out.append(best[0])
    return out[0], out[1]


def emulation_ctas(world, bus_gbps=720.0, per_cta_gbps=29.0):
    """CTAs for the emulated collectives (K11) of an N-rank job: enough to move
    a reduce-scatter's HBM bytes (the N fp32 segments read + this rank's
    segment written, (1 + 1/N) x the bucket) at the modelled bus rate, at the
    ~29 GB/s per CTA K11 sustained on B200 (32 CTAs hold an 8B block's RS at
    N = 8 to its modelled time; 16 did not).  32 at N = 8, 42 at N = 4, 75 at
    N = 2."""
    import math
    if world < 2:
        return 32
    rate = (1.0 + 1.0 / world) * bus_gbps * world / (world - 1)
    return int(min(148, max(32, math.ceil(rate / per_cta_gbps))))


def emulation_ctas_p2p(world, bus_gbps=720.0, per_cta_gbps=29.0):
    """CTAs for the paced peer-memory kernels (K8 / K9 under
    fsdp_comm_emulation): K8 reads all N segments (the simulated peers live in
    local HBM) and writes the full parameters, 2 x the bucket within the link
    time of (N - 1) / N of it -> 2 x bus x N / (N - 1) of HBM traffic; 57 CTAs
    at N = 8."""
    import math
    if world < 2:
        return 32
    rate = 2.0 * bus_gbps * world / (world - 1)
    return int(min(148, max(32, math.ceil(rate / per_cta_gbps))))


def time_bucket_collectives(specs, world, rank, ctx, compute, comm, reps=20, warmup=5, p2p=False,
                            exchange=None, max_over_ranks=None, seed=11, windows=False):
    """One bucket holding all of ``specs``, alone: a forward AG, a backward AG
    and an RS per step through fsdp_run_schedule with FSDP_SCHED_TIMING -- the
    AG / RS log entries are CUDA events around the collective alone on the comm
    stream (NCCL, or K8 / K9 with FSDP_SCHED_P2P).  Median over `reps` steps
    after `warmup`, max over ranks.  Returns dict(ag_bytes, rs_bytes, ag_ns,
    rs_ns): full bucket bytes in the planner's definition (G8: N * seg, bf16
    AG / fp32 RS) and the collective's device time."""
    plan = [list(range(len(specs)))]
    windows = windows and p2p
    st = RankState(specs, world, rank, plan, plan, ctx, seed=seed, ipc=p2p and world > 1 and not windows,
                   windows=windows)
    try:
        if windows:
            st.setup_p2p_windows()
        elif p2p:
            if world > 1:
                st.setup_p2p_ipc(exchange)
            else:
                st.setup_p2p_simulated()
        flags = L.SCHED_REORDER | L.SCHED_TIMING | (L.SCHED_P2P if p2p else 0)
        ag, rs = [], []
        for i in range(warmup + reps):
            rep = st.step(flags, compute, comm, want_log=True)
            if i >= warmup:
                ag += [e[4] for e in rep["log"] if e[1] == L.OP_AG]
                rs += [e[4] for e in rep["log"] if e[1] == L.OP_RS]
        st.check_p2p()
        t_ag, t_rs = float(np.median(ag)), float(np.median(rs))
        if max_over_ranks is not None:
            t_ag, t_rs = max_over_ranks(t_ag), max_over_ranks(t_rs)
        return dict(ag_bytes=world * st.fwd[0].ag_seg, rs_bytes=world * st.bwd[0].rs_seg, ag_ns=t_ag, rs_ns=t_rs)
    finally:
        torch.cuda.synchronize()
        if p2p:
            st.close_ipc()
            if exchange is not None and world > 1:
                exchange(None)          # every rank closed its mappings of ours
            st.free_ipc()
        st.close_nccl_mem()
        del st
        torch.cuda.empty_cache()


def fit_link(rows, key_bytes, key_ns, big=64 << 20):
    """alpha / beta of T(n) = alpha + beta n from a size sweep (SURVEY
    §8(d)): alpha = the measured time at the smallest size; beta = the
    least-squares slope over sizes >= `big`; both rounded to the planner's
    integer units (ns, fs per byte; G9).  Returns (alpha_ns, beta_fs_per_byte)."""
    small = min(rows, key=lambda r: r[key_bytes])
    pts = [(r[key_bytes], r[key_ns]) for r in rows if r[key_bytes] >= big]
    beta = 0.0
    if len(pts) >= 2:
        x = np.array([p[0] for p in pts], dtype=np.float64)
        y = np.array([p[1] for p in pts], dtype=np.float64)
        beta = float(np.polyfit(x, y, 1)[0])
    return int(round(small[key_ns])), max(0, int(round(beta * 1e6)))


def calibrate_proxy(ctx, stream, ctas_per_sm=1, smem=0, probe_iters=200000):
    """Proxy duration model on this device, now (clocks vary): K7 timed (median
    of 5) at probe_iters and probe_iters / 10 -> (ns per iteration, fixed ns
    per launch), an affine fit: the 16 waves of short CTAs cost a fixed
    launch / drain time on top of the iterations (a pure ratio ran
    100 us - 1 ms ops 10-13 % long)."""
    lo = probe_iters // 10
    t_hi = F.proxy_calibrate(ctx, probe_iters, ctas_per_sm, smem, 5, stream)
    t_lo = F.proxy_calibrate(ctx, lo, ctas_per_sm, smem, 5, stream)
    slope = (t_hi - t_lo) / (probe_iters - lo)
    if slope <= 0:
        return (t_hi / probe_iters, 0.0)
    return (slope, max(0.0, t_lo - slope * lo))


def proxy_iters(t_ns_per_bucket, cal):
    """Iterations of K7 that take t ns: cal = calibrate_proxy's (ns per
    iteration, fixed ns) or a plain ns-per-iteration; the fixed part is taken
    off ops longer than twice it (shorter ops keep half their time)."""
    slope, fixed = cal if isinstance(cal, tuple) else (cal, 0.0)
    return [int(round(max(t - fixed, 0.5 * t) / slope)) if t > 0 else 0 for t in t_ns_per_bucket]


def bucket_times(plan, t_per_param):
    return [sum(t_per_param[j] for j in b) for b in plan]


def np_dtype(dt):
    return np.uint16 if dt == L.BF16 else np.float32


def memory_sizes(st):
    """Per-bucket bytes of the G40 memory model (fsdp_simulate_memory), in each
    phase's execution order: flat AG (N x segment), full parameters, full
    gradients (bf16), flat RS input (N x fp32 segment)."""
    def full(b):
        return sum(st.full_numel[j] * st.ep for j in b.members)
    return dict(ag_fwd=[st.world * b.ag_seg for b in st.fwd], full_fwd=[full(b) for b in st.fwd],
                ag_bwd=[st.world * b.ag_seg for b in st.bwd], full_bwd=[full(b) for b in st.bwd],
                grad_bwd=[sum(st.full_numel[j] * 2 for j in b.members) for b in st.bwd],
                rs_bwd=[st.world * b.rs_seg for b in st.bwd])


def predict_memory(st, flags):
    """Peak bytes of the step's FSDP buffers under the G40 allocate-on-produce /
    free-after-last-use model, for the op sequence this rank's step enqueues
    with `flags` (host dry run); and the bytes this library's static pools hold
    instead (two slots of each kind)."""
    rep = F.run_schedule(None, None, None, n_fwd=len(st.fwd), n_bwd=len(st.bwd),
                         flags=(flags & (L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT |
                                         L.SCHED_BWD_AG_BEFORE_WAIT)) | L.SCHED_DRY_RUN)
    sz = memory_sizes(st)
    peak, _ = F.simulate_memory(rep["log"], sz["ag_fwd"], sz["full_fwd"], sz["ag_bwd"], sz["full_bwd"],
                                sz["grad_bwd"], sz["rs_bwd"])
    pools = 2 * (st.slot_bytes + st.gslot_bytes + st.ag_st[0].numel() + st.rs_st[0].numel())
    return peak, pools


def predict_exposure(st, flags, compute, comm, proxy_fwd, proxy_bwd, link_ag, link_rs, ctas_per_sm=1, smem=0,
                     gemm=None, hook=None):
    """Two-stream prediction of the N-rank step (fsdp_simulate_schedule): one
    timed step of this rank gives every compute-stream op its MEASURED
    duration; every collective takes alpha + beta n of its full bucket bytes
    (fsdp_comm_time_ns).  Returns (total_ns, exposed_ns).  A model: no SM /
    HBM contention between the copies and the collectives."""
    rep = st.step(flags | L.SCHED_TIMING, compute, comm, proxy_fwd, proxy_bwd, ctas_per_sm, smem, want_log=True,
                  gemm=gemm, hook=hook)
    return simulate_n_rank(st, rep["log"], link_ag, link_rs)


def simulate_n_rank(st, log, link_ag, link_rs):
    """The N-rank step from one timed step's log of this rank: compute-stream
    ops at their measured durations, except the copies a rank with a
    communicator does not run -- the AG copy-in of segment-layout storage (the
    collective sends from it) and the RS read-out into segment-layout gradient
    storage (the collective writes it) -- which a layout-only rank still runs
    (K1 own rows / K6) and which are charged 0 here; collectives at
    alpha + beta n.  Returns (total_ns, exposed_ns)."""
    durs = []
    q = {}
    for ph, op, b, _s, ns, _t in log:
        bk = (st.fwd if ph == 0 else st.bwd)[b]
        if (ph, b) not in q:
            q[(ph, b)] = bk.query()
        info = q[(ph, b)]
        if op == L.OP_AG:
            durs.append(F.comm_time_ns(st.world * bk.ag_seg, link_ag))
        elif op == L.OP_RS:
            durs.append(F.comm_time_ns(st.world * bk.rs_seg, link_rs))
        elif (op == L.OP_PACK_AG and info["ag_zero_copy"] and not info["ag_grouped"]) or \
                (op == L.OP_COPYOUT_RS and info["rs_zero_copy"]):
            durs.append(0)
        else:
            durs.append(max(ns, 0))
    tot, exp, _, _ = F.simulate_schedule(log, durs)
    return tot, exp
