"""Python names for the C ABI (include/fsdp.h).  Marshalling only.

Pointers are plain integers (e.g. ``tensor.data_ptr()``), streams are
``torch.cuda.Stream.cuda_stream`` integers (0 = legacy default stream).  No
logic of the method lives here: sharding, layout, planning, scheduling and all
data movement happen in libfsdp_b200.so.
"""
import ctypes as C

from . import _lib as L
from ._lib import check


def abi_version():
    return L.lib.fsdp_abi_version()


def nccl_get_unique_id():
    buf = (C.c_uint8 * 128)()
    check(L.lib.fsdp_nccl_get_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def shard(world, rank, desc, dtype, full_ptr=None, shard_ptr=None, stream=0):
    """fsdp_shard: metadata always, K0 copy when both pointers are given."""
    d = L.descs([desc])
    info = L.ShardInfo()
    check(L.lib.fsdp_shard(world, rank, d, dtype, full_ptr, shard_ptr, C.byref(info), stream or None))
    return dict(shard_rows=info.shard_rows, row_begin=info.row_begin, valid_rows=info.valid_rows,
                shard_numel=info.shard_numel)


def layout(members, world, elem_bytes, align=16):
    d = L.descs(members)
    offs = (C.c_int64 * len(members))()
    seg = C.c_int64()
    check(L.lib.fsdp_layout(d, len(members), world, elem_bytes, align, offs, C.byref(seg)))
    return list(offs), seg.value


def plan_buckets(params, world, t_compute_ns, ag, rs, mem_max, mode, phase, param_dtype=L.BF16,
                 align=16, mem_bytes=None, reduce_bytes=4, want_trace=False):
    """fsdp_plan_buckets.  params: (dim0, row_numel, module_id) in forward order.
    Returns (buckets, trace): buckets = lists of forward indices in the phase's
    execution order; trace = list of dicts (one per decision) if requested."""
    params = list(params)
    P = len(params)
    d = L.descs(params)
    tc = L.i64_array(t_compute_ns) if t_compute_ns is not None else None
    mb = L.i64_array(mem_bytes) if mem_bytes is not None else None
    pin = L.PlanIn()
    pin.params = d
    pin.t_compute_ns = tc
    pin.mem_bytes = mb
    pin.ag = L.Link(int(ag[0]), int(ag[1]))
    pin.rs = L.Link(int(rs[0]), int(rs[1]))
    pin.mem_max_bytes = int(mem_max)
    pin.n_params, pin.world, pin.align_bytes = P, world, align
    pin.mode, pin.phase, pin.param_dtype, pin.reduce_bytes, pin.reserved = mode, phase, param_dtype, reduce_bytes, 0
    bb = (C.c_int32 * (P + 1))()
    nb = C.c_int32()
    tr = (L.PlanTrace * max(P - 1, 1))() if want_trace else None
    check(L.lib.fsdp_plan_buckets(C.byref(pin), bb, C.byref(nb), tr))
    order = list(range(P)) if phase == L.PHASE_FWD else list(range(P - 1, -1, -1))
    buckets = [order[bb[b]:bb[b + 1]] for b in range(nb.value)]
    trace = None
    if want_trace:
        trace = [dict(param=t.param, t_lhs=t.t_lhs_ns, t_rhs=t.t_rhs_ns, m_lhs=t.m_lhs, m_rhs=t.m_rhs,
                      accept=bool(t.accept)) for t in tr[:P - 1]]
    return buckets, trace


def plan_search(params, world, t_compute_ns, ag, rs, mem_max, phase, start_plan, cost, param_dtype=L.BF16,
                align=16, mem_bytes=None, reduce_bytes=4):
    """fsdp_plan_search.  start_plan: buckets (forward indices, execution order)
    of this phase, e.g. from plan_buckets; cost: dict(unpack_bytes_per_us,
    pack_rs_bytes_per_us, copy_launch_ns, compute_overhead_ns, sched_flags,
    max_moves).  Returns (buckets, predicted phase ns)."""
    params = list(params)
    P = len(params)
    pin = L.PlanIn()
    keep = [L.descs(params), L.i64_array(t_compute_ns), L.i64_array(mem_bytes) if mem_bytes is not None else None]
    pin.params, pin.t_compute_ns, pin.mem_bytes = keep
    pin.ag = L.Link(int(ag[0]), int(ag[1]))
    pin.rs = L.Link(int(rs[0]), int(rs[1]))
    pin.mem_max_bytes = int(mem_max)
    pin.n_params, pin.world, pin.align_bytes = P, world, align
    pin.mode, pin.phase, pin.param_dtype, pin.reduce_bytes, pin.reserved = L.PLAN_GREEDY, phase, param_dtype, \
        reduce_bytes, 0
    starts = [0]
    for b in start_plan:
        starts.append(starts[-1] + len(b))
    sb = (C.c_int32 * len(starts))(*starts)
    c = L.SearchCost(int(cost["unpack_bytes_per_us"]), int(cost["pack_rs_bytes_per_us"]),
                     int(cost["copy_launch_ns"]), int(cost["compute_overhead_ns"]), int(cost["sched_flags"]),
                     int(cost.get("max_moves", 0)))
    bb = (C.c_int32 * (P + 1))()
    nb = C.c_int32()
    t = C.c_int64()
    check(L.lib.fsdp_plan_search(C.byref(pin), C.byref(c), sb, len(starts) - 1, bb, C.byref(nb), C.byref(t)))
    order = list(range(P)) if phase == L.PHASE_FWD else list(range(P - 1, -1, -1))
    return [order[bb[b]:bb[b + 1]] for b in range(nb.value)], t.value


class Ctx:
    """fsdp_ctx_create / fsdp_ctx_destroy."""

    def __init__(self, world, rank, device=0, nccl_uid=None, borrowed_comm=None, nccl_config=None):
        """nccl_config: dict(min_ctas, max_ctas, nvls_ctas, cta_policy) ->
        fsdp_ctx_create_config (needs nccl_uid)."""
        self.world, self.rank, self.device = world, rank, device
        self.has_nccl = nccl_uid is not None or bool(borrowed_comm)   # a communicator is held
        h = C.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = (C.c_uint8 * 128).from_buffer_copy(nccl_uid)
        uidp = C.cast(uid, C.c_void_p) if uid is not None else None
        if nccl_config is not None:
            cfg = L.NcclConfig(int(nccl_config.get("min_ctas", 0)), int(nccl_config.get("max_ctas", 0)),
                               int(nccl_config.get("nvls_ctas", 0)), int(nccl_config.get("cta_policy", -1)))
            check(L.lib.fsdp_ctx_create_config(C.byref(h), world, rank, device, uidp, C.byref(cfg)))
        else:
            check(L.lib.fsdp_ctx_create(C.byref(h), world, rank, device, uidp, borrowed_comm))
        self.h = h

    def nccl_estimate_ns(self, op, full_bytes):
        """fsdp_nccl_estimate_ns: NCCL's own estimate (ncclGroupSimulateEnd) for
        one AG (op = OP_AG, bf16) or RS (op = OP_RS, fp32) of full_bytes."""
        ns = C.c_int64()
        check(L.lib.fsdp_nccl_estimate_ns(self.h, int(op), int(full_bytes), C.byref(ns)))
        return ns.value

    def split(self, color, key):
        """fsdp_ctx_split: the sub-mesh ctx (a collective over this ctx's
        communicator); None for color -1."""
        h = C.c_void_p()
        check(L.lib.fsdp_ctx_split(self.h, int(color), int(key), C.byref(h)))
        if not h.value:
            return None
        sub = Ctx.__new__(Ctx)
        sub.device, sub.h = self.device, h
        n, r = C.c_int32(), C.c_int32()
        check(L.lib.fsdp_ctx_info(h, C.byref(n), C.byref(r)))
        sub.world, sub.rank = n.value, r.value
        sub.has_nccl = True
        return sub

    def close(self):
        if self.h:
            check(L.lib.fsdp_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Bucket:
    """fsdp_bucket_create / fsdp_bucket_destroy.  Pointer lists hold ints."""

    def __init__(self, ctx, params, shards=None, fulls=None, full_grads=None, grad_shards=None,
                 param_dtype=L.BF16, grad_dtype=L.BF16, align=16, flags=0):
        self.ctx = ctx
        self._keep = [L.descs(params), L.ptr_array(shards), L.ptr_array(fulls),
                      L.ptr_array(full_grads), L.ptr_array(grad_shards)]
        d = L.BucketDesc()
        d.params, d.shards, d.fulls, d.full_grads, d.grad_shards = self._keep
        d.k, d.align_bytes, d.param_dtype, d.grad_dtype = len(params), align, param_dtype, grad_dtype
        d.flags, d.reserved = flags, 0
        h = C.c_void_p()
        ag, rs = C.c_int64(), C.c_int64()
        check(L.lib.fsdp_bucket_create(ctx.h, C.byref(d), C.byref(h), C.byref(ag), C.byref(rs)))
        self.h = h
        self.ag_seg, self.rs_seg = ag.value, rs.value

    def set_grad_accumulation(self, on):
        """fsdp_bucket_set_grad_accumulation: later reduce-scatters add into
        the gradient shards (on) or overwrite them (off, the default)."""
        check(L.lib.fsdp_bucket_set_grad_accumulation(self.h, 1 if on else 0))

    def query(self):
        """fsdp_bucket_query: segment sizes, zero-copy flags, per-kernel
        algorithmic bytes per launch (K1, K3, K4, K6; 0 = not launched)."""
        i = L.BucketInfo()
        check(L.lib.fsdp_bucket_query(self.h, C.byref(i)))
        return dict(ag_seg=i.ag_seg_bytes, rs_seg=i.rs_seg_bytes, kernel_bytes=list(i.kernel_bytes),
                    kernel_chunks=list(i.kernel_chunks), ag_zero_copy=bool(i.ag_zero_copy),
                    rs_zero_copy=bool(i.rs_zero_copy), p2p_bytes=list(i.p2p_bytes), ag_direct=bool(i.ag_direct),
                    ag_grouped=bool(i.ag_grouped))

    def close(self):
        if self.h:
            check(L.lib.fsdp_bucket_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allgather_bucket(ctx, bucket, staging_ptr, compute=0, comm=0, flags=L.ISSUE | L.WAIT):
    check(L.lib.fsdp_allgather_bucket(ctx.h, bucket.h, staging_ptr, compute or None, comm or None, flags))


def reduce_scatter_bucket(ctx, bucket, staging_ptr, compute=0, comm=0, flags=L.ISSUE | L.WAIT):
    check(L.lib.fsdp_reduce_scatter_bucket(ctx.h, bucket.h, staging_ptr, compute or None, comm or None, flags))


def bucket_launch_kernel(ctx, bucket, op, staging_ptr, stream=0):
    """fsdp_bucket_launch_kernel: one data kernel of the bucket alone (op =
    OP_PACK_AG / OP_UNPACK / OP_PACK_RS / OP_COPYOUT_RS) as the step launches
    it; returns 1 if a kernel was enqueued, 0 if the step skips it."""
    n = C.c_int32()
    check(L.lib.fsdp_bucket_launch_kernel(ctx.h, bucket.h, int(op), staging_ptr, stream or None, C.byref(n)))
    return n.value


def run_schedule(ctx, fwd, bwd, ag_staging=(0, 0), rs_staging=(0, 0), compute=0, comm=0, flags=0,
                 proxy_iters_fwd=None, proxy_iters_bwd=None, proxy_ctas_per_sm=1, proxy_smem_bytes=0,
                 n_fwd=None, n_bwd=None, want_log=True, p2p=None, io=None, gemm=None, hook=None,
                 emulate=None, _capture=None):
    """fsdp_run_schedule.  fwd / bwd: Bucket lists in execution order (or
    counts via n_fwd / n_bwd with FSDP_SCHED_DRY_RUN and ctx=None).  Returns the
    step report as a dict (log as a list of (phase, op, bucket, stream, ns)).
    p2p (with FSDP_SCHED_P2P): dict with ag_peers (rows of world pointers),
    rs_peers, ready_slots, done_slots, ready_flags, done_flags, epoch_base,
    timeout_ns, error_flag.
    emulate (fsdp_comm_emulation): dict(ag=(alpha, beta), rs=(alpha, beta),
    ctas) -- emulated N-rank collectives on a layout-only ctx (timing only).
    hook (fsdp_compute_hook): a Python callable hook(phase, bucket, stream)
    that enqueues the bucket's model compute on `stream` (a cudaStream_t
    handle); an exception inside it aborts the step and is re-raised here."""
    nf = len(fwd) if fwd is not None else (n_fwd or 0)
    nb = len(bwd) if bwd is not None else (n_bwd or 0)
    s = L.Schedule()
    fw = L.ptr_array([b.h.value for b in fwd]) if fwd else None
    bw = L.ptr_array([b.h.value for b in bwd]) if bwd else None
    pf = L.i64_array(proxy_iters_fwd)
    pb = L.i64_array(proxy_iters_bwd)
    s.fwd, s.bwd, s.proxy_iters_fwd, s.proxy_iters_bwd = fw, bw, pf, pb
    s.ag_staging[0], s.ag_staging[1] = ag_staging
    s.rs_staging[0], s.rs_staging[1] = rs_staging
    s.compute, s.comm = compute or None, comm or None
    s.n_fwd, s.n_bwd, s.flags = nf, nb, flags
    s.proxy_ctas_per_sm, s.proxy_smem_bytes, s.reserved = proxy_ctas_per_sm, proxy_smem_bytes, 0
    keep = []
    if p2p is not None:
        ps = L.P2PSchedule()
        arrs = [L.ptr_array([x for row in p2p["ag_peers"] for x in row]),
                L.ptr_array([x for row in p2p.get("rs_peers", []) for x in row]),
                L.ptr_array(p2p["ready_slots"]), L.ptr_array(p2p["done_slots"])]
        keep += arrs
        ps.ag_peers, ps.rs_peers, ps.ready_slots, ps.done_slots = arrs
        ps.ready_flags, ps.done_flags = p2p["ready_flags"], p2p["done_flags"]
        ps.epoch_base, ps.timeout_ns = int(p2p["epoch_base"]), int(p2p.get("timeout_ns", 10**10))
        ps.error_flag = p2p.get("error_flag") or None
        ps.epoch_counter = p2p.get("epoch_counter") or None
        ps.max_ctas, ps.grad_slots = int(p2p.get("max_ctas", 0)), int(p2p.get("grad_slots", 0))
        keep.append(ps)
        s.p2p = C.pointer(ps)
    if io is not None:
        # io: dict(fwd_host_shards=[ptr or 0 per forward bucket], bwd_host_grads=[...], h2d=stream, d2h=stream)
        hio = L.HostIO()
        a = L.ptr_array(io.get("fwd_host_shards"))
        g = L.ptr_array(io.get("bwd_host_grads"))
        keep += [a, g, hio]
        hio.fwd_host_shards, hio.bwd_host_grads = a, g
        hio.h2d, hio.d2h = io.get("h2d") or None, io.get("d2h") or None
        hio.async_d2h, hio.reserved = 1 if io.get("async_d2h") else 0, 0
        s.io = C.pointer(hio)
    if gemm is not None:
        # gemm: dict(tokens, x, dy, y, workspace, workspace_bytes) -- fsdp_gemm_compute
        gc = L.GemmCompute(int(gemm["tokens"]), gemm["x"], gemm["dy"], gemm["y"], gemm.get("workspace") or None,
                           int(gemm.get("workspace_bytes", 0)))
        keep.append(gc)
        s.gemm = C.pointer(gc)
    hook_exc = []
    if hook is not None:
        def _fn(user, phase, bucket, stream):
            try:
                hook(phase, bucket, stream or 0)
                return 0
            except BaseException as e:  # reported through the status, re-raised below
                hook_exc.append(e)
                return 1
        cb = L.COMPUTE_FN(_fn)
        hk = L.ComputeHook(cb, None)
        keep += [cb, hk]
        s.hook = C.pointer(hk)
    if emulate is not None:
        # emulate: dict(ag=(alpha_ns, beta_fs), rs=(alpha_ns, beta_fs), ctas) -- fsdp_comm_emulation
        em = L.CommEmulation(L.Link(*[int(x) for x in emulate["ag"]]), L.Link(*[int(x) for x in emulate["rs"]]),
                             int(emulate.get("ctas", 16)), 0)
        keep.append(em)
        s.emulate = C.pointer(em)
    if _capture is not None:     # StepGraph: capture instead of run
        h = C.c_void_p()
        check(L.lib.fsdp_step_graph_create(ctx.h, C.byref(s), C.byref(h)))
        return h
    cap = 5 * nf + 9 * nb + 4
    log = (L.LogEntry * cap)() if want_log else None
    rep = L.StepReport()
    rep.log, rep.log_capacity = log, cap if want_log else 0
    st = L.lib.fsdp_run_schedule(ctx.h if ctx is not None else None, C.byref(s), C.byref(rep))
    if hook_exc:
        raise hook_exc[0]
    check(st)
    out = dict(step_ns=rep.step_ns, op_ns=list(rep.op_ns), op_count=list(rep.op_count),
               kernel_launches=rep.kernel_launches, collectives=rep.collectives, log_len=rep.log_len)
    if want_log:
        out["log"] = [(e.phase, e.op, e.bucket, e.stream, e.ns, e.start_ns) for e in log[:rep.log_len]]
    return out


def simulate_memory(seq, ag_fwd, full_fwd, ag_bwd, full_bwd, grad_bwd, rs_bwd):
    """fsdp_simulate_memory.  seq: (phase, op, bucket, stream[, ...]) tuples;
    per-bucket byte lists in each phase's execution order.  Returns
    (peak_bytes, live bytes after each entry)."""
    n = len(seq)
    arr = (L.LogEntry * max(n, 1))()
    for i, e in enumerate(seq):
        arr[i].ns, arr[i].phase, arr[i].op, arr[i].bucket, arr[i].stream = -1, e[0], e[1], e[2], e[3]
    keep = [L.i64_array(x) for x in (ag_fwd, full_fwd, ag_bwd, full_bwd, grad_bwd, rs_bwd)]
    sz = L.MemSizes(*keep, len(ag_fwd), len(ag_bwd))
    peak = C.c_int64()
    live = (C.c_int64 * max(n, 1))()
    check(L.lib.fsdp_simulate_memory(arr, n, C.byref(sz), C.byref(peak), live))
    return peak.value, list(live[:n])


class StepGraph:
    """fsdp_step_graph_*: one step (same arguments as run_schedule) captured
    into a CUDA graph; .launch(stream) replays it."""

    def __init__(self, ctx, fwd, bwd, **kw):
        self.h = run_schedule(ctx, fwd, bwd, want_log=False, _capture=True, **kw)
        k, c = C.c_int32(), C.c_int32()
        check(L.lib.fsdp_step_graph_info(self.h, C.byref(k), C.byref(c)))
        self.kernel_launches, self.collectives = k.value, c.value

    def launch(self, stream=0):
        check(L.lib.fsdp_step_graph_launch(self.h, stream or None))

    def close(self):
        if self.h:
            check(L.lib.fsdp_step_graph_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def proxy_launch(ctx, iters, ctas_per_sm=1, smem_bytes=0, stream=0):
    check(L.lib.fsdp_proxy_launch(ctx.h, int(iters), ctas_per_sm, smem_bytes, stream or None))


def proxy_calibrate(ctx, iters, ctas_per_sm=1, smem_bytes=0, reps=5, stream=0):
    ns = C.c_int64()
    check(L.lib.fsdp_proxy_calibrate(ctx.h, int(iters), ctas_per_sm, smem_bytes, reps, stream or None,
                                     C.byref(ns)))
    return ns.value


# ------------------------------------------------ peer-memory (fused) path
def p2p_allgather_bucket(ctx, bucket, peer_segs, stream=0):
    """fsdp_p2p_allgather_bucket: peer_segs[q] = rank q's segment-layout shard storage."""
    check(L.lib.fsdp_p2p_allgather_bucket(ctx.h, bucket.h, L.ptr_array(peer_segs), stream or None))


def p2p_reduce_scatter_bucket(ctx, bucket, peer_grads, stream=0):
    """fsdp_p2p_reduce_scatter_bucket: peer_grads[q] = rank q's full_grads[0]."""
    check(L.lib.fsdp_p2p_reduce_scatter_bucket(ctx.h, bucket.h, L.ptr_array(peer_grads), stream or None))


def p2p_signal(ctx, slots, value, stream=0):
    check(L.lib.fsdp_p2p_signal(ctx.h, L.ptr_array([s or 0 for s in slots]), int(value), stream or None))


def p2p_wait(ctx, flags_ptr, value, timeout_ns=10**9, error_flag_ptr=0, stream=0):
    check(L.lib.fsdp_p2p_wait(ctx.h, flags_ptr, int(value), int(timeout_ns), error_flag_ptr or None, stream or None))


def ipc_alloc(nbytes):
    """Returns (device pointer, 64-byte IPC handle)."""
    p = C.c_void_p()
    h = (C.c_uint8 * 64)()
    check(L.lib.fsdp_ipc_alloc(int(nbytes), C.byref(p), C.cast(h, C.c_void_p)))
    return p.value, bytes(h)


def ipc_open(handle):
    p = C.c_void_p()
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    check(L.lib.fsdp_ipc_open(C.cast(h, C.c_void_p), C.byref(p)))
    return p.value


def ipc_close(ptr):
    check(L.lib.fsdp_ipc_close(ptr))


def ipc_free(ptr):
    check(L.lib.fsdp_ipc_free(ptr))


def mem_alloc(ctx, nbytes):
    """fsdp_mem_alloc: ncclMemAlloc'd device memory (NVLS / symmetric-capable)."""
    p = C.c_void_p()
    check(L.lib.fsdp_mem_alloc(ctx.h, int(nbytes), C.byref(p)))
    return p.value


def mem_free(ctx, ptr):
    check(L.lib.fsdp_mem_free(ctx.h, ptr))


def register_buffer(ctx, ptr, nbytes, mode=L.REG_LOCAL):
    """fsdp_register_buffer: REG_LOCAL (ncclCommRegister) or REG_SYMMETRIC
    (collective ncclCommWindowRegister)."""
    check(L.lib.fsdp_register_buffer(ctx.h, ptr, int(nbytes), int(mode)))


def window_peer_pointers(ctx, base):
    """fsdp_window_peer_pointers: every rank's copy of the symmetric window
    registered at `base` (list of world addresses, this process's VA)."""
    out = (C.c_void_p * ctx.world)()
    check(L.lib.fsdp_window_peer_pointers(ctx.h, base, out))
    return [int(x or 0) for x in out]


def window_multimem_pointer(ctx, base):
    """fsdp_window_multimem_pointer: the window's NVLS multicast address
    (collective on the first call per ctx)."""
    mc = C.c_void_p()
    check(L.lib.fsdp_window_multimem_pointer(ctx.h, base, C.byref(mc)))
    return mc.value


class Nvls:
    """NVLS multicast team memory (fsdp_nvls_*).  Rank 0: Nvls(ctx, nbytes);
    others: Nvls(ctx, nbytes, handle=<rank 0's .handle>); then, after every
    rank constructed its object (a host barrier), .bind() -> (uc, mc, nbytes).

    Where the platform has no fabric handles the library exports a POSIX file
    descriptor instead; rank 0 then serves it to the peers over an abstract
    unix socket (SCM_RIGHTS, one connection per peer: ctx world - 1) and each
    peer writes the descriptor it received into the handle before importing
    (include/fsdp.h, fsdp_nvls_handle).  Plumbing only: no bytes of the
    collective pass through here."""

    def __init__(self, ctx, nbytes, handle=None, timeout_s=120.0):
        import struct
        self.ctx = ctx
        h = C.c_void_p()
        self._server = None
        if handle is None:
            buf = (C.c_uint8 * L.NVLS_HANDLE_BYTES)()
            check(L.lib.fsdp_nvls_create(ctx.h, int(nbytes), C.cast(buf, C.c_void_p), C.byref(h)))
            self.handle = bytes(buf)
            kind, fd, _pid, _ = struct.unpack_from("<iiii", self.handle)
            if kind == L.NVLS_POSIX_FD and ctx.world > 1:
                self._serve_fd(fd, ctx.world - 1, timeout_s)
        else:
            hb = bytearray(handle)
            kind, fd, pid, _ = struct.unpack_from("<iiii", hb)
            if kind == L.NVLS_POSIX_FD:
                struct.pack_into("<i", hb, 4, self._receive_fd(pid, fd, timeout_s))
            buf = (C.c_uint8 * L.NVLS_HANDLE_BYTES).from_buffer_copy(bytes(hb))
            check(L.lib.fsdp_nvls_import(ctx.h, C.cast(buf, C.c_void_p), int(nbytes), C.byref(h)))
            self.handle = bytes(handle)
        self.h = h
        self.uc = self.mc = None
        self.nbytes = int(nbytes)

    @staticmethod
    def _sock_name(pid, fd):
        return "\0fsdp_nvls.%d.%d" % (pid, fd)

    def _serve_fd(self, fd, peers, timeout_s):
        import os
        import socket
        import threading
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(self._sock_name(os.getpid(), fd))
        srv.listen(peers)
        srv.settimeout(timeout_s)

        def run():
            try:
                for _ in range(peers):
                    conn, _ = srv.accept()
                    with conn:
                        socket.send_fds(conn, [b"fd"], [fd])
            finally:
                srv.close()
                os.close(fd)   # every peer holds its own copy now
        self._server = threading.Thread(target=run, daemon=True)
        self._server.start()

    def _receive_fd(self, pid, fd, timeout_s):
        import socket
        import time
        t0 = time.time()
        while True:
            s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            try:
                s.connect(self._sock_name(pid, fd))
                _, fds, _, _ = socket.recv_fds(s, 16, 1)
                return fds[0]
            except (ConnectionRefusedError, FileNotFoundError):
                if time.time() - t0 > timeout_s:
                    raise
                time.sleep(0.05)
            finally:
                s.close()

    def bind(self):
        if self._server is not None:
            self._server.join()      # every peer took its descriptor
            self._server = None
        uc, mc, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(L.lib.fsdp_nvls_bind(self.h, C.byref(uc), C.byref(mc), C.byref(n)))
        self.uc, self.mc, self.nbytes = uc.value, mc.value, n.value
        return self.uc, self.mc, self.nbytes

    def close(self):
        if self.h:
            check(L.lib.fsdp_nvls_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nvls_reduce_scatter_bucket(ctx, bucket, mc_staging, stream=0):
    """K10: grad shards = the switch-reduced own segment of the staging."""
    check(L.lib.fsdp_nvls_reduce_scatter_bucket(ctx.h, bucket.h, mc_staging, stream or None))


# ------------------------------------------------------ cost model / prediction
def comm_time_ns(nbytes, link):
    """fsdp_comm_time_ns: alpha + ceil(n * beta_fs / 1e6)."""
    ns = C.c_int64()
    check(L.lib.fsdp_comm_time_ns(int(nbytes), C.byref(L.Link(int(link[0]), int(link[1]))), C.byref(ns)))
    return ns.value


def simulate_schedule(seq, durations):
    """fsdp_simulate_schedule.  seq: (phase, op, bucket, stream[, ...]) tuples,
    durations: ns per entry.  Returns (total_ns, exposed_ns, starts, ends)."""
    n = len(seq)
    arr = (L.LogEntry * max(n, 1))()
    for i, e in enumerate(seq):
        arr[i].ns, arr[i].phase, arr[i].op, arr[i].bucket, arr[i].stream = -1, e[0], e[1], e[2], e[3]
    d = (C.c_int64 * max(n, 1))(*[int(x) for x in durations])
    tot, exp = C.c_int64(), C.c_int64()
    st, en = (C.c_int64 * max(n, 1))(), (C.c_int64 * max(n, 1))()
    check(L.lib.fsdp_simulate_schedule(arr, n, d, C.byref(tot), C.byref(exp), st, en))
    return tot.value, exp.value, list(st[:n]), list(en[:n])
