// fsdp_run_schedule: the reordered (Table 6) or vanilla op
// sequence of one training step, executed on a compute and a comm stream.
// Also the compute proxy (K7) launch and calibration.
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

#include "internal.h"

using namespace fsdp;

namespace {

struct Op {
  int32_t phase, op, bucket;
};

bool is_comm(int32_t op) { return op == FSDP_OP_AG || op == FSDP_OP_RS; }
// ops that run on the copy stream with FSDP_SCHED_COPY_STREAM (the waits too:
// the copy-out after them is what consumes the collective's result)
bool is_copy_side(int32_t op) {
  return op == FSDP_OP_PACK_AG || op == FSDP_OP_WAIT_AG || op == FSDP_OP_UNPACK || op == FSDP_OP_PACK_RS ||
         op == FSDP_OP_WAIT_RS || op == FSDP_OP_COPYOUT_RS;
}
// [lo, hi) of the memory a bucket's full parameters (grads = false) or full
// gradients (grads = true) occupy
std::pair<uintptr_t, uintptr_t> full_range(const fsdp_bucket* b, bool grads) {
  uintptr_t lo = UINTPTR_MAX, hi = 0;
  const std::vector<void*>& ptrs = grads ? b->grads : b->fulls;
  for (size_t j = 0; j < ptrs.size() && j < b->members.size(); ++j) {
    if (!ptrs[j]) continue;
    const uintptr_t p = reinterpret_cast<uintptr_t>(ptrs[j]);
    const uintptr_t n = static_cast<uintptr_t>(b->members[j].dim0 * b->members[j].row_numel *
                                               (grads ? b->grad_bytes : b->param_bytes));
    lo = std::min(lo, p);
    hi = std::max(hi, p + n);
  }
  return {lo, hi};
}
bool overlaps(std::pair<uintptr_t, uintptr_t> a, std::pair<uintptr_t, uintptr_t> b) {
  return a.first < b.second && b.first < a.second;
}

// NVTX range names (host-side enqueue ranges; visible in nsys / ncu --nvtx).
const char* const kOpNames[FSDP_N_OPS] = {"fsdp:PACK_AG", "fsdp:AG",        "fsdp:WAIT_AG", "fsdp:UNPACK",
                                          "fsdp:COMPUTE_F", "fsdp:COMPUTE_B", "fsdp:PACK_RS", "fsdp:RS",
                                          "fsdp:WAIT_RS", "fsdp:COPYOUT_RS"};

struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Forward: prefetch depth 1; AG(k+1) before Wa(k) or after Wa(k) and its
// copy-out.  Vanilla: AG(k) right before Wa(k).
void forward_ops(std::vector<Op>& s, int32_t K, bool reorder, bool before) {
  if (!reorder) {
    for (int32_t b = 0; b < K; ++b)
      for (int32_t op : {FSDP_OP_PACK_AG, FSDP_OP_AG, FSDP_OP_WAIT_AG, FSDP_OP_UNPACK, FSDP_OP_COMPUTE_F})
        s.push_back({0, op, b});
    return;
  }
  if (K > 0) {
    s.push_back({0, FSDP_OP_PACK_AG, 0});
    s.push_back({0, FSDP_OP_AG, 0});
  }
  for (int32_t b = 0; b < K; ++b) {
    auto prefetch = [&] {
      if (b + 1 < K) {
        s.push_back({0, FSDP_OP_PACK_AG, b + 1});
        s.push_back({0, FSDP_OP_AG, b + 1});
      }
    };
    if (before) prefetch();
    s.push_back({0, FSDP_OP_WAIT_AG, b});
    s.push_back({0, FSDP_OP_UNPACK, b});
    if (!before) prefetch();
    s.push_back({0, FSDP_OP_COMPUTE_F, b});
  }
}

// Backward: re-gather with AG(j+1) after (default) or before Wa(j);
// "Wr12 is placed before RS34": Wr(j-1) and its read-out precede RS(j).
void backward_ops(std::vector<Op>& s, int32_t K, bool reorder, bool before, bool keep_first) {
  // keep_first (G42): bucket 0 reuses the last forward bucket's gathered
  // parameters -- its PACK_AG / AG / WAIT_AG / UNPACK are left out
  const size_t start = s.size();
  if (!reorder) {
    for (int32_t b = 0; b < K; ++b)
      for (int32_t op : {FSDP_OP_PACK_AG, FSDP_OP_AG, FSDP_OP_WAIT_AG, FSDP_OP_UNPACK, FSDP_OP_COMPUTE_B,
                         FSDP_OP_PACK_RS, FSDP_OP_RS, FSDP_OP_WAIT_RS, FSDP_OP_COPYOUT_RS})
        s.push_back({1, op, b});
  } else {
    if (K > 0) {
      s.push_back({1, FSDP_OP_PACK_AG, 0});
      s.push_back({1, FSDP_OP_AG, 0});
    }
    for (int32_t b = 0; b < K; ++b) {
      auto prefetch = [&] {
        if (b + 1 < K) {
          s.push_back({1, FSDP_OP_PACK_AG, b + 1});
          s.push_back({1, FSDP_OP_AG, b + 1});
        }
      };
      if (before) prefetch();
      s.push_back({1, FSDP_OP_WAIT_AG, b});
      s.push_back({1, FSDP_OP_UNPACK, b});
      if (!before) prefetch();
      s.push_back({1, FSDP_OP_COMPUTE_B, b});
      s.push_back({1, FSDP_OP_PACK_RS, b});
      if (b >= 1) {
        s.push_back({1, FSDP_OP_WAIT_RS, b - 1});
        s.push_back({1, FSDP_OP_COPYOUT_RS, b - 1});
      }
      s.push_back({1, FSDP_OP_RS, b});
    }
    if (K > 0) {
      s.push_back({1, FSDP_OP_WAIT_RS, K - 1});
      s.push_back({1, FSDP_OP_COPYOUT_RS, K - 1});
    }
  }
  if (keep_first)
    s.erase(std::remove_if(s.begin() + static_cast<std::ptrdiff_t>(start), s.end(),
                           [](const Op& o) {
                             return o.bucket == 0 && (o.op == FSDP_OP_PACK_AG || o.op == FSDP_OP_AG ||
                                                      o.op == FSDP_OP_WAIT_AG || o.op == FSDP_OP_UNPACK);
                           }),
            s.end());
}

int64_t max_seg(fsdp_bucket* const* bs, int32_t n, bool ag) {
  int64_t m = 0;
  for (int32_t i = 0; i < n; ++i) m = std::max(m, ag ? bs[i]->ag_seg : bs[i]->rs_seg);
  return m;
}

fsdp_status grow_events(fsdp_ctx* c, size_t n) {
  while (c->timing_events.size() < n) {
    cudaEvent_t e;
    FSDP_CUDA_TRY(cudaEventCreate(&e));
    c->timing_events.push_back(e);
  }
  return FSDP_OK;
}

}  // namespace

extern "C" fsdp_status fsdp_run_schedule(fsdp_ctx* ctx, const fsdp_schedule* s, fsdp_step_report* out) {
  if (!s) return fail(FSDP_ERR_INVALID_ARG, "NULL schedule");
  const uint32_t known = FSDP_SCHED_REORDER | FSDP_SCHED_FWD_AG_BEFORE_WAIT | FSDP_SCHED_BWD_AG_BEFORE_WAIT |
                         FSDP_SCHED_NO_COMM | FSDP_SCHED_DRY_RUN | FSDP_SCHED_TIMING | FSDP_SCHED_P2P |
                         FSDP_SCHED_KEEP_LAST_GATHERED | FSDP_SCHED_COPY_STREAM;
  if (s->flags & ~known) return fail(FSDP_ERR_INVALID_ARG, "unknown schedule flag");
  const bool copy_stream = s->flags & FSDP_SCHED_COPY_STREAM;
  if (copy_stream && (s->flags & FSDP_SCHED_P2P))
    return fail(FSDP_ERR_INVALID_ARG, "FSDP_SCHED_COPY_STREAM is not for FSDP_SCHED_P2P");
  if (s->n_fwd < 0 || s->n_bwd < 0) return fail(FSDP_ERR_INVALID_ARG, "negative bucket count");
  const bool p2p = s->flags & FSDP_SCHED_P2P;
  const bool dry = s->flags & FSDP_SCHED_DRY_RUN;
  const bool timing = (s->flags & FSDP_SCHED_TIMING) && !dry;
  const bool with_comm = !(s->flags & FSDP_SCHED_NO_COMM);

  std::vector<Op> seq;
  seq.reserve(5 * s->n_fwd + 9 * s->n_bwd + 4);
  const bool reorder = s->flags & FSDP_SCHED_REORDER;
  forward_ops(seq, s->n_fwd, reorder, s->flags & FSDP_SCHED_FWD_AG_BEFORE_WAIT);
  const bool keep_last = (s->flags & FSDP_SCHED_KEEP_LAST_GATHERED) && s->n_fwd > 0 && s->n_bwd > 0;
  backward_ops(seq, s->n_bwd, reorder, s->flags & FSDP_SCHED_BWD_AG_BEFORE_WAIT, keep_last);

  if (out) {
    if (out->log && out->log_capacity < static_cast<int32_t>(seq.size()))
      return fail(FSDP_ERR_INVALID_ARG, "log_capacity smaller than the step's op sequence");
    out->log_len = static_cast<int32_t>(seq.size());
    out->step_ns = -1;
    out->kernel_launches = 0;
    out->collectives = 0;
    for (int i = 0; i < FSDP_N_OPS; ++i) {
      out->op_ns[i] = timing ? 0 : -1;
      out->op_count[i] = 0;
    }
    for (size_t i = 0; i < seq.size(); ++i) {
      out->op_count[seq[i].op]++;
      if (out->log) {
        fsdp_log_entry& e = out->log[i];
        e.ns = -1;
        e.start_ns = -1;
        e.phase = seq[i].phase;
        e.op = seq[i].op;
        e.bucket = seq[i].bucket;
        e.stream = is_comm(seq[i].op) ? 1 : (copy_stream && is_copy_side(seq[i].op)) ? 2 : 0;
      }
    }
  }
  if (dry) return FSDP_OK;

  // ---- validation before any enqueue
  if (!ctx) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx");
  if ((s->n_fwd && !s->fwd) || (s->n_bwd && !s->bwd)) return fail(FSDP_ERR_INVALID_ARG, "NULL bucket array");
  for (int32_t i = 0; i < s->n_fwd; ++i)
    if (!s->fwd[i] || s->fwd[i]->ctx != ctx || !s->fwd[i]->has_shards || !s->fwd[i]->has_fulls)
      return fail(FSDP_ERR_INVALID_ARG, "forward bucket missing, foreign or without AG pointers");
  for (int32_t i = 0; i < s->n_bwd; ++i)
    if (!s->bwd[i] || s->bwd[i]->ctx != ctx || !s->bwd[i]->has_shards || !s->bwd[i]->has_fulls ||
        !s->bwd[i]->has_grads || !s->bwd[i]->has_gshards)
      return fail(FSDP_ERR_INVALID_ARG, "backward bucket missing, foreign or without AG/RS pointers");
  if (keep_last) {
    // the first backward bucket must bind exactly the last forward bucket's gathered parameters
    const fsdp_bucket* f = s->fwd[s->n_fwd - 1];
    const fsdp_bucket* g = s->bwd[0];
    bool same = f->fulls == g->fulls && f->members.size() == g->members.size() && f->param_bytes == g->param_bytes;
    for (size_t j = 0; same && j < f->members.size(); ++j)
      same = f->members[j].dim0 == g->members[j].dim0 && f->members[j].row_numel == g->members[j].row_numel;
    if (!same)
      return fail(FSDP_ERR_INVALID_ARG,
                  "FSDP_SCHED_KEEP_LAST_GATHERED: the first backward bucket does not bind the last forward "
                  "bucket's full parameters");
  }
  if (p2p) {
    const fsdp_p2p_schedule* pp = s->p2p;
    if (!pp || !pp->ag_peers || (s->n_bwd && !pp->rs_peers) || !pp->ready_slots || !pp->done_slots ||
        !pp->ready_flags || !pp->done_flags)
      return fail(FSDP_ERR_INVALID_ARG, "FSDP_SCHED_P2P needs a complete fsdp_p2p_schedule");
    if (ctx->world > kMaxPeers) return fail(FSDP_ERR_UNSUPPORTED, "peer-memory path supports world <= 16");
    if (pp->max_ctas < 0 || pp->grad_slots < 0 || pp->grad_slots == 1)
      return fail(FSDP_ERR_INVALID_ARG, "bad fsdp_p2p_schedule.max_ctas / grad_slots");
    for (int32_t i = 0; i < s->n_fwd + s->n_bwd; ++i) {
      fsdp_bucket* b = i < s->n_fwd ? s->fwd[i] : s->bwd[i - s->n_fwd];
      if (!b->ag_zero_copy) return fail(FSDP_ERR_INVALID_ARG, "FSDP_SCHED_P2P needs FSDP_BUCKET_SEGMENT_SHARDS buckets");
      for (int32_t q = 0; q < ctx->world; ++q) {
        const void* p = pp->ag_peers[static_cast<int64_t>(i) * ctx->world + q];
        if (!p || reinterpret_cast<uintptr_t>(p) % 16) return fail(FSDP_ERR_INVALID_ARG, "bad ag_peers entry");
      }
    }
    for (int32_t i = 0; i < s->n_bwd; ++i)
      if (s->bwd[i]->gshard_bf16)
        return fail(FSDP_ERR_INVALID_ARG, "FSDP_SCHED_P2P writes fp32 gradient shards (FSDP_BUCKET_BF16_GRAD_SHARDS)");
    for (int32_t i = 0; i < s->n_bwd; ++i)
      for (int32_t q = 0; q < ctx->world; ++q) {
        const void* p = pp->rs_peers[static_cast<int64_t>(i) * ctx->world + q];
        if (!p || reinterpret_cast<uintptr_t>(p) % 16) return fail(FSDP_ERR_INVALID_ARG, "bad rs_peers entry");
      }
    for (int32_t q = 0; q < ctx->world; ++q)
      if (reinterpret_cast<uintptr_t>(pp->ready_slots[q]) % 8 || reinterpret_cast<uintptr_t>(pp->done_slots[q]) % 8)
        return fail(FSDP_ERR_INVALID_ARG, "flag slot not 8-B aligned");
  } else {
    if ((s->n_fwd || s->n_bwd) && (!s->ag_staging[0] || !s->ag_staging[1]))
      return fail(FSDP_ERR_INVALID_ARG, "NULL AG staging slot");
    if (s->n_bwd && (!s->rs_staging[0] || !s->rs_staging[1]))
      return fail(FSDP_ERR_INVALID_ARG, "NULL RS staging slot");
  }
  for (int i = 0; i < 2; ++i)
    if (reinterpret_cast<uintptr_t>(s->ag_staging[i]) % 16 || reinterpret_cast<uintptr_t>(s->rs_staging[i]) % 16)
      return fail(FSDP_ERR_INVALID_ARG, "staging slot not 16-B aligned");
  if (s->proxy_ctas_per_sm < 0 || s->proxy_smem_bytes < 0)
    return fail(FSDP_ERR_INVALID_ARG, "bad proxy footprint");
  (void)max_seg;  // slot sizes are the caller's contract (>= world * largest segment)
  if (s->hook && !s->hook->fn) return fail(FSDP_ERR_INVALID_ARG, "compute hook without fn");
  if (s->gemm && !s->hook) {
    const fsdp_gemm_compute* g = s->gemm;
    if (g->tokens < 1 || g->tokens > INT32_MAX || !g->x || !g->dy || !g->y || g->workspace_bytes < 0 ||
        (g->workspace_bytes && !g->workspace))
      return fail(FSDP_ERR_INVALID_ARG, "bad fsdp_gemm_compute");
    for (int32_t j = 0; j < s->n_bwd; ++j)
      if (s->bwd[j]->grad_bytes != 2) return fail(FSDP_ERR_INVALID_ARG, "linear-layer compute needs bf16 gradients");
  }
  if (s->io) {
    if ((s->io->async_d2h != 0 && s->io->async_d2h != 1) || s->io->reserved != 0)
      return fail(FSDP_ERR_INVALID_ARG, "host I/O: async_d2h must be 0 or 1, reserved 0");
    if (s->io->async_d2h && (s->flags & FSDP_SCHED_P2P))
      return fail(FSDP_ERR_INVALID_ARG, "host I/O: async_d2h is not for FSDP_SCHED_P2P");
    for (int32_t k = 0; k < s->n_fwd; ++k)
      if (s->io->fwd_host_shards && s->io->fwd_host_shards[k] && !s->fwd[k]->ag_zero_copy)
        return fail(FSDP_ERR_INVALID_ARG, "host I/O: forward buckets need FSDP_BUCKET_SEGMENT_SHARDS");
    for (int32_t j = 0; j < s->n_bwd; ++j)
      if (s->io->bwd_host_grads && s->io->bwd_host_grads[j] && !s->bwd[j]->rs_zero_copy)
        return fail(FSDP_ERR_INVALID_ARG, "host I/O: backward buckets need FSDP_BUCKET_SEGMENT_GRAD_SHARDS");
  }

  if (s->emulate) {
    const fsdp_comm_emulation* em = s->emulate;
    if (ctx->comm) return fail(FSDP_ERR_INVALID_ARG, "emulated collectives need a ctx without a communicator");
    if (em->ctas < 1 || em->ctas > 4 * ctx->sm_count || em->reserved != 0 || em->ag.alpha_ns < 0 || em->ag.beta_fs_per_byte < 0 ||
        em->rs.alpha_ns < 0 || em->rs.beta_fs_per_byte < 0)
      return fail(FSDP_ERR_INVALID_ARG, "bad fsdp_comm_emulation");
    for (int32_t i = 0; i < s->n_fwd + s->n_bwd; ++i) {
      const fsdp_bucket* bk = i < s->n_fwd ? s->fwd[i] : s->bwd[i - s->n_fwd];
      if (bk->ag_grouped)
        return fail(FSDP_ERR_INVALID_ARG, "emulated collectives do not cover FSDP_BUCKET_GROUPED_AG");
      // K11 moves 16-B units: segments built with align_bytes < 16 may not be
      auto mis = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 != 0; };
      if (bk->ag_seg % 16 != 0 || (i >= s->n_fwd && bk->rs_seg % 16 != 0) ||
          (bk->ag_zero_copy && mis(bk->shard_seg)) || (bk->ag_direct && mis(bk->full0)) ||
          (i >= s->n_fwd && bk->rs_zero_copy && mis(bk->gshard_seg)))
        return fail(FSDP_ERR_INVALID_ARG,
                    "emulated collectives need 16-B multiple segments (align_bytes 16) and 16-B aligned buffers");
    }
  }
  // the emulated collectives (fsdp_comm_emulation) stand in for a communicator for this call only
  struct EmulGuard {
    fsdp_ctx* c;
    ~EmulGuard() { c->emul = nullptr; }
  } emul_guard{ctx};
  ctx->emul = p2p ? nullptr : s->emulate;

  FSDP_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t cs = static_cast<cudaStream_t>(s->compute);
  cudaStream_t ms = resolve_comm(ctx, s->comm);
  const int proxy_grid = ctx->sm_count * std::max(1, s->proxy_ctas_per_sm);
  if (timing) FSDP_TRY(grow_events(ctx, 2 * seq.size() + 2));
  cudaEvent_t* ev = timing ? ctx->timing_events.data() : nullptr;
  if (timing) FSDP_CUDA_TRY(cudaEventRecord(ev[0], cs));

  int launches = 0, colls = 0;
  // ---- peer-memory mode: epoch protocol of include/fsdp.h (FSDP_SCHED_P2P)
  const fsdp_p2p_schedule* pp = p2p ? s->p2p : nullptr;
  // emulated NVLink (fsdp_comm_emulation) for the peer-memory kernels: a grid of
  // emulate->ctas CTAs that stay for alpha + beta n (AG: the gathered bf16
  // bucket; RS: the bucket's gradients in their dtype, the bytes K9 pulls)
  const int p2p_ctas = (pp && s->emulate) ? s->emulate->ctas
                       : (pp && pp->max_ctas > 0) ? std::min(pp->max_ctas, ctx->max_ctas) : ctx->max_ctas;
  // K9 keeps half of K8's bytes in flight per thread (peers in batches of 4
  // x 16 B vs 8 x 16 B), so under a cap it gets twice the CTAs: the same
  // bytes in flight against NVLink latency
  const int p2p_ctas_rs = (pp && !s->emulate && pp->max_ctas > 0) ? std::min(2 * pp->max_ctas, ctx->max_ctas)
                                                                  : p2p_ctas;
  auto p2p_hold = [&](fsdp_bucket* bk, bool rs) -> int64_t {
    if (!pp || !s->emulate) return 0;
    int64_t ns = 0;
    if (rs) fsdp_comm_time_ns(ctx->world * bk->rs_seg / 4 * bk->grad_bytes, &s->emulate->rs, &ns);
    else fsdp_comm_time_ns(ctx->world * bk->ag_seg, &s->emulate->ag, &ns);
    return ns;
  };
  PeerTable ready_slots{}, done_slots{};
  auto epoch = [&](int64_t b) { return pp->epoch_base + 2 + static_cast<uint64_t>(b); };
  const uint64_t* ebase = pp ? pp->epoch_counter : nullptr;  // device epoch counter (nullable)
  auto p2p_wait = [&](const void* flags, uint64_t v, cudaStream_t st) -> fsdp_status {
    FSDP_CUDA_TRY(launch_p2p_wait(flags, ctx->world, v, pp->timeout_ns, pp->error_flag, st, ebase));
    ++launches;
    return FSDP_OK;
  };
  auto p2p_signal = [&](const PeerTable& slots, uint64_t v, cudaStream_t st) -> fsdp_status {
    FSDP_CUDA_TRY(launch_p2p_signal(slots, ctx->world, v, st, ebase));
    ++launches;
    return FSDP_OK;
  };
  auto peer_row = [&](const void* const* rows, int64_t row) {
    PeerTable t{};
    for (int32_t q = 0; q < ctx->world; ++q) t.p[q] = static_cast<const char*>(rows[row * ctx->world + q]);
    return t;
  };
  // ---- FSDP_SCHED_COPY_STREAM: pack / copy-out kernels on a third stream
  // (xs); events per bucket position p (forward k -> k, backward j -> n_fwd + j):
  // [3p] unpacked (xs), [3p + 1] computed (cs), [3p + 2] grads packed (xs);
  // [3P] the copy stream's end of step
  cudaStream_t xs = cs;
  cudaEvent_t* xev = nullptr;
  const int32_t P = s->n_fwd + s->n_bwd;
  if (copy_stream) {
    if (!ctx->own_copy_stream) {
      int lo = 0, hi = 0;
      FSDP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      FSDP_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->own_copy_stream, cudaStreamNonBlocking, hi));
    }
    xs = ctx->own_copy_stream;
    while (ctx->copy_events.size() < static_cast<size_t>(3 * P + 2)) {
      cudaEvent_t e;
      FSDP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->copy_events.push_back(e);
    }
    xev = ctx->copy_events.data();
    // the copy stream starts where the compute stream stands
    FSDP_CUDA_TRY(cudaEventRecord(xev[3 * P + 1], cs));
    FSDP_CUDA_TRY(cudaStreamWaitEvent(xs, xev[3 * P + 1], 0));
  }
  auto pos = [&](const Op& o) { return o.phase == 0 ? o.bucket : s->n_fwd + o.bucket; };
  auto bucket_at = [&](int32_t p) { return p < s->n_fwd ? s->fwd[p] : s->bwd[p - s->n_fwd]; };
  std::vector<char> computed(copy_stream ? P : 0, 0), grads_packed(copy_stream ? P : 0, 0);
  // stream `st` waits for the last earlier COMPUTE (grads = false) / PACK_RS
  // (grads = true) whose bucket's full-parameter / full-gradient memory
  // overlaps position p's
  auto wait_last_user = [&](int32_t p, bool grads, cudaStream_t st) -> fsdp_status {
    const auto mine = full_range(bucket_at(p), grads);
    for (int32_t q = p - 1; q >= 0; --q) {
      if (grads && q < s->n_fwd) break;
      if (!overlaps(mine, full_range(bucket_at(q), grads))) continue;
      const char done = grads ? grads_packed[q] : computed[q];
      // an overlapping bucket whose compute is not enqueued yet (the prefetch
      // of the next bucket into the memory the current one is computing on):
      // the two-slot contract of the schedule is broken
      if (!done)
        return fail(FSDP_ERR_INVALID_ARG,
                    "FSDP_SCHED_COPY_STREAM: adjacent buckets share full-parameter memory (prefetch needs two slots)");
      FSDP_CUDA_TRY(cudaStreamWaitEvent(st, xev[3 * q + (grads ? 2 : 1)], 0));
      break;
    }
    return FSDP_OK;
  };

  // ---- host I/O (fsdp_host_io): per-bucket H2D of shards, D2H of gradient shards
  const fsdp_host_io* io = s->io;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t* iev = nullptr;  // [0] step start, [1 + k] forward bucket k loaded, [1 + n_fwd + j] grads of j final, [last] d2h done
  if (io) {
    h2d = io->h2d ? static_cast<cudaStream_t>(io->h2d) : ctx->own_h2d;
    d2h = io->d2h ? static_cast<cudaStream_t>(io->d2h) : ctx->own_d2h;
    if (!h2d) {
      FSDP_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->own_h2d, cudaStreamNonBlocking));
      h2d = ctx->own_h2d;
    }
    if (!d2h) {
      FSDP_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->own_d2h, cudaStreamNonBlocking));
      d2h = ctx->own_d2h;
    }
    const size_t need = 2 + static_cast<size_t>(s->n_fwd + s->n_bwd);
    while (ctx->io_events.size() < need) {
      cudaEvent_t e;
      FSDP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->io_events.push_back(e);
    }
    iev = ctx->io_events.data();
    // the previous step's readers of the shard storage are ordered before the
    // H2D that overwrites it: after that step's last UNPACK (so this step's
    // loads overlap the previous step's gradient D2H, PCIe being full duplex),
    // else -- first step, peer-memory mode (peers read the storage until their
    // step ends), after a captured step -- after everything enqueued on compute
    if (!pp && ctx->shards_released_valid) {
      FSDP_CUDA_TRY(cudaStreamWaitEvent(h2d, ctx->ev_shards_released, 0));
    } else {
      FSDP_CUDA_TRY(cudaEventRecord(iev[0], cs));
      FSDP_CUDA_TRY(cudaStreamWaitEvent(h2d, iev[0], 0));
    }
    for (int32_t k = 0; k < s->n_fwd; ++k) {
      if (!io->fwd_host_shards || !io->fwd_host_shards[k]) continue;
      FSDP_CUDA_TRY(cudaMemcpyAsync(s->fwd[k]->shard_seg, io->fwd_host_shards[k], static_cast<size_t>(s->fwd[k]->ag_seg),
                                    cudaMemcpyHostToDevice, h2d));
      FSDP_CUDA_TRY(cudaEventRecord(iev[1 + k], h2d));
    }
  }
  auto io_before = [&](const Op& o) -> fsdp_status {
    if (io && o.op == FSDP_OP_PACK_AG && o.phase == 0 && io->fwd_host_shards && io->fwd_host_shards[o.bucket])
      FSDP_CUDA_TRY(cudaStreamWaitEvent(xs, iev[1 + o.bucket], 0));
    if (o.op == FSDP_OP_PACK_RS) {
      // an earlier step's asynchronous D2H of this bucket's gradient shards
      // must finish before anything of this step rewrites them
      fsdp_bucket* bb = s->bwd[o.bucket];
      if (bb->d2h_pending) {
        FSDP_CUDA_TRY(cudaStreamWaitEvent(xs, bb->ev_d2h_done, 0));
        bb->d2h_pending = false;
      }
    }
    return FSDP_OK;
  };
  // the step's last reader of the shard storage: its last UNPACK (after its
  // WAIT_AG, hence after every all-gather that sent from the storage)
  int64_t last_unpack = -1;
  for (size_t i = 0; i < seq.size(); ++i)
    if (seq[i].op == FSDP_OP_UNPACK) last_unpack = static_cast<int64_t>(i);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FSDP_CUDA_TRY(cudaStreamIsCapturing(cs, &cap));
  const bool track_release = !pp && cap == cudaStreamCaptureStatusNone;
  ctx->shards_released_valid = false;
  if (track_release && !ctx->ev_shards_released)
    FSDP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_shards_released, cudaEventDisableTiming));
  auto mark_release = [&](size_t i) -> fsdp_status {
    if (track_release && static_cast<int64_t>(i) == last_unpack) {
      FSDP_CUDA_TRY(cudaEventRecord(ctx->ev_shards_released, xs));
      ctx->shards_released_valid = true;
    }
    return FSDP_OK;
  };
  auto io_after = [&](const Op& o) -> fsdp_status {
    if (io && o.op == FSDP_OP_COPYOUT_RS && io->bwd_host_grads && io->bwd_host_grads[o.bucket]) {
      fsdp_bucket* bb = s->bwd[o.bucket];
      cudaEvent_t e = iev[1 + s->n_fwd + o.bucket];
      FSDP_CUDA_TRY(cudaEventRecord(e, xs));
      FSDP_CUDA_TRY(cudaStreamWaitEvent(d2h, e, 0));
      FSDP_CUDA_TRY(cudaMemcpyAsync(io->bwd_host_grads[o.bucket], bb->gshard_seg, static_cast<size_t>(bb->rs_seg),
                                    cudaMemcpyDeviceToHost, d2h));
      if (io->async_d2h) {
        FSDP_CUDA_TRY(cudaEventRecord(bb->ev_d2h_done, d2h));
        bb->d2h_pending = true;
      }
    }
    return FSDP_OK;
  };

  if (pp && with_comm) {
    for (int32_t q = 0; q < ctx->world; ++q) {
      ready_slots.p[q] = static_cast<const char*>(pp->ready_slots[q]);
      done_slots.p[q] = static_cast<const char*>(pp->done_slots[q]);
    }
    FSDP_TRY(p2p_signal(ready_slots, pp->epoch_base + 1, cs));  // my shards are final
    FSDP_TRY(p2p_wait(pp->ready_flags, pp->epoch_base + 1, cs));
  }
  // the compute of a bucket: linear-layer GEMMs (fsdp_gemm_compute) or the K7 proxy
  auto compute = [&](const Op& o, fsdp_bucket* b) -> fsdp_status {
    if (s->hook) {
      const int32_t rc = s->hook->fn(s->hook->user, o.phase, o.bucket, static_cast<fsdp_stream_t>(cs));
      if (rc != 0) return fail(FSDP_ERR_INVALID_ARG, "compute hook failed (rc " + std::to_string(rc) + ")");
      return FSDP_OK;
    }
    if (s->gemm) return bucket_compute(ctx, b, s->gemm, o.op == FSDP_OP_COMPUTE_B, cs, &launches);
    const int64_t* it = o.op == FSDP_OP_COMPUTE_F ? s->proxy_iters_fwd : s->proxy_iters_bwd;
    if (it && it[o.bucket] > 0) {
      FSDP_CUDA_TRY(launch_proxy(it[o.bucket], proxy_grid, s->proxy_smem_bytes, ctx->sink, cs));
      ++launches;
    }
    return FSDP_OK;
  };
  NvtxRange step_range("fsdp:step");
  for (size_t i = 0; i < seq.size(); ++i) {
    const Op& o = seq[i];
    fsdp_bucket* b = (o.phase == 0 ? s->fwd : s->bwd)[o.bucket];
    NvtxRange op_range(kOpNames[o.op]);
    FSDP_TRY(io_before(o));
    if (pp) {
      // the peer-memory path: same sequence, different work per op
      const bool comm_op = is_comm(o.op);
      const bool skipped = !with_comm && (comm_op || o.op == FSDP_OP_WAIT_AG || o.op == FSDP_OP_WAIT_RS);
      cudaStream_t on = comm_op ? ms : cs;
      if (timing && !skipped) {
        if (comm_op) FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, o.op == FSDP_OP_AG ? b->ev_ag_packed : b->ev_rs_packed, 0));
        FSDP_CUDA_TRY(cudaEventRecord(ev[2 + 2 * i], on));
      }
      switch (o.op) {
        case FSDP_OP_PACK_AG:
          if (with_comm) FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_packed, cs));
          break;
        case FSDP_OP_AG:
          if (with_comm) {
            FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, b->ev_ag_packed, 0));
            const int64_t row = o.phase == 0 ? o.bucket : s->n_fwd + o.bucket;
            FSDP_CUDA_TRY(launch_p2p_allgather(b->p2p_ag, peer_row(pp->ag_peers, row), ms, p2p_ctas,
                                               p2p_hold(b, false)));
            FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_done, ms));
            ++launches;
            ++colls;
          }
          break;
        case FSDP_OP_WAIT_AG:
          if (with_comm) FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, b->ev_ag_done, 0));
          break;
        case FSDP_OP_COMPUTE_F:
        case FSDP_OP_COMPUTE_B: {
          // the backward of bucket b overwrites gradient slot b % G: peers must be done with b - G
          const int32_t gslots = pp->grad_slots > 0 ? pp->grad_slots : 2;
          if (o.op == FSDP_OP_COMPUTE_B && with_comm && o.bucket >= gslots)
            FSDP_TRY(p2p_wait(pp->done_flags, epoch(o.bucket - gslots), cs));
          FSDP_TRY(compute(o, b));
          break;
        }
        case FSDP_OP_PACK_RS:
          if (with_comm) {
            FSDP_TRY(p2p_signal(ready_slots, epoch(o.bucket), cs));  // my gradients of b are final
            FSDP_CUDA_TRY(cudaEventRecord(b->ev_rs_packed, cs));
          }
          break;
        case FSDP_OP_RS:
          if (with_comm) {
            FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, b->ev_rs_packed, 0));
            const float inv = 1.0f / static_cast<float>(ctx->world);
#if FSDP_P2P_FUSED_SYNC
            if (ebase) return fail(FSDP_ERR_UNSUPPORTED, "fused-sync build: no device epoch counter");
            // one launch: wait "ready" >= E(b), reduce, last CTA signals "consumed" E(b)
            P2PSync sync{static_cast<const unsigned long long*>(pp->ready_flags), epoch(o.bucket),
                         static_cast<long long>(pp->timeout_ns), pp->error_flag, done_slots, epoch(o.bucket),
                         ctx->p2p_counter};
            FSDP_CUDA_TRY(launch_p2p_reduce_scatter(b->p2p_rs, peer_row(pp->rs_peers, o.bucket), ctx->world, inv,
                                                    b->grad_accumulate, ms, p2p_ctas_rs, &sync, p2p_hold(b, true)));
            ++launches;
#else
            FSDP_TRY(p2p_wait(pp->ready_flags, epoch(o.bucket), ms));
            FSDP_CUDA_TRY(launch_p2p_reduce_scatter(b->p2p_rs, peer_row(pp->rs_peers, o.bucket), ctx->world, inv,
                                                    b->grad_accumulate, ms, p2p_ctas_rs, nullptr, p2p_hold(b, true)));
            ++launches;
            FSDP_TRY(p2p_signal(done_slots, epoch(o.bucket), ms));  // done reading peers' b
#endif
            FSDP_CUDA_TRY(cudaEventRecord(b->ev_rs_done, ms));
            ++colls;
          }
          break;
        case FSDP_OP_WAIT_RS:
          if (with_comm) FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, b->ev_rs_done, 0));
          break;
        default:  // UNPACK, COPYOUT_RS: the peer kernels wrote the destinations
          break;
      }
      if (timing && !skipped) FSDP_CUDA_TRY(cudaEventRecord(ev[3 + 2 * i], on));
      FSDP_TRY(io_after(o));
      continue;
    }
    char* ag_st = static_cast<char*>(s->ag_staging[o.bucket & 1]);
    char* rs_st = static_cast<char*>(s->rs_staging[o.bucket & 1]);
    const bool comm_op = is_comm(o.op);
    const bool skipped = !with_comm && (comm_op || o.op == FSDP_OP_WAIT_AG || o.op == FSDP_OP_WAIT_RS);
    const int32_t p = pos(o);
    cudaStream_t on = comm_op ? ms : is_copy_side(o.op) ? xs : cs;
    if (copy_stream) {
      // cross-stream data dependencies of the copy stream (include/fsdp.h)
      if (o.op == FSDP_OP_UNPACK || (o.op == FSDP_OP_PACK_AG && (b->ag_direct || b->ag_grouped)))
        FSDP_TRY(wait_last_user(p, false, xs));                 // full-parameter memory free
      if (o.op == FSDP_OP_COMPUTE_F || o.op == FSDP_OP_COMPUTE_B) {
        const bool has_unpack = !(keep_last && o.phase == 1 && o.bucket == 0);
        if (has_unpack) FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, xev[3 * p], 0));     // unpacked
        if (o.op == FSDP_OP_COMPUTE_B) FSDP_TRY(wait_last_user(p, true, cs));      // full-gradient memory free
      }
      if (o.op == FSDP_OP_PACK_RS) FSDP_CUDA_TRY(cudaStreamWaitEvent(xs, xev[3 * p + 1], 0));  // computed
    }
    if (timing && !skipped) {
      if (comm_op) {
        // start after the pack this collective depends on
        FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, o.op == FSDP_OP_AG ? b->ev_ag_packed : b->ev_rs_packed, 0));
      }
      FSDP_CUDA_TRY(cudaEventRecord(ev[2 + 2 * i], on));
    }
    switch (o.op) {
      case FSDP_OP_PACK_AG: FSDP_TRY(ag_pack(ctx, b, ag_st, xs, with_comm, &launches)); break;
      case FSDP_OP_AG: FSDP_TRY(ag_collective(ctx, b, ag_st, ms, with_comm, &colls)); break;
      case FSDP_OP_WAIT_AG: FSDP_TRY(ag_wait(ctx, b, xs, with_comm)); break;
      case FSDP_OP_UNPACK: FSDP_TRY(ag_unpack(ctx, b, ag_st, xs, &launches)); break;
      case FSDP_OP_COMPUTE_F:
      case FSDP_OP_COMPUTE_B: {
        FSDP_TRY(compute(o, b));
        break;
      }
      case FSDP_OP_PACK_RS: FSDP_TRY(rs_pack(ctx, b, rs_st, xs, with_comm, &launches)); break;
      case FSDP_OP_RS: FSDP_TRY(rs_collective(ctx, b, rs_st, ms, with_comm, &colls)); break;
      case FSDP_OP_WAIT_RS: FSDP_TRY(rs_wait(ctx, b, xs, with_comm)); break;
      case FSDP_OP_COPYOUT_RS: FSDP_TRY(rs_copyout(ctx, b, rs_st, xs, with_comm, &launches)); break;
    }
    if (copy_stream) {
      if (o.op == FSDP_OP_UNPACK) FSDP_CUDA_TRY(cudaEventRecord(xev[3 * p], xs));
      if (o.op == FSDP_OP_COMPUTE_F || o.op == FSDP_OP_COMPUTE_B) {
        FSDP_CUDA_TRY(cudaEventRecord(xev[3 * p + 1], cs));
        computed[p] = 1;
      }
      if (o.op == FSDP_OP_PACK_RS) {
        FSDP_CUDA_TRY(cudaEventRecord(xev[3 * p + 2], xs));
        grads_packed[p] = 1;
      }
    }
    if (timing && !skipped) FSDP_CUDA_TRY(cudaEventRecord(ev[3 + 2 * i], on));
    FSDP_TRY(io_after(o));
    FSDP_TRY(mark_release(i));
  }
  if (copy_stream) {
    // the step ends on the compute stream after the copy stream's last op
    FSDP_CUDA_TRY(cudaEventRecord(xev[3 * P], xs));
    FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, xev[3 * P], 0));
  }
  if (io && s->n_bwd > 0 && !io->async_d2h) {
    // the step ends when its gradient shards are on the host
    cudaEvent_t e = iev[1 + s->n_fwd + s->n_bwd];
    FSDP_CUDA_TRY(cudaEventRecord(e, d2h));
    FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, e, 0));
  }
  if (pp && with_comm) {
    // step end: peers are done with every gradient slot and every shard of mine
    if (s->n_bwd > 0) FSDP_TRY(p2p_wait(pp->done_flags, epoch(s->n_bwd - 1), cs));
    FSDP_TRY(p2p_signal(ready_slots, epoch(s->n_bwd), cs));
    FSDP_TRY(p2p_wait(pp->ready_flags, epoch(s->n_bwd), cs));
    if (pp->epoch_counter) {  // the next step (or replay) starts past this step's epochs
      FSDP_CUDA_TRY(launch_p2p_epoch_advance(pp->epoch_counter, static_cast<uint64_t>(s->n_bwd) + 2, cs));
      ++launches;
    }
  }
  if (timing) FSDP_CUDA_TRY(cudaEventRecord(ev[1], cs));
  FSDP_TRY(check_async_error(ctx));

  if (out) {
    out->kernel_launches = launches;
    out->collectives = colls;
  }
  if (timing) {
    FSDP_CUDA_TRY(cudaEventSynchronize(ev[1]));
    float ms_total = 0.f;
    FSDP_CUDA_TRY(cudaEventElapsedTime(&ms_total, ev[0], ev[1]));
    if (out) {
      out->step_ns = static_cast<int64_t>(ms_total * 1e6);
      for (size_t i = 0; i < seq.size(); ++i) {
        const Op& o = seq[i];
        const bool skipped = !with_comm && (is_comm(o.op) || o.op == FSDP_OP_WAIT_AG || o.op == FSDP_OP_WAIT_RS);
        if (skipped) continue;
        float t = 0.f;
        FSDP_CUDA_TRY(cudaEventElapsedTime(&t, ev[2 + 2 * i], ev[3 + 2 * i]));
        const int64_t ns = static_cast<int64_t>(t * 1e6);
        out->op_ns[o.op] += ns;
        if (out->log) {
          out->log[i].ns = ns;
          float t0 = 0.f;
          FSDP_CUDA_TRY(cudaEventElapsedTime(&t0, ev[0], ev[2 + 2 * i]));
          out->log[i].start_ns = static_cast<int64_t>(t0 * 1e6);
        }
      }
    }
  }
  if (timing && pp && with_comm && pp->error_flag) {
    // the step has completed (synchronised above): a timed-out epoch wait means
    // a kernel went ahead without its peers -- the results are invalid
    int32_t flag = 0;
    FSDP_CUDA_TRY(cudaMemcpy(&flag, pp->error_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag) return fail(FSDP_ERR_CUDA, "peer-memory epoch wait timed out: this step's results are invalid");
  }
  return FSDP_OK;
}

// ---------------------------------------------------------------- step graph
struct fsdp_step_graph {
  int32_t device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t kernel_launches = 0, collectives = 0;
};

extern "C" fsdp_status fsdp_step_graph_destroy(fsdp_step_graph* g) {
  if (!g) return FSDP_OK;
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_step_graph_create(fsdp_ctx* ctx, const fsdp_schedule* s, fsdp_step_graph** out) {
  if (!ctx || !s || !out) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (s->flags & (FSDP_SCHED_TIMING | FSDP_SCHED_DRY_RUN))
    return fail(FSDP_ERR_INVALID_ARG, "step graph: no TIMING or DRY_RUN");
  if ((s->flags & FSDP_SCHED_P2P) && (!s->p2p || !s->p2p->epoch_counter))
    return fail(FSDP_ERR_INVALID_ARG, "step graph with FSDP_SCHED_P2P needs a device epoch_counter");
  if (s->io) return fail(FSDP_ERR_INVALID_ARG, "step graph: host I/O is not captured");
  if (!s->compute) return fail(FSDP_ERR_INVALID_ARG, "step graph: needs a non-default compute stream");
  FSDP_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t cs = static_cast<cudaStream_t>(s->compute);
  (void)resolve_comm(ctx, s->comm);  // create a library-owned comm stream before capture
  fsdp_step_report rep{};
  // the whole step -- kernels, NCCL collectives, cross-stream events -- is
  // recorded from `compute`; the comm stream joins through the event waits
  FSDP_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  fsdp_status st = fsdp_run_schedule(ctx, s, &rep);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &graph);
  if (st != FSDP_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(FSDP_ERR_CUDA, std::string("step graph capture: ") + cudaGetErrorString(e));
  fsdp_step_graph* g = new fsdp_step_graph();
  g->device = ctx->device;
  g->graph = graph;
  g->kernel_launches = rep.kernel_launches;
  g->collectives = rep.collectives;
  // keep the captured per-kernel stream priorities (the comm stream's NCCL
  // kernels must still overtake compute-stream CTAs, as in the eager step)
  e = cudaGraphInstantiate(&g->exec, graph, cudaGraphInstantiateFlagUseNodePriority);
  if (e != cudaSuccess) {
    fsdp_step_graph_destroy(g);
    return fail(FSDP_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  }
  *out = g;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_step_graph_launch(fsdp_step_graph* g, fsdp_stream_t stream) {
  if (!g) return fail(FSDP_ERR_INVALID_ARG, "NULL graph");
  FSDP_CUDA_TRY(cudaSetDevice(g->device));
  FSDP_CUDA_TRY(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_step_graph_info(const fsdp_step_graph* g, int32_t* kernel_launches,
                                            int32_t* collectives) {
  if (!g) return fail(FSDP_ERR_INVALID_ARG, "NULL graph");
  if (kernel_launches) *kernel_launches = g->kernel_launches;
  if (collectives) *collectives = g->collectives;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_proxy_launch(fsdp_ctx* ctx, int64_t iters, int32_t ctas_per_sm, int32_t smem_bytes,
                                         fsdp_stream_t stream) {
  if (!ctx || iters < 0 || ctas_per_sm < 1 || smem_bytes < 0)
    return fail(FSDP_ERR_INVALID_ARG, "bad proxy arguments");
  FSDP_CUDA_TRY(cudaSetDevice(ctx->device));
  if (iters == 0) return FSDP_OK;
  FSDP_CUDA_TRY(launch_proxy(iters, ctx->sm_count * ctas_per_sm, smem_bytes, ctx->sink,
                             static_cast<cudaStream_t>(stream)));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_proxy_calibrate(fsdp_ctx* ctx, int64_t iters, int32_t ctas_per_sm, int32_t smem_bytes,
                                            int32_t reps, fsdp_stream_t stream, int64_t* ns_out) {
  if (!ctx || iters < 1 || ctas_per_sm < 1 || smem_bytes < 0 || reps < 1 || !ns_out)
    return fail(FSDP_ERR_INVALID_ARG, "bad calibration arguments");
  FSDP_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t a, b;
  FSDP_CUDA_TRY(cudaEventCreate(&a));
  FSDP_CUDA_TRY(cudaEventCreate(&b));
  std::vector<float> t;
  fsdp_status status = FSDP_OK;
  for (int32_t r = 0; r < reps + 1 && status == FSDP_OK; ++r) {  // first rep warms up
    cudaError_t e = cudaEventRecord(a, st);
    if (e == cudaSuccess) e = launch_proxy(iters, ctx->sm_count * ctas_per_sm, smem_bytes, ctx->sink, st);
    if (e == cudaSuccess) e = cudaEventRecord(b, st);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess) status = fail(FSDP_ERR_CUDA, std::string("proxy calibration: ") + cudaGetErrorString(e));
    if (r > 0) t.push_back(ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (status != FSDP_OK) return status;
  std::sort(t.begin(), t.end());
  *ns_out = static_cast<int64_t>(t[t.size() / 2] * 1e6);
  return FSDP_OK;
}
