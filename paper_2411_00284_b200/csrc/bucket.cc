// Bucket handles and the per-bucket collectives:
//   fsdp_allgather_bucket      -- AG bucketing, P:177 (copy-in, AG + Wa, copy-out)
//   fsdp_reduce_scatter_bucket -- RS bucketing, P:179 (chunk/concat, RS + Wr avg, read-out)
// Copies are the sm_100a kernels of kernels.cu on the compute stream; the
// collectives are in-place NCCL calls on the comm stream, ordered by events.
#include <cstring>

#include "internal.h"

using namespace fsdp;

namespace {

cudaStream_t comm_stream(fsdp_ctx* c, fsdp_stream_t s) {
  if (s) return static_cast<cudaStream_t>(s);
  if (!c->own_comm_stream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->own_comm_stream, cudaStreamNonBlocking, hi);
  }
  return c->own_comm_stream;
}

void destroy_bucket(fsdp_bucket* b) {
  release(&b->ag_pack);
  release(&b->rs_accum);
  release(&b->nvls_rs);
  release(&b->ag_unpack);
  release(&b->rs_pack);
  release(&b->rs_copyout);
  release(&b->p2p_ag);
  release(&b->p2p_rs);
  for (cudaEvent_t* e : {&b->ev_ag_packed, &b->ev_ag_done, &b->ev_rs_packed, &b->ev_rs_done, &b->ev_d2h_done})
    if (*e) cudaEventDestroy(*e);
  delete b;
}

}  // namespace

extern "C" fsdp_status fsdp_bucket_create(fsdp_ctx* ctx, const fsdp_bucket_desc* d, fsdp_bucket** out,
                                          int64_t* ag_seg_bytes, int64_t* rs_seg_bytes) {
  if (!ctx || !d || !out) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const int32_t k = d->k;
  if (k < 1 || !d->params) return fail(FSDP_ERR_INVALID_ARG, "bucket needs >= 1 member");
  if (d->align_bytes < 1) return fail(FSDP_ERR_INVALID_ARG, "align_bytes < 1");
  if (d->reserved != 0 || (d->flags & ~(FSDP_BUCKET_SEGMENT_SHARDS | FSDP_BUCKET_SEGMENT_GRAD_SHARDS |
                                        FSDP_BUCKET_FP32_MASTER | FSDP_BUCKET_GROUPED_AG |
                                        FSDP_BUCKET_BF16_GRAD_SHARDS)))
    return fail(FSDP_ERR_INVALID_ARG, "unknown bucket flags");
  const int32_t ep = dtype_bytes(d->param_dtype), eg = dtype_bytes(d->grad_dtype);
  if (!ep || !eg) return fail(FSDP_ERR_INVALID_ARG, "unsupported dtype");
  // fp32 master shards, cast to bf16 by the pack
  const bool master = d->flags & FSDP_BUCKET_FP32_MASTER;
  if (master && (d->param_dtype != FSDP_BF16 || (d->flags & FSDP_BUCKET_SEGMENT_SHARDS)))
    return fail(FSDP_ERR_INVALID_ARG, "FSDP_BUCKET_FP32_MASTER needs param_dtype BF16 and no SEGMENT_SHARDS");
  // bf16 gradient shards: K6 rounds the fp32 RS output (G41)
  const bool gs_bf16 = d->flags & FSDP_BUCKET_BF16_GRAD_SHARDS;
  if (gs_bf16 && (d->flags & FSDP_BUCKET_SEGMENT_GRAD_SHARDS))
    return fail(FSDP_ERR_INVALID_ARG, "FSDP_BUCKET_BF16_GRAD_SHARDS excludes SEGMENT_GRAD_SHARDS");
  for (int32_t j = 0; j < k; ++j) {
    const fsdp_param_desc& p = d->params[j];
    if (p.dim0 < 1 || p.row_numel < 1 || p.reserved != 0)
      return fail(FSDP_ERR_INVALID_ARG, "bad param descriptor");
    if (d->shards && !d->shards[j]) return fail(FSDP_ERR_INVALID_ARG, "NULL shard pointer");
    if (d->fulls && !d->fulls[j]) return fail(FSDP_ERR_INVALID_ARG, "NULL full pointer");
    if (d->full_grads && !d->full_grads[j]) return fail(FSDP_ERR_INVALID_ARG, "NULL grad pointer");
    if (d->grad_shards && !d->grad_shards[j])
      return fail(FSDP_ERR_INVALID_ARG, "NULL grad shard pointer");
  }
  const int32_t N = ctx->world, r = ctx->rank;
  std::vector<int64_t> ag_off(k), rs_off(k);
  int64_t ag_seg = 0, rs_seg = 0;
  layout(d->params, k, N, ep, d->align_bytes, ag_off.data(), &ag_seg);
  layout(d->params, k, N, 4, d->align_bytes, rs_off.data(), &rs_seg);

  // Segment-layout storage ("zero-copy"): if the caller keeps this rank's
  // shards exactly where its AG segment would hold them (shards[j] ==
  // shards[0] + off_j), the segment already exists in memory: ISSUE needs no
  // pack (the all-gather sends from the storage, out of place) and WAIT reads
  // this rank's rows straight from it.  Likewise gradient shards stored at
  // grad_shards[0] + off'_j let the reduce-scatter write its result in place
  // of the copy-out (with a communicator).  The alignment gaps of such
  // storage are zeroed once here, so the bytes on the wire match the packed
  // form.
  const bool ag_zc = d->flags & FSDP_BUCKET_SEGMENT_SHARDS;
  const bool rs_zc = d->flags & FSDP_BUCKET_SEGMENT_GRAD_SHARDS;
  if ((ag_zc && !d->shards) || (rs_zc && !d->grad_shards))
    return fail(FSDP_ERR_INVALID_ARG, "segment-layout flag without the matching pointer array");
  if ((ag_zc && reinterpret_cast<uintptr_t>(d->shards[0]) % 16) ||
      (rs_zc && reinterpret_cast<uintptr_t>(d->grad_shards[0]) % 16))
    return fail(FSDP_ERR_INVALID_ARG, "segment-layout storage not 16-B aligned");
  for (int32_t j = 0; j < k; ++j) {
    if (ag_zc && reinterpret_cast<uintptr_t>(d->shards[j]) !=
                     reinterpret_cast<uintptr_t>(d->shards[0]) + static_cast<uintptr_t>(ag_off[j]))
      return fail(FSDP_ERR_INVALID_ARG, "FSDP_BUCKET_SEGMENT_SHARDS: shards do not follow the segment offsets");
    if (rs_zc && reinterpret_cast<uintptr_t>(d->grad_shards[j]) !=
                     reinterpret_cast<uintptr_t>(d->grad_shards[0]) + static_cast<uintptr_t>(rs_off[j]))
      return fail(FSDP_ERR_INVALID_ARG,
                  "FSDP_BUCKET_SEGMENT_GRAD_SHARDS: grad shards do not follow the segment offsets");
  }

  // Direct gather: a one-parameter bucket without padding (N | d and no
  // alignment gap) has a gathered buffer byte-identical to the full parameter,
  // so the all-gather writes the full parameter itself -- no staging, no
  // copy-out (the per-parameter collective of the paper's unbucketed graph).
  const bool direct = k == 1 && d->fulls && d->params[0].dim0 % N == 0 &&
                      ag_seg == (d->params[0].dim0 / N) * d->params[0].row_numel * ep;
  // Grouped all-gather (FSDP_BUCKET_GROUPED_AG): one NCCL group of per-member
  // out-of-place all-gathers, shard j -> full j; needs N | d_j for every member.
  const bool grouped = d->flags & FSDP_BUCKET_GROUPED_AG;
  if (grouped) {
    if (!d->shards || !d->fulls || master)
      return fail(FSDP_ERR_INVALID_ARG, "FSDP_BUCKET_GROUPED_AG needs shards and fulls, no FP32_MASTER");
    for (int32_t j = 0; j < k; ++j)
      if (d->params[j].dim0 % N)
        return fail(FSDP_ERR_INVALID_ARG, "FSDP_BUCKET_GROUPED_AG needs every dim0 divisible by the world size");
  }

  TableBuilder pack, unpack, rpack, rcopy, raccum, nvls, gaps, p2p_ag, p2p_rs;
  std::vector<TableBuilder> p2p_ag_by_peer(static_cast<size_t>(N));  // K8 chunks per source rank
  for (int32_t j = 0; j < k; ++j) {
    const fsdp_param_desc& p = d->params[j];
    const ShardRows own = shard_rows(p.dim0, N, r);
    const int64_t R = p.row_numel;
    const int64_t ag_end = (j + 1 < k) ? ag_off[j + 1] : ag_seg;
    const int64_t rs_end = (j + 1 < k) ? rs_off[j + 1] : rs_seg;
    if (d->shards && grouped) {
      // layout-only ctx: this rank's rows straight into the full parameter
      // (with a communicator the group's all-gathers write every row)
      const int64_t nb = own.c * R * ep;
      pack.copy(reinterpret_cast<uint64_t>(d->shards[j]),
                reinterpret_cast<uint64_t>(d->fulls[j]) + static_cast<uint64_t>(r * nb), nb, kAbsDst);
      if (ag_zc)
        gaps.zero(reinterpret_cast<uint64_t>(d->shards[0]) + ag_off[j] + nb, ag_end - ag_off[j] - nb);
    } else if (d->shards && direct) {
      // own rows straight into the full parameter (used unless the collective
      // sends from segment storage itself)
      const uint64_t src = reinterpret_cast<uint64_t>(d->shards[0]);
      const uint64_t dst = reinterpret_cast<uint64_t>(d->fulls[0]) + static_cast<uint64_t>(r * ag_seg);
      if (master) pack.narrow(src, dst, ag_seg / 2, kAbsDst);
      else pack.copy(src, dst, ag_seg, kAbsDst);
    } else if (d->shards) {
      const int64_t nb = own.c * R * ep;
      if (ag_zc) {
        gaps.zero(reinterpret_cast<uint64_t>(d->shards[0]) + ag_off[j] + nb, ag_end - ag_off[j] - nb);
      } else {
        // K1: this rank's whole padded shard into segment r, alignment gap zeroed
        // (fp32 master shards rounded to bf16 on the way).
        const uint64_t dst = static_cast<uint64_t>(r * ag_seg + ag_off[j]);
        if (master) pack.narrow(reinterpret_cast<uint64_t>(d->shards[j]), dst, own.c * R);
        else pack.copy(reinterpret_cast<uint64_t>(d->shards[j]), dst, nb);
        pack.zero(dst + nb, ag_end - ag_off[j] - nb);
      }
    }
    if (rs_zc) {
      const int64_t nb = own.c * R * 4;
      gaps.zero(reinterpret_cast<uint64_t>(d->grad_shards[0]) + rs_off[j] + nb, rs_end - rs_off[j] - nb);
    }
    for (int32_t q = 0; q < N; ++q) {
      const ShardRows s = shard_rows(p.dim0, N, q);
      if (d->fulls && s.v > 0 && !direct && !grouped) {
        // K3: valid rows of rank q's chunk -> rows [q c, q c + v) of the full param
        // (this rank's rows from its segment-layout storage when zero-copy).
        const uint64_t dst = reinterpret_cast<uint64_t>(d->fulls[j]) + static_cast<uint64_t>(s.begin * R * ep);
        if (ag_zc && q == r)
          unpack.copy(reinterpret_cast<uint64_t>(d->shards[j]), dst, s.v * R * ep, kAbsSrc);
        else
          unpack.copy(static_cast<uint64_t>(q * ag_seg + ag_off[j]), dst, s.v * R * ep);
      }
      if (d->full_grads) {
        // K4: rows of chunk q, widened and scaled, into segment q; pads +0.0.
        const uint64_t dst = static_cast<uint64_t>(q * rs_seg + rs_off[j]);
        const uint64_t src = reinterpret_cast<uint64_t>(d->full_grads[j]) +
                             static_cast<uint64_t>(s.begin * R * eg);
        if (eg == 2) rpack.widen(src, dst, s.v * R);
        else rpack.scale(src, dst, s.v * R);
        rpack.zero(dst + s.v * R * 4, rs_end - rs_off[j] - s.v * R * 4);
      }
    }
    if (ag_zc && d->fulls) {
      // K8 (peer-memory AG): valid rows of rank q's shard, read at offset off_j of
      // rank q's segment storage, into rows [q c, q c + v) of the full param.
      for (int32_t q = 0; q < N; ++q) {
        const ShardRows s = shard_rows(p.dim0, N, q);
        if (s.v > 0)
          p2p_ag_by_peer[q].copy(static_cast<uint64_t>(ag_off[j]),
                                 reinterpret_cast<uint64_t>(d->fulls[j]) + static_cast<uint64_t>(s.begin * R * ep),
                                 s.v * R * ep, static_cast<uint32_t>(q) << kPeerShift);
      }
    }
    if (d->full_grads && d->grad_shards && !gs_bf16) {
      // K9 (peer-memory RS): rows of chunk r at the same offset from full_grads[0]
      // on every rank, summed in rank order into the fp32 shard; pad rows +0.0.
      const uint64_t rel = reinterpret_cast<uint64_t>(d->full_grads[j]) - reinterpret_cast<uint64_t>(d->full_grads[0]);
      const uint64_t dst = reinterpret_cast<uint64_t>(d->grad_shards[j]);
      p2p_rs.peer_reduce(rel + static_cast<uint64_t>(own.begin * R * eg), dst, own.v * R, eg, N);
      p2p_rs.zero(dst + static_cast<uint64_t>(own.v * R * 4), (own.c - own.v) * R * 4);
    }
    if (d->grad_shards && gs_bf16) {
      // K6: own segment r -> bf16 gradient shard [c, R], one RNE rounding (G41)
      rcopy.narrow(static_cast<uint64_t>(r * rs_seg + rs_off[j]), reinterpret_cast<uint64_t>(d->grad_shards[j]),
                   own.c * R);
    } else if (d->grad_shards) {
      // K6: own segment r -> fp32 gradient shard [c, R].
      rcopy.copy(static_cast<uint64_t>(r * rs_seg + rs_off[j]),
                 reinterpret_cast<uint64_t>(d->grad_shards[j]), own.c * R * 4);
      // K6 in accumulation mode: grad shard += own segment (pad rows add +0.0)
      raccum.accum(static_cast<uint64_t>(r * rs_seg + rs_off[j]),
                   reinterpret_cast<uint64_t>(d->grad_shards[j]), own.c * R);
      // K10 (NVLS): own segment summed across GPUs by the switch -> grad shard
      nvls.nvls(static_cast<uint64_t>(r * rs_seg + rs_off[j]), reinterpret_cast<uint64_t>(d->grad_shards[j]),
                own.c * R);
    }
  }
  // K8 chunk order: round-robin over the source ranks, starting at this rank's
  // successor.  CTAs take chunks in table order, so at any moment a rank reads
  // from every peer at once and the ranks start on different peers -- no
  // peer's NVLink egress is the one all N - 1 readers queue on (as with every
  // rank walking the sources 0, 1, ... in step).
  // Runs of kPeerRun consecutive chunks (256 KiB) keep each source's reads
  // and each destination's writes DRAM-page friendly.
  {
    constexpr size_t kPeerRun = 8;
    std::vector<size_t> next(static_cast<size_t>(N), 0);
    for (bool more = true; more;) {
      more = false;
      for (int32_t t = 1; t <= N; ++t) {
        const int32_t q = (r + t) % N;
        TableBuilder& src = p2p_ag_by_peer[q];
        for (size_t u = 0; u < kPeerRun && next[q] < src.chunks.size(); ++u) {
          p2p_ag.chunks.push_back(src.chunks[next[q]++]);
          more = true;
        }
      }
    }
    for (const TableBuilder& tb : p2p_ag_by_peer) p2p_ag.bytes_moved += tb.bytes_moved;
  }
  FSDP_CUDA_TRY(cudaSetDevice(ctx->device));
  fsdp_bucket* b = new fsdp_bucket();
  b->ctx = ctx;
  b->device = ctx->device;
  b->k = k;
  b->ag_seg = ag_seg;
  b->rs_seg = rs_seg;
  b->param_bytes = ep;
  b->grad_bytes = eg;
  b->has_shards = d->shards != nullptr;
  b->has_fulls = d->fulls != nullptr;
  b->has_grads = d->full_grads != nullptr;
  b->has_gshards = d->grad_shards != nullptr;
  b->ag_zero_copy = ag_zc;
  b->rs_zero_copy = rs_zc;
  b->ag_direct = direct;
  b->ag_grouped = grouped;
  b->gshard_bf16 = gs_bf16;
  if (grouped)
    for (int32_t j = 0; j < k; ++j) {
      b->shard_ptrs.push_back(d->shards[j]);
      b->own_bytes.push_back((d->params[j].dim0 / N) * d->params[j].row_numel * ep);
    }
  b->full0 = d->fulls ? static_cast<char*>(d->fulls[0]) : nullptr;
  b->members.assign(d->params, d->params + k);
  for (int32_t j = 0; j < k; ++j) {
    b->fulls.push_back(d->fulls ? d->fulls[j] : nullptr);
    b->grads.push_back(d->full_grads ? const_cast<void*>(d->full_grads[j]) : nullptr);
  }
  b->shard_seg = ag_zc ? static_cast<char*>(d->shards[0]) : nullptr;
  b->gshard_seg = rs_zc ? static_cast<char*>(d->grad_shards[0]) : nullptr;
  fsdp_status st = FSDP_OK;
  if (!gaps.chunks.empty()) {
    // one-time zero fill of the storage's alignment gaps (setup, synchronous)
    DevTable g;
    st = upload(gaps, &g);
    if (st == FSDP_OK) {
      cudaError_t e = launch_table(KK_SHARD, g, nullptr, 1.0f, nullptr, ctx->max_ctas);
      if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
      if (e != cudaSuccess) st = fail(FSDP_ERR_CUDA, std::string("gap fill: ") + cudaGetErrorString(e));
    }
    release(&g);
  }
  if (st == FSDP_OK) st = upload(pack, &b->ag_pack);
  if (st == FSDP_OK) st = upload(unpack, &b->ag_unpack);
  if (st == FSDP_OK) st = upload(rpack, &b->rs_pack);
  if (st == FSDP_OK) st = upload(rcopy, &b->rs_copyout);
  if (st == FSDP_OK) st = upload(raccum, &b->rs_accum);
  if (st == FSDP_OK) st = upload(nvls, &b->nvls_rs);
  if (st == FSDP_OK && N <= kMaxPeers) st = upload(p2p_ag, &b->p2p_ag);
  if (st == FSDP_OK && N <= kMaxPeers) st = upload(p2p_rs, &b->p2p_rs);
  for (cudaEvent_t* e : {&b->ev_ag_packed, &b->ev_ag_done, &b->ev_rs_packed, &b->ev_rs_done, &b->ev_d2h_done}) {
    if (st != FSDP_OK) break;
    cudaError_t err = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    if (err != cudaSuccess) st = fail(FSDP_ERR_CUDA, cudaGetErrorString(err));
  }
  if (st != FSDP_OK) {
    destroy_bucket(b);
    return st;
  }
  if (ag_seg_bytes) *ag_seg_bytes = ag_seg;
  if (rs_seg_bytes) *rs_seg_bytes = rs_seg;
  *out = b;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_bucket_query(const fsdp_bucket* b, fsdp_bucket_info* out) {
  if (!b || !out) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  out->ag_seg_bytes = b->ag_seg;
  out->rs_seg_bytes = b->rs_seg;
  const fsdp::DevTable* t[4] = {&b->ag_pack, &b->ag_unpack, &b->rs_pack, &b->rs_copyout};
  for (int i = 0; i < 4; ++i) {
    out->kernel_bytes[i] = t[i]->n ? t[i]->bytes_moved : 0;
    out->kernel_chunks[i] = t[i]->n;
  }
  // with a communicator and zero-copy RS storage the copy-out never launches
  if (b->rs_zero_copy && b->ctx && b->ctx->comm) out->kernel_bytes[3] = 0;
  out->ag_zero_copy = b->ag_zero_copy ? 1 : 0;
  out->rs_zero_copy = b->rs_zero_copy ? 1 : 0;
  out->p2p_bytes[0] = b->p2p_ag.n ? b->p2p_ag.bytes_moved : 0;
  out->p2p_bytes[1] = b->p2p_rs.n ? b->p2p_rs.bytes_moved : 0;
  out->ag_direct = b->ag_direct ? 1 : 0;
  // a direct bucket with segment storage and a communicator never packs
  if (b->ag_direct && b->ag_zero_copy && b->ctx && b->ctx->comm) out->kernel_bytes[0] = 0;
  // a grouped bucket with a communicator never packs (the group sends from the shards)
  if (b->ag_grouped && b->ctx && b->ctx->comm) out->kernel_bytes[0] = 0;
  out->ag_grouped = b->ag_grouped ? 1 : 0;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_bucket_destroy(fsdp_bucket* b) {
  if (!b) return FSDP_OK;
  cudaSetDevice(b->device);
  destroy_bucket(b);
  return FSDP_OK;
}

namespace fsdp {

// Per-bucket steps, shared by the public calls and the schedule executor.
// `launches` / `colls` (nullable) count enqueued kernels / collectives;
// with_comm = false (FSDP_SCHED_NO_COMM) skips collectives and waits.
static bool comm_on(fsdp_ctx* c, bool with_comm) { return with_comm && (c->comm != nullptr || c->emul != nullptr); }

fsdp_status ag_pack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches) {
  // segment storage: the collective sends from it, no pack -- except for a
  // direct-gather bucket when no collective will write this rank's rows
  const bool skip = b->ag_grouped  ? comm_on(c, with_comm)
                    : b->ag_direct ? (b->ag_zero_copy && comm_on(c, with_comm))
                                   : b->ag_zero_copy;
  if (!skip) {
    FSDP_CUDA_TRY(launch_table(KK_AG_PACK, b->ag_pack, staging, 1.0f, cs, c->max_ctas));
    if (b->ag_pack.n && launches) ++*launches;
  }
  // the collective starts after everything enqueued on compute so far
  if (comm_on(c, with_comm)) FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_packed, cs));
  return FSDP_OK;
}

fsdp_status ag_collective(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t ms, bool with_comm, int* colls) {
  if (!comm_on(c, with_comm)) return FSDP_OK;
  FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, b->ev_ag_packed, 0));
  if (b->ag_grouped) {
    // one NCCL group: shard j (this rank's c_j rows) -> rows of every rank in full j
    FSDP_NCCL_TRY(ncclGroupStart());
    for (size_t j = 0; j < b->shard_ptrs.size(); ++j) {
      ncclResult_t r = ncclAllGather(b->shard_ptrs[j], b->fulls[j], static_cast<size_t>(b->own_bytes[j]), ncclInt8,
                                     c->comm, ms);
      if (r != ncclSuccess) {
        ncclGroupEnd();
        return fail(FSDP_ERR_NCCL, std::string("ncclAllGather (grouped): ") + ncclGetErrorString(r));
      }
    }
    FSDP_NCCL_TRY(ncclGroupEnd());
    FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_done, ms));
    if (colls) ++*colls;
    return FSDP_OK;
  }
  // In place (sendbuff = recvbuff + rank * sendcount), or out of place from
  // segment-layout shard storage; bytes as ncclInt8.
  // A direct-gather bucket gathers into the full parameter itself.
  char* recv = b->ag_direct ? b->full0 : staging;
  const char* send = b->ag_zero_copy ? b->shard_seg : recv + c->rank * b->ag_seg;
  if (!c->comm) {  // emulated collective (fsdp_comm_emulation): K11 on the comm stream
    int64_t ns = 0;
    FSDP_TRY(fsdp_comm_time_ns(c->world * b->ag_seg, &c->emul->ag, &ns));
    FSDP_CUDA_TRY(launch_comm_emulation(false, send, recv, b->ag_seg, c->world, c->rank, ns, c->emul->ctas, ms));
    FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_done, ms));
    if (colls) ++*colls;
    return FSDP_OK;
  }
  FSDP_NCCL_TRY(ncclAllGather(send, recv, static_cast<size_t>(b->ag_seg), ncclInt8, c->comm, ms));
  FSDP_CUDA_TRY(cudaEventRecord(b->ev_ag_done, ms));
  if (colls) ++*colls;
  return FSDP_OK;
}

// Asynchronous NCCL failures (a peer died, a network error) surface here, at
// every WAIT and at the end of each scheduled step.
fsdp_status check_async_error(fsdp_ctx* c) {
  if (!c->comm) return FSDP_OK;
  ncclResult_t ae = ncclSuccess;
  FSDP_NCCL_TRY(ncclCommGetAsyncError(c->comm, &ae));
  if (ae != ncclSuccess && ae != ncclInProgress)
    return fail(FSDP_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ae));
  return FSDP_OK;
}

fsdp_status ag_wait(fsdp_ctx* c, fsdp_bucket* b, cudaStream_t cs, bool with_comm) {
  if (comm_on(c, with_comm)) {
    FSDP_TRY(check_async_error(c));
    FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, b->ev_ag_done, 0));
  }
  return FSDP_OK;
}

fsdp_status ag_unpack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, int* launches) {
  FSDP_CUDA_TRY(launch_table(KK_AG_UNPACK, b->ag_unpack, staging, 1.0f, cs, c->max_ctas));
  if (b->ag_unpack.n && launches) ++*launches;
  return FSDP_OK;
}

fsdp_status rs_pack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches) {
  const float inv = 1.0f / static_cast<float>(c->world);  // fl32(1/N), correctly rounded
  b->rs_accum_issued = b->grad_accumulate;  // latched for the matching collective / copy-out
  FSDP_CUDA_TRY(launch_table(KK_RS_PACK, b->rs_pack, staging, inv, cs, c->max_ctas));
  if (b->rs_pack.n && launches) ++*launches;
  if (comm_on(c, with_comm)) FSDP_CUDA_TRY(cudaEventRecord(b->ev_rs_packed, cs));
  return FSDP_OK;
}

fsdp_status rs_collective(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t ms, bool with_comm, int* colls) {
  if (!comm_on(c, with_comm)) return FSDP_OK;
  FSDP_CUDA_TRY(cudaStreamWaitEvent(ms, b->ev_rs_packed, 0));
  // fp32 sum of pre-scaled chunks; in place (recvbuff = sendbuff + rank *
  // recvcount) or straight into segment-layout gradient-shard storage.
  // (accumulation needs the result beside the shards, so it goes to staging)
  char* recv = (b->rs_zero_copy && !b->rs_accum_issued) ? b->gshard_seg : staging + c->rank * b->rs_seg;
  if (!c->comm) {  // emulated collective (fsdp_comm_emulation): K11 on the comm stream
    int64_t ns = 0;
    FSDP_TRY(fsdp_comm_time_ns(c->world * b->rs_seg, &c->emul->rs, &ns));
    FSDP_CUDA_TRY(launch_comm_emulation(true, staging, recv, b->rs_seg, c->world, c->rank, ns, c->emul->ctas, ms));
    FSDP_CUDA_TRY(cudaEventRecord(b->ev_rs_done, ms));
    if (colls) ++*colls;
    return FSDP_OK;
  }
  FSDP_NCCL_TRY(ncclReduceScatter(staging, recv, static_cast<size_t>(b->rs_seg / 4), ncclFloat32, ncclSum,
                                  c->comm, ms));
  FSDP_CUDA_TRY(cudaEventRecord(b->ev_rs_done, ms));
  if (colls) ++*colls;
  return FSDP_OK;
}

fsdp_status rs_wait(fsdp_ctx* c, fsdp_bucket* b, cudaStream_t cs, bool with_comm) {
  if (comm_on(c, with_comm)) {
    FSDP_TRY(check_async_error(c));
    FSDP_CUDA_TRY(cudaStreamWaitEvent(cs, b->ev_rs_done, 0));
  }
  return FSDP_OK;
}

fsdp_status rs_copyout(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches) {
  // with a communicator and segment-layout storage the collective already
  // wrote the result in place: nothing to copy
  if (b->rs_accum_issued) {
    FSDP_CUDA_TRY(launch_table(KK_RS_COPYOUT, b->rs_accum, staging, 1.0f, cs, c->max_ctas));
    if (b->rs_accum.n && launches) ++*launches;
    return FSDP_OK;
  }
  if (b->rs_zero_copy && comm_on(c, with_comm)) return FSDP_OK;
  FSDP_CUDA_TRY(launch_table(KK_RS_COPYOUT, b->rs_copyout, staging, 1.0f, cs, c->max_ctas));
  if (b->rs_copyout.n && launches) ++*launches;
  return FSDP_OK;
}

cudaStream_t resolve_comm(fsdp_ctx* c, fsdp_stream_t s) { return comm_stream(c, s); }

}  // namespace fsdp

static fsdp_status check_call(fsdp_ctx* c, fsdp_bucket* b, void* staging, uint32_t flags) {
  if (!c || !b || !staging) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (b->ctx != c) return fail(FSDP_ERR_INVALID_ARG, "bucket belongs to another ctx");
  if (reinterpret_cast<uintptr_t>(staging) % 16) return fail(FSDP_ERR_INVALID_ARG, "staging not 16-B aligned");
  if (!(flags & 3u) || (flags & ~7u) || ((flags & FSDP_NO_COLLECTIVE) && (flags & FSDP_WAIT)))
    return fail(FSDP_ERR_INVALID_ARG, "flags must be ISSUE and/or WAIT (NO_COLLECTIVE only with ISSUE alone)");
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_allgather_bucket(fsdp_ctx* c, fsdp_bucket* b, void* staging,
                                             fsdp_stream_t compute, fsdp_stream_t comm, uint32_t flags) {
  FSDP_TRY(check_call(c, b, staging, flags));
  if ((flags & FSDP_ISSUE) && !b->has_shards) return fail(FSDP_ERR_INVALID_ARG, "ISSUE needs bound shards");
  if ((flags & FSDP_WAIT) && !b->has_fulls) return fail(FSDP_ERR_INVALID_ARG, "WAIT needs bound fulls");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t cs = static_cast<cudaStream_t>(compute);
  cudaStream_t ms = resolve_comm(c, comm);
  char* st = static_cast<char*>(staging);
  if (flags & FSDP_ISSUE) {
    const bool coll = !(flags & FSDP_NO_COLLECTIVE);
    FSDP_TRY(ag_pack(c, b, st, cs, coll, nullptr));
    FSDP_TRY(ag_collective(c, b, st, ms, coll, nullptr));
  }
  if (flags & FSDP_WAIT) {
    FSDP_TRY(ag_wait(c, b, cs, true));
    FSDP_TRY(ag_unpack(c, b, st, cs, nullptr));
  }
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_reduce_scatter_bucket(fsdp_ctx* c, fsdp_bucket* b, void* staging,
                                                  fsdp_stream_t compute, fsdp_stream_t comm,
                                                  uint32_t flags) {
  FSDP_TRY(check_call(c, b, staging, flags));
  if ((flags & FSDP_ISSUE) && !b->has_grads) return fail(FSDP_ERR_INVALID_ARG, "ISSUE needs bound full_grads");
  if ((flags & FSDP_WAIT) && !b->has_gshards) return fail(FSDP_ERR_INVALID_ARG, "WAIT needs bound grad_shards");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t cs = static_cast<cudaStream_t>(compute);
  cudaStream_t ms = resolve_comm(c, comm);
  char* st = static_cast<char*>(staging);
  if (flags & FSDP_ISSUE) {
    const bool coll = !(flags & FSDP_NO_COLLECTIVE);
    FSDP_TRY(rs_pack(c, b, st, cs, coll, nullptr));
    FSDP_TRY(rs_collective(c, b, st, ms, coll, nullptr));
  }
  if (flags & FSDP_WAIT) {
    FSDP_TRY(rs_wait(c, b, cs, true));
    FSDP_TRY(rs_copyout(c, b, st, cs, true, nullptr));
  }
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_bucket_launch_kernel(fsdp_ctx* c, fsdp_bucket* b, int32_t op, void* staging,
                                                 fsdp_stream_t stream, int32_t* launched) {
  if (launched) *launched = 0;
  if (!c || !b || !staging) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (b->ctx != c) return fail(FSDP_ERR_INVALID_ARG, "bucket belongs to another ctx");
  if (reinterpret_cast<uintptr_t>(staging) % 16) return fail(FSDP_ERR_INVALID_ARG, "staging not 16-B aligned");
  const bool ag = op == FSDP_OP_PACK_AG || op == FSDP_OP_UNPACK;
  if (!ag && op != FSDP_OP_PACK_RS && op != FSDP_OP_COPYOUT_RS)
    return fail(FSDP_ERR_INVALID_ARG, "op must be PACK_AG, UNPACK, PACK_RS or COPYOUT_RS");
  if ((op == FSDP_OP_PACK_AG && !b->has_shards) || (op == FSDP_OP_UNPACK && !b->has_fulls) ||
      (op == FSDP_OP_PACK_RS && !b->has_grads) || (op == FSDP_OP_COPYOUT_RS && !b->has_gshards))
    return fail(FSDP_ERR_INVALID_ARG, "the op's buffers are not bound");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  char* st = static_cast<char*>(staging);
  int n = 0;
  switch (op) {
    case FSDP_OP_PACK_AG: {
      // the step's skip rule (ag_pack) with the ctx's collective state
      const bool coll = comm_on(c, true);
      const bool skip = b->ag_grouped ? coll : b->ag_direct ? (b->ag_zero_copy && coll) : b->ag_zero_copy;
      if (!skip) {
        FSDP_CUDA_TRY(launch_table(KK_AG_PACK, b->ag_pack, st, 1.0f, cs, c->max_ctas));
        n = b->ag_pack.n ? 1 : 0;
      }
      break;
    }
    case FSDP_OP_UNPACK:
      FSDP_TRY(ag_unpack(c, b, st, cs, &n));
      break;
    case FSDP_OP_PACK_RS:
      FSDP_CUDA_TRY(launch_table(KK_RS_PACK, b->rs_pack, st, 1.0f / static_cast<float>(c->world), cs, c->max_ctas));
      n = b->rs_pack.n ? 1 : 0;
      break;
    default:
      FSDP_TRY(rs_copyout(c, b, st, cs, true, &n));
  }
  if (launched) *launched = n;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_bucket_set_grad_accumulation(fsdp_bucket* b, int32_t on) {
  if (!b) return fail(FSDP_ERR_INVALID_ARG, "NULL bucket");
  if (on != 0 && on != 1) return fail(FSDP_ERR_INVALID_ARG, "on must be 0 or 1");
  if (on && b->gshard_bf16)
    return fail(FSDP_ERR_INVALID_ARG, "gradient accumulation needs fp32 gradient shards (FSDP_BUCKET_BF16_GRAD_SHARDS)");
  b->grad_accumulate = on != 0;
  return FSDP_OK;
}
