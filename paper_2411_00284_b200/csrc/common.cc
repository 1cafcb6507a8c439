// Errors, shard math, bucket layout, run tables,
// context, and fsdp_shard / fsdp_layout.
#include <algorithm>
#include <cstring>

#include "internal.h"

namespace fsdp {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }

fsdp_status fail(fsdp_status st, const std::string& msg) {
  g_error = msg;
  return st;
}

ShardRows shard_rows(int64_t d, int32_t world, int32_t rank) {
  ShardRows s;
  s.c = (d + world - 1) / world;
  int64_t start = static_cast<int64_t>(rank) * s.c;
  s.v = std::max<int64_t>(0, std::min<int64_t>(d - start, s.c));
  s.begin = std::min<int64_t>(start, d);
  return s;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

int32_t dtype_bytes(int32_t dt) {
  if (dt == FSDP_BF16) return 2;
  if (dt == FSDP_FP32) return 4;
  return 0;
}

void layout(const fsdp_param_desc* m, int32_t k, int32_t world, int64_t e, int64_t a, int64_t* offs,
            int64_t* seg) {
  int64_t cur = 0;
  for (int32_t j = 0; j < k; ++j) {
    if (offs) offs[j] = cur;
    int64_t c = (m[j].dim0 + world - 1) / world;
    cur = align_up(cur + c * m[j].row_numel * e, a);
  }
  *seg = cur;
}

// Largest power-of-two unit <= 16 dividing all three values.
static uint32_t unit_of(uint64_t a, uint64_t b, uint64_t n) {
  uint64_t x = a | b | n;
  for (uint32_t u = 16; u > 1; u >>= 1)
    if ((x & (u - 1)) == 0) return u;
  return 1;
}

static void push(std::vector<Chunk>& v, uint64_t src, uint64_t dst, uint32_t n, uint32_t op,
                 uint32_t unit) {
  Chunk c;
  c.src = src;
  c.dst = dst;
  c.n = n;
  c.op_unit = op | (unit << 8);
  v.push_back(c);
}

void TableBuilder::copy(uint64_t src, uint64_t dst, int64_t bytes, uint32_t flags) {
  if (bytes <= 0) return;
  bytes_moved += 2 * bytes;
  uint32_t u = unit_of(src, dst, static_cast<uint64_t>(bytes));
  for (int64_t off = 0; off < bytes; off += kChunkBytes) {
    int64_t nb = std::min<int64_t>(kChunkBytes, bytes - off);
    push(chunks, src + off, dst + off, static_cast<uint32_t>(nb / u), OP_COPY | flags, u);
  }
}

void TableBuilder::zero(uint64_t dst, int64_t bytes) {
  if (bytes <= 0) return;
  bytes_moved += bytes;
  uint32_t u = unit_of(0, dst, static_cast<uint64_t>(bytes));
  for (int64_t off = 0; off < bytes; off += kChunkBytes) {
    int64_t nb = std::min<int64_t>(kChunkBytes, bytes - off);
    push(chunks, 0, dst + off, static_cast<uint32_t>(nb / u), OP_ZERO, u);
  }
}

// bf16 src (2 B/elem) -> fp32 dst (4 B/elem).  Vector body when both ends are
// 16-B aligned: groups of 8 elements (16 B in, 32 B out); scalar tail.
void TableBuilder::widen(uint64_t src, uint64_t dst, int64_t elems) {
  if (elems <= 0) return;
  bytes_moved += 6 * elems;
  int64_t body = 0;
  if (src % 16 == 0 && dst % 16 == 0) body = elems / 8 * 8;
  const int64_t per_chunk = kChunkBytes / 4;  // elems per chunk (32 KiB of fp32 out)
  for (int64_t e = 0; e < body; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + 2 * e, dst + 4 * e, static_cast<uint32_t>(ne / 8), OP_WIDEN, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + 2 * e, dst + 4 * e, static_cast<uint32_t>(ne), OP_WIDEN, 2);
  }
}

void TableBuilder::scale(uint64_t src, uint64_t dst, int64_t elems) {
  if (elems <= 0) return;
  bytes_moved += 8 * elems;
  int64_t body = 0;
  if (src % 16 == 0 && dst % 16 == 0) body = elems / 4 * 4;
  const int64_t per_chunk = kChunkBytes / 4;
  for (int64_t e = 0; e < body; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne / 4), OP_SCALE, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne), OP_SCALE, 4);
  }
}

// fp32 src (4 B/elem) -> bf16 dst (2 B/elem), round to nearest even.  Vector
// body: groups of 8 elements (32 B in, 16 B out) when both ends are 16-B
// aligned; scalar tail.
void TableBuilder::narrow(uint64_t src, uint64_t dst, int64_t elems, uint32_t flags) {
  if (elems <= 0) return;
  bytes_moved += 6 * elems;
  int64_t body = 0;
  if (src % 16 == 0 && dst % 16 == 0) body = elems / 8 * 8;
  const int64_t per_chunk = kChunkBytes / 4;  // elems per chunk (32 KiB of fp32 in)
  for (int64_t e = 0; e < body; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + 4 * e, dst + 2 * e, static_cast<uint32_t>(ne / 8), OP_NARROW | flags, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + 4 * e, dst + 2 * e, static_cast<uint32_t>(ne), OP_NARROW | flags, 4);
  }
}

// fp32 dst = dst + src (gradient accumulation): 12 B per element.
void TableBuilder::accum(uint64_t src, uint64_t dst, int64_t elems) {
  if (elems <= 0) return;
  bytes_moved += 12 * elems;
  int64_t body = 0;
  if (src % 16 == 0 && dst % 16 == 0) body = elems / 4 * 4;
  const int64_t per_chunk = kChunkBytes / 4;
  for (int64_t e = 0; e < body; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne / 4), OP_ACCUM, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne), OP_ACCUM, 4);
  }
}

// K10 (NVLS): fp32 elements reduced by the switch; 4 B read per rank
// through the multicast address (counted once, the local copy) + 4 B written.
void TableBuilder::nvls(uint64_t src, uint64_t dst, int64_t elems) {
  if (elems <= 0) return;
  bytes_moved += 8 * elems;
  int64_t body = 0;
  if (src % 16 == 0 && dst % 16 == 0) body = elems / 4 * 4;
  const int64_t per_chunk = kChunkBytes / 4;
  for (int64_t e = 0; e < body; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne / 4), OP_NVLS, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + 4 * e, dst + 4 * e, static_cast<uint32_t>(ne), OP_NVLS, 4);
  }
}

void TableBuilder::peer_reduce(uint64_t src, uint64_t dst, int64_t elems, int eb, int world) {
  if (elems <= 0) return;
  bytes_moved += elems * (static_cast<int64_t>(eb) * world + 4);  // every peer's elements + fp32 write
  const uint32_t op = eb == 2 ? OP_PEER_REDUCE_BF16 : OP_PEER_REDUCE_F32;
  const int64_t g = eb == 2 ? 8 : 4;  // elements per 16-B load
  const int64_t body = (src % 16 == 0 && dst % 16 == 0) ? elems / g * g : 0;
  const int64_t per_chunk = kChunkBytes / 4;  // fp32 outputs per chunk
  for (int64_t e = 0; e < body; e += per_chunk) {
    const int64_t ne = std::min<int64_t>(per_chunk, body - e);
    push(chunks, src + eb * e, dst + 4 * e, static_cast<uint32_t>(ne / g), op, 16);
  }
  for (int64_t e = body; e < elems; e += per_chunk) {
    const int64_t ne = std::min<int64_t>(per_chunk, elems - e);
    push(chunks, src + eb * e, dst + 4 * e, static_cast<uint32_t>(ne), op, static_cast<uint32_t>(eb));
  }
}

fsdp_status upload(const TableBuilder& tb, DevTable* out) {
  out->n = static_cast<int32_t>(tb.chunks.size());
  out->bytes_moved = tb.bytes_moved;
  out->d = nullptr;
  if (tb.chunks.size() > static_cast<size_t>(INT32_MAX))
    return fail(FSDP_ERR_UNSUPPORTED, "run table too large");
  if (out->n == 0) return FSDP_OK;
  size_t bytes = tb.chunks.size() * sizeof(Chunk);
  FSDP_CUDA_TRY(cudaMalloc(&out->d, bytes));
  FSDP_CUDA_TRY(cudaMemcpy(out->d, tb.chunks.data(), bytes, cudaMemcpyHostToDevice));
  return FSDP_OK;
}

void release(DevTable* t) {
  if (t->d) cudaFree(t->d);
  t->d = nullptr;
  t->n = 0;
}

static bool valid_desc(const fsdp_param_desc& p) {
  return p.dim0 >= 1 && p.row_numel >= 1 && p.reserved == 0;
}

}  // namespace fsdp

using namespace fsdp;

extern "C" {

const char* fsdp_last_error(void) { return g_error.c_str(); }

int32_t fsdp_abi_version(void) { return FSDP_ABI_VERSION; }

fsdp_status fsdp_nccl_get_unique_id(void* uid128) {
  if (!uid128) return fail(FSDP_ERR_INVALID_ARG, "uid128 is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId id;
  FSDP_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(uid128, &id, sizeof(id));
  return FSDP_OK;
}

static fsdp_status ctx_create(fsdp_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                              const void* nccl_uid, void* borrowed_comm, const fsdp_nccl_config* cfg) {
  if (!out) return fail(FSDP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(FSDP_ERR_INVALID_ARG, "bad world/rank");
  if (nccl_uid && borrowed_comm)
    return fail(FSDP_ERR_INVALID_ARG, "give either nccl_uid or borrowed_comm, not both");
  int ndev = 0;
  FSDP_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(FSDP_ERR_INVALID_ARG, "bad cuda_device");
  FSDP_CUDA_TRY(cudaSetDevice(cuda_device));
  FSDP_CUDA_TRY(preload_kernels());
  fsdp_ctx* c = new fsdp_ctx();
  c->world = world;
  c->rank = rank;
  c->device = cuda_device;
  c->sm_count = device_sm_count(cuda_device);
  if (c->sm_count <= 0) c->sm_count = 148;
  c->max_ctas = c->sm_count * FSDP_CTAS_PER_SM;
  // proxy sink (4096 floats) followed by the fused-K9 grid counter (zeroed)
  cudaError_t e = cudaMalloc(&c->sink, 4096 * sizeof(float) + 256);
  if (e == cudaSuccess) {
    c->p2p_counter = reinterpret_cast<unsigned int*>(c->sink + 4096);
    e = cudaMemset(c->p2p_counter, 0, 256);
  }
  if (e != cudaSuccess) {
    if (c->sink) cudaFree(c->sink);
    delete c;
    return fail(FSDP_ERR_CUDA, std::string("cudaMalloc sink: ") + cudaGetErrorString(e));
  }
  if (nccl_uid) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_uid, sizeof(id));
    ncclResult_t r;
    if (cfg) {
      ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
      if (cfg->min_ctas > 0) nc.minCTAs = cfg->min_ctas;
      if (cfg->max_ctas > 0) nc.maxCTAs = cfg->max_ctas;
      if (cfg->nvls_ctas > 0) nc.nvlsCTAs = cfg->nvls_ctas;
      if (cfg->cta_policy >= 0) nc.CTAPolicy = cfg->cta_policy;
      r = ncclCommInitRankConfig(&c->comm, world, id, rank, &nc);
    } else {
      r = ncclCommInitRank(&c->comm, world, id, rank);
    }
    if (r != ncclSuccess) {
      cudaFree(c->sink);
      delete c;
      return fail(FSDP_ERR_NCCL, std::string(cfg ? "ncclCommInitRankConfig: " : "ncclCommInitRank: ") +
                                     ncclGetErrorString(r));
    }
    c->owns_comm = true;
  } else if (borrowed_comm) {
    c->comm = static_cast<ncclComm_t>(borrowed_comm);
  }
  *out = c;
  return FSDP_OK;
}

fsdp_status fsdp_ctx_create(fsdp_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                            const void* nccl_uid, void* borrowed_comm) {
  return ctx_create(out, world, rank, cuda_device, nccl_uid, borrowed_comm, nullptr);
}

fsdp_status fsdp_ctx_create_config(fsdp_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                                   const void* nccl_uid, const fsdp_nccl_config* cfg) {
  if (cfg) {
    if (!nccl_uid) return fail(FSDP_ERR_INVALID_ARG, "an NCCL config needs nccl_uid (the library builds the comm)");
    if (cfg->min_ctas > 0 && cfg->max_ctas > 0 && cfg->min_ctas > cfg->max_ctas)
      return fail(FSDP_ERR_INVALID_ARG, "min_ctas > max_ctas");
  }
  return ctx_create(out, world, rank, cuda_device, nccl_uid, nullptr, cfg);
}

fsdp_status fsdp_nccl_estimate_ns(fsdp_ctx* c, int32_t op, int64_t full_bytes, int64_t* ns) {
  if (!c || !ns) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (!c->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_nccl_estimate_ns needs a ctx with a communicator");
  if (op != FSDP_OP_AG && op != FSDP_OP_RS) return fail(FSDP_ERR_INVALID_ARG, "op must be FSDP_OP_AG or FSDP_OP_RS");
  const int64_t es = op == FSDP_OP_AG ? 2 : 4;
  if (full_bytes < 0 || full_bytes % (c->world * es)) return fail(FSDP_ERR_INVALID_ARG, "bad full_bytes");
  const size_t per_rank = static_cast<size_t>(full_bytes / c->world / es);
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  // nothing is launched: any non-NULL device pointer stands in for the buffers
  void* dummy = c->sink;
  ncclSimInfo_t si = NCCL_SIM_INFO_INITIALIZER;
  FSDP_NCCL_TRY(ncclGroupStart());
  ncclResult_t r = op == FSDP_OP_AG
                       ? ncclAllGather(dummy, dummy, per_rank, ncclBfloat16, c->comm, nullptr)
                       : ncclReduceScatter(dummy, dummy, per_rank, ncclFloat32, ncclSum, c->comm, nullptr);
  ncclResult_t r2 = ncclGroupSimulateEnd(&si);
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(FSDP_ERR_NCCL, std::string("ncclGroupSimulateEnd: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
  if (!(si.estimatedTime >= 0.0f))  // NCCL_UNDEF_FLOAT: no model for this communicator (e.g. world 1)
    return fail(FSDP_ERR_UNSUPPORTED, "NCCL gave no time estimate for this communicator");
  *ns = static_cast<int64_t>(static_cast<double>(si.estimatedTime) * 1000.0 + 0.5);
  return FSDP_OK;
}

fsdp_status fsdp_ctx_info(const fsdp_ctx* c, int32_t* world, int32_t* rank) {
  if (!c) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return FSDP_OK;
}

fsdp_status fsdp_ctx_split(fsdp_ctx* parent, int32_t color, int32_t key, fsdp_ctx** out) {
  if (!parent || !out) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (!parent->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_ctx_split needs a ctx with a communicator");
  if (color < 0 && color != NCCL_SPLIT_NOCOLOR) return fail(FSDP_ERR_INVALID_ARG, "color < 0");
  FSDP_CUDA_TRY(cudaSetDevice(parent->device));
  ncclComm_t sub = nullptr;
  FSDP_NCCL_TRY(ncclCommSplit(parent->comm, color, key, &sub, nullptr));
  if (!sub) return FSDP_OK;  // NCCL_SPLIT_NOCOLOR: this rank is in no sub-mesh
  int n = 0, r = 0;
  ncclResult_t nr = ncclCommCount(sub, &n);
  if (nr == ncclSuccess) nr = ncclCommUserRank(sub, &r);
  if (nr != ncclSuccess) {
    ncclCommDestroy(sub);
    return fail(FSDP_ERR_NCCL, std::string("sub-communicator query: ") + ncclGetErrorString(nr));
  }
  fsdp_status st = fsdp_ctx_create(out, n, r, parent->device, nullptr, sub);
  if (st != FSDP_OK) {
    ncclCommDestroy(sub);
    return st;
  }
  (*out)->owns_comm = true;
  return FSDP_OK;
}

fsdp_status fsdp_ctx_destroy(fsdp_ctx* c) {
  if (!c) return FSDP_OK;
  cudaSetDevice(c->device);
  for (cudaEvent_t ev : c->timing_events) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->io_events) cudaEventDestroy(ev);
  if (c->ev_shards_released) cudaEventDestroy(c->ev_shards_released);
  if (c->gemm_cache) gemm_cache_destroy(c->gemm_cache);
  if (c->own_comm_stream) cudaStreamDestroy(c->own_comm_stream);
  if (c->own_copy_stream) cudaStreamDestroy(c->own_copy_stream);
  for (cudaEvent_t ev : c->copy_events) cudaEventDestroy(ev);
  if (c->own_h2d) cudaStreamDestroy(c->own_h2d);
  if (c->own_d2h) cudaStreamDestroy(c->own_d2h);
  if (c->sink) cudaFree(c->sink);
  release_devcomm(c);                  // before the windows and the communicator go
  release_registrations(c, nullptr);  // before the communicator goes
  fsdp_status st = FSDP_OK;
  if (c->owns_comm && c->comm) {
    ncclResult_t r = ncclCommDestroy(c->comm);
    if (r != ncclSuccess) st = fail(FSDP_ERR_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  }
  delete c;
  return st;
}

fsdp_status fsdp_shard(int32_t world, int32_t rank, const fsdp_param_desc* p, fsdp_dtype dt,
                       const void* full_dev, void* shard_dev, fsdp_shard_info* info,
                       fsdp_stream_t stream) {
  if (!p || !info) return fail(FSDP_ERR_INVALID_ARG, "NULL param or info");
  if (world < 1 || rank < 0 || rank >= world) return fail(FSDP_ERR_INVALID_ARG, "bad world/rank");
  if (!valid_desc(*p)) return fail(FSDP_ERR_INVALID_ARG, "bad param descriptor");
  int32_t e = dtype_bytes(dt);
  if (!e) return fail(FSDP_ERR_INVALID_ARG, "unsupported dtype");
  if ((full_dev == nullptr) != (shard_dev == nullptr))
    return fail(FSDP_ERR_INVALID_ARG, "full_dev and shard_dev must be both set or both NULL");
  ShardRows s = shard_rows(p->dim0, world, rank);
  info->shard_rows = s.c;
  info->row_begin = s.begin;
  info->valid_rows = s.v;
  info->shard_numel = s.c * p->row_numel;
  if (!full_dev) return FSDP_OK;
  TableBuilder tb;
  const int64_t row_bytes = p->row_numel * e;
  uint64_t src = reinterpret_cast<uint64_t>(full_dev) + static_cast<uint64_t>(s.begin * row_bytes);
  uint64_t dst = reinterpret_cast<uint64_t>(shard_dev);
  tb.copy(src, dst, s.v * row_bytes);
  tb.zero(dst + static_cast<uint64_t>(s.v * row_bytes), (s.c - s.v) * row_bytes);
  if (tb.chunks.empty()) return FSDP_OK;
  // One-shot table, allocated, filled and freed in stream order so that it
  // outlives the kernel without a host synchronisation.
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevTable t;
  t.n = static_cast<int32_t>(tb.chunks.size());
  const size_t bytes = tb.chunks.size() * sizeof(Chunk);
  FSDP_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t.d), bytes, st));
  FSDP_CUDA_TRY(cudaMemcpyAsync(t.d, tb.chunks.data(), bytes, cudaMemcpyHostToDevice, st));
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = device_sm_count(dev);
  cudaError_t err = launch_table(KK_SHARD, t, nullptr, 1.0f, st, (sms > 0 ? sms : 148) * FSDP_CTAS_PER_SM);
  cudaError_t err2 = cudaFreeAsync(t.d, st);
  if (err != cudaSuccess) return fail(FSDP_ERR_CUDA, std::string("shard kernel: ") + cudaGetErrorString(err));
  if (err2 != cudaSuccess) return fail(FSDP_ERR_CUDA, std::string("cudaFreeAsync: ") + cudaGetErrorString(err2));
  return FSDP_OK;
}

fsdp_status fsdp_layout(const fsdp_param_desc* members, int32_t k, int32_t world, int32_t elem_bytes,
                        int32_t align_bytes, int64_t* offs, int64_t* seg_bytes) {
  if (!members || k < 1 || world < 1 || elem_bytes < 1 || align_bytes < 1 || !seg_bytes)
    return fail(FSDP_ERR_INVALID_ARG, "bad layout arguments");
  for (int32_t j = 0; j < k; ++j)
    if (!valid_desc(members[j])) return fail(FSDP_ERR_INVALID_ARG, "bad param descriptor");
  layout(members, k, world, elem_bytes, align_bytes, offs, seg_bytes);
  return FSDP_OK;
}

}  // extern "C"
