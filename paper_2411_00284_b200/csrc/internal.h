// Internal declarations of the B200-native SimpleFSDP hot path.
// Not part of the ABI; see include/fsdp.h for the public contract.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "fsdp.h"

namespace fsdp {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
fsdp_status fail(fsdp_status st, const std::string& msg);

#define FSDP_CUDA_TRY(expr)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return ::fsdp::fail(e_ == cudaErrorMemoryAllocation ? FSDP_ERR_OOM : FSDP_ERR_CUDA, \
                          std::string(#expr) + ": " + cudaGetErrorString(e_));           \
  } while (0)

#define FSDP_NCCL_TRY(expr)                                                              \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return ::fsdp::fail(FSDP_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define FSDP_TRY(expr)                 \
  do {                                 \
    fsdp_status s_ = (expr);           \
    if (s_ != FSDP_OK) return s_;      \
  } while (0)

// ------------------------------------------------------------ shard math
struct ShardRows {
  int64_t c, begin, v;  // rows per rank, first owned row, owned rows
};
ShardRows shard_rows(int64_t d, int32_t world, int32_t rank);
int64_t align_up(int64_t x, int64_t a);
int32_t dtype_bytes(int32_t dt);  // 0 if unknown
// Segment layout of k members (forward order): offsets and segment bytes.
void layout(const fsdp_param_desc* m, int32_t k, int32_t world, int64_t elem_bytes, int64_t align,
            int64_t* offs, int64_t* seg);

// ------------------------------------------------------------ run tables
// A chunk is <= kChunkBytes of destination data processed by one CTA.
// Addresses are absolute device addresses, or offsets from the staging base
// passed at launch for the side a kernel treats as relative.
#ifndef FSDP_CHUNK_KB
#define FSDP_CHUNK_KB 32
#endif
#ifndef FSDP_CTAS_PER_SM
// LSU-engine grid cap per SM.  1024 = in practice one CTA per chunk: the
// hardware block scheduler then balances the chunks dynamically, which
// measured 6529 GB/s on K3 vs 5901 for a persistent 8-CTA/SM grid
// (profiles/r01_kernel_sweep.md).
#define FSDP_CTAS_PER_SM 1024
#endif
constexpr uint32_t kChunkBytes = FSDP_CHUNK_KB * 1024;
#ifndef FSDP_P2P_FUSED_SYNC
// Scheduled peer-memory RS: epoch wait + signal fused into K9 (1) or separate
// 1-warp launches around it (0, default).  Measured equal step time on one
// B200 (13.57 vs 13.52 ms, profiles/r01_summary.md); the separate wait is kept
// because a fused K9 waiting for a late peer would hold every SM spinning and
// starve this rank's compute stream, while a 1-warp wait kernel does not.
#define FSDP_P2P_FUSED_SYNC 0
#endif

enum ChunkOp : uint32_t {
  OP_COPY = 0,   // n units of `unit` bytes
  OP_ZERO = 1,   // n units of `unit` bytes at dst
  OP_WIDEN = 2,  // bf16 -> fp32 * scale; unit 16: n groups of 8 elems, unit 2: n elems
  OP_SCALE = 3,  // fp32 * scale;        unit 16: n groups of 4 elems, unit 4: n elems
  // peer-memory reduce (K9): src = offset into every peer's gradient region;
  // unit 16: n groups of 8 bf16 / 4 fp32 elements, unit 2 / 4: n elements
  OP_PEER_REDUCE_BF16 = 4,
  OP_PEER_REDUCE_F32 = 5,
  OP_NARROW = 6,  // fp32 -> bf16 RNE; unit 16: n groups of 8 elems (32 B in, 16 B out), unit 4: n elems
  OP_ACCUM = 7,   // fp32 dst = dst + src;  unit 16: n groups of 4 elems, unit 4: n elems
  OP_NVLS = 8,    // K10: fp32 dst (+)= multimem.ld_reduce.add(src); unit 16: n groups of 4, unit 4: n elems
};
// Peer-memory copy (K8): OP_COPY chunks whose src is an offset into peer q's
// segment, q in op_unit bits 24..31.
constexpr uint32_t kPeerShift = 24;
constexpr int kMaxPeers = 16;
struct PeerTable {
  const char* p[kMaxPeers];
};

struct Chunk {
  uint64_t src;
  uint64_t dst;
  uint32_t n;
  uint32_t op_unit;  // op | unit << 8 | kAbsSrc
};
// Chunk flag: src is an absolute address even in a kernel whose source side is
// staging-relative (K3 reading this rank's rows straight from segment-layout
// shard storage, see fsdp_bucket_create).
constexpr uint32_t kAbsSrc = 1u << 16;
// Chunk flag: dst is an absolute address even in a kernel whose destination
// side is staging-relative (K1 of a direct-gather bucket writing the full
// parameter).
constexpr uint32_t kAbsDst = 1u << 17;
static_assert(sizeof(Chunk) == 24, "chunk layout");

// Builder that splits runs into chunks (host side).
struct TableBuilder {
  std::vector<Chunk> chunks;
  int64_t bytes_moved = 0;  // algorithmic bytes (read + write)
  void copy(uint64_t src, uint64_t dst, int64_t bytes, uint32_t flags = 0);
  void zero(uint64_t dst, int64_t bytes);
  void widen(uint64_t src, uint64_t dst, int64_t elems);  // bf16 -> f32 * s
  void scale(uint64_t src, uint64_t dst, int64_t elems);  // f32 -> f32 * s
  void narrow(uint64_t src, uint64_t dst, int64_t elems, uint32_t flags = 0);  // f32 -> bf16 RNE
  void accum(uint64_t src, uint64_t dst, int64_t elems);  // f32 dst += src
  void nvls(uint64_t src, uint64_t dst, int64_t elems);   // f32 dst = switch-reduced src
  // K9: rank-order sum over peers of `elems` gradient elements of elem_bytes
  // (2 = bf16, 4 = fp32) at offset src of every peer region -> fp32 at dst
  void peer_reduce(uint64_t src, uint64_t dst, int64_t elems, int elem_bytes, int world);
};

struct DevTable {
  Chunk* d = nullptr;
  int32_t n = 0;
  int64_t bytes_moved = 0;
};
fsdp_status upload(const TableBuilder& tb, DevTable* out);
void release(DevTable* t);

// Kernel launchers (kernels.cu).  `base` is the staging buffer for the side
// that is relative; grid = min(n, max_ctas).
enum KernelKind { KK_SHARD = 0, KK_AG_PACK, KK_AG_UNPACK, KK_RS_PACK, KK_RS_COPYOUT };
cudaError_t launch_table(KernelKind kind, const DevTable& t, char* base, float scale, cudaStream_t s,
                         int max_ctas);
cudaError_t launch_proxy(int64_t iters, int grid, int smem, float* sink, cudaStream_t s);
// K11: emulated collective (fsdp_comm_emulation).  AG: `src` (seg bytes) copied
// into the N - 1 slots q != rank of `dst` (N x seg); RS: dst (seg bytes) = sum
// over q of the fp32 slots of `src` (N x seg); then hold until target_ns.
cudaError_t launch_comm_emulation(bool reduce, const char* src, char* dst, int64_t seg, int32_t world, int32_t rank,
                                  int64_t target_ns, int ctas, cudaStream_t s);
// hold_ns > 0 (emulated NVLink, fsdp_comm_emulation): each CTA stays until
// hold_ns after it began, so the kernel lasts the modelled link time.
cudaError_t launch_p2p_allgather(const DevTable& t, const PeerTable& pt, cudaStream_t s, int max_ctas,
                                 int64_t hold_ns = 0);
// Epoch handshake fused into K9 (scheduled step): wait for wait_flags[q] >=
// wait_value before reading, store signal_value into every signal_slots[q]
// once the whole grid is done; counter: a zeroed device word per stream.
struct P2PSync {
  const unsigned long long* wait_flags;
  unsigned long long wait_value;
  long long timeout_ns;
  int* err;
  PeerTable signal_slots;
  unsigned long long signal_value;
  unsigned int* counter;  // NULL = no fused handshake
};
cudaError_t launch_p2p_reduce_scatter(const DevTable& t, const PeerTable& pt, int world, float scale,
                                      bool accumulate, cudaStream_t s, int max_ctas, const P2PSync* sync = nullptr,
                                      int64_t hold_ns = 0);
// K10: src offsets relative to the multicast mapping of the RS staging.
cudaError_t launch_nvls_reduce(const DevTable& t, const char* mc_base, bool accumulate, cudaStream_t s,
                               int max_ctas);
// base (nullable): device epoch counter added to `value` at run time
cudaError_t launch_p2p_signal(const PeerTable& slots, int world, uint64_t value, cudaStream_t s,
                              const uint64_t* base = nullptr);
cudaError_t launch_p2p_wait(const void* flags, int world, uint64_t value, int64_t timeout_ns, int* err,
                            cudaStream_t s, const uint64_t* base = nullptr);
cudaError_t launch_p2p_epoch_advance(uint64_t* base, uint64_t inc, cudaStream_t s);
int device_sm_count(int device);
cudaError_t preload_kernels();  // defeat lazy loading (see kernels.cu)

// Per-bucket steps shared by the public calls and the schedule executor
// (bucket.cc).  `launches` / `colls` (nullable) count enqueued kernels and
// collectives; with_comm = false skips the collective and the event wait.
}  // namespace fsdp
struct fsdp_ctx;
struct fsdp_bucket;
namespace fsdp {
fsdp_status ag_pack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches);
fsdp_status ag_collective(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t ms, bool with_comm, int* colls);
fsdp_status ag_wait(fsdp_ctx* c, fsdp_bucket* b, cudaStream_t cs, bool with_comm);
fsdp_status ag_unpack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, int* launches);
fsdp_status rs_pack(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches);
// The gradient-accumulation mode (fsdp_bucket_set_grad_accumulation) is
// latched by rs_pack and used by the matching rs_collective / rs_copyout.
fsdp_status rs_collective(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t ms, bool with_comm, int* colls);
fsdp_status rs_wait(fsdp_ctx* c, fsdp_bucket* b, cudaStream_t cs, bool with_comm);
fsdp_status rs_copyout(fsdp_ctx* c, fsdp_bucket* b, char* staging, cudaStream_t cs, bool with_comm, int* launches);
cudaStream_t resolve_comm(fsdp_ctx* c, fsdp_stream_t s);
fsdp_status check_async_error(fsdp_ctx* c);  // ncclCommGetAsyncError, if the ctx has a comm
// gemm.cc
fsdp_status bucket_compute(fsdp_ctx* c, fsdp_bucket* b, const fsdp_gemm_compute* g, bool backward, cudaStream_t s,
                           int* launches);
void gemm_cache_destroy(void* p);
}  // namespace fsdp

struct fsdp_ctx {
  int32_t world = 1, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  bool owns_comm = false;
  cudaStream_t own_comm_stream = nullptr;
  // FSDP_SCHED_COPY_STREAM: the pack / copy-out kernels' stream and the
  // per-call cross-stream events (unpacked / computed / grads packed per bucket)
  cudaStream_t own_copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_events;
  // NCCL device communicator with an LSA multicast mapping (ncclwin.cu,
  // fsdp_window_multimem_pointer); ncclDevComm_t behind a void*
  void* devcomm = nullptr;
  bool devcomm_ready = false;
  void* devcomm_mc_base = nullptr;
  int sm_count = 148;
  int max_ctas = 148 * 8;
  float* sink = nullptr;
  unsigned int* p2p_counter = nullptr;  // fused K9 handshake (zeroed; comm stream only)
  std::vector<cudaEvent_t> timing_events;  // pool for FSDP_SCHED_TIMING
  std::vector<cudaEvent_t> io_events;      // pool for host I/O ordering (fsdp_host_io)
  cudaStream_t own_h2d = nullptr, own_d2h = nullptr;
  // recorded on the compute stream after the last reader of the shard storage
  // in a scheduled step (its last UNPACK); the next step's host-I/O H2D waits
  // on it instead of on the whole previous step (fsdp_host_io)
  cudaEvent_t ev_shards_released = nullptr;
  bool shards_released_valid = false;
  void* gemm_cache = nullptr;              // cuBLASLt handle + plans (gemm.cc)
  const fsdp_comm_emulation* emul = nullptr;  // set by fsdp_run_schedule for the call (emulated collectives)
  // NCCL registrations (ncclmem.cc): base pointer -> local handle / window
  std::vector<std::pair<void*, void*>> nccl_regs;
  std::vector<std::pair<void*, ncclWindow_t>> nccl_wins;
};
namespace fsdp {
void release_registrations(fsdp_ctx* c, void* base);  // base NULL = all
void release_devcomm(fsdp_ctx* c);                      // the device communicator, if any
}

struct fsdp_bucket {
  fsdp_ctx* ctx = nullptr;
  int32_t device = 0;  // copied from the ctx: destroy must not read a destroyed ctx
  int32_t k = 0;
  int64_t ag_seg = 0, rs_seg = 0;
  int32_t param_bytes = 2, grad_bytes = 2;
  // which pointer arrays were bound: K1 shards, K3 fulls, K4 full_grads, K6 grad_shards
  bool has_shards = false, has_fulls = false, has_grads = false, has_gshards = false;
  // segment-layout ("zero-copy") storage, see fsdp_bucket_create
  bool ag_zero_copy = false, rs_zero_copy = false;
  char* shard_seg = nullptr;   // this rank's AG segment in shard storage
  char* gshard_seg = nullptr;  // this rank's RS segment in grad-shard storage
  bool ag_direct = false;      // gathered buffer == the (single) full parameter
  bool ag_grouped = false;     // FSDP_BUCKET_GROUPED_AG: per-member AGs in one NCCL group
  bool gshard_bf16 = false;    // FSDP_BUCKET_BF16_GRAD_SHARDS: K6 rounds the fp32 RS output to bf16
  std::vector<const void*> shard_ptrs;  // grouped: shards[j]
  std::vector<int64_t> own_bytes;       // grouped: c_j * R_j * e_p
  char* full0 = nullptr;       // fulls[0]
  // members and their full-parameter / full-gradient pointers (linear-layer compute)
  std::vector<fsdp_param_desc> members;
  std::vector<void*> fulls, grads;
  fsdp::DevTable ag_pack, ag_unpack, rs_pack, rs_copyout;
  fsdp::DevTable rs_accum;           // K6 variant: grad_shards += own segment (accumulation)
  fsdp::DevTable nvls_rs;            // K10: own segment through the NVLS multicast mapping
  bool grad_accumulate = false;      // fsdp_bucket_set_grad_accumulation
  bool rs_accum_issued = false;      // mode latched by the last rs_pack
  fsdp::DevTable p2p_ag, p2p_rs;  // K8 / K9 tables (peer-memory path)
  cudaEvent_t ev_ag_packed = nullptr, ev_ag_done = nullptr;
  cudaEvent_t ev_rs_packed = nullptr, ev_rs_done = nullptr;
  // host I/O with async_d2h: this bucket's gradient-shard D2H (d2h stream),
  // which its next gradient-shard writer waits for
  cudaEvent_t ev_d2h_done = nullptr;
  bool d2h_pending = false;
};
