// Peer-memory ("fused") collectives: all-gather + copy-out (K8) and
// gradient widen + 1/N + reduce-scatter + copy-out (K9) as single kernels that
// read peers' buffers directly (NVLink P2P through CUDA IPC mappings), plus
// release/acquire epoch signalling and the IPC plumbing.  P:177.
#include <cstring>

#include "internal.h"

using namespace fsdp;

namespace {

fsdp_status peer_table(fsdp_ctx* c, const void* const* ptrs, PeerTable* pt, bool allow_null, uintptr_t align = 16) {
  if (!ptrs) return fail(FSDP_ERR_INVALID_ARG, "NULL peer array");
  if (c->world > kMaxPeers) return fail(FSDP_ERR_UNSUPPORTED, "peer-memory path supports world <= 16");
  std::memset(pt, 0, sizeof(*pt));
  for (int32_t q = 0; q < c->world; ++q) {
    if (!ptrs[q] && !allow_null) return fail(FSDP_ERR_INVALID_ARG, "NULL peer pointer");
    if (reinterpret_cast<uintptr_t>(ptrs[q]) % align) return fail(FSDP_ERR_INVALID_ARG, "peer pointer misaligned");
    pt->p[q] = static_cast<const char*>(ptrs[q]);
  }
  return FSDP_OK;
}

}  // namespace

extern "C" fsdp_status fsdp_p2p_allgather_bucket(fsdp_ctx* c, fsdp_bucket* b, const void* const* peer_segs,
                                                 fsdp_stream_t stream) {
  if (!c || !b) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (b->ctx != c) return fail(FSDP_ERR_INVALID_ARG, "bucket belongs to another ctx");
  if (!b->ag_zero_copy || !b->has_fulls)
    return fail(FSDP_ERR_INVALID_ARG, "peer all-gather needs FSDP_BUCKET_SEGMENT_SHARDS storage and fulls");
  PeerTable pt;
  FSDP_TRY(peer_table(c, peer_segs, &pt, false));
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_CUDA_TRY(launch_p2p_allgather(b->p2p_ag, pt, static_cast<cudaStream_t>(stream), c->max_ctas));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_p2p_reduce_scatter_bucket(fsdp_ctx* c, fsdp_bucket* b, const void* const* peer_grads,
                                                      fsdp_stream_t stream) {
  if (!c || !b) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (b->ctx != c) return fail(FSDP_ERR_INVALID_ARG, "bucket belongs to another ctx");
  if (!b->has_grads || !b->has_gshards)
    return fail(FSDP_ERR_INVALID_ARG, "peer reduce-scatter needs full_grads and grad_shards");
  if (b->gshard_bf16) return fail(FSDP_ERR_INVALID_ARG, "peer reduce-scatter writes fp32 gradient shards");
  PeerTable pt;
  FSDP_TRY(peer_table(c, peer_grads, &pt, false));
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  const float inv = 1.0f / static_cast<float>(c->world);  // fl32(1/N)
  FSDP_CUDA_TRY(launch_p2p_reduce_scatter(b->p2p_rs, pt, c->world, inv, b->grad_accumulate,
                                          static_cast<cudaStream_t>(stream), c->max_ctas));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_p2p_signal(fsdp_ctx* c, void* const* slots, uint64_t value, fsdp_stream_t stream) {
  if (!c) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx");
  PeerTable pt;
  FSDP_TRY(peer_table(c, const_cast<const void* const*>(slots), &pt, true, 8));
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_CUDA_TRY(launch_p2p_signal(pt, c->world, value, static_cast<cudaStream_t>(stream)));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_p2p_wait(fsdp_ctx* c, const void* flags, uint64_t value, int64_t timeout_ns,
                                     int32_t* error_flag, fsdp_stream_t stream) {
  if (!c || !flags) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (reinterpret_cast<uintptr_t>(flags) % 8) return fail(FSDP_ERR_INVALID_ARG, "flags not 8-B aligned");
  if (c->world > 32) return fail(FSDP_ERR_UNSUPPORTED, "wait supports world <= 32");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_CUDA_TRY(launch_p2p_wait(flags, c->world, value, timeout_ns, error_flag, static_cast<cudaStream_t>(stream)));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle64) {
  if (bytes < 1 || !dev_ptr || !handle64) return fail(FSDP_ERR_INVALID_ARG, "bad ipc_alloc arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  FSDP_CUDA_TRY(cudaMalloc(dev_ptr, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, *dev_ptr);
  if (e != cudaSuccess) {
    cudaFree(*dev_ptr);
    *dev_ptr = nullptr;
    return fail(FSDP_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  std::memcpy(handle64, &h, sizeof(h));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(FSDP_ERR_INVALID_ARG, "bad ipc_open arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  FSDP_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return FSDP_OK;
  FSDP_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return FSDP_OK;
  FSDP_CUDA_TRY(cudaFree(dev_ptr));
  return FSDP_OK;
}
