// Peer and multicast addresses of NCCL symmetric windows (include/fsdp.h,
// "NCCL symmetric windows for the peer-memory path"): the NCCL 2.28 device
// API (nccl_device.h) maps every rank's window of a symmetric registration
// into this process's address space (cuMem + NCCL's own handle exchange);
// ncclGetPeerPointer / the window's multicast offset are evaluated on the
// device by a one-warp kernel and handed back to the host, so that K8 / K9 /
// K10 read peers through the same kind of pointer table as with CUDA IPC.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace fsdp;

namespace {

__global__ void fsdp_window_peers_kernel(ncclWindow_t w, int world, unsigned long long* out) {
  const int q = threadIdx.x;
  if (q < world) out[q] = reinterpret_cast<unsigned long long>(ncclGetPeerPointer(w, 0, q));
}

__global__ void fsdp_window_mc_offset_kernel(ncclWindow_t w, unsigned long long* out) {
  if (threadIdx.x == 0) out[0] = static_cast<unsigned long long>(w->mcOffset4K) * 4096ull;
}

ncclWindow_t find_window(fsdp_ctx* c, const void* base) {
  for (auto& pw : c->nccl_wins)
    if (pw.first == base) return pw.second;
  return nullptr;
}

}  // namespace

extern "C" fsdp_status fsdp_window_peer_pointers(fsdp_ctx* c, const void* base, void** peer_ptrs) {
  if (!c || !base || !peer_ptrs) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (!c->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_window_peer_pointers needs a ctx with a communicator");
  ncclWindow_t w = find_window(c, base);
  if (!w) return fail(FSDP_ERR_INVALID_ARG, "no symmetric window registered at this base (fsdp_register_buffer)");
  // every rank must be a load/store-accessible (NVLink) peer: the LSA team is the world
  const ncclTeam_t lsa = ncclTeamLsa(c->comm);
  if (lsa.nRanks != c->world)
    return fail(FSDP_ERR_UNSUPPORTED, "ranks outside this rank's NVLink domain (LSA team " +
                                          std::to_string(lsa.nRanks) + " of " + std::to_string(c->world) + ")");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  unsigned long long* d = nullptr;
  FSDP_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long) * static_cast<size_t>(c->world)));
  (void)cudaGetLastError();
  fsdp_window_peers_kernel<<<1, 32 * ((c->world + 31) / 32)>>>(w, c->world, d);
  cudaError_t e = cudaGetLastError();
  std::vector<unsigned long long> h(static_cast<size_t>(c->world));
  if (e == cudaSuccess)
    e = cudaMemcpy(h.data(), d, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(FSDP_ERR_CUDA, std::string("window peer pointers: ") + cudaGetErrorString(e));
  for (int q = 0; q < c->world; ++q) peer_ptrs[q] = reinterpret_cast<void*>(h[static_cast<size_t>(q)]);
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_window_multimem_pointer(fsdp_ctx* c, const void* base, void** mc_ptr) {
  if (!c || !base || !mc_ptr) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  *mc_ptr = nullptr;
  if (!c->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_window_multimem_pointer needs a ctx with a communicator");
  ncclWindow_t w = find_window(c, base);
  if (!w) return fail(FSDP_ERR_INVALID_ARG, "no symmetric window registered at this base (fsdp_register_buffer)");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  if (!c->devcomm_ready) {
    // the device communicator with a multicast (NVLS) mapping over the LSA team
    ncclDevCommRequirements_t req;
    std::memset(&req, 0, sizeof req);
    req.lsaMultimem = true;
    ncclDevComm_t dc;
    const ncclResult_t r = ncclDevCommCreate(c->comm, &req, &dc);
    if (r != ncclSuccess)
      return fail(FSDP_ERR_UNSUPPORTED, std::string("ncclDevCommCreate(lsaMultimem): ") + ncclGetErrorString(r));
    c->devcomm_mc_base = dc.lsaMultimem.mcBasePtr;
    c->devcomm_ready = true;
    c->devcomm = new ncclDevComm_t(dc);
  }
  if (!c->devcomm_mc_base) return fail(FSDP_ERR_UNSUPPORTED, "NCCL gave no multicast mapping (NVLS unavailable)");
  unsigned long long* d = nullptr;
  FSDP_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long)));
  (void)cudaGetLastError();
  fsdp_window_mc_offset_kernel<<<1, 32>>>(w, d);
  cudaError_t e = cudaGetLastError();
  unsigned long long off = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&off, d, sizeof(off), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(FSDP_ERR_CUDA, std::string("window multicast offset: ") + cudaGetErrorString(e));
  *mc_ptr = static_cast<char*>(c->devcomm_mc_base) + off;
  return FSDP_OK;
}

namespace fsdp {
void release_devcomm(fsdp_ctx* c) {
  if (c->devcomm) {
    ncclDevCommDestroy(c->comm, static_cast<const ncclDevComm_t*>(c->devcomm));
    delete static_cast<ncclDevComm_t*>(c->devcomm);
    c->devcomm = nullptr;
  }
  c->devcomm_ready = false;
  c->devcomm_mc_base = nullptr;
}
}  // namespace fsdp
