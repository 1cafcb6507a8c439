// NCCL buffer registration (include/fsdp.h, "NCCL buffer registration"):
// cuMem-backed allocations and local / symmetric-window registrations with the
// ctx's communicator, so the path's collectives can run zero-copy on NVSwitch.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <string>

#include "internal.h"

using namespace fsdp;

namespace fsdp {
void release_registrations(fsdp_ctx* c, void* base) {
  if (!c || !c->comm) return;
  auto& regs = c->nccl_regs;
  for (auto it = regs.begin(); it != regs.end();) {
    if (!base || it->first == base) {
      ncclCommDeregister(c->comm, it->second);
      it = regs.erase(it);
    } else {
      ++it;
    }
  }
  auto& wins = c->nccl_wins;
  for (auto it = wins.begin(); it != wins.end();) {
    if (!base || it->first == base) {
      ncclCommWindowDeregister(c->comm, it->second);
      it = wins.erase(it);
    } else {
      ++it;
    }
  }
}
}  // namespace fsdp

extern "C" fsdp_status fsdp_mem_alloc(fsdp_ctx* c, int64_t bytes, void** dev_ptr) {
  if (!c || !dev_ptr || bytes < 1) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx / pointer or bytes < 1");
  *dev_ptr = nullptr;
  if (!c->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_mem_alloc needs a ctx with a communicator");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_NCCL_TRY(ncclMemAlloc(dev_ptr, static_cast<size_t>(bytes)));
  if (reinterpret_cast<uintptr_t>(*dev_ptr) % 4096) {
    ncclMemFree(*dev_ptr);
    *dev_ptr = nullptr;
    return fail(FSDP_ERR_CUDA, "ncclMemAlloc returned memory not 4096-B aligned");
  }
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_mem_free(fsdp_ctx* c, void* dev_ptr) {
  if (!c) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx");
  if (!dev_ptr) return FSDP_OK;
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  release_registrations(c, dev_ptr);
  FSDP_NCCL_TRY(ncclMemFree(dev_ptr));
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_register_buffer(fsdp_ctx* c, void* dev_ptr, int64_t bytes, int32_t mode) {
  if (!c || !dev_ptr || bytes < 1) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx / pointer or bytes < 1");
  if (!c->comm) return fail(FSDP_ERR_INVALID_ARG, "fsdp_register_buffer needs a ctx with a communicator");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  if (mode == FSDP_REG_LOCAL) {
    void* h = nullptr;
    FSDP_NCCL_TRY(ncclCommRegister(c->comm, dev_ptr, static_cast<size_t>(bytes), &h));
    c->nccl_regs.emplace_back(dev_ptr, h);
    return FSDP_OK;
  }
  if (mode == FSDP_REG_SYMMETRIC) {
    if (reinterpret_cast<uintptr_t>(dev_ptr) % NCCL_WIN_REQUIRED_ALIGNMENT)
      return fail(FSDP_ERR_INVALID_ARG, "symmetric window needs a 4096-B aligned pointer (fsdp_mem_alloc)");
    ncclWindow_t w = nullptr;
    FSDP_NCCL_TRY(
        ncclCommWindowRegister(c->comm, dev_ptr, static_cast<size_t>(bytes), &w, NCCL_WIN_COLL_SYMMETRIC));
    c->nccl_wins.emplace_back(dev_ptr, w);
    return FSDP_OK;
  }
  return fail(FSDP_ERR_INVALID_ARG, "mode must be FSDP_REG_LOCAL or FSDP_REG_SYMMETRIC");
}
