// NVLink SHARP (NVLS) multicast memory for the reduce-scatter (include/fsdp.h,
// "NVLS multicast"; SURVEY §8(f) NEXT #1 "multimem reduce"): a CUDA multicast
// object spanning the ranks' GPUs, each rank's physical staging bound to it,
// and a unicast plus a multicast mapping.  A multimem.ld_reduce through the
// multicast mapping makes the NVSwitch sum the same address across every
// GPU's staging, so one load returns the reduced value (kernel K10).
//
// Driver entry points come from cudaGetDriverEntryPoint (the library links the
// CUDA runtime statically and has no link-time libcuda dependency).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <unistd.h>

#include "internal.h"

using namespace fsdp;

namespace {

struct Driver {
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) memGranularity = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceAttr = nullptr;
  bool ok = false;
  std::string why;
};

template <typename F>
bool entry(const char* name, F* fn, std::string* why) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    *why = std::string("driver entry point ") + name + " not found";
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    x.ok = entry("cuMulticastCreate", &x.mcCreate, &x.why) && entry("cuMulticastAddDevice", &x.mcAddDevice, &x.why) &&
           entry("cuMulticastBindMem", &x.mcBindMem, &x.why) && entry("cuMulticastUnbind", &x.mcUnbind, &x.why) &&
           entry("cuMulticastGetGranularity", &x.mcGranularity, &x.why) &&
           entry("cuMemCreate", &x.memCreate, &x.why) && entry("cuMemRelease", &x.memRelease, &x.why) &&
           entry("cuMemAddressReserve", &x.addrReserve, &x.why) && entry("cuMemAddressFree", &x.addrFree, &x.why) &&
           entry("cuMemMap", &x.memMap, &x.why) && entry("cuMemUnmap", &x.memUnmap, &x.why) &&
           entry("cuMemSetAccess", &x.memSetAccess, &x.why) &&
           entry("cuMemGetAllocationGranularity", &x.memGranularity, &x.why) &&
           entry("cuMemExportToShareableHandle", &x.exportHandle, &x.why) &&
           entry("cuMemImportFromShareableHandle", &x.importHandle, &x.why) &&
           entry("cuDeviceGet", &x.deviceGet, &x.why) && entry("cuDeviceGetAttribute", &x.deviceAttr, &x.why);
    return x;
  }();
  return d;
}

#define FSDP_CU_TRY(expr)                                                                               \
  do {                                                                                                  \
    CUresult r_ = (expr);                                                                               \
    if (r_ != CUDA_SUCCESS)                                                                             \
      return ::fsdp::fail(r_ == CUDA_ERROR_NOT_SUPPORTED ? FSDP_ERR_UNSUPPORTED : FSDP_ERR_CUDA,        \
                          std::string(#expr) + ": CUresult " + std::to_string(static_cast<int>(r_))); \
  } while (0)

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct fsdp_nvls {
  int32_t device = 0, world = 1;
  size_t size = 0;
  CUmemGenericAllocationHandle mc = 0, uc = 0;
  CUdeviceptr uc_ptr = 0, mc_ptr = 0;
  bool added = false, bound = false, uc_mapped = false, mc_mapped = false;
};

static fsdp_status nvls_begin(fsdp_ctx* c, int64_t bytes, fsdp_nvls** out, CUmulticastObjectProp* prop,
                              unsigned handle_types) {
  if (!c || !out || bytes < 1) return fail(FSDP_ERR_INVALID_ARG, "NULL ctx / out or bytes < 1");
  *out = nullptr;
  const Driver& d = drv();
  if (!d.ok) return fail(FSDP_ERR_UNSUPPORTED, d.why);
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_CUDA_TRY(cudaFree(nullptr));  // the primary context exists
  int mc_ok = 0;
  CUdevice dev;
  FSDP_CU_TRY(d.deviceGet(&dev, c->device));
  FSDP_CU_TRY(d.deviceAttr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  if (!mc_ok) return fail(FSDP_ERR_UNSUPPORTED, "device does not support multicast (NVLS)");
  std::memset(prop, 0, sizeof(*prop));
  prop->numDevices = static_cast<unsigned>(c->world);
  // a team of one needs no shareable handle; larger teams export one (fabric or POSIX fd)
  prop->handleTypes = c->world > 1 ? handle_types : 0;
  size_t g = 0;
  prop->size = static_cast<size_t>(bytes);
  FSDP_CU_TRY(d.mcGranularity(&g, prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  size_t g2 = 0;
  FSDP_CU_TRY(d.memGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  prop->size = round_up(static_cast<size_t>(bytes), std::max(g, g2));
  fsdp_nvls* m = new fsdp_nvls();
  m->device = c->device;
  m->world = c->world;
  m->size = prop->size;
  *out = m;
  return FSDP_OK;
}

static fsdp_status add_device(fsdp_nvls* m) {
  const Driver& d = drv();
  CUdevice dev;
  FSDP_CU_TRY(d.deviceGet(&dev, m->device));
  FSDP_CU_TRY(d.mcAddDevice(m->mc, dev));
  m->added = true;
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_nvls_destroy(fsdp_nvls* m) {
  if (!m) return FSDP_OK;
  const Driver& d = drv();
  if (d.ok) {
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    if (m->mc_mapped) d.memUnmap(m->mc_ptr, m->size);
    if (m->uc_mapped) d.memUnmap(m->uc_ptr, m->size);
    if (m->mc_ptr) d.addrFree(m->mc_ptr, m->size);
    if (m->uc_ptr) d.addrFree(m->uc_ptr, m->size);
    if (m->bound) {
      CUdevice dev;
      if (d.deviceGet(&dev, m->device) == CUDA_SUCCESS) d.mcUnbind(m->mc, dev, 0, m->size);
    }
    if (m->uc) d.memRelease(m->uc);
    if (m->mc) d.memRelease(m->mc);
  }
  delete m;
  return FSDP_OK;
}

// One attempt at the multicast object with the given shareable handle type;
// on success the handle is exported into h.
static CUresult create_exported(fsdp_nvls* m, CUmulticastObjectProp* prop, int world, unsigned type,
                                fsdp_nvls_handle* h, const char** what) {
  const Driver& d = drv();
  prop->handleTypes = world > 1 ? type : 0;
  *what = "cuMulticastCreate";
  CUresult r = d.mcCreate(&m->mc, prop);
  if (r != CUDA_SUCCESS || world == 1) return r;
  if (type == CU_MEM_HANDLE_TYPE_FABRIC) {
    CUmemFabricHandle fh;
    *what = "cuMemExportToShareableHandle(FABRIC)";
    r = d.exportHandle(&fh, m->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    if (r == CUDA_SUCCESS) {
      h->type = FSDP_NVLS_FABRIC;
      std::memcpy(h->fabric, &fh, sizeof(fh));
    }
  } else {
    int fd = -1;
    *what = "cuMemExportToShareableHandle(POSIX_FD)";
    r = d.exportHandle(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r == CUDA_SUCCESS) {
      h->type = FSDP_NVLS_POSIX_FD;
      h->fd = fd;
      h->pid = static_cast<int32_t>(getpid());
    }
  }
  if (r != CUDA_SUCCESS) {
    d.memRelease(m->mc);
    m->mc = 0;
  }
  return r;
}

extern "C" fsdp_status fsdp_nvls_create(fsdp_ctx* c, int64_t bytes, void* handle_out, fsdp_nvls** out) {
  if (!handle_out) return fail(FSDP_ERR_INVALID_ARG, "NULL handle_out");
  CUmulticastObjectProp prop;
  FSDP_TRY(nvls_begin(c, bytes, out, &prop, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  fsdp_nvls* m = *out;
  fsdp_nvls_handle h;
  std::memset(&h, 0, sizeof h);
  h.fd = -1;
  const char* what = "";
  // a fabric handle where the platform provides one (IMEX / NVSwitch fabric
  // manager), else a POSIX file descriptor for the caller to pass on
  CUresult r = create_exported(m, &prop, c->world, CU_MEM_HANDLE_TYPE_FABRIC, &h, &what);
  if (r != CUDA_SUCCESS && c->world > 1)
    r = create_exported(m, &prop, c->world, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, &h, &what);
  std::memcpy(handle_out, &h, sizeof h);
  // A device can report multicast support while the platform refuses the
  // object (e.g. a GPU whose NVSwitch fabric partition holds only itself:
  // CUDA_ERROR_INVALID_VALUE for every property set): unsupported here.
  const bool refused = r == CUDA_ERROR_NOT_SUPPORTED || r == CUDA_ERROR_NOT_PERMITTED ||
                       (r == CUDA_ERROR_INVALID_VALUE && m->mc == 0);
  fsdp_status st = r == CUDA_SUCCESS ? add_device(m)
                                     : fail(refused ? FSDP_ERR_UNSUPPORTED : FSDP_ERR_CUDA,
                                            std::string(what) + ": CUresult " + std::to_string(r) +
                                                (refused ? " (multicast object refused by the platform)" : ""));
  if (st != FSDP_OK) {
    fsdp_nvls_destroy(m);
    *out = nullptr;
  }
  return st;
}

extern "C" fsdp_status fsdp_nvls_import(fsdp_ctx* c, const void* handle, int64_t bytes, fsdp_nvls** out) {
  if (!handle) return fail(FSDP_ERR_INVALID_ARG, "NULL handle");
  fsdp_nvls_handle h;
  std::memcpy(&h, handle, sizeof h);
  if (h.type != FSDP_NVLS_FABRIC && h.type != FSDP_NVLS_POSIX_FD)
    return fail(FSDP_ERR_INVALID_ARG, "NVLS handle of unknown type");
  if (h.type == FSDP_NVLS_POSIX_FD && h.fd < 0) return fail(FSDP_ERR_INVALID_ARG, "NVLS POSIX handle without fd");
  CUmulticastObjectProp prop;
  FSDP_TRY(nvls_begin(c, bytes, out, &prop, h.type == FSDP_NVLS_FABRIC ? CU_MEM_HANDLE_TYPE_FABRIC
                                                                       : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  fsdp_nvls* m = *out;
  CUresult r;
  if (h.type == FSDP_NVLS_FABRIC) {
    CUmemFabricHandle fh;
    std::memcpy(&fh, h.fabric, sizeof(fh));
    r = drv().importHandle(&m->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC);
  } else {
    r = drv().importHandle(&m->mc, reinterpret_cast<void*>(static_cast<intptr_t>(h.fd)),
                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(h.fd);  // ownership taken (include/fsdp.h)
  }
  fsdp_status st = r == CUDA_SUCCESS ? add_device(m)
                                     : fail(FSDP_ERR_CUDA, "cuMemImportFromShareableHandle: CUresult " + std::to_string(r));
  if (st != FSDP_OK) {
    fsdp_nvls_destroy(m);
    *out = nullptr;
  }
  return st;
}

extern "C" fsdp_status fsdp_nvls_bind(fsdp_nvls* m, void** uc_ptr, void** mc_ptr, int64_t* bytes) {
  if (!m || !uc_ptr || !mc_ptr) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (m->bound) return fail(FSDP_ERR_INVALID_ARG, "already bound");
  const Driver& d = drv();
  FSDP_CUDA_TRY(cudaSetDevice(m->device));
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  FSDP_CU_TRY(d.memCreate(&m->uc, m->size, &ap, 0));
  CUdevice dev;
  FSDP_CU_TRY(d.deviceGet(&dev, m->device));
  FSDP_CU_TRY(d.mcBindMem(m->mc, 0, m->uc, 0, m->size, 0));
  m->bound = true;
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  FSDP_CU_TRY(d.addrReserve(&m->uc_ptr, m->size, 0, 0, 0));
  FSDP_CU_TRY(d.memMap(m->uc_ptr, m->size, 0, m->uc, 0));
  m->uc_mapped = true;
  FSDP_CU_TRY(d.memSetAccess(m->uc_ptr, m->size, &acc, 1));
  FSDP_CU_TRY(d.addrReserve(&m->mc_ptr, m->size, 0, 0, 0));
  FSDP_CU_TRY(d.memMap(m->mc_ptr, m->size, 0, m->mc, 0));
  m->mc_mapped = true;
  FSDP_CU_TRY(d.memSetAccess(m->mc_ptr, m->size, &acc, 1));
  *uc_ptr = reinterpret_cast<void*>(m->uc_ptr);
  *mc_ptr = reinterpret_cast<void*>(m->mc_ptr);
  if (bytes) *bytes = static_cast<int64_t>(m->size);
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_nvls_reduce_scatter_bucket(fsdp_ctx* c, fsdp_bucket* b, const void* mc_staging,
                                                       fsdp_stream_t stream) {
  if (!c || !b || !mc_staging) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  if (b->ctx != c) return fail(FSDP_ERR_INVALID_ARG, "bucket belongs to another ctx");
  if (!b->has_gshards) return fail(FSDP_ERR_INVALID_ARG, "NVLS reduce-scatter needs bound grad_shards");
  if (b->gshard_bf16) return fail(FSDP_ERR_INVALID_ARG, "NVLS reduce-scatter writes fp32 gradient shards");
  if (reinterpret_cast<uintptr_t>(mc_staging) % 16) return fail(FSDP_ERR_INVALID_ARG, "staging not 16-B aligned");
  FSDP_CUDA_TRY(cudaSetDevice(c->device));
  FSDP_CUDA_TRY(launch_nvls_reduce(b->nvls_rs, static_cast<const char*>(mc_staging), b->grad_accumulate,
                                   static_cast<cudaStream_t>(stream), c->max_ctas));
  return FSDP_OK;
}
