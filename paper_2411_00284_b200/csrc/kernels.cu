// sm_100a kernels of the SimpleFSDP hot path (HBM-bound; no tensor cores: the
// path has no dense contraction).
//
//   K0 fsdp_shard_kernel       full param -> padded dim-0 shard
//   K1 fsdp_ag_pack_kernel     shards -> rank segment of the AG bucket  ("flattens and concatenates")
//   K3 fsdp_ag_unpack_kernel   gathered bucket -> full params           ("copy out ... original tensor size")
//   K4 fsdp_rs_pack_kernel     full grads -> rank-major fp32 chunks x 1/N ("splits ... into chunks", P:302/311 fp32 avg)
//   K6 fsdp_rs_copyout_kernel  own RS segment -> grad shards            ("read out from RS12")
//   K7 fsdp_compute_proxy_kernel  calibrated stand-in for layer compute (measurement device)
//
// Every data kernel walks a host-built table of <= 32 KiB chunks with a grid
// of at most (SMs x 8) CTAs of 256 threads; one CTA owns a whole chunk, so the
// per-chunk branch is CTA-uniform.  Aligned chunks move 16 B per thread per
// access with 8 independent loads in flight per thread before the stores
// (8 x 256 x 16 B = one 32 KiB chunk per pass); misaligned runs (odd toy
// shapes, 1-D norms at N = 3) fall back to the widest unit that divides their
// addresses and size.  Arithmetic is IEEE round-to-nearest with no FTZ and no
// contraction: widen is exact, then one __fmul_rn by fl32(1/N).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fsdp {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void copy16(const char* src, char* dst, uint32_t n) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  uint32_t base = 0;
  // Full passes: kUnroll independent 16-B loads in flight, immediate offsets.
  for (; base + kThreads * kUnroll <= n; base += kThreads * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(s + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(d + base + u * kThreads, v[u]);
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += kThreads)
    st_v4(d - threadIdx.x + i, ld_stream(s - threadIdx.x + i));
}

template <typename T>
__device__ __forceinline__ void copy_units(const char* src, char* dst, uint32_t n) {
  const T* s = reinterpret_cast<const T*>(src);
  T* d = reinterpret_cast<T*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) d[i] = s[i];
}

template <typename T>
__device__ __forceinline__ void zero_units(char* dst, uint32_t n) {
  T* d = reinterpret_cast<T*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) d[i] = T{};
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// 8 bf16 (16 B) -> 8 fp32 (32 B), each * scale.
__device__ __forceinline__ uint4 widen_lo(const uint4& v, float scale) {
  uint4 a;
  a.x = __float_as_uint(__fmul_rn(bf16_lo(v.x), scale));
  a.y = __float_as_uint(__fmul_rn(bf16_hi(v.x), scale));
  a.z = __float_as_uint(__fmul_rn(bf16_lo(v.y), scale));
  a.w = __float_as_uint(__fmul_rn(bf16_hi(v.y), scale));
  return a;
}
__device__ __forceinline__ uint4 widen_hi(const uint4& v, float scale) {
  uint4 b;
  b.x = __float_as_uint(__fmul_rn(bf16_lo(v.z), scale));
  b.y = __float_as_uint(__fmul_rn(bf16_hi(v.z), scale));
  b.z = __float_as_uint(__fmul_rn(bf16_lo(v.w), scale));
  b.w = __float_as_uint(__fmul_rn(bf16_hi(v.w), scale));
  return b;
}

__device__ __forceinline__ void widen16(const char* src, char* dst, uint32_t n, float scale) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + 2 * threadIdx.x;
  constexpr int U = kUnroll / 2;
  uint32_t base = 0;
  for (; base + kThreads * U <= n; base += kThreads * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(s + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      st_v4(d + 2 * (base + u * kThreads), widen_lo(v[u], scale));
      st_v4(d + 2 * (base + u * kThreads) + 1, widen_hi(v[u], scale));
    }
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += kThreads) {
    uint4 v = ld_stream(s - threadIdx.x + i);
    st_v4(d - 2 * threadIdx.x + 2 * i, widen_lo(v, scale));
    st_v4(d - 2 * threadIdx.x + 2 * i + 1, widen_hi(v, scale));
  }
}

__device__ __forceinline__ void widen1(const char* src, char* dst, uint32_t n, float scale) {
  const uint16_t* s = reinterpret_cast<const uint16_t*>(src);
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += kThreads)
    d[i] = __fmul_rn(__uint_as_float(static_cast<uint32_t>(s[i]) << 16), scale);
}

__device__ __forceinline__ uint4 scale4(const uint4& v, float scale) {
  uint4 a;
  a.x = __float_as_uint(__fmul_rn(__uint_as_float(v.x), scale));
  a.y = __float_as_uint(__fmul_rn(__uint_as_float(v.y), scale));
  a.z = __float_as_uint(__fmul_rn(__uint_as_float(v.z), scale));
  a.w = __float_as_uint(__fmul_rn(__uint_as_float(v.w), scale));
  return a;
}

__device__ __forceinline__ void scale16(const char* src, char* dst, uint32_t n, float scale) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  uint32_t base = 0;
  for (; base + kThreads * kUnroll <= n; base += kThreads * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(s + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(d + base + u * kThreads, scale4(v[u], scale));
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += kThreads)
    st_v4(d - threadIdx.x + i, scale4(ld_stream(s - threadIdx.x + i), scale));
}

__device__ __forceinline__ void scale1(const char* src, char* dst, uint32_t n, float scale) {
  const float* s = reinterpret_cast<const float*>(src);
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) d[i] = __fmul_rn(s[i], scale);
}

template <bool kSrcRel, bool kDstRel>
__device__ __forceinline__ void run_table(const Chunk* __restrict__ tab, int n, char* base,
                                          float scale) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    const char* src = kSrcRel ? base + ch.src : reinterpret_cast<const char*>(ch.src);
    char* dst = kDstRel ? base + ch.dst : reinterpret_cast<char*>(ch.dst);
    const uint32_t op = ch.op_unit & 0xFFu;
    const uint32_t unit = ch.op_unit >> 8;
    if (op == OP_COPY) {
      switch (unit) {
        case 16: copy16(src, dst, ch.n); break;
        case 8: copy_units<uint2>(src, dst, ch.n); break;
        case 4: copy_units<uint32_t>(src, dst, ch.n); break;
        case 2: copy_units<uint16_t>(src, dst, ch.n); break;
        default: copy_units<uint8_t>(src, dst, ch.n); break;
      }
    } else if (op == OP_ZERO) {
      switch (unit) {
        case 16: zero_units<uint4>(dst, ch.n); break;
        case 8: zero_units<uint2>(dst, ch.n); break;
        case 4: zero_units<uint32_t>(dst, ch.n); break;
        case 2: zero_units<uint16_t>(dst, ch.n); break;
        default: zero_units<uint8_t>(dst, ch.n); break;
      }
    } else if (op == OP_WIDEN) {
      if (unit == 16) widen16(src, dst, ch.n, scale);
      else widen1(src, dst, ch.n, scale);
    } else {
      if (unit == 16) scale16(src, dst, ch.n, scale);
      else scale1(src, dst, ch.n, scale);
    }
  }
}

}  // namespace

// K0: full parameter -> padded shard (absolute -> absolute).
__global__ void __launch_bounds__(kThreads, 4) fsdp_shard_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table<false, false>(tab, n, base, s);
}
// K1: shards -> segment `rank` of the AG staging buffer (absolute -> staging).
__global__ void __launch_bounds__(kThreads, 4) fsdp_ag_pack_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table<false, true>(tab, n, base, s);
}
// K3: gathered staging -> full parameters (staging -> absolute).
__global__ void __launch_bounds__(kThreads, 4) fsdp_ag_unpack_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table<true, false>(tab, n, base, s);
}
// K4: full gradients -> fp32 rank-major chunks * fl32(1/N) (absolute -> staging).
__global__ void __launch_bounds__(kThreads, 4) fsdp_rs_pack_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table<false, true>(tab, n, base, s);
}
// K6: own reduce-scatter segment -> fp32 gradient shards (staging -> absolute).
__global__ void __launch_bounds__(kThreads, 4) fsdp_rs_copyout_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table<true, false>(tab, n, base, s);
}

// K7: persistent compute proxy.  Four independent FMA chains per thread; the
// result is consumed behind an impossible branch so the loop survives.
__global__ void __launch_bounds__(kThreads) fsdp_compute_proxy_kernel(long long iters, float* sink) {
  extern __shared__ float smem[];
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  const float m = 0.9999999f, c = 1e-7f;
  for (long long i = 0; i < iters; ++i) {
    a0 = fmaf(a0, m, c);
    a1 = fmaf(a1, m, c);
    a2 = fmaf(a2, m, c);
    a3 = fmaf(a3, m, c);
  }
  float r = a0 + a1 + a2 + a3;
  if (r == -1.0f) {
    smem[threadIdx.x] = r;
    sink[blockIdx.x] = smem[(threadIdx.x + 1) % kThreads];
  }
}

cudaError_t launch_table(KernelKind kind, const DevTable& t, char* base, float scale, cudaStream_t s,
                         int max_ctas) {
  if (t.n == 0) return cudaSuccess;
  int grid = t.n < max_ctas ? t.n : max_ctas;
  switch (kind) {
    case KK_SHARD: fsdp_shard_kernel<<<grid, kThreads, 0, s>>>(t.d, t.n, base, scale); break;
    case KK_AG_PACK: fsdp_ag_pack_kernel<<<grid, kThreads, 0, s>>>(t.d, t.n, base, scale); break;
    case KK_AG_UNPACK: fsdp_ag_unpack_kernel<<<grid, kThreads, 0, s>>>(t.d, t.n, base, scale); break;
    case KK_RS_PACK: fsdp_rs_pack_kernel<<<grid, kThreads, 0, s>>>(t.d, t.n, base, scale); break;
    case KK_RS_COPYOUT: fsdp_rs_copyout_kernel<<<grid, kThreads, 0, s>>>(t.d, t.n, base, scale); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_proxy(int64_t iters, int grid, int smem, float* sink, cudaStream_t s) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fsdp_compute_proxy_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  fsdp_compute_proxy_kernel<<<grid, kThreads, smem, s>>>(static_cast<long long>(iters), sink);
  return cudaGetLastError();
}

int device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return n;
}

}  // namespace fsdp
