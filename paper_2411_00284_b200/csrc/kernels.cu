// sm_100a kernels of the SimpleFSDP hot path (HBM-bound; no tensor cores: the
// path has no dense contraction).
//
//   K0 fsdp_shard_kernel       full param -> padded dim-0 shard
//   K1 fsdp_ag_pack_kernel     shards -> rank segment of the AG bucket  ("flattens and concatenates";
//                              fp32 master shards rounded to bf16 on the way)
//   K3 fsdp_ag_unpack_kernel   gathered bucket -> full params           ("copy out ... original tensor size")
//   K4 fsdp_rs_pack_kernel     full grads -> rank-major fp32 chunks x 1/N ("splits ... into chunks", P:302/311 fp32 avg)
//   K6 fsdp_rs_copyout_kernel  own RS segment -> grad shards            ("read out from RS12";
//                              or added to them: gradient accumulation)
//   K7 fsdp_compute_proxy_kernel  calibrated stand-in for layer compute (measurement device)
//
// Every data kernel walks a host-built table of <= kChunkBytes chunks; one CTA
// owns a whole chunk, so the per-chunk branch is CTA-uniform.
//
// Two engines:
//  * LSU engine (run_table, the default): one CTA of FSDP_THREADS threads per
//    32 KiB chunk (grid = chunks; the block scheduler balances them), aligned
//    chunks move 16 B per thread per access with FSDP_UNROLL independent loads
//    in flight per thread before the stores; K4 writes its 32 widened bytes
//    per thread with one 256-bit STG.  Measured on B200 (8B block, N = 8):
//    K3 6529 GB/s and K4 6643 GB/s vs 6585 GB/s for torch's copy_ on the same
//    box (profiles/r01_kernel_sweep.md).
//  * Bulk-copy (TMA) engine (run_table_bulk, FSDP_BULK, off by default: it
//    measured 5.9 TB/s at best on K3): one warp per CTA; lane 0
//    streams 16-B-aligned copy chunks global -> shared -> global with
//    cp.async.bulk through a ring of FSDP_BULK_STAGES shared-memory stages
//    (mbarrier complete_tx for loads, bulk groups for stores), so a handful of
//    instructions keep up to (stages - 1) x 32 KiB of loads in flight per CTA.
// Misaligned runs (odd toy shapes, 1-D norms at N = 3) fall back to the widest
// unit that divides their addresses and size.  Arithmetic is IEEE
// round-to-nearest with no FTZ and no contraction: widen is exact, then one
// __fmul_rn by fl32(1/N).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.h"

#ifndef FSDP_THREADS
#define FSDP_THREADS 256
#endif
#ifndef FSDP_UNROLL
#define FSDP_UNROLL 8
#endif
#ifndef FSDP_MIN_BLOCKS
#define FSDP_MIN_BLOCKS 4
#endif
#ifndef FSDP_ST_HINT
#define FSDP_ST_HINT 0  // 0: st.global, 1: st.global.cs (evict-first streaming)
#endif
#ifndef FSDP_LD_HINT
#define FSDP_LD_HINT 0  // 0: ld.global.nc.L1::no_allocate, 1: ld.global.cs
#endif
#ifndef FSDP_WIDEN_V8
#define FSDP_WIDEN_V8 1  // K4: one 256-bit store per 8 widened elements
#endif
#ifndef FSDP_K9_TEMPLATED
#define FSDP_K9_TEMPLATED 0  // K9: compile-time world (all peers' loads in flight) vs batches of 4
#endif
#ifndef FSDP_K9_MIN_BLOCKS
#define FSDP_K9_MIN_BLOCKS FSDP_MIN_BLOCKS
#endif
#ifndef FSDP_PDL
#define FSDP_PDL 1  // K0-K6: programmatic dependent launch (launch overlaps the previous kernel's tail)
#endif
#ifndef FSDP_PROXY_WAVES
#define FSDP_PROXY_WAVES 16  // K7: short CTAs per (SM x ctas_per_sm) slot
#endif
#ifndef FSDP_PROXY_MIN_ITERS
#define FSDP_PROXY_MIN_ITERS 512  // K7: fewest iterations per CTA before another wave is added
#endif
#ifndef FSDP_BULK
#define FSDP_BULK 0  // bulk engine for: 0 none, 1 K3, 2 all pure-copy kernels (K0, K1, K3, K6)
#endif
#ifndef FSDP_BULK_STAGES
#define FSDP_BULK_STAGES 6
#endif
#ifndef FSDP_BULK_LAG
#define FSDP_BULK_LAG 0  // bulk engine: stores kept in flight before a stage is reloaded
#endif
#define FSDP_STR2(x) #x
#define FSDP_STR(x) FSDP_STR2(x)
#ifndef FSDP_BULK_CTAS_PER_SM
#define FSDP_BULK_CTAS_PER_SM 1  // resident bulk CTAs per SM the smem ring is sized for
#endif
#ifndef FSDP_BULK_GRID_PER_SM
#define FSDP_BULK_GRID_PER_SM FSDP_BULK_CTAS_PER_SM  // bulk-engine grid cap per SM
#endif

namespace fsdp {
namespace {

constexpr int kThreads = FSDP_THREADS;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Emulated link time (fsdp_comm_emulation): the CTA stays until hold_ns after t0.
__device__ __forceinline__ void hold_until(unsigned long long t0, long long hold_ns) {
  if (hold_ns <= 0) return;
  if (threadIdx.x == 0)
    while (global_ns() - t0 < static_cast<unsigned long long>(hold_ns)) __nanosleep(256);
  __syncthreads();
}
constexpr int kUnroll = FSDP_UNROLL;
constexpr int kStages = FSDP_BULK_STAGES;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
#if FSDP_LD_HINT == 1
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#endif
  return r;
}

__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
#if FSDP_ST_HINT == 1
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
#else
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
#endif
}

template <int NT>
__device__ __forceinline__ void copy16(const char* src, char* dst, uint32_t n) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  uint32_t base = 0;
  // Full passes: kUnroll independent 16-B loads in flight, immediate offsets.
  for (; base + NT * kUnroll <= n; base += NT * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(s + base + u * NT);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(d + base + u * NT, v[u]);
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += NT) st_v4(d - threadIdx.x + i, ld_stream(s - threadIdx.x + i));
}

template <int NT, typename T>
__device__ __forceinline__ void copy_units(const char* src, char* dst, uint32_t n) {
  const T* s = reinterpret_cast<const T*>(src);
  T* d = reinterpret_cast<T*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT) d[i] = s[i];
}

template <int NT, typename T>
__device__ __forceinline__ void zero_units(char* dst, uint32_t n) {
  T* d = reinterpret_cast<T*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT) d[i] = T{};
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

// The 32 widened bytes of one thread go out as one 256-bit store (sm_100
// STG.256), so a warp's store covers 1 KiB contiguously; two 128-bit stores
// would each cover every other 16 B of that range.  Needs 32-B alignment of
// the destination, which the table builder guarantees for OP_WIDEN unit 16.
template <bool kV8>
__device__ __forceinline__ void st_widened(uint4* p, const uint4& v, float scale) {
  if (kV8) {
    const uint4 a = widen_lo(v, scale), b = widen_hi(v, scale);
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y),
                 "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
  } else {
    st_v4(p, widen_lo(v, scale));
    st_v4(p + 1, widen_hi(v, scale));
  }
}

template <int NT, bool kV8>
__device__ __forceinline__ void widen16_impl(const char* src, char* dst, uint32_t n, float scale) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + 2 * threadIdx.x;
  constexpr int U = kUnroll / 2 > 0 ? kUnroll / 2 : 1;
  uint32_t base = 0;
  for (; base + NT * U <= n; base += NT * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(s + base + u * NT);
#pragma unroll
    for (int u = 0; u < U; ++u) st_widened<kV8>(d + 2 * (base + u * NT), v[u], scale);
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += NT)
    st_widened<kV8>(d - 2 * threadIdx.x + 2 * i, ld_stream(s - threadIdx.x + i), scale);
}

template <int NT>
__device__ __forceinline__ void widen16(const char* src, char* dst, uint32_t n, float scale) {
  if (FSDP_WIDEN_V8 && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) widen16_impl<NT, true>(src, dst, n, scale);
  else widen16_impl<NT, false>(src, dst, n, scale);
}

template <int NT>
__device__ __forceinline__ void widen1(const char* src, char* dst, uint32_t n, float scale) {
  const uint16_t* s = reinterpret_cast<const uint16_t*>(src);
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT)
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

template <int NT>
__device__ __forceinline__ void scale16(const char* src, char* dst, uint32_t n, float scale) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  uint32_t base = 0;
  for (; base + NT * kUnroll <= n; base += NT * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(s + base + u * NT);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(d + base + u * NT, scale4(v[u], scale));
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += NT)
    st_v4(d - threadIdx.x + i, scale4(ld_stream(s - threadIdx.x + i), scale));
}

template <int NT>
__device__ __forceinline__ void scale1(const char* src, char* dst, uint32_t n, float scale) {
  const float* s = reinterpret_cast<const float*>(src);
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT) d[i] = __fmul_rn(s[i], scale);
}

// Two fp32 -> one bf16x2 word, round to nearest even (cvt.rn.bf16x2.f32 puts
// its first source in the upper half): `lo` lands at the lower address.
__device__ __forceinline__ uint32_t narrow2(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(hi)), "f"(__uint_as_float(lo)));
  return r;
}

// fp32 master shard -> bf16 (mixed precision): n groups of 8 elements,
// 32 B in (two 16-B loads), 16 B out.
template <int NT>
__device__ __forceinline__ void narrow16(const char* src, char* dst, uint32_t n) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + 2 * threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  constexpr int U = kUnroll / 2 > 0 ? kUnroll / 2 : 1;
  auto pack = [](const uint4& a, const uint4& b) {
    return make_uint4(narrow2(a.x, a.y), narrow2(a.z, a.w), narrow2(b.x, b.y), narrow2(b.z, b.w));
  };
  uint32_t base = 0;
  for (; base + NT * U <= n; base += NT * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = ld_stream(s + 2 * (base + u * NT));
      b[u] = ld_stream(s + 2 * (base + u * NT) + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st_v4(d + base + u * NT, pack(a[u], b[u]));
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += NT) {
    const uint4* si = s - 2 * threadIdx.x + 2 * i;
    st_v4(d - threadIdx.x + i, pack(ld_stream(si), ld_stream(si + 1)));
  }
}

template <int NT>
__device__ __forceinline__ void narrow1(const char* src, char* dst, uint32_t n) {
  const float* s = reinterpret_cast<const float*>(src);
  uint16_t* d = reinterpret_cast<uint16_t*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT)
    d[i] = static_cast<uint16_t>(narrow2(__float_as_uint(s[i]), 0u) & 0xFFFFu);
}

// Gradient accumulation: fp32 dst = dst + src, one rounding per element.
__device__ __forceinline__ uint4 add4(const uint4& a, const uint4& b) {
  return make_uint4(__float_as_uint(__fadd_rn(__uint_as_float(a.x), __uint_as_float(b.x))),
                    __float_as_uint(__fadd_rn(__uint_as_float(a.y), __uint_as_float(b.y))),
                    __float_as_uint(__fadd_rn(__uint_as_float(a.z), __uint_as_float(b.z))),
                    __float_as_uint(__fadd_rn(__uint_as_float(a.w), __uint_as_float(b.w))));
}

template <int NT>
__device__ __forceinline__ void accum16(const char* src, char* dst, uint32_t n) {
  const uint4* s = reinterpret_cast<const uint4*>(src) + threadIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst) + threadIdx.x;
  constexpr int U = kUnroll / 2 > 0 ? kUnroll / 2 : 1;
  uint32_t base = 0;
  for (; base + NT * U <= n; base += NT * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = *(d + base + u * NT);  // existing shard: plain (cached) load, it is rewritten next
      b[u] = ld_stream(s + base + u * NT);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st_v4(d + base + u * NT, add4(a[u], b[u]));
  }
  for (uint32_t i = base + threadIdx.x; i < n; i += NT)
    st_v4(d - threadIdx.x + i, add4(*(d - threadIdx.x + i), ld_stream(s - threadIdx.x + i)));
}

template <int NT>
__device__ __forceinline__ void accum1(const char* src, char* dst, uint32_t n) {
  const float* s = reinterpret_cast<const float*>(src);
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += NT) d[i] = __fadd_rn(d[i], s[i]);
}

template <bool kSrcRel>
__device__ __forceinline__ const char* src_of(const Chunk& ch, char* base) {
  return (kSrcRel && !(ch.op_unit & kAbsSrc)) ? base + ch.src : reinterpret_cast<const char*>(ch.src);
}

template <bool kDstRel>
__device__ __forceinline__ char* dst_of(const Chunk& ch, char* base) {
  return (kDstRel && !(ch.op_unit & kAbsDst)) ? base + ch.dst : reinterpret_cast<char*>(ch.dst);
}

template <int NT>
__device__ __forceinline__ void process_chunk(const Chunk& ch, const char* src, char* dst, float scale) {
  const uint32_t op = ch.op_unit & 0xFFu;
  const uint32_t unit = (ch.op_unit >> 8) & 0xFFu;
  if (op == OP_COPY) {
    switch (unit) {
      case 16: copy16<NT>(src, dst, ch.n); break;
      case 8: copy_units<NT, uint2>(src, dst, ch.n); break;
      case 4: copy_units<NT, uint32_t>(src, dst, ch.n); break;
      case 2: copy_units<NT, uint16_t>(src, dst, ch.n); break;
      default: copy_units<NT, uint8_t>(src, dst, ch.n); break;
    }
  } else if (op == OP_ZERO) {
    switch (unit) {
      case 16: zero_units<NT, uint4>(dst, ch.n); break;
      case 8: zero_units<NT, uint2>(dst, ch.n); break;
      case 4: zero_units<NT, uint32_t>(dst, ch.n); break;
      case 2: zero_units<NT, uint16_t>(dst, ch.n); break;
      default: zero_units<NT, uint8_t>(dst, ch.n); break;
    }
  } else if (op == OP_WIDEN) {
    if (unit == 16) widen16<NT>(src, dst, ch.n, scale);
    else widen1<NT>(src, dst, ch.n, scale);
  } else if (op == OP_NARROW) {
    if (unit == 16) narrow16<NT>(src, dst, ch.n);
    else narrow1<NT>(src, dst, ch.n);
  } else if (op == OP_ACCUM) {
    if (unit == 16) accum16<NT>(src, dst, ch.n);
    else accum1<NT>(src, dst, ch.n);
  } else {
    if (unit == 16) scale16<NT>(src, dst, ch.n, scale);
    else scale1<NT>(src, dst, ch.n, scale);
  }
}

template <bool kSrcRel, bool kDstRel>
__device__ __forceinline__ void run_table(const Chunk* __restrict__ tab, int n, char* base, float scale) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    const char* src = src_of<kSrcRel>(ch, base);
    char* dst = dst_of<kDstRel>(ch, base);
    process_chunk<kThreads>(ch, src, dst, scale);
  }
}

// ------------------------------------------------------------ bulk engine
__device__ __forceinline__ bool is_bulk(const Chunk& ch) {
  return (ch.op_unit & 0xFFu) == OP_COPY && ((ch.op_unit >> 8) & 0xFFu) == 16;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <bool kSrcRel, bool kDstRel>
__device__ __forceinline__ void run_table_bulk(const Chunk* __restrict__ tab, int n, char* base, float scale) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  __shared__ __align__(8) unsigned long long bars[kStages];
  // pass 1: chunks the bulk engine does not take (zero fill, misaligned), by the whole warp
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    if (is_bulk(ch)) continue;
    const char* src = src_of<kSrcRel>(ch, base);
    char* dst = dst_of<kDstRel>(ch, base);
    process_chunk<32>(ch, src, dst, scale);
  }
  if (threadIdx.x != 0) return;
  // pass 2: lane 0 streams the 16-B-aligned copy chunks through the stage ring
  const uint32_t smem0 = static_cast<uint32_t>(__cvta_generic_to_shared(bulk_smem));
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  char* dsts[kStages];
  uint32_t lens[kStages];
  int next = blockIdx.x;  // next table index to consider for loading
  auto advance = [&](int c) {
    while (c < n && !is_bulk(tab[c])) c += gridDim.x;
    return c;
  };
  next = advance(next);
  int loaded = 0, stored = 0;
  // prologue: fill the ring
  while (loaded < kStages && next < n) {
    const Chunk ch = tab[next];
    const int s = loaded % kStages;
    const uint32_t bytes = ch.n * 16u;
    dsts[s] = dst_of<kDstRel>(ch, base);
    lens[s] = bytes;
    bulk_load(smem0 + s * kChunkBytes, src_of<kSrcRel>(ch, base), bytes,
              bar0 + 8 * s);
    ++loaded;
    next = advance(next + gridDim.x);
  }
  // Stage of chunk c is reloaded (with chunk c + kStages) right after store
  // c + kLag is issued, once all but the kLag most recent stores have read
  // shared memory: kLag stores and kStages - 1 - kLag loads stay in flight.
  constexpr int kLag = FSDP_BULK_LAG;
  static_assert(kLag >= 0 && kLag < kStages, "bulk lag");
  while (stored < loaded) {
    const int s = stored % kStages;
    mbar_wait(bar0 + 8 * s, (stored / kStages) & 1);
    bulk_store(dsts[s], smem0 + s * kChunkBytes, lens[s]);
    ++stored;
    const int c = stored - 1 - kLag;
    if (c >= 0 && next < n && loaded == c + kStages) {
      asm volatile("cp.async.bulk.wait_group.read " FSDP_STR(FSDP_BULK_LAG) ";" ::: "memory");
      const int rs = c % kStages;
      const Chunk ch = tab[next];
      const uint32_t bytes = ch.n * 16u;
      dsts[rs] = dst_of<kDstRel>(ch, base);
      lens[rs] = bytes;
      bulk_load(smem0 + rs * kChunkBytes, src_of<kSrcRel>(ch, base), bytes, bar0 + 8 * rs);
      ++loaded;
      next = advance(next + gridDim.x);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

#define FSDP_LSU_BOUNDS __launch_bounds__(kThreads, FSDP_MIN_BLOCKS)

// K0: full parameter -> padded shard (absolute -> absolute).
// Programmatic dependent launch (launched with programmaticStreamSerialization,
// launch_table): every CTA first waits until the kernels it depends on have
// completed and their writes are visible (griddepcontrol.wait), then lets the
// next kernel of the stream start launching (griddepcontrol.launch_dependents)
// -- once every CTA of this grid is resident the next grid's CTAs fill the
// SM slots this one's tail frees, instead of after a launch gap.
__device__ __forceinline__ void pdl_enter() {
#if FSDP_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__global__ void FSDP_LSU_BOUNDS fsdp_shard_kernel(const Chunk* tab, int n, char* base, float s) {
  pdl_enter();
  run_table<false, false>(tab, n, base, s);
}
// K1: shards -> segment `rank` of the AG staging buffer (absolute -> staging).
__global__ void FSDP_LSU_BOUNDS fsdp_ag_pack_kernel(const Chunk* tab, int n, char* base, float s) {
  pdl_enter();
  run_table<false, true>(tab, n, base, s);
}
// K3: gathered staging -> full parameters (staging -> absolute).
__global__ void FSDP_LSU_BOUNDS fsdp_ag_unpack_kernel(const Chunk* tab, int n, char* base, float s) {
  pdl_enter();
  run_table<true, false>(tab, n, base, s);
}
// K4: full gradients -> fp32 rank-major chunks * fl32(1/N) (absolute -> staging).
__global__ void FSDP_LSU_BOUNDS fsdp_rs_pack_kernel(const Chunk* tab, int n, char* base, float s) {
  pdl_enter();
  run_table<false, true>(tab, n, base, s);
}
// K6: own reduce-scatter segment -> fp32 gradient shards (staging -> absolute).
__global__ void FSDP_LSU_BOUNDS fsdp_rs_copyout_kernel(const Chunk* tab, int n, char* base, float s) {
  pdl_enter();
  run_table<true, false>(tab, n, base, s);
}

// Bulk-copy (TMA) variants of the pure-copy kernels.
__global__ void __launch_bounds__(32) fsdp_shard_bulk_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table_bulk<false, false>(tab, n, base, s);
}
__global__ void __launch_bounds__(32) fsdp_ag_pack_bulk_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table_bulk<false, true>(tab, n, base, s);
}
__global__ void __launch_bounds__(32) fsdp_ag_unpack_bulk_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table_bulk<true, false>(tab, n, base, s);
}
__global__ void __launch_bounds__(32) fsdp_rs_copyout_bulk_kernel(const Chunk* tab, int n, char* base, float s) {
  run_table_bulk<true, false>(tab, n, base, s);
}

// ------------------------------------------------ peer-memory collectives
namespace {

// K8 body: chunk src is an offset into peer q's segment (q in op_unit bits 24..31).
__device__ __forceinline__ void run_peer_copy(const Chunk* __restrict__ tab, int n, const PeerTable& pt) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    const char* src = pt.p[ch.op_unit >> 24] + ch.src;
    process_chunk<kThreads>(ch, src, reinterpret_cast<char*>(ch.dst), 1.0f);
  }
}

// fp32 accumulate of one 16-B gradient vector from one peer, rank order kept
// by the caller: acc = acc + fl32(x * scale) (first peer: acc = fl32(x * scale)).
template <bool kBf16>
__device__ __forceinline__ void acc_vec(float (&acc)[8], const uint4& v, float scale, bool first) {
  float x[8];
  if (kBf16) {
    x[0] = bf16_lo(v.x); x[1] = bf16_hi(v.x); x[2] = bf16_lo(v.y); x[3] = bf16_hi(v.y);
    x[4] = bf16_lo(v.z); x[5] = bf16_hi(v.z); x[6] = bf16_lo(v.w); x[7] = bf16_hi(v.w);
  } else {
    x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y); x[2] = __uint_as_float(v.z);
    x[3] = __uint_as_float(v.w);
  }
  constexpr int K = kBf16 ? 8 : 4;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float t = __fmul_rn(x[k], scale);
    acc[k] = first ? t : __fadd_rn(acc[k], t);
  }
}

// K9 body: this rank's gradient shard = rank-order fp32 sum over every peer
// (with `accum`: the existing shard + that sum, gradient accumulation).
// Vector chunks: n groups of 8 bf16 (or 4 fp32) elements.  Compile-time world:
// all W peers' 16-B loads are issued before the first add (W loads in flight
// per thread), then added strictly in rank order.
__device__ __forceinline__ void add_existing(float (&acc)[8], const char* dst, uint32_t i, bool bf16) {
  const uint4* d = reinterpret_cast<const uint4*>(dst) + (bf16 ? 2 * i : i);
  const uint4 a = d[0];
  acc[0] = __fadd_rn(__uint_as_float(a.x), acc[0]);
  acc[1] = __fadd_rn(__uint_as_float(a.y), acc[1]);
  acc[2] = __fadd_rn(__uint_as_float(a.z), acc[2]);
  acc[3] = __fadd_rn(__uint_as_float(a.w), acc[3]);
  if (bf16) {
    const uint4 b = d[1];
    acc[4] = __fadd_rn(__uint_as_float(b.x), acc[4]);
    acc[5] = __fadd_rn(__uint_as_float(b.y), acc[5]);
    acc[6] = __fadd_rn(__uint_as_float(b.z), acc[6]);
    acc[7] = __fadd_rn(__uint_as_float(b.w), acc[7]);
  }
}

template <bool kBf16, int W>
__device__ __forceinline__ void peer_reduce16_w(const PeerTable& pt, uint64_t off, char* dst, uint32_t n,
                                                float scale, bool accum) {
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
    const uint64_t o = off + 16ull * i;
    uint4 v[W];
#pragma unroll
    for (int q = 0; q < W; ++q) v[q] = ld_stream(reinterpret_cast<const uint4*>(pt.p[q] + o));
    float acc[8];
#pragma unroll
    for (int q = 0; q < W; ++q) acc_vec<kBf16>(acc, v[q], scale, q == 0);
    if (accum) add_existing(acc, dst, i, kBf16);
    uint4 a, b;
    a.x = __float_as_uint(acc[0]); a.y = __float_as_uint(acc[1]); a.z = __float_as_uint(acc[2]);
    a.w = __float_as_uint(acc[3]);
    if (kBf16) {
      b.x = __float_as_uint(acc[4]); b.y = __float_as_uint(acc[5]); b.z = __float_as_uint(acc[6]);
      b.w = __float_as_uint(acc[7]);
      if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(reinterpret_cast<uint4*>(dst) + 2 * i),
                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
      } else {
        uint4* d = reinterpret_cast<uint4*>(dst) + 2 * i;
        st_v4(d, a);
        st_v4(d + 1, b);
      }
    } else {
      st_v4(reinterpret_cast<uint4*>(dst) + i, a);
    }
  }
}

template <bool kBf16>
__device__ __forceinline__ void peer_reduce16(const PeerTable& pt, int world, uint64_t off, char* dst,
                                              uint32_t n, float scale, bool accum) {
  if (FSDP_K9_TEMPLATED) {
    switch (world) {
      case 1: return peer_reduce16_w<kBf16, 1>(pt, off, dst, n, scale, accum);
      case 2: return peer_reduce16_w<kBf16, 2>(pt, off, dst, n, scale, accum);
      case 4: return peer_reduce16_w<kBf16, 4>(pt, off, dst, n, scale, accum);
      case 8: return peer_reduce16_w<kBf16, 8>(pt, off, dst, n, scale, accum);
      default: break;
    }
  }
  constexpr int K = kBf16 ? 8 : 4;
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
    float acc[8];
    const uint64_t o = off + 16ull * i;
    for (int q0 = 0; q0 < world; q0 += 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u < world) v[u] = ld_stream(reinterpret_cast<const uint4*>(pt.p[q0 + u] + o));
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u < world) acc_vec<kBf16>(acc, v[u], scale, q0 + u == 0);
    }
    if (accum) add_existing(acc, dst, i, kBf16);
    uint4 a, b;
    a.x = __float_as_uint(acc[0]); a.y = __float_as_uint(acc[1]); a.z = __float_as_uint(acc[2]);
    a.w = __float_as_uint(acc[3]);
    if (kBf16) {
      b.x = __float_as_uint(acc[4]); b.y = __float_as_uint(acc[5]); b.z = __float_as_uint(acc[6]);
      b.w = __float_as_uint(acc[7]);
      uint4* d = reinterpret_cast<uint4*>(dst) + 2 * i;
      if (FSDP_WIDEN_V8 && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d), "r"(a.x), "r"(a.y),
                     "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
      } else {
        st_v4(d, a);
        st_v4(d + 1, b);
      }
    } else {
      st_v4(reinterpret_cast<uint4*>(dst) + i, a);
    }
    (void)K;
  }
}

template <bool kBf16>
__device__ __forceinline__ void peer_reduce1(const PeerTable& pt, int world, uint64_t off, char* dst, uint32_t n,
                                             float scale, bool accum) {
  float* d = reinterpret_cast<float*>(dst);
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
    float acc = 0.f;
    for (int q = 0; q < world; ++q) {
      float x;
      if (kBf16) {
        x = __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(pt.p[q] + off + 2ull * i)) << 16);
      } else {
        x = *reinterpret_cast<const float*>(pt.p[q] + off + 4ull * i);
      }
      const float t = __fmul_rn(x, scale);
      acc = q == 0 ? t : __fadd_rn(acc, t);
    }
    d[i] = accum ? __fadd_rn(d[i], acc) : acc;
  }
}

__device__ __forceinline__ void run_peer_reduce(const Chunk* __restrict__ tab, int n, const PeerTable& pt, int world,
                                                float scale, bool accum) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    const uint32_t op = ch.op_unit & 0xFFu, unit = (ch.op_unit >> 8) & 0xFFu;
    char* dst = reinterpret_cast<char*>(ch.dst);
    if (op == OP_ZERO && accum) {
      // pad rows while accumulating: dst + (+0.0), like every other element
      float* d = reinterpret_cast<float*>(dst);
      const uint32_t nf = ch.n * unit / 4;
      for (uint32_t i = threadIdx.x; i < nf; i += kThreads) d[i] = __fadd_rn(d[i], 0.0f);
    } else if (op == OP_ZERO) {
      process_chunk<kThreads>(ch, nullptr, dst, 1.0f);
    } else if (op == OP_PEER_REDUCE_BF16) {
      if (unit == 16) peer_reduce16<true>(pt, world, ch.src, dst, ch.n, scale, accum);
      else peer_reduce1<true>(pt, world, ch.src, dst, ch.n, scale, accum);
    } else {
      if (unit == 16) peer_reduce16<false>(pt, world, ch.src, dst, ch.n, scale, accum);
      else peer_reduce1<false>(pt, world, ch.src, dst, ch.n, scale, accum);
    }
  }
}

}  // namespace

// K8: fused all-gather + copy-out over peer memory.
__global__ void FSDP_LSU_BOUNDS fsdp_p2p_allgather_kernel(const Chunk* tab, int n, const __grid_constant__ PeerTable pt,
                                                          long long hold_ns) {
  pdl_enter();
  const unsigned long long t0 = hold_ns > 0 ? global_ns() : 0ull;
  run_peer_copy(tab, n, pt);
  hold_until(t0, hold_ns);
}
namespace {
// Spin (lanes q < world of the calling warp) until flags[q] >= value at system
// scope, or timeout_ns elapses (then *err = 1 and return: the caller proceeds
// rather than hang).
__device__ __forceinline__ void wait_flags(const unsigned long long* flags, int world, unsigned long long value,
                                           long long timeout_ns, int* err) {
  const int q = threadIdx.x & 31;
  bool timed_out = false;
  if (q < world) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
      if (v >= value) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (timeout_ns > 0 && static_cast<long long>(t - t0) > timeout_ns) {
        timed_out = true;
        break;
      }
      __nanosleep(200);
    }
  }
  if (__any_sync(0xFFFFFFFFu, timed_out) && q == 0 && err) *err = 1;
}

__device__ __forceinline__ void store_flags(const PeerTable& slots, int world, unsigned long long value) {
  for (int q = 0; q < world; ++q) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(const_cast<char*>(slots.p[q]));
    if (p) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(value) : "memory");
  }
}
}  // namespace

// K9: fused gradient widen + 1/N + reduce-scatter + copy-out over peer memory.
// With sync.counter set (the scheduled step) the epoch handshake is fused in
// too: every CTA first waits for the peers' "gradients ready" flags, and the
// last CTA to finish publishes "done reading" to every peer -- no separate
// wait / signal launches around the reduction.
__global__ void __launch_bounds__(kThreads, FSDP_K9_MIN_BLOCKS) fsdp_p2p_reduce_scatter_kernel(
    const Chunk* tab, int n, const __grid_constant__ PeerTable pt, int world, float scale, int accum,
    const __grid_constant__ P2PSync sync, long long hold_ns) {
  pdl_enter();
  if (sync.counter) {
    if (threadIdx.x < 32) wait_flags(sync.wait_flags, world, sync.wait_value, sync.timeout_ns, sync.err);
    __syncthreads();
  }
  const unsigned long long t0 = hold_ns > 0 ? global_ns() : 0ull;
  run_peer_reduce(tab, n, pt, world, scale, accum != 0);
  hold_until(t0, hold_ns);
  if (sync.counter) {
    __syncthreads();  // every thread of this CTA is done reading peer memory
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned int prev = atomicAdd(sync.counter, 1u);
      if (prev == gridDim.x - 1) {  // last CTA: all reads of the grid are done
        __threadfence_system();
        store_flags(sync.signal_slots, world, sync.signal_value);
        *sync.counter = 0u;  // ready for the next launch (stream-ordered)
      }
    }
  }
}

// K10: NVLS reduce-scatter read-out.  Chunk src = offset of this rank's rows in
// the RS staging, read through its multicast mapping: multimem.ld_reduce makes
// the NVSwitch return the fp32 sum of that address over every GPU of the team;
// dst = the gradient shard (absolute), accumulated into when accum.
__global__ void FSDP_LSU_BOUNDS fsdp_nvls_reduce_scatter_kernel(const Chunk* tab, int n, const char* mc_base,
                                                                 int accum) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const Chunk ch = tab[c];
    const char* src = mc_base + ch.src;
    char* dst = reinterpret_cast<char*>(ch.dst);
    const uint32_t unit = (ch.op_unit >> 8) & 0xFFu;
    if (unit == 16) {
      for (uint32_t i = threadIdx.x; i < ch.n; i += kThreads) {
        uint4 v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + 16ull * i)
                     : "memory");
        uint4* d = reinterpret_cast<uint4*>(dst) + i;
        if (accum) v = add4(*d, v);
        st_v4(d, v);
      }
    } else {
      float* d = reinterpret_cast<float*>(dst);
      for (uint32_t i = threadIdx.x; i < ch.n; i += kThreads) {
        uint32_t v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];"
                     : "=r"(v)
                     : "l"(src + 4ull * i)
                     : "memory");
        d[i] = accum ? __fadd_rn(d[i], __uint_as_float(v)) : __uint_as_float(v);
      }
    }
  }
}

// Epoch values are value + *base when `base` (a device-resident epoch
// counter, see fsdp_p2p_schedule.epoch_counter) is set: a captured step then
// replays with fresh epochs.
__global__ void fsdp_p2p_signal_kernel(const __grid_constant__ PeerTable slots, int world, unsigned long long value,
                                       const unsigned long long* base) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  store_flags(slots, world, value + (base ? *base : 0ull));
}

__global__ void fsdp_p2p_wait_kernel(const unsigned long long* flags, int world, unsigned long long value,
                                     long long timeout_ns, int* err, const unsigned long long* base) {
  wait_flags(flags, world, value + (base ? *base : 0ull), timeout_ns, err);
  __threadfence_system();
}

// The step's last p2p kernel: advance the device epoch counter by the epochs
// one step uses, for the next step (replay).
__global__ void fsdp_p2p_epoch_advance_kernel(unsigned long long* base, unsigned long long inc) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *base += inc;
}

// K7: compute proxy.  Four independent FMA chains per thread; the result is
// consumed behind an impossible branch so the loop survives.  The work is cut
// into FSDP_PROXY_WAVES short CTAs per (SM x ctas_per_sm) slot, like the tiles
// of a real GEMM: the block scheduler balances them over whatever SM room is
// free, so a concurrent kernel (a collective, a copy) stretches the proxy in
// proportion to the room it takes -- one long CTA per SM instead measured up to
// 7.7x longer whenever the scheduler had to double CTAs up on some SMs.
__global__ void __launch_bounds__(256) fsdp_compute_proxy_kernel(long long iters, float* sink) {
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
    sink[blockIdx.x] = smem[(threadIdx.x + 1) % 256];
  }
}

namespace {
constexpr int kBulkSmem = kStages * static_cast<int>(kChunkBytes);

bool use_bulk(KernelKind kind) {
  if (FSDP_BULK == 0) return false;
  if (FSDP_BULK == 1) return kind == KK_AG_UNPACK;
  return kind != KK_RS_PACK;
}

template <typename K>
cudaError_t launch_bulk(KernelKind kind, K kernel, int grid, const DevTable& t, char* base, float scale,
                        cudaStream_t s) {
  static bool configured[8] = {};
  if (!configured[kind]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem);
    if (e != cudaSuccess) return e;
    configured[kind] = true;
  }
  kernel<<<grid, 32, kBulkSmem, s>>>(t.d, t.n, base, scale);
  return cudaSuccess;
}
}  // namespace

// Launch configuration of the PDL kernels (kThreads threads, no dynamic smem,
// programmatic stream serialization when FSDP_PDL); `attr` is the caller's storage.
static cudaLaunchConfig_t pdl_config(int grid, cudaStream_t s, cudaLaunchAttribute (&attr)[1]) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = FSDP_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

cudaError_t launch_table(KernelKind kind, const DevTable& t, char* base, float scale, cudaStream_t s,
                         int max_ctas) {
  if (t.n == 0) return cudaSuccess;
  // This library's runtime instance is private to it, and every runtime call
  // it makes is checked where it is made, so a pending error here is stale.
  (void)cudaGetLastError();
  if (use_bulk(kind)) {
    const int sms = max_ctas / FSDP_CTAS_PER_SM;
    const int cap = sms * FSDP_BULK_GRID_PER_SM;
    const int grid = t.n < cap ? t.n : cap;
    cudaError_t e = cudaSuccess;
    switch (kind) {
      case KK_SHARD: e = launch_bulk(kind, fsdp_shard_bulk_kernel, grid, t, base, scale, s); break;
      case KK_AG_PACK: e = launch_bulk(kind, fsdp_ag_pack_bulk_kernel, grid, t, base, scale, s); break;
      case KK_AG_UNPACK: e = launch_bulk(kind, fsdp_ag_unpack_bulk_kernel, grid, t, base, scale, s); break;
      case KK_RS_COPYOUT: e = launch_bulk(kind, fsdp_rs_copyout_bulk_kernel, grid, t, base, scale, s); break;
      default: break;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  const int grid = t.n < max_ctas ? t.n : max_ctas;
  void (*fn)(const Chunk*, int, char*, float) = nullptr;
  switch (kind) {
    case KK_SHARD: fn = fsdp_shard_kernel; break;
    case KK_AG_PACK: fn = fsdp_ag_pack_kernel; break;
    case KK_AG_UNPACK: fn = fsdp_ag_unpack_kernel; break;
    case KK_RS_PACK: fn = fsdp_rs_pack_kernel; break;
    case KK_RS_COPYOUT: fn = fsdp_rs_copyout_kernel; break;
  }
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = pdl_config(grid, s, attr);
  const Chunk* tab = t.d;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, tab, t.n, base, scale);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_p2p_allgather(const DevTable& t, const PeerTable& pt, cudaStream_t s, int max_ctas,
                                 int64_t hold_ns) {
  if (t.n == 0) return cudaSuccess;
  (void)cudaGetLastError();
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = pdl_config(t.n < max_ctas ? t.n : max_ctas, s, attr);
  const Chunk* tab = t.d;
  const long long hold = hold_ns;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fsdp_p2p_allgather_kernel, tab, t.n, pt, hold);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_p2p_reduce_scatter(const DevTable& t, const PeerTable& pt, int world, float scale,
                                      bool accumulate, cudaStream_t s, int max_ctas, const P2PSync* sync,
                                      int64_t hold_ns) {
  P2PSync none{};
  if (t.n == 0 && !sync) return cudaSuccess;
  (void)cudaGetLastError();
  // a fused handshake needs >= 1 CTA even for an empty table
  const int grid = t.n == 0 ? 1 : (t.n < max_ctas ? t.n : max_ctas);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = pdl_config(grid, s, attr);
  const Chunk* tab = t.d;
  const int acc = accumulate ? 1 : 0;
  const P2PSync sy = sync ? *sync : none;
  const long long hold = hold_ns;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fsdp_p2p_reduce_scatter_kernel, tab, t.n, pt, world, scale, acc, sy, hold);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_nvls_reduce(const DevTable& t, const char* mc_base, bool accumulate, cudaStream_t s,
                               int max_ctas) {
  if (t.n == 0) return cudaSuccess;
  (void)cudaGetLastError();
  fsdp_nvls_reduce_scatter_kernel<<<t.n < max_ctas ? t.n : max_ctas, kThreads, 0, s>>>(t.d, t.n, mc_base,
                                                                                     accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_p2p_signal(const PeerTable& slots, int world, uint64_t value, cudaStream_t s,
                              const uint64_t* base) {
  (void)cudaGetLastError();
  fsdp_p2p_signal_kernel<<<1, 32, 0, s>>>(slots, world, static_cast<unsigned long long>(value),
                                          reinterpret_cast<const unsigned long long*>(base));
  return cudaGetLastError();
}

cudaError_t launch_p2p_epoch_advance(uint64_t* base, uint64_t inc, cudaStream_t s) {
  (void)cudaGetLastError();
  fsdp_p2p_epoch_advance_kernel<<<1, 32, 0, s>>>(reinterpret_cast<unsigned long long*>(base),
                                                 static_cast<unsigned long long>(inc));
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const void* flags, int world, uint64_t value, int64_t timeout_ns, int* err,
                            cudaStream_t s, const uint64_t* base) {
  (void)cudaGetLastError();
  fsdp_p2p_wait_kernel<<<1, 32, 0, s>>>(static_cast<const unsigned long long*>(flags), world,
                                        static_cast<unsigned long long>(value), static_cast<long long>(timeout_ns),
                                        err, reinterpret_cast<const unsigned long long*>(base));
  return cudaGetLastError();
}

// K11: an emulated collective (measurement device, fsdp_comm_emulation).

// src / dst may alias (the RS runs in place: dst = this rank's slot of src),
// so neither is __restrict__; each output element is read from every slot by
// the one thread that then writes it.  seg is a multiple of 16 (checked by
// fsdp_run_schedule) and both pointers are 16-B aligned.
__global__ void __launch_bounds__(512) fsdp_comm_emulate_kernel(int reduce, const char* src, char* dst, long long seg,
                                                                 int world, int rank, long long target_ns) {
  const unsigned long long t0 = global_ns();
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;
  if (!reduce) {
    // this rank's segment into every slot (16-B units); its own slot only when
    // the gather runs out of place (send != recv + rank * seg), as NCCL's would
    const uint4* s = reinterpret_cast<const uint4*>(src);
    const long long n = seg / 16;
    const bool in_place = src == dst + static_cast<long long>(rank) * seg;
    for (int q = 0; q < world; ++q) {
      if (q == rank && in_place) continue;
      uint4* d = reinterpret_cast<uint4*>(dst + static_cast<long long>(q) * seg);
      for (long long i = tid; i < n; i += nth) d[i] = s[i];
    }
  } else {
    // fp32 sum of the N slots into this rank's output
    const float4* s = reinterpret_cast<const float4*>(src);
    float4* d = reinterpret_cast<float4*>(dst);
    const long long n = seg / 16;
    for (long long i = tid; i < n; i += nth) {
      float4 a = s[i];
      for (int q = 1; q < world; ++q) {
        const float4 b = s[static_cast<long long>(q) * n + i];
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      d[i] = a;
    }
  }
  // hold the SMs for the collective's modelled duration, like NCCL's CTAs
  if (threadIdx.x == 0)
    while (global_ns() - t0 < static_cast<unsigned long long>(target_ns)) __nanosleep(256);
  __syncthreads();
}

cudaError_t launch_comm_emulation(bool reduce, const char* src, char* dst, int64_t seg, int32_t world, int32_t rank,
                                  int64_t target_ns, int ctas, cudaStream_t s) {
  (void)cudaGetLastError();
  fsdp_comm_emulate_kernel<<<ctas, 512, 0, s>>>(reduce ? 1 : 0, src, dst, seg, world, rank, target_ns);
  return cudaGetLastError();
}

cudaError_t launch_proxy(int64_t iters, int grid, int smem, float* sink, cudaStream_t s) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fsdp_compute_proxy_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  (void)cudaGetLastError();
  // up to FSDP_PROXY_WAVES waves of short CTAs; a short op gets fewer waves
  // (>= FSDP_PROXY_MIN_ITERS iterations per CTA) so that a 3 us norm is not
  // charged the scheduling of thousands of near-empty CTAs
  const long long it = static_cast<long long>(iters);
  const long long waves = std::max(1LL, std::min<long long>(FSDP_PROXY_WAVES, it / FSDP_PROXY_MIN_ITERS));
  const long long per_cta = (it + waves - 1) / waves;
  fsdp_compute_proxy_kernel<<<static_cast<unsigned>(grid * waves), 256, smem, s>>>(per_cta, sink);
  return cudaGetLastError();
}

// CUDA loads kernels lazily by default (CUDA_MODULE_LOADING=LAZY): the first
// launch of a kernel loads it, and loading waits for the device, so a first
// launch enqueued while an epoch wait kernel spins (peer-memory path) would
// only start once the wait times out.  Load every kernel up front.
cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      reinterpret_cast<const void*>(fsdp_comm_emulate_kernel),
      reinterpret_cast<const void*>(fsdp_shard_kernel), reinterpret_cast<const void*>(fsdp_ag_pack_kernel),
      reinterpret_cast<const void*>(fsdp_ag_unpack_kernel), reinterpret_cast<const void*>(fsdp_rs_pack_kernel),
      reinterpret_cast<const void*>(fsdp_rs_copyout_kernel), reinterpret_cast<const void*>(fsdp_shard_bulk_kernel),
      reinterpret_cast<const void*>(fsdp_ag_pack_bulk_kernel), reinterpret_cast<const void*>(fsdp_ag_unpack_bulk_kernel),
      reinterpret_cast<const void*>(fsdp_rs_copyout_bulk_kernel), reinterpret_cast<const void*>(fsdp_p2p_allgather_kernel),
      reinterpret_cast<const void*>(fsdp_p2p_reduce_scatter_kernel), reinterpret_cast<const void*>(fsdp_p2p_signal_kernel),
      reinterpret_cast<const void*>(fsdp_nvls_reduce_scatter_kernel),
      reinterpret_cast<const void*>(fsdp_p2p_epoch_advance_kernel),
      reinterpret_cast<const void*>(fsdp_p2p_wait_kernel), reinterpret_cast<const void*>(fsdp_compute_proxy_kernel)};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return n;
}

}  // namespace fsdp
