/* The C ABI used from plain C, no Python and no torch: three simulated ranks
 * of an FSDP job on one GPU (layout-only contexts), one bucket of three
 * parameters with uneven dim 0.
 *   1. fsdp_plan_buckets (GREEDY) and fsdp_layout on the host;
 *   2. fsdp_shard (K0) cuts every rank's shards from the full parameters;
 *   3. fsdp_allgather_bucket: every rank's ISSUE (K1) packs its segment of one
 *      shared staging buffer -- exactly what an all-gather leaves on every
 *      rank -- then WAIT (K3) rebuilds the full parameters: must equal them
 *      bit for bit (all_gather(shard(p)) == p);
 *   4. fsdp_reduce_scatter_bucket: ISSUE (K4) packs fp32(g) * fl32(1/N); the
 *      host adds the segments in rank order (standing in for NCCL) and WAIT
 *      (K6) reads this rank's averaged shard out;
 *   5. fsdp_run_schedule: one step of rank 0 with a C compute hook.
 * Device memory comes from the CUDA driver API.  Exit code 0 and "OK" on
 * success.  Built by __graft_entry__.build(); run by tests/test_gpu_c_abi.py. */
#include <cuda.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fsdp.h"

#define WORLD 3
#define K 3

#define CK(x)                                                              \
  do {                                                                     \
    CUresult r_ = (x);                                                     \
    if (r_ != CUDA_SUCCESS) {                                              \
      fprintf(stderr, "%s:%d CUDA driver error %d\n", __FILE__, __LINE__, (int)r_); \
      exit(2);                                                             \
    }                                                                      \
  } while (0)
#define FK(x)                                                               \
  do {                                                                      \
    fsdp_status s_ = (x);                                                   \
    if (s_ != FSDP_OK) {                                                    \
      fprintf(stderr, "%s:%d fsdp error %d: %s\n", __FILE__, __LINE__, (int)s_, fsdp_last_error()); \
      exit(3);                                                              \
    }                                                                       \
  } while (0)

/* fsdp_compute_hook: a model's compute enqueue point.  A real model would
 * launch its forward / backward kernels on `stream` here. */
typedef struct {
  int calls[2];
  int bad_stream;
  void* expect;
} hook_state;
static int32_t demo_hook(void* user, int32_t phase, int32_t bucket, fsdp_stream_t stream) {
  hook_state* h = (hook_state*)user;
  if (phase < 0 || phase > 1 || bucket != 0) return 1;
  h->calls[phase]++;
  if (stream != h->expect) h->bad_stream = 1;
  return 0;
}

static void* dalloc(size_t n) {
  CUdeviceptr p;
  CK(cuMemAlloc(&p, n < 16 ? 16 : n));
  CK(cuMemsetD8(p, 0xA5, n < 16 ? 16 : n));
  return (void*)(uintptr_t)p;
}
static void h2d(void* d, const void* h, size_t n) { CK(cuMemcpyHtoD((CUdeviceptr)(uintptr_t)d, h, n)); }
static void d2h(void* h, const void* d, size_t n) { CK(cuMemcpyDtoH(h, (CUdeviceptr)(uintptr_t)d, n)); }

int main(void) {
  CUdevice dev;
  CUcontext cctx;
  CK(cuInit(0));
  CK(cuDeviceGet(&dev, 0));
  CK(cuDevicePrimaryCtxRetain(&cctx, dev));
  CK(cuCtxSetCurrent(cctx));
  if (fsdp_abi_version() != FSDP_ABI_VERSION) return 4;

  const fsdp_param_desc p[K] = {{37, 5, 0, 0}, {8, 16, 0, 0}, {4096, 1, 1, 0}};
  /* 1. host-side plan and layout */
  int64_t tc[K] = {1000, 50000, 10};
  fsdp_plan_in in;
  memset(&in, 0, sizeof in);
  in.params = p;
  in.t_compute_ns = tc;
  in.ag.alpha_ns = 100;
  in.ag.beta_fs_per_byte = 1000000;
  in.rs = in.ag;
  in.mem_max_bytes = 1 << 30;
  in.n_params = K;
  in.world = WORLD;
  in.align_bytes = 16;
  in.mode = FSDP_PLAN_GREEDY;
  in.phase = FSDP_PHASE_FWD;
  in.param_dtype = FSDP_BF16;
  in.reduce_bytes = 4;
  int32_t begin[K + 1], nb = 0;
  FK(fsdp_plan_buckets(&in, begin, &nb, NULL));
  int64_t offs[K], seg = 0, roffs[K], rseg = 0;
  FK(fsdp_layout(p, K, WORLD, 2, 16, offs, &seg));
  FK(fsdp_layout(p, K, WORLD, 4, 16, roffs, &rseg));
  printf("greedy forward plan: %d bucket(s); AG segment %lld B, RS segment %lld B\n", nb, (long long)seg,
         (long long)rseg);

  /* full parameters (bf16 bit patterns) and gradients (bf16 1.0 everywhere) */
  uint16_t* host_full[K];
  void* dev_full[K];
  void* dev_grad[WORLD][K];
  for (int j = 0; j < K; ++j) {
    size_t n = (size_t)(p[j].dim0 * p[j].row_numel);
    host_full[j] = (uint16_t*)malloc(2 * n);
    for (size_t i = 0; i < n; ++i) host_full[j][i] = (uint16_t)((i * 2654435761u + 977u * j) >> 7);
    dev_full[j] = dalloc(2 * n);
    h2d(dev_full[j], host_full[j], 2 * n);
    uint16_t* ones = (uint16_t*)malloc(2 * n);
    for (size_t i = 0; i < n; ++i) ones[i] = 0x3F80; /* 1.0 */
    for (int r = 0; r < WORLD; ++r) {
      dev_grad[r][j] = dalloc(2 * n);
      h2d(dev_grad[r][j], ones, 2 * n);
    }
    free(ones);
  }

  /* 2. contexts, shards, buckets */
  fsdp_ctx* ctx[WORLD];
  fsdp_bucket* b[WORLD];
  void* shards[WORLD][K];
  void* outs[WORLD][K];
  void* gsh[WORLD][K];
  for (int r = 0; r < WORLD; ++r) {
    FK(fsdp_ctx_create(&ctx[r], WORLD, r, 0, NULL, NULL));
    for (int j = 0; j < K; ++j) {
      fsdp_shard_info si;
      FK(fsdp_shard(WORLD, r, &p[j], FSDP_BF16, NULL, NULL, &si, NULL));
      shards[r][j] = dalloc(2 * (size_t)si.shard_numel);
      FK(fsdp_shard(WORLD, r, &p[j], FSDP_BF16, dev_full[j], shards[r][j], &si, NULL));
      outs[r][j] = dalloc(2 * (size_t)(p[j].dim0 * p[j].row_numel));
      gsh[r][j] = dalloc(4 * (size_t)si.shard_numel);
    }
    fsdp_bucket_desc d;
    memset(&d, 0, sizeof d);
    d.params = p;
    d.shards = shards[r];
    d.fulls = outs[r];
    d.full_grads = (const void* const*)dev_grad[r];
    d.grad_shards = gsh[r];
    d.k = K;
    d.align_bytes = 16;
    d.param_dtype = FSDP_BF16;
    d.grad_dtype = FSDP_BF16;
    int64_t ag = 0, rs = 0;
    FK(fsdp_bucket_create(ctx[r], &d, &b[r], &ag, &rs));
    if (ag != seg || rs != rseg) return 5;
  }

  /* 3. all-gather */
  void* ag_st = dalloc((size_t)(WORLD * seg));
  for (int r = 0; r < WORLD; ++r) FK(fsdp_allgather_bucket(ctx[r], b[r], ag_st, NULL, NULL, FSDP_ISSUE));
  int bad = 0;
  for (int r = 0; r < WORLD; ++r) {
    FK(fsdp_allgather_bucket(ctx[r], b[r], ag_st, NULL, NULL, FSDP_WAIT));
    CK(cuCtxSynchronize());
    for (int j = 0; j < K; ++j) {
      size_t n = (size_t)(p[j].dim0 * p[j].row_numel);
      uint16_t* got = (uint16_t*)malloc(2 * n);
      d2h(got, outs[r][j], 2 * n);
      if (memcmp(got, host_full[j], 2 * n) != 0) ++bad;
      free(got);
    }
  }
  printf("all-gather: %s\n", bad ? "MISMATCH" : "bit-exact on every rank");

  /* 4. reduce-scatter(avg) */
  void* rs_st[WORLD];
  float* packed[WORLD];
  const size_t rs_elems = (size_t)(WORLD * rseg / 4);
  for (int r = 0; r < WORLD; ++r) {
    rs_st[r] = dalloc((size_t)(WORLD * rseg));
    FK(fsdp_reduce_scatter_bucket(ctx[r], b[r], rs_st[r], NULL, NULL, FSDP_ISSUE));
  }
  CK(cuCtxSynchronize());
  for (int r = 0; r < WORLD; ++r) {
    packed[r] = (float*)malloc(4 * rs_elems);
    d2h(packed[r], rs_st[r], 4 * rs_elems);
  }
  const float inv = 1.0f / (float)WORLD;
  const float want = (inv + inv) + inv; /* rank-order fp32 sum of the pre-scaled 1.0s */
  for (int q = 0; q < WORLD; ++q) {
    float* mine = (float*)malloc((size_t)rseg);
    for (size_t i = 0; i < (size_t)rseg / 4; ++i) {
      float acc = packed[0][q * rseg / 4 + i];
      for (int r = 1; r < WORLD; ++r) acc = acc + packed[r][q * rseg / 4 + i];
      mine[i] = acc;
    }
    h2d((char*)rs_st[q] + q * rseg, mine, (size_t)rseg);
    free(mine);
    FK(fsdp_reduce_scatter_bucket(ctx[q], b[q], rs_st[q], NULL, NULL, FSDP_WAIT));
    CK(cuCtxSynchronize());
    for (int j = 0; j < K; ++j) {
      fsdp_shard_info si;
      FK(fsdp_shard(WORLD, q, &p[j], FSDP_BF16, NULL, NULL, &si, NULL));
      float* g = (float*)malloc(4 * (size_t)si.shard_numel);
      d2h(g, gsh[q][j], 4 * (size_t)si.shard_numel);
      for (int64_t i = 0; i < si.shard_numel; ++i) {
        const float w = i < si.valid_rows * p[j].row_numel ? want : 0.0f;
        if (memcmp(&g[i], &w, 4) != 0) {
          ++bad;
          break;
        }
      }
      free(g);
    }
  }
  printf("reduce-scatter(avg): %s\n", bad ? "MISMATCH" : "bit-exact on every rank");

  /* 5. one scheduled step of rank 0 (fsdp_run_schedule) with the model's
   *    compute supplied by a C callback (fsdp_compute_hook): the step
   *    re-gathers the bucket before each use, so the parameters must again
   *    be bit-exact, and the hook must run once per phase on the compute stream */
  {
    CUstream cs, ms;
    CK(cuStreamCreate(&cs, CU_STREAM_NON_BLOCKING));
    CK(cuStreamCreate(&ms, CU_STREAM_NON_BLOCKING));
    hook_state hs;
    memset(&hs, 0, sizeof hs);
    hs.expect = (void*)cs;
    fsdp_compute_hook hk = {demo_hook, &hs};
    for (int j = 0; j < K; ++j) CK(cuMemsetD8((CUdeviceptr)(uintptr_t)outs[0][j], 0x5C, 2 * (size_t)(p[j].dim0 * p[j].row_numel)));
    void* ag_st2 = dalloc((size_t)(WORLD * seg));
    void* rs_st2 = dalloc((size_t)(WORLD * rseg));
    fsdp_schedule sc;
    memset(&sc, 0, sizeof sc);
    sc.fwd = &b[0];
    sc.bwd = &b[0];
    sc.n_fwd = 1;
    sc.n_bwd = 1;
    sc.ag_staging[0] = ag_st;
    sc.ag_staging[1] = ag_st2;
    sc.rs_staging[0] = rs_st[0];
    sc.rs_staging[1] = rs_st2;
    sc.compute = (void*)cs;
    sc.comm = (void*)ms;
    sc.flags = FSDP_SCHED_REORDER | FSDP_SCHED_FWD_AG_BEFORE_WAIT;
    sc.proxy_ctas_per_sm = 1;
    sc.hook = &hk;
    fsdp_step_report rep;
    memset(&rep, 0, sizeof rep);
    FK(fsdp_run_schedule(ctx[0], &sc, &rep));
    CK(cuCtxSynchronize());
    int sbad = hs.calls[0] != 1 || hs.calls[1] != 1 || hs.bad_stream || rep.op_count[FSDP_OP_COMPUTE_F] != 1 ||
               rep.op_count[FSDP_OP_COMPUTE_B] != 1;
    for (int j = 0; j < K; ++j) {
      size_t n = (size_t)(p[j].dim0 * p[j].row_numel);
      uint16_t* got = (uint16_t*)malloc(2 * n);
      d2h(got, outs[0][j], 2 * n);
      /* rank 0 of a layout-only ctx gathers only its own rows: compare those */
      fsdp_shard_info si;
      FK(fsdp_shard(WORLD, 0, &p[j], FSDP_BF16, NULL, NULL, &si, NULL));
      if (memcmp(got, host_full[j], 2 * (size_t)(si.valid_rows * p[j].row_numel)) != 0) ++sbad;
      free(got);
    }
    printf("scheduled step with a C compute hook: %s\n", sbad ? "MISMATCH" : "hook ran per phase, re-gather bit-exact");
    bad += sbad;
    CK(cuStreamDestroy(cs));
    CK(cuStreamDestroy(ms));
  }

  for (int r = 0; r < WORLD; ++r) {
    FK(fsdp_bucket_destroy(b[r]));
    FK(fsdp_ctx_destroy(ctx[r]));
  }
  printf("%s\n", bad ? "FAILED" : "OK");
  return bad ? 1 : 0;
}
