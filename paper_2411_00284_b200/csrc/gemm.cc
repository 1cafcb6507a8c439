// Linear-layer compute for fsdp_run_schedule (fsdp_gemm_compute): cuBLASLt
// bf16 GEMMs with fp32 accumulation (a plain library GEMM: the hot path of this
// library is the data movement around it).  Plans and heuristic algorithms are
// cached per shape in the ctx.
#include <cublasLt.h>

#include <map>
#include <tuple>

#include "internal.h"

namespace fsdp {

namespace {

struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo{};
  bool has_algo = false;
};

using Key = std::tuple<int, int, int, int, int, int, int, int, int64_t>;  // ta tb m n k lda ldb ldc ws

struct Cache {
  cublasLtHandle_t lt = nullptr;
  std::map<Key, Plan> plans;
  ~Cache() {
    for (auto& kv : plans) {
      Plan& p = kv.second;
      if (p.desc) cublasLtMatmulDescDestroy(p.desc);
      if (p.a) cublasLtMatrixLayoutDestroy(p.a);
      if (p.b) cublasLtMatrixLayoutDestroy(p.b);
      if (p.c) cublasLtMatrixLayoutDestroy(p.c);
    }
    if (lt) cublasLtDestroy(lt);
  }
};

fsdp_status lt_fail(cublasStatus_t st, const char* what) {
  return fail(FSDP_ERR_CUDA, std::string("cuBLASLt ") + what + " failed: status " + std::to_string(static_cast<int>(st)));
}

}  // namespace

void gemm_cache_destroy(void* p) { delete static_cast<Cache*>(p); }

// C (m x n, col-major, ldc) = op(A) (m x k) . op(B) (k x n); bf16 in/out, fp32 accumulate.
fsdp_status gemm_bf16(fsdp_ctx* c, bool ta, bool tb, int m, int n, int k, const void* A, int lda, const void* B,
                      int ldb, void* C, int ldc, void* ws, int64_t ws_bytes, cudaStream_t s) {
  if (!c->gemm_cache) c->gemm_cache = new Cache();
  Cache* cache = static_cast<Cache*>(c->gemm_cache);
  cublasStatus_t st;
  if (!cache->lt && (st = cublasLtCreate(&cache->lt)) != CUBLAS_STATUS_SUCCESS) return lt_fail(st, "create");
  const Key key(ta, tb, m, n, k, lda, ldb, ldc, ws_bytes);
  auto it = cache->plans.find(key);
  if (it == cache->plans.end()) {
    Plan p;
    const cublasOperation_t opa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, opb = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
    if ((st = cublasLtMatmulDescCreate(&p.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F)) != CUBLAS_STATUS_SUCCESS)
      return lt_fail(st, "desc");
    cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &opa, sizeof(opa));
    cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &opb, sizeof(opb));
    cublasLtMatrixLayoutCreate(&p.a, CUDA_R_16BF, ta ? k : m, ta ? m : k, lda);
    cublasLtMatrixLayoutCreate(&p.b, CUDA_R_16BF, tb ? n : k, tb ? k : n, ldb);
    cublasLtMatrixLayoutCreate(&p.c, CUDA_R_16BF, m, n, ldc);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    uint64_t wsb = static_cast<uint64_t>(ws_bytes);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    cublasLtMatmulHeuristicResult_t res;
    int found = 0;
    st = cublasLtMatmulAlgoGetHeuristic(cache->lt, p.desc, p.a, p.b, p.c, p.c, pref, 1, &res, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st == CUBLAS_STATUS_SUCCESS && found > 0) {
      p.algo = res.algo;
      p.has_algo = true;
    }
    it = cache->plans.emplace(key, p).first;
  }
  const float alpha = 1.0f, beta = 0.0f;
  Plan& p = it->second;
  st = cublasLtMatmul(cache->lt, p.desc, &alpha, A, p.a, B, p.b, &beta, C, p.c, C, p.c,
                      p.has_algo ? &p.algo : nullptr, ws, static_cast<size_t>(ws_bytes), s);
  if (st != CUBLAS_STATUS_SUCCESS) return lt_fail(st, "matmul");
  return FSDP_OK;
}

// The linear-layer compute of one bucket (see fsdp_gemm_compute in fsdp.h).
fsdp_status bucket_compute(fsdp_ctx* c, fsdp_bucket* b, const fsdp_gemm_compute* g, bool backward, cudaStream_t s,
                           int* launches) {
  const int T = static_cast<int>(g->tokens);
  for (size_t j = 0; j < b->members.size(); ++j) {
    const fsdp_param_desc& p = b->members[j];
    if (p.row_numel <= 1) continue;
    const int out = static_cast<int>(p.dim0), in = static_cast<int>(p.row_numel);
    const void* W = b->fulls[j];
    if (!backward) {
      // Y' (out x T) = Wc^T . Xc,   Wc = W as col-major (in x out)
      FSDP_TRY(gemm_bf16(c, true, false, out, T, in, W, in, g->x, in, g->y, out, g->workspace, g->workspace_bytes, s));
      ++*launches;
    } else {
      // dX' (in x T) = Wc . dYc;   dWc (in x out) = Xc . dYc^T  -> full gradient (row-major [out, in])
      FSDP_TRY(gemm_bf16(c, false, false, in, T, out, W, in, g->dy, out, g->y, in, g->workspace, g->workspace_bytes, s));
      FSDP_TRY(gemm_bf16(c, false, true, in, out, T, g->x, in, g->dy, out, b->grads[j], in, g->workspace,
                         g->workspace_bytes, s));
      *launches += 2;
    }
  }
  return FSDP_OK;
}

}  // namespace fsdp
