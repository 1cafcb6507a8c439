// fsdp_plan_buckets: manual wrapping and Algorithm 1 greedy
// auto-wrapping (Table 1 variables P:226-243).  Host-only,
// integer nanoseconds and bytes, O(P) over the parameters (each candidate's
// T_AG is kept incrementally from the open bucket's segment bytes).
#include <vector>

#include "internal.h"

using namespace fsdp;

namespace {

// T(n) = alpha + ceil(n * beta_fs / 1e6)   (integer units)
int64_t comm_ns(const fsdp_link& l, int64_t n) {
  __int128 p = static_cast<__int128>(n) * l.beta_fs_per_byte;
  return l.alpha_ns + static_cast<int64_t>((p + 999999) / 1000000);
}

}  // namespace

extern "C" fsdp_status fsdp_plan_buckets(const fsdp_plan_in* in, int32_t* bucket_begin,
                                         int32_t* n_buckets, fsdp_plan_trace* trace) {
  if (!in || !bucket_begin || !n_buckets) return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  const int32_t P = in->n_params;
  if (P < 1 || !in->params) return fail(FSDP_ERR_INVALID_ARG, "need >= 1 parameter");
  if (in->world < 1 || in->align_bytes < 1) return fail(FSDP_ERR_INVALID_ARG, "bad world/align");
  if (in->phase != FSDP_PHASE_FWD && in->phase != FSDP_PHASE_BWD)
    return fail(FSDP_ERR_INVALID_ARG, "bad phase");
  if (in->mode < FSDP_PLAN_PER_PARAM || in->mode > FSDP_PLAN_GREEDY)
    return fail(FSDP_ERR_INVALID_ARG, "bad mode");
  const int64_t ep = dtype_bytes(in->param_dtype);
  const int64_t er = in->reduce_bytes;
  if (!ep || er < 1) return fail(FSDP_ERR_INVALID_ARG, "bad dtype");
  for (int32_t j = 0; j < P; ++j) {
    const fsdp_param_desc& p = in->params[j];
    if (p.dim0 < 1 || p.row_numel < 1 || p.reserved != 0)
      return fail(FSDP_ERR_INVALID_ARG, "bad param descriptor");
  }
  const bool timed = in->mode == FSDP_PLAN_GREEDY || in->mode == FSDP_PLAN_SIZE_CAP;
  if (timed && !in->t_compute_ns && in->mode == FSDP_PLAN_GREEDY)
    return fail(FSDP_ERR_INVALID_ARG, "GREEDY needs t_compute_ns");
  const bool bwd = in->phase == FSDP_PHASE_BWD;
  const int64_t N = in->world, A = in->align_bytes;
  auto fwd_index = [&](int32_t pos) { return bwd ? P - 1 - pos : pos; };

  // Per-parameter quantities by forward index.
  std::vector<int64_t> ag_bytes(P), rs_bytes(P), mem(P), tc(P, 0);
  for (int32_t j = 0; j < P; ++j) {
    const int64_t c = (in->params[j].dim0 + N - 1) / N;
    const int64_t elems = c * in->params[j].row_numel;
    ag_bytes[j] = align_up(elems * ep, A);  // aligned member footprint in a segment
    rs_bytes[j] = align_up(elems * er, A);
    mem[j] = in->mem_bytes ? in->mem_bytes[j] : N * elems * ep;
    if (in->t_compute_ns) tc[j] = in->t_compute_ns[j];
  }

  int32_t nb = 0;
  bucket_begin[0] = 0;
  auto close_at = [&](int32_t pos) { bucket_begin[++nb] = pos; };

  if (in->mode == FSDP_PLAN_PER_PARAM || in->mode == FSDP_PLAN_MANUAL) {
    for (int32_t pos = 1; pos < P; ++pos) {
      const int32_t i = fwd_index(pos), prev = fwd_index(pos - 1);
      const bool merge = in->mode == FSDP_PLAN_MANUAL &&
                         in->params[i].module_id == in->params[prev].module_id;
      if (trace) {
        fsdp_plan_trace& t = trace[pos - 1];
        t.t_lhs_ns = t.t_rhs_ns = t.m_lhs = t.m_rhs = 0;
        t.param = i;
        t.accept = merge ? 1 : 0;
      }
      if (!merge) close_at(pos);
    }
    close_at(P);
    *n_buckets = nb;
    return FSDP_OK;
  }

  // Greedy state (Table 1): the open bucket b_j = positions [open_begin, pos).
  int32_t open_begin = 0;
  int64_t open_ag_seg = ag_bytes[fwd_index(0)];  // segment bytes of b_j
  int64_t open_mem = mem[fwd_index(0)];          // M_c
  int64_t t_c = 0;                               // T_c: compute of b_{j-1}
  int64_t t_rs_prev = 0;                         // T^RS_m: RS of b_{j-2}
  int64_t prev_closed_rs_seg = -1;               // RS segment bytes of b_{j-1}
  for (int32_t pos = 1; pos < P; ++pos) {
    const int32_t i = fwd_index(pos);
    const int64_t t_lhs = comm_ns(in->ag, N * (open_ag_seg + ag_bytes[i])) + (bwd ? t_rs_prev : 0);
    const int64_t m_lhs = open_mem + mem[i];
    const bool time_ok = in->mode == FSDP_PLAN_SIZE_CAP || t_lhs <= t_c;
    const bool mem_ok = m_lhs <= in->mem_max_bytes;
    const bool accept = time_ok && mem_ok;
    if (trace) {
      fsdp_plan_trace& t = trace[pos - 1];
      t.t_lhs_ns = t_lhs;
      t.t_rhs_ns = t_c;
      t.m_lhs = m_lhs;
      t.m_rhs = in->mem_max_bytes;
      t.param = i;
      t.accept = accept ? 1 : 0;
    }
    if (accept) {
      open_ag_seg += ag_bytes[i];
      open_mem += mem[i];
      continue;
    }
    // Close b_j = [open_begin, pos): it becomes b_{j-1} for the new bucket.
    int64_t closed_tc = 0, closed_rs_seg = 0;
    for (int32_t q = open_begin; q < pos; ++q) {
      closed_tc += tc[fwd_index(q)];
      closed_rs_seg += rs_bytes[fwd_index(q)];
    }
    t_rs_prev = (bwd && prev_closed_rs_seg >= 0) ? comm_ns(in->rs, N * prev_closed_rs_seg) : 0;
    prev_closed_rs_seg = closed_rs_seg;
    t_c = closed_tc;
    close_at(pos);
    open_begin = pos;
    open_ag_seg = ag_bytes[i];
    open_mem = mem[i];
  }
  close_at(P);
  *n_buckets = nb;
  return FSDP_OK;
}
