// Cost model and two-stream timeline prediction of an op sequence
// (the paper's auto-wrap estimates exposure from exactly these inputs: T_c per
// compute node and alpha + beta n per collective).  Host-only.
#include <algorithm>
#include <map>
#include <tuple>

#include "internal.h"

using namespace fsdp;

extern "C" fsdp_status fsdp_comm_time_ns(int64_t nbytes, const fsdp_link* l, int64_t* ns) {
  if (!l || !ns || nbytes < 0 || l->alpha_ns < 0 || l->beta_fs_per_byte < 0)
    return fail(FSDP_ERR_INVALID_ARG, "bad comm_time arguments");
  const __int128 p = static_cast<__int128>(nbytes) * l->beta_fs_per_byte;
  *ns = l->alpha_ns + static_cast<int64_t>((p + 999999) / 1000000);
  return FSDP_OK;
}

extern "C" fsdp_status fsdp_simulate_schedule(const fsdp_log_entry* seq, int32_t n, const int64_t* dur,
                                              int64_t* total_ns, int64_t* exposed_ns, int64_t* start_ns,
                                              int64_t* end_ns) {
  if (n < 0 || (n && (!seq || !dur)) || !total_ns || !exposed_ns)
    return fail(FSDP_ERR_INVALID_ARG, "bad simulate arguments");
  using Key = std::tuple<int32_t, int32_t, int32_t>;  // phase, op, bucket
  std::map<Key, int64_t> done;                      // finish time of packs and collectives
  int64_t t_cmp = 0, t_comm = 0, exposed = 0;
  for (int32_t i = 0; i < n; ++i) {
    const fsdp_log_entry& e = seq[i];
    int64_t s = 0, f = 0;
    if (e.op == FSDP_OP_AG || e.op == FSDP_OP_RS) {
      const int32_t pk = e.op == FSDP_OP_AG ? FSDP_OP_PACK_AG : FSDP_OP_PACK_RS;
      auto it = done.find(Key(e.phase, pk, e.bucket));
      if (it == done.end()) return fail(FSDP_ERR_INVALID_ARG, "collective before its pack");
      s = std::max(t_comm, it->second);
      f = s + dur[i];
      t_comm = f;
      done[Key(e.phase, e.op, e.bucket)] = f;
    } else if (e.op == FSDP_OP_WAIT_AG || e.op == FSDP_OP_WAIT_RS) {
      const int32_t co = e.op == FSDP_OP_WAIT_AG ? FSDP_OP_AG : FSDP_OP_RS;
      auto it = done.find(Key(e.phase, co, e.bucket));
      if (it == done.end()) return fail(FSDP_ERR_INVALID_ARG, "wait before its collective");
      s = t_cmp;
      if (it->second > t_cmp) {
        exposed += it->second - t_cmp;
        t_cmp = it->second;
      }
      f = t_cmp;
    } else {
      if (dur[i] < 0) return fail(FSDP_ERR_INVALID_ARG, "negative duration");
      s = t_cmp;
      t_cmp += dur[i];
      f = t_cmp;
      if (e.op == FSDP_OP_PACK_AG || e.op == FSDP_OP_PACK_RS) done[Key(e.phase, e.op, e.bucket)] = f;
    }
    if (start_ns) start_ns[i] = s;
    if (end_ns) end_ns[i] = f;
  }
  *total_ns = std::max(t_cmp, t_comm);
  *exposed_ns = exposed;
  return FSDP_OK;
}

// Memory curve of the FSDP buffers (reading G40): allocate on produce, free
// after the last use, peak after each op's allocation.
extern "C" fsdp_status fsdp_simulate_memory(const fsdp_log_entry* seq, int32_t n, const fsdp_mem_sizes* sz,
                                            int64_t* peak_bytes, int64_t* live_out) {
  if (n < 0 || (n && !seq) || !sz || !peak_bytes || sz->n_fwd < 0 || sz->n_bwd < 0)
    return fail(FSDP_ERR_INVALID_ARG, "bad simulate_memory arguments");
  if ((sz->n_fwd && (!sz->ag_fwd || !sz->full_fwd)) ||
      (sz->n_bwd && (!sz->ag_bwd || !sz->full_bwd || !sz->grad_bwd || !sz->rs_bwd)))
    return fail(FSDP_ERR_INVALID_ARG, "simulate_memory: NULL size array");
  int64_t live = 0, peak = 0;
  // a backward bucket 0 without UNPACK reuses the last forward bucket's
  // parameters (G42): that bucket's COMPUTE_F frees nothing
  bool has_unpack0 = false, has_compute_b0 = false;
  int32_t last_f = -1;
  for (int32_t i = 0; i < n; ++i) {
    const fsdp_log_entry& e = seq[i];
    if (e.phase == 1 && e.bucket == 0 && e.op == FSDP_OP_UNPACK) has_unpack0 = true;
    if (e.phase == 1 && e.bucket == 0 && e.op == FSDP_OP_COMPUTE_B) has_compute_b0 = true;
    if (e.phase == 0 && e.op == FSDP_OP_COMPUTE_F) last_f = std::max(last_f, e.bucket);
  }
  const bool keep = has_compute_b0 && !has_unpack0;
  for (int32_t i = 0; i < n; ++i) {
    const fsdp_log_entry& e = seq[i];
    const bool fwd = e.phase == 0;
    if ((e.phase != 0 && e.phase != 1) || e.bucket < 0 || e.bucket >= (fwd ? sz->n_fwd : sz->n_bwd))
      return fail(FSDP_ERR_INVALID_ARG, "simulate_memory: bucket out of range");
    const int32_t b = e.bucket;
    const int64_t ag = fwd ? sz->ag_fwd[b] : sz->ag_bwd[b];
    const int64_t full = fwd ? sz->full_fwd[b] : sz->full_bwd[b];
    const int64_t grad = fwd ? 0 : sz->grad_bwd[b];
    const int64_t rs = fwd ? 0 : sz->rs_bwd[b];
    if (ag < 0 || full < 0 || grad < 0 || rs < 0) return fail(FSDP_ERR_INVALID_ARG, "simulate_memory: negative size");
    auto alloc = [&](int64_t x) {
      live += x;
      peak = std::max(peak, live);
    };
    switch (e.op) {
      case FSDP_OP_PACK_AG: alloc(ag); break;
      case FSDP_OP_UNPACK: alloc(full); live -= ag; break;
      case FSDP_OP_COMPUTE_F:
        if (!(keep && b == last_f)) live -= full;
        break;
      case FSDP_OP_COMPUTE_B: alloc(grad); live -= full; break;
      case FSDP_OP_PACK_RS: alloc(rs); live -= grad; break;
      case FSDP_OP_COPYOUT_RS: live -= rs; break;
      default: break;  // AG, RS, WAIT_*: in place
    }
    if (live < 0) return fail(FSDP_ERR_INVALID_ARG, "simulate_memory: a buffer freed before it was allocated");
    if (live_out) live_out[i] = live;
  }
  *peak_bytes = peak;
  return FSDP_OK;
}
