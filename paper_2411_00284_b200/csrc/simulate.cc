// Cost model and two-stream timeline prediction of an op sequence
// (the paper's auto-wrap estimates exposure from exactly these inputs: T_c per
// compute node and alpha + beta n per collective).  Host-only.
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
