// fsdp_plan_search: simulator-guided bucket plans (beyond Algorithm 1).
//
// Algorithm 1 merges a parameter while its all-gather fits the
// previous bucket's compute window -- one local test per decision -- and the
// paper concedes it can lose to manual wrapping.  This planner
// scores WHOLE-phase candidate partitions with the library's own two-stream
// timeline (fsdp_simulate_schedule over the op sequence fsdp_run_schedule
// would enqueue) and hill-climbs: for the current best partition it tries, in
// a fixed order, removing each inner boundary (merge), moving it by -1 / +1,
// then adding a boundary inside each bucket at its midpoint, first and last
// position (split); the first candidate that is feasible (every bucket's M <=
// M_max, or a single parameter) and strictly faster becomes the new best, and
// the scan restarts.  It stops when no move improves (or after max_moves).
// Deterministic; the reference implementation of the same moves is
// tools/plan_search.py (tests/test_plan_search_host.py checks they agree).
#include <algorithm>
#include <map>
#include <utility>
#include <vector>

#include "internal.h"

using namespace fsdp;

namespace {

struct BucketCost {
  int64_t unpack, compute, pack_rs, ag, rs, mem;
};

struct Model {
  const fsdp_plan_in* in;
  const fsdp_search_cost* cost;
  int32_t P;
  bool bwd;
  std::vector<int32_t> order;  // phase position -> forward index
  std::map<std::pair<int32_t, int32_t>, BucketCost> cache;
  std::map<int32_t, std::vector<fsdp_log_entry>> seqs;

  fsdp_status bucket(int32_t a, int32_t b, BucketCost* out) {
    auto key = std::make_pair(a, b);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return FSDP_OK;
    }
    std::vector<fsdp_param_desc> m;
    for (int32_t pos = a; pos < b; ++pos) m.push_back(in->params[order[pos]]);
    if (bwd) std::reverse(m.begin(), m.end());  // members in forward order
    const int32_t N = in->world;
    const int64_t ep = dtype_bytes(in->param_dtype);
    std::vector<int64_t> offs(m.size());
    int64_t ag_seg = 0, rs_seg = 0;
    layout(m.data(), static_cast<int32_t>(m.size()), N, ep, in->align_bytes, offs.data(), &ag_seg);
    layout(m.data(), static_cast<int32_t>(m.size()), N, in->reduce_bytes, in->align_bytes, offs.data(), &rs_seg);
    int64_t full = 0, mem = 0, tc = 0;
    for (int32_t pos = a; pos < b; ++pos) {
      const int32_t j = order[pos];
      const fsdp_param_desc& p = in->params[j];
      full += p.dim0 * p.row_numel * ep;
      mem += in->mem_bytes ? in->mem_bytes[j] : N * ((p.dim0 + N - 1) / N) * p.row_numel * ep;
      tc += in->t_compute_ns ? in->t_compute_ns[j] : 0;
    }
    const bool direct = m.size() == 1 && m[0].dim0 % N == 0 && ag_seg == (m[0].dim0 / N) * m[0].row_numel * ep;
    BucketCost c;
    // durations in ns from bytes per microsecond: bytes * 1000 / (bytes/us), integer
    c.unpack = direct ? 0 : 2 * full * 1000 / cost->unpack_bytes_per_us + cost->copy_launch_ns;
    c.pack_rs = bwd ? (full / ep) * (2 + in->reduce_bytes) * 1000 / cost->pack_rs_bytes_per_us + cost->copy_launch_ns
                    : 0;
    c.compute = tc + cost->compute_overhead_ns;
    FSDP_TRY(fsdp_comm_time_ns(N * ag_seg, &in->ag, &c.ag));
    c.rs = 0;
    if (bwd) FSDP_TRY(fsdp_comm_time_ns(N * rs_seg, &in->rs, &c.rs));
    c.mem = mem;
    cache[key] = c;
    *out = c;
    return FSDP_OK;
  }

  fsdp_status sequence(int32_t k, const std::vector<fsdp_log_entry>** out) {
    auto it = seqs.find(k);
    if (it == seqs.end()) {
      fsdp_schedule s{};
      s.n_fwd = bwd ? 0 : k;
      s.n_bwd = bwd ? k : 0;
      s.flags = (cost->sched_flags & (FSDP_SCHED_REORDER | FSDP_SCHED_FWD_AG_BEFORE_WAIT |
                                      FSDP_SCHED_BWD_AG_BEFORE_WAIT)) | FSDP_SCHED_DRY_RUN;
      std::vector<fsdp_log_entry> log(static_cast<size_t>(10 * k + 8));
      fsdp_step_report rep{};
      rep.log = log.data();
      rep.log_capacity = static_cast<int32_t>(log.size());
      FSDP_TRY(fsdp_run_schedule(nullptr, &s, &rep));
      log.resize(static_cast<size_t>(rep.log_len));
      it = seqs.emplace(k, std::move(log)).first;
    }
    *out = &it->second;
    return FSDP_OK;
  }

  // predicted phase time of a partition (cuts: 0 = c_0 < c_1 < ... < c_K = P); -1 if infeasible
  fsdp_status time(const std::vector<int32_t>& cuts, int64_t* t) {
    const int32_t K = static_cast<int32_t>(cuts.size()) - 1;
    std::vector<BucketCost> bs(static_cast<size_t>(K));
    for (int32_t i = 0; i < K; ++i) {
      FSDP_TRY(bucket(cuts[i], cuts[i + 1], &bs[i]));
      if (bs[i].mem > in->mem_max_bytes && cuts[i + 1] - cuts[i] > 1) {
        *t = -1;
        return FSDP_OK;
      }
    }
    const std::vector<fsdp_log_entry>* seq = nullptr;
    FSDP_TRY(sequence(K, &seq));
    std::vector<int64_t> dur(seq->size(), 0);
    for (size_t i = 0; i < seq->size(); ++i) {
      const fsdp_log_entry& e = (*seq)[i];
      const BucketCost& c = bs[e.bucket];
      switch (e.op) {
        case FSDP_OP_UNPACK: dur[i] = c.unpack; break;
        case FSDP_OP_COMPUTE_F:
        case FSDP_OP_COMPUTE_B: dur[i] = c.compute; break;
        case FSDP_OP_PACK_RS: dur[i] = c.pack_rs; break;
        case FSDP_OP_AG: dur[i] = c.ag; break;
        case FSDP_OP_RS: dur[i] = c.rs; break;
        default: break;
      }
    }
    int64_t exposed = 0;
    return fsdp_simulate_schedule(seq->data(), static_cast<int32_t>(seq->size()), dur.data(), t, &exposed, nullptr,
                                  nullptr);
  }
};

}  // namespace

extern "C" fsdp_status fsdp_plan_search(const fsdp_plan_in* in, const fsdp_search_cost* cost,
                                        const int32_t* start_begin, int32_t n_start, int32_t* bucket_begin,
                                        int32_t* n_buckets, int64_t* predicted_ns) {
  if (!in || !cost || !start_begin || !bucket_begin || !n_buckets)
    return fail(FSDP_ERR_INVALID_ARG, "NULL argument");
  const int32_t P = in->n_params;
  if (P < 1 || !in->params || in->world < 1 || in->align_bytes < 1 || in->reduce_bytes < 1 ||
      !dtype_bytes(in->param_dtype) || (in->phase != FSDP_PHASE_FWD && in->phase != FSDP_PHASE_BWD))
    return fail(FSDP_ERR_INVALID_ARG, "bad fsdp_plan_in");
  for (int32_t j = 0; j < P; ++j) {
    const fsdp_param_desc& p = in->params[j];
    if (p.dim0 < 1 || p.row_numel < 1 || p.reserved != 0) return fail(FSDP_ERR_INVALID_ARG, "bad param descriptor");
  }
  if (cost->unpack_bytes_per_us < 1 || cost->pack_rs_bytes_per_us < 1 || cost->copy_launch_ns < 0 ||
      cost->compute_overhead_ns < 0 || cost->max_moves < 0)
    return fail(FSDP_ERR_INVALID_ARG, "bad fsdp_search_cost");
  if (n_start < 1 || n_start > P || start_begin[0] != 0 || start_begin[n_start] != P)
    return fail(FSDP_ERR_INVALID_ARG, "start plan must partition the phase's positions 0..P");
  for (int32_t i = 0; i < n_start; ++i)
    if (start_begin[i + 1] <= start_begin[i]) return fail(FSDP_ERR_INVALID_ARG, "start plan boundaries not increasing");

  Model md;
  md.in = in;
  md.cost = cost;
  md.P = P;
  md.bwd = in->phase == FSDP_PHASE_BWD;
  md.order.resize(static_cast<size_t>(P));
  for (int32_t pos = 0; pos < P; ++pos) md.order[pos] = md.bwd ? P - 1 - pos : pos;

  std::vector<int32_t> best(start_begin, start_begin + n_start + 1);
  int64_t best_t = 0;
  FSDP_TRY(md.time(best, &best_t));
  if (best_t < 0) return fail(FSDP_ERR_INVALID_ARG, "start plan exceeds mem_max_bytes");
  int32_t moves = 0;
  for (bool improved = true; improved && (cost->max_moves == 0 || moves < cost->max_moves);) {
    improved = false;
    std::vector<std::vector<int32_t>> cands;
    const int32_t nb = static_cast<int32_t>(best.size());
    for (int32_t i = 1; i < nb - 1; ++i) {
      std::vector<int32_t> c = best;  // merge
      c.erase(c.begin() + i);
      cands.push_back(std::move(c));
      for (int32_t d : {-1, 1}) {  // shift
        const int32_t v = best[i] + d;
        if (best[i - 1] < v && v < best[i + 1]) {
          std::vector<int32_t> s = best;
          s[i] = v;
          cands.push_back(std::move(s));
        }
      }
    }
    for (int32_t i = 0; i < nb - 1; ++i) {  // split at the midpoint, first and last position (ascending, unique)
      const int32_t a = best[i], b = best[i + 1];
      std::vector<int32_t> pts{a + (b - a) / 2, a + 1, b - 1};
      std::sort(pts.begin(), pts.end());
      pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
      for (int32_t v : pts)
        if (a < v && v < b) {
          std::vector<int32_t> s = best;
          s.insert(s.begin() + i + 1, v);
          cands.push_back(std::move(s));
        }
    }
    for (const auto& c : cands) {
      int64_t t = 0;
      FSDP_TRY(md.time(c, &t));
      if (t >= 0 && t < best_t) {
        best = c;
        best_t = t;
        improved = true;
        ++moves;
        break;
      }
    }
  }
  *n_buckets = static_cast<int32_t>(best.size()) - 1;
  for (size_t i = 0; i < best.size(); ++i) bucket_begin[i] = best[i];
  if (predicted_ns) *predicted_ns = best_t;
  return FSDP_OK;
}
