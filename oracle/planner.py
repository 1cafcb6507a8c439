"""O8 -- bucket planning (test infrastructure; see oracle/__init__.py).

Algorithm 1 with the variables of Table 1, written
step by step in the paper's order:

  forward  (l.4-5):   bucket i iff  T^AG_(m+mi) <= T_c            and  M_c + M_ci <= M_max
  backward (l.10-11): bucket i iff  T^RS_m + T^AG_(m+mi) <= T_c   and  M_c + M_ci <= M_max

Readings:
  * phase execution order: forward-use order for FWD, its reverse for BWD;
    one independent plan per phase (Alg. 1's isForward / isBackward branches);
  * T^AG_(m+mi) = alpha + beta * n of the merged bucket (one alpha: P:175),
    n = N * seg(bucket) in param dtype (G8);
  * T_c ("current step's computation time") = total compute of the previously
    closed bucket, whose compute the open bucket's prefetch overlaps;
    0 before any bucket has closed, so the first bucket is its first parameter (G10);
  * T^RS_m ("last step's bucketed RS") = RS time of the bucket closed before the
    previous one, b_{j-2}, which shares the comm stream with AG(b_j) during the
    compute of b_{j-1} (G11);
  * M_c = sum of M_ci over the open bucket (G13); M_ci defaults to the padded
    gathered bytes N c_i R_i e_p;
  * ties accept (<=, as printed; G15).

Other modes: MANUAL = one bucket per wrapped module: maximal runs of
equal module id in phase order; PER_PARAM = singletons (the unbucketed
baseline); SIZE_CAP = GREEDY with the time test disabled (bucket-size sweep).
"""
from .cost import comm_time
from .layout import bucket_layout

PER_PARAM, MANUAL, SIZE_CAP, GREEDY = "per_param", "manual", "size_cap", "greedy"
FWD, BWD = "fwd", "bwd"


class PlanInput:
    """Mirror of the planner's inputs.

    params: list of (dim0, row_numel, module_id) in forward-use order.
    t_compute_ns / mem_bytes: per parameter, indexed by forward index.
    ag / rs: (alpha_ns, beta_fs_per_byte).
    """

    def __init__(self, params, world, t_compute_ns, ag, rs, mem_max, mode, phase,
                 param_bytes=2, reduce_bytes=4, align=16, mem_bytes=None):
        self.params = list(params)
        self.world = world
        self.t_compute_ns = list(t_compute_ns)
        self.ag = ag
        self.rs = rs
        self.mem_max = mem_max
        self.mode = mode
        self.phase = phase
        self.param_bytes = param_bytes
        self.reduce_bytes = reduce_bytes
        self.align = align
        if mem_bytes is None:
            mem_bytes = [world * (-(-d // world)) * r * param_bytes for d, r, _ in self.params]
        self.mem_bytes = list(mem_bytes)

    def order(self):
        n = len(self.params)
        return list(range(n)) if self.phase == FWD else list(range(n - 1, -1, -1))

    def dims(self, members):
        return [self.params[j][:2] for j in sorted(members)]

    def t_ag(self, members):
        _, seg = bucket_layout(self.dims(members), self.world, self.param_bytes, self.align)
        return comm_time(self.world * seg, *self.ag)

    def t_rs(self, members):
        _, seg = bucket_layout(self.dims(members), self.world, self.reduce_bytes, self.align)
        return comm_time(self.world * seg, *self.rs)

    def mem(self, members):
        return sum(self.mem_bytes[j] for j in members)

    def t_c(self, members):
        return sum(self.t_compute_ns[j] for j in members)


def plan(pi):
    """Returns (buckets, trace).

    buckets: list of lists of forward indices, in the phase's execution order
    (each list in phase order).  trace: one record per decision i = 2..P:
    dict(param, t_lhs, t_rhs, m_lhs, m_rhs, accept).
    """
    q = pi.order()
    if not q:
        return [], []
    trace = []
    if pi.mode == PER_PARAM:
        for i in q[1:]:
            trace.append(dict(param=i, t_lhs=0, t_rhs=0, m_lhs=0, m_rhs=0, accept=False))
        return [[i] for i in q], trace
    if pi.mode == MANUAL:
        buckets = [[q[0]]]
        for i in q[1:]:
            same = pi.params[i][2] == pi.params[buckets[-1][-1]][2]
            trace.append(dict(param=i, t_lhs=0, t_rhs=0, m_lhs=0, m_rhs=0, accept=same))
            if same:
                buckets[-1].append(i)
            else:
                buckets.append([i])
        return buckets, trace
    if pi.mode not in (GREEDY, SIZE_CAP):
        raise ValueError(pi.mode)

    closed = []          # closed buckets b_1 .. b_{j-1}
    open_b = [q[0]]      # b_j, seeded unconditionally with q_1
    t_c = 0              # T_c: compute of b_{j-1} (0 before any close)
    t_rs_last = 0        # T^RS_m: RS of b_{j-2} (backward only)
    for i in q[1:]:
        cand = open_b + [i]
        t_lhs = pi.t_ag(cand) + (t_rs_last if pi.phase == BWD else 0)
        t_rhs = t_c
        m_lhs = pi.mem(open_b) + pi.mem_bytes[i]
        m_rhs = pi.mem_max
        time_ok = (t_lhs <= t_rhs) or pi.mode == SIZE_CAP
        mem_ok = m_lhs <= m_rhs
        accept = time_ok and mem_ok
        trace.append(dict(param=i, t_lhs=t_lhs, t_rhs=t_rhs, m_lhs=m_lhs, m_rhs=m_rhs,
                          accept=accept))
        if accept:
            open_b = cand
        else:
            closed.append(open_b)
            t_c = pi.t_c(closed[-1])
            t_rs_last = pi.t_rs(closed[-2]) if (pi.phase == BWD and len(closed) >= 2) else 0
            open_b = [i]
    closed.append(open_b)
    return closed, trace


def bucket_begin(buckets):
    """Phase-position prefix offsets: bucket b covers positions [bb[b], bb[b+1])."""
    bb = [0]
    for b in buckets:
        bb.append(bb[-1] + len(b))
    return bb
