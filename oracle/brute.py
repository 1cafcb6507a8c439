"""O8(iii)/(iv) -- plan verifier and exhaustive search (test infrastructure; see
oracle/__init__.py).

The verifier restates Algorithm 1 as properties of a finished plan,
independently of the planner's loop:
  (a) every non-seed member of bucket b_j passes both inequalities evaluated on
      the prefix of b_j ending at it, with window T_c(b_{j-1}) and RS term
      T^RS(b_{j-2}) (backward);
  (b) every close is forced: adding the first member of b_{j+1} to b_j fails
      one of the inequalities.
These two properties characterise the greedy output uniquely, so exhaustive
enumeration of the 2^(P-1) contiguous partitions must find exactly one
plan that passes, and it must equal the planner's.
"""
from itertools import product

from .planner import BWD, SIZE_CAP


def contiguous_partitions(seq):
    """All 2^(P-1) ways to cut ``seq`` into contiguous non-empty runs."""
    n = len(seq)
    if n == 0:
        yield []
        return
    for cuts in product((0, 1), repeat=n - 1):
        parts, cur = [], [seq[0]]
        for c, x in zip(cuts, seq[1:]):
            if c:
                parts.append(cur)
                cur = [x]
            else:
                cur.append(x)
        parts.append(cur)
        yield parts


def _ok(pi, members, window, rs_term):
    t = pi.t_ag(members) + (rs_term if pi.phase == BWD else 0)
    time_ok = t <= window or pi.mode == SIZE_CAP
    return time_ok and pi.mem(members) <= pi.mem_max


def verify_greedy(pi, buckets):
    """True iff ``buckets`` (phase order) satisfies properties (a) and (b)."""
    for j, b in enumerate(buckets):
        window = pi.t_c(buckets[j - 1]) if j >= 1 else 0
        rs_term = pi.t_rs(buckets[j - 2]) if (pi.phase == BWD and j >= 2) else 0
        for k in range(1, len(b)):
            if not _ok(pi, b[:k + 1], window, rs_term):
                return False
        if j + 1 < len(buckets):
            if _ok(pi, b + [buckets[j + 1][0]], window, rs_term):
                return False
    return True
