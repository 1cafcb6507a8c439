"""O9 / O10 pins: Fig. 2 prose orderings and SPEC's examples
(S:292-294), linear-extension validity, simulator hand traces (S:411-413,
S:421/S:531), exposed = total - compute busy, FIFO non-interference
(S:309), reorder <= vanilla, and optimum <= greedy on brute-force instances."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import schedule as S
from oracle.brute import contiguous_partitions
from oracle.planner import BWD, FWD, GREEDY, PER_PARAM, PlanInput, plan
from oracle.sim import simulate


def _idx(seq, ph, op, b):
    return seq.index((ph, op, b, 1 if op in S.COMM_OPS else 0))


def test_fig2_forward_prefetch_before_wait():
    seq = S.forward_sequence(2, True, S.BEFORE)
    # "AG34 is reordered in front of Wa12"
    assert _idx(seq, 0, S.AG, 1) < _idx(seq, 0, S.WAIT_AG, 0)
    comm = [e for e in seq if e[3] == 1]
    assert comm == [(0, S.AG, 0, 1), (0, S.AG, 1, 1)]


def test_fig2_backward_after_wait_and_wr_before_next_rs():
    seq = S.backward_sequence(3, True, S.AFTER)
    # "AG34 is placed after Wa12" (and its copy-out, G33)
    assert _idx(seq, 1, S.UNPACK, 0) < _idx(seq, 1, S.AG, 1)
    # "The Wr12 is placed before RS34"
    for b in range(2):
        assert _idx(seq, 1, S.WAIT_RS, b) < _idx(seq, 1, S.RS, b + 1)
    # RS(b) issued before the next bucket's AG-wait: it overlaps later compute
    assert _idx(seq, 1, S.RS, 0) < _idx(seq, 1, S.WAIT_AG, 1)


def test_single_bucket_reorder_equals_vanilla_forward():
    assert S.forward_sequence(1, True) == S.forward_sequence(1, False)


@given(kf=st.integers(0, 12), kb=st.integers(0, 12), reorder=st.booleans(),
       fp=st.sampled_from([S.BEFORE, S.AFTER]), bp=st.sampled_from([S.BEFORE, S.AFTER]))
@settings(max_examples=300, deadline=None)
def test_sequences_are_linear_extensions(kf, kb, reorder, fp, bp):
    seq = S.step_sequence(kf, kb, reorder, fp, bp)
    assert S.dependencies_respected(seq)
    assert sum(1 for e in seq if e[1] == S.AG) == kf + kb       # alpha count = buckets
    assert sum(1 for e in seq if e[1] == S.RS) == kb
    assert all((e[3] == 1) == (e[1] in S.COMM_OPS) for e in seq)
    # prefetch depth (G16 = 1, P:189 'prefetch bucket i+1 during compute of
    # bucket i'): when WAIT_AG k of a phase is enqueued, exactly k + 1 AGs of
    # that phase have been issued (vanilla, or reorder with the AG placed after
    # the wait) or k + 2 (reorder with the AG placed before the wait), never more;
    # under reorder AG k+1 is always issued before COMPUTE k.
    for ph, kk, place in ((0, kf, fp), (1, kb, bp)):
        for k in range(kk):
            w = _idx(seq, ph, S.WAIT_AG, k)
            issued = sum(1 for e in seq[:w] if e[0] == ph and e[1] == S.AG)
            ahead = 1 if (reorder and place == S.BEFORE and k + 1 < kk) else 0
            assert issued == k + 1 + ahead
            if reorder and k + 1 < kk:
                comp = S.COMPUTE_F if ph == 0 else S.COMPUTE_B
                assert _idx(seq, ph, S.AG, k + 1) < _idx(seq, ph, comp, k)
            if not reorder and k + 1 < kk:
                comp = S.COMPUTE_F if ph == 0 else S.COMPUTE_B
                assert _idx(seq, ph, S.AG, k + 1) > _idx(seq, ph, comp, k)


def _two_bucket(ex):
    ag = ex["ag_ns"]
    cp = ex["compute_ns"]
    seq = S.forward_sequence(len(ag), ex["reorder"], S.BEFORE)

    def dur(ph, op, b):
        return cp[b] if op == S.COMPUTE_F else 0
    return simulate(seq, dur, lambda ph, op, b: ag[b])


def test_sim_hand_traces(golden):
    for ex in golden("spec_examples.json")["sim_traces"]:
        if ex["case"] == "compute_only":
            r = simulate([(0, S.COMPUTE_F, 0, 0)], lambda *a: ex["compute_ns"], lambda *a: 0)
        else:
            r = _two_bucket(ex)
        assert r["total"] == ex["total_ns"], ex["cite"]
        assert r["exposed"] == ex["exposed_ns"], ex["cite"]
        assert r["total"] - r["compute_busy"] == r["exposed"]
        if "comm_events" in ex:
            assert [[e[4], e[5]] for e in r["events"] if e[3] == 1] == ex["comm_events"]
            assert [[e[4], e[5]] for e in r["events"] if e[1] == S.COMPUTE_F] == ex["compute_events"]


def _rand_durations(seed, kf, kb):
    rng = np.random.Generator(np.random.Philox(seed))
    table = {}

    def dur(ph, op, b):
        key = (ph, op, b)
        if key not in table:
            table[key] = int(rng.integers(0, 3000 if op not in (S.COMPUTE_F, S.COMPUTE_B) else 20000))
        return table[key]
    coll = {}

    def tc(ph, op, b):
        key = (ph, op, b)
        if key not in coll:
            coll[key] = int(rng.integers(1, 30000))
        return coll[key]
    return dur, tc


@given(kf=st.integers(1, 10), kb=st.integers(1, 10), seed=st.integers(0, 2**31),
       fp=st.sampled_from([S.BEFORE, S.AFTER]), bp=st.sampled_from([S.BEFORE, S.AFTER]))
@settings(max_examples=500, deadline=None)
def test_reorder_never_worse_than_vanilla_and_accounting(kf, kb, seed, fp, bp):
    dur, tc = _rand_durations(seed, kf, kb)
    rv = simulate(S.step_sequence(kf, kb, False), dur, tc)
    rr = simulate(S.step_sequence(kf, kb, True, fp, bp), dur, tc)
    for r in (rv, rr):
        assert r["total"] - r["compute_busy"] == r["exposed"]
        assert r["total"] >= max(r["compute_busy"], r["comm_busy"])
    assert rr["compute_busy"] == rv["compute_busy"]
    assert rr["exposed"] <= rv["exposed"]
    # vanilla exposes every collective in full
    assert rv["exposed"] == rv["comm_busy"]


@given(kf=st.integers(2, 8), seed=st.integers(0, 2**31))
@settings(max_examples=200, deadline=None)
def test_fifo_non_interference(kf, seed):
    # moving AG(k+1) before Wait(k) never changes when Wait(k) completes
    dur, tc = _rand_durations(seed, kf, 0)
    before = simulate(S.forward_sequence(kf, True, S.BEFORE), dur, tc)
    after = simulate(S.forward_sequence(kf, True, S.AFTER), dur, tc)
    ends_b = {e[2]: e[5] for e in before["events"] if e[1] == S.AG}
    ends_a = {e[2]: e[5] for e in after["events"] if e[1] == S.AG}
    assert ends_b[0] == ends_a[0]
    assert before["total"] <= after["total"]  # Table 6 direction with copy-outs > 0


def _plan_exposure(pi, buckets, t_c_per_param, copy_ns_per_byte=0):
    """Simulated exposure of one phase for a plan (phase-order buckets)."""
    k = len(buckets)
    seq = S.forward_sequence(k, True) if pi.phase == FWD else S.backward_sequence(k, True)

    def dur(ph, op, b):
        if op in (S.COMPUTE_F, S.COMPUTE_B):
            return sum(t_c_per_param[j] for j in buckets[b])
        return 0

    def tc(ph, op, b):
        return pi.t_ag(buckets[b]) if op == S.AG else pi.t_rs(buckets[b])
    return simulate(seq, dur, tc)


@given(P=st.integers(1, 8), seed=st.integers(0, 2**31), phase=st.sampled_from([FWD, BWD]))
@settings(max_examples=200, deadline=None)
def test_optimum_le_greedy(P, seed, phase):
    rng = np.random.Generator(np.random.Philox(seed))
    params = [(int(rng.integers(1, 40)), int(rng.integers(1, 40)), i) for i in range(P)]
    tc = [int(x) for x in rng.integers(0, 20000, size=P)]
    pi = PlanInput(params, 4, tc, (int(rng.integers(0, 5000)), int(rng.integers(0, 10**6))),
                   (int(rng.integers(0, 5000)), int(rng.integers(0, 10**6))), 10**18, GREEDY, phase)
    greedy, _ = plan(pi)
    g = _plan_exposure(pi, greedy, tc)["total"]
    best = min(_plan_exposure(pi, p, tc)["total"] for p in contiguous_partitions(pi.order()))
    assert best <= g
    pp = PlanInput(params, 4, tc, pi.ag, pi.rs, 10**18, PER_PARAM, phase)
    singles, _ = plan(pp)
    assert best <= _plan_exposure(pp, singles, tc)["total"]


# ------------------------------------------------------------ memory curve (G40)
from oracle.sim import memory_curve  # noqa: E402


def _mem(seq, A, Fp, G, R):
    return memory_curve(seq, lambda ph, b: A[ph][b], lambda ph, b: Fp[ph][b], lambda b: G[b], lambda b: R[b])


def test_memory_hand_example():
    """Two buckets per phase, worked by hand from the G40 rules.
    A = flat AG, F = full params (same in both phases), G = full grads, R = RS input.
    Forward vanilla: 20 | 180 -> 160 | 0 | 10 | 90 -> 80 | 0                      peak 180
    Forward before:  20, 30 | UNPACK 0: 190 -> 170 | C0: 10 | UNPACK 1: 90 -> 80 | 0   peak 190
    Backward vanilla (fwd-order buckets reversed: b0 = A 10 / F 80 / G 80 / R 320,
    b1 = A 20 / F 160 / G 160 / R 640):
      b0: 10 | 90 -> 80 | +G 160 -> 80 | +R 400 -> 320 | 0
      b1: 20 | 180 -> 160 | +G 320 -> 160 | +R 800 -> 640 | 0                      peak 800"""
    A = {0: [20, 10], 1: [10, 20]}
    Fp = {0: [160, 80], 1: [80, 160]}
    G, R = [80, 160], [320, 640]
    assert _mem(S.forward_sequence(2, reorder=False), A, Fp, G, R)["peak"] == 180
    assert _mem(S.forward_sequence(2, reorder=True, placement=S.BEFORE), A, Fp, G, R)["peak"] == 190
    assert _mem(S.forward_sequence(2, reorder=True, placement=S.AFTER), A, Fp, G, R)["peak"] == 180
    r = _mem(S.backward_sequence(2, reorder=False), A, Fp, G, R)
    assert r["peak"] == 800 and r["final"] == 0


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 9), st.integers(0, 10 ** 6))
def test_memory_closed_forms(k, seed):
    """Per-phase peaks in closed form (derived from the G40 rules, not by
    walking the sequence):
      forward vanilla          max_k A_k + F_k
      forward before           max_k A_k + A_{k+1} + F_k          (A_K = 0)
      forward after            max_k max(A_k + F_k, F_k + A_{k+1})
      backward vanilla         max_j max(A_j + F_j, F_j + G_j, G_j + R_j)"""
    rng = np.random.default_rng(seed)
    A = {p: [int(x) for x in rng.integers(1, 10 ** 6, k)] for p in (0, 1)}
    Fp = {p: [int(x) for x in rng.integers(1, 10 ** 7, k)] for p in (0, 1)}
    G = [int(x) for x in rng.integers(1, 10 ** 7, k)]
    R = [int(x) for x in rng.integers(1, 10 ** 7, k)]
    A0n = A[0] + [0]
    assert _mem(S.forward_sequence(k, reorder=False), A, Fp, G, R)["peak"] == max(
        A[0][i] + Fp[0][i] for i in range(k))
    assert _mem(S.forward_sequence(k, reorder=True, placement=S.BEFORE), A, Fp, G, R)["peak"] == max(
        A0n[i] + A0n[i + 1] + Fp[0][i] for i in range(k))
    assert _mem(S.forward_sequence(k, reorder=True, placement=S.AFTER), A, Fp, G, R)["peak"] == max(
        max(A0n[i] + Fp[0][i], Fp[0][i] + A0n[i + 1]) for i in range(k))
    assert _mem(S.backward_sequence(k, reorder=False), A, Fp, G, R)["peak"] == max(
        max(A[1][j] + Fp[1][j], Fp[1][j] + G[j], G[j] + R[j]) for j in range(k))


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 8), st.integers(1, 8), st.integers(0, 10 ** 6),
       st.sampled_from([S.BEFORE, S.AFTER]), st.sampled_from([S.BEFORE, S.AFTER]))
def test_memory_conservation_and_reorder_costs_memory(kf, kb, seed, fp, bp):
    """Every allocation is freed by the end of the step; prefetching (reorder)
    never lowers the peak below the vanilla order's (Table 5: +reorder raises
    memory)."""
    rng = np.random.default_rng(seed)
    A = {0: [int(x) for x in rng.integers(1, 10 ** 6, kf)], 1: [int(x) for x in rng.integers(1, 10 ** 6, kb)]}
    Fp = {0: [int(x) for x in rng.integers(1, 10 ** 7, kf)], 1: [int(x) for x in rng.integers(1, 10 ** 7, kb)]}
    G = [int(x) for x in rng.integers(1, 10 ** 7, kb)]
    R = [int(x) for x in rng.integers(1, 10 ** 7, kb)]
    van = _mem(S.step_sequence(kf, kb, reorder=False), A, Fp, G, R)
    reo = _mem(S.step_sequence(kf, kb, reorder=True, fwd_placement=fp, bwd_placement=bp), A, Fp, G, R)
    assert van["final"] == 0 and reo["final"] == 0
    assert min(van["live"]) >= 0 and min(reo["live"]) >= 0
    assert reo["peak"] >= van["peak"]


# ------------------------------------------------- keep the last gathered (G42)
def test_keep_first_hand_sequence():
    """k_fwd = k_bwd = 2, reordered, default placements: the backward loses
    exactly bucket 0's PACK_AG / AG / WAIT_AG / UNPACK; COMPUTE_B 0 follows the
    forward's last COMPUTE_F."""
    F_, B_ = 0, 1
    # full: PACK_AG 0, AG 0 | WAIT_AG 0, UNPACK 0, PACK_AG 1, AG 1, COMPUTE_B 0, PACK_RS 0, RS 0 |
    #       WAIT_AG 1, UNPACK 1, COMPUTE_B 1, PACK_RS 1, WAIT_RS 0, COPYOUT_RS 0, RS 1 | WAIT_RS 1, COPYOUT_RS 1
    want = [(B_, S.PACK_AG, 1), (B_, S.AG, 1), (B_, S.COMPUTE_B, 0), (B_, S.PACK_RS, 0), (B_, S.RS, 0),
            (B_, S.WAIT_AG, 1), (B_, S.UNPACK, 1), (B_, S.COMPUTE_B, 1), (B_, S.PACK_RS, 1),
            (B_, S.WAIT_RS, 0), (B_, S.COPYOUT_RS, 0), (B_, S.RS, 1), (B_, S.WAIT_RS, 1), (B_, S.COPYOUT_RS, 1)]
    got = [e[:3] for e in S.backward_sequence(2, True, S.AFTER, keep_first=True)]
    assert got == want
    full = [e[:3] for e in S.backward_sequence(2, True, S.AFTER)]
    assert [e for e in full if not (e[2] == 0 and e[1] in (S.PACK_AG, S.AG, S.WAIT_AG, S.UNPACK))] == got
    seq = S.step_sequence(2, 2, keep_first=True)
    assert S.dependencies_respected(seq)
    i_f = seq.index((F_, S.COMPUTE_F, 1, 0))
    i_b = seq.index((B_, S.COMPUTE_B, 0, 0))
    assert i_f < i_b


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 8), st.integers(1, 8), st.booleans(), st.integers(0, 10 ** 6),
       st.sampled_from([S.BEFORE, S.AFTER]), st.sampled_from([S.BEFORE, S.AFTER]))
def test_keep_first_never_costs_time_or_leaks_memory(kf, kb, reorder, seed, fp, bp):
    rng = np.random.default_rng(seed)
    base = S.step_sequence(kf, kb, reorder, fp, bp)
    keep = S.step_sequence(kf, kb, reorder, fp, bp, keep_first=True)
    assert S.dependencies_respected(keep) and len(keep) == len(base) - 4
    dur = {e[:3]: int(rng.integers(0, 50000)) for e in base}
    f = lambda ph, op, b: dur[(ph, op, b)]   # noqa: E731
    assert simulate(keep, f, f)["total"] <= simulate(base, f, f)["total"]
    A = {p: [int(x) for x in rng.integers(1, 10 ** 6, n)] for p, n in ((0, kf), (1, kb))}
    Fp = {0: [int(x) for x in rng.integers(1, 10 ** 7, kf)], 1: None}
    Fp[1] = [int(x) for x in rng.integers(1, 10 ** 7, kb)]
    Fp[1][0] = Fp[0][kf - 1]            # bucket 0 of the backward = the forward's last bucket
    G = [int(x) for x in rng.integers(1, 10 ** 7, kb)]
    R = [int(x) for x in rng.integers(1, 10 ** 7, kb)]
    r = _mem(keep, A, Fp, G, R)
    assert r["final"] == 0 and min(r["live"]) >= 0
