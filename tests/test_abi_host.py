"""CPU tests of the C ABI: the library loads and exports every symbol
include/fsdp.h declares; host-only entry points (shard metadata, layout,
plan, dry-run schedule) are bit-exact / sequence-equal against the oracle.
No GPU needed: these calls never touch the device."""
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import schedule as OS
from oracle.layout import bucket_layout
from oracle.planner import BWD, FWD, GREEDY, MANUAL, PER_PARAM, SIZE_CAP, PlanInput, plan
from oracle.shard import shard_rows
from workloads import llama, toy_mlp
from workloads.compute_model import per_param_compute_ns

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {PER_PARAM: L.PLAN_PER_PARAM, MANUAL: L.PLAN_MANUAL, SIZE_CAP: L.PLAN_SIZE_CAP, GREEDY: L.PLAN_GREEDY}
PHASES = {FWD: L.PHASE_FWD, BWD: L.PHASE_BWD}


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fsdp.h")).read()
    declared = set(re.findall(r"\b(fsdp_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(L.EXPORTED)
    for name in declared:
        assert hasattr(L.lib, name), name
    assert F.abi_version() == 5


@given(d=st.integers(1, 10**6), world=st.integers(1, 64), data=st.data())
@settings(max_examples=300, deadline=None)
def test_shard_metadata_matches_oracle(d, world, data):
    r = data.draw(st.integers(0, world - 1))
    info = F.shard(world, r, (d, 7, 0), L.BF16)
    c, begin, v = shard_rows(d, world, r)
    assert (info["shard_rows"], info["row_begin"], info["valid_rows"], info["shard_numel"]) == (c, begin, v, 7 * c)


def test_shard_rejects_bad_args():
    with pytest.raises(F.FsdpError):
        F.shard(2, 2, (10, 1, 0), L.BF16)
    with pytest.raises(F.FsdpError):
        F.shard(2, 0, (0, 1, 0), L.BF16)
    with pytest.raises(F.FsdpError):
        F.shard(2, 0, (4, 1, 0), L.BF16, full_ptr=1234, shard_ptr=None)


@given(dims=st.lists(st.tuples(st.integers(1, 500), st.integers(1, 300)), min_size=1, max_size=12),
       world=st.integers(1, 9), e=st.sampled_from([2, 4]), a=st.sampled_from([1, 2, 16, 256]))
@settings(max_examples=300, deadline=None)
def test_layout_matches_oracle(dims, world, e, a):
    offs, seg = F.layout([(d, r, 0) for d, r in dims], world, e, a)
    o2, s2 = bucket_layout(dims, world, e, a)
    assert offs == o2 and seg == s2


def _both_plans(pi, param_dtype):
    ob, otr = plan(pi)
    cb, ctr = F.plan_buckets(pi.params, pi.world, pi.t_compute_ns, pi.ag, pi.rs, pi.mem_max,
                             MODES[pi.mode], PHASES[pi.phase], param_dtype=param_dtype, align=pi.align,
                             mem_bytes=pi.mem_bytes, reduce_bytes=pi.reduce_bytes, want_trace=True)
    return ob, otr, cb, ctr


def _assert_same(ob, otr, cb, ctr, mode):
    assert cb == ob
    if mode in (GREEDY, SIZE_CAP):
        assert [dict(param=t["param"], t_lhs=t["t_lhs"], t_rhs=t["t_rhs"], m_lhs=t["m_lhs"],
                     m_rhs=t["m_rhs"], accept=t["accept"]) for t in ctr] == otr
    else:
        assert [(t["param"], t["accept"]) for t in ctr] == [(t["param"], t["accept"]) for t in otr]


@given(P=st.integers(1, 40), world=st.integers(1, 9), seed=st.integers(0, 2**31),
       phase=st.sampled_from([FWD, BWD]), mode=st.sampled_from([PER_PARAM, MANUAL, SIZE_CAP, GREEDY]),
       bf16=st.booleans(), a=st.sampled_from([1, 16]))
@settings(max_examples=500, deadline=None)
def test_plan_bit_exact_fuzz(P, world, seed, phase, mode, bf16, a):
    rng = np.random.Generator(np.random.Philox(seed))
    params = [(int(rng.integers(1, 300)), int(rng.integers(1, 200)), int(rng.integers(0, 4)))
              for _ in range(P)]
    tc = [int(x) for x in rng.integers(0, 200000, size=P)]
    mem = None if rng.integers(0, 2) else [int(x) for x in rng.integers(1, 10**6, size=P)]
    pi = PlanInput(params, world, tc, (int(rng.integers(0, 20000)), int(rng.integers(0, 10**6))),
                   (int(rng.integers(0, 20000)), int(rng.integers(0, 10**6))),
                   int(rng.integers(1, 4 * 10**6)), mode, phase, param_bytes=2 if bf16 else 4,
                   align=a, mem_bytes=mem)
    _assert_same(*_both_plans(pi, L.BF16 if bf16 else L.FP32), mode)


@pytest.mark.parametrize("model", ["8b", "70b"])
@pytest.mark.parametrize("tokens", [1024, 8192])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_plan_bit_exact_llama(model, tokens, world):
    ps = llama(model)
    params = [(p.dim0, p.row_numel, p.module_id) for p in ps]
    f, b = per_param_compute_ns(ps, tokens)
    # alpha/beta of an NVLink-class link: 20 us, 1.5 ps/B (~670 GB/s)
    for phase, tc in ((FWD, f), (BWD, b)):
        for mode, mmax in ((GREEDY, 2 * 10**9), (GREEDY, 10**18), (SIZE_CAP, 500 * 10**6), (MANUAL, 0)):
            pi = PlanInput(params, world, tc, (20000, 1500), (20000, 1500), mmax, mode, phase)
            _assert_same(*_both_plans(pi, L.BF16), mode)


def test_plan_hand_examples(golden):
    for key, phase in (("forward", FWD), ("backward", BWD)):
        ex = golden("alg1_hand_examples.json")[key]
        pi = PlanInput([(1, 500000, i) for i in range(7)], 1, [ex["t_c_ns"]] * 7, (10000, ex["beta_ag_fs"]),
                       (10000, ex["beta_rs_fs"]), 3_000_000, GREEDY, phase, mem_bytes=[10**6] * 7)
        ob, otr, cb, ctr = _both_plans(pi, L.BF16)
        _assert_same(ob, otr, cb, ctr, GREEDY)
        pos = {j: k + 1 for k, j in enumerate(pi.order())}
        assert [[pos[j] for j in bb] for bb in cb] == ex["buckets"]


def test_plan_world3_hand_examples(golden):
    """C++ planner against the world-3 hand-worked Alg. 1 examples (G8 / G13 world factor)."""
    g = golden("alg1_world3_examples.json")
    st_ = g["setup"]
    params = [(d, r, i) for i, (d, r) in enumerate(st_["params_forward_order"])]
    for key in ("forward_time", "forward_memory", "backward"):
        ex = g[key]
        pi = PlanInput(params, st_["world"], ex["t_c_ns"], (st_["alpha_ns"], st_["beta_ag_fs"]),
                       (st_["alpha_ns"], st_["beta_rs_fs"]), ex["mem_max"], GREEDY,
                       FWD if ex["phase"] == "fwd" else BWD)
        ob, otr, cb, ctr = _both_plans(pi, L.BF16)
        _assert_same(ob, otr, cb, ctr, GREEDY)
        assert [[j + 1 for j in bb] for bb in cb] == ex["buckets"]
        assert [(t["param"] + 1, t["t_lhs"], t["t_rhs"], t["m_lhs"], bool(t["accept"])) for t in ctr] == \
            [(t["param"], t["t_lhs"], t["t_rhs"], t["m_lhs"], t["accept"]) for t in ex["trace"]]
        # the library's own default M_i (mem_bytes NULL): N ceil(d/N) R e_p
        cb2, ctr2 = F.plan_buckets(pi.params, 3, pi.t_compute_ns, pi.ag, pi.rs, pi.mem_max, L.PLAN_GREEDY,
                                   PHASES[pi.phase], param_dtype=L.BF16, want_trace=True)
        assert (cb2, ctr2) == (cb, ctr)


def test_plan_rejects_bad_input():
    with pytest.raises(F.FsdpError):
        F.plan_buckets([], 2, [], (0, 0), (0, 0), 0, L.PLAN_GREEDY, L.PHASE_FWD)
    with pytest.raises(F.FsdpError):
        F.plan_buckets([(0, 1, 0)], 2, [0], (0, 0), (0, 0), 0, L.PLAN_GREEDY, L.PHASE_FWD)


@given(kf=st.integers(0, 40), kb=st.integers(0, 40), reorder=st.booleans(), fb=st.booleans(), bb=st.booleans(),
       keep=st.booleans())
@settings(max_examples=300, deadline=None)
def test_dry_run_schedule_log_equals_oracle(kf, kb, reorder, fb, bb, keep):
    flags = L.SCHED_DRY_RUN | (L.SCHED_REORDER if reorder else 0)
    flags |= (L.SCHED_FWD_AG_BEFORE_WAIT if fb else 0) | (L.SCHED_BWD_AG_BEFORE_WAIT if bb else 0)
    flags |= L.SCHED_KEEP_LAST_GATHERED if keep else 0
    rep = F.run_schedule(None, None, None, flags=flags, n_fwd=kf, n_bwd=kb)
    got = [e[:4] for e in rep["log"]]
    want = OS.step_sequence(kf, kb, reorder, OS.BEFORE if fb else OS.AFTER, OS.BEFORE if bb else OS.AFTER,
                            keep_first=keep)
    assert got == want
    assert all(e[4] == -1 for e in rep["log"])


@given(n=st.integers(0, 10**12), alpha=st.integers(0, 10**7), beta=st.integers(0, 10**8))
@settings(max_examples=300, deadline=None)
def test_comm_time_matches_oracle(n, alpha, beta):
    from oracle.cost import comm_time
    assert F.comm_time_ns(n, (alpha, beta)) == comm_time(n, alpha, beta)


@given(kf=st.integers(0, 12), kb=st.integers(0, 12), reorder=st.booleans(), fb=st.booleans(), bb=st.booleans(),
       seed=st.integers(0, 2**31))
@settings(max_examples=300, deadline=None)
def test_simulator_matches_oracle(kf, kb, reorder, fb, bb, seed):
    from oracle.sim import simulate
    seq = OS.step_sequence(kf, kb, reorder, OS.BEFORE if fb else OS.AFTER, OS.BEFORE if bb else OS.AFTER)
    rng = np.random.Generator(np.random.Philox(seed))
    dur = [int(x) for x in rng.integers(0, 50000, size=len(seq))]
    table = {e[:3]: d for e, d in zip(seq, dur)}
    ref = simulate(seq, lambda ph, op, b: table[(ph, op, b)], lambda ph, op, b: table[(ph, op, b)])
    tot, exp, starts, ends = F.simulate_schedule(seq, dur)
    assert (tot, exp) == (ref["total"], ref["exposed"])
    ev = {(e[0], e[1], e[2]): (e[4], e[5]) for e in ref["events"]}
    for e, s, f in zip(seq, starts, ends):
        if e[:3] in ev and e[1] not in (OS.WAIT_AG, OS.WAIT_RS):
            assert (s, f) == ev[e[:3]]


@given(kf=st.integers(0, 12), kb=st.integers(0, 12), reorder=st.booleans(), fb=st.booleans(), bb=st.booleans(),
       seed=st.integers(0, 2**31))
@settings(max_examples=300, deadline=None)
def test_memory_model_matches_oracle(kf, kb, reorder, fb, bb, seed):
    """fsdp_simulate_memory == oracle.sim.memory_curve (G40, G42), peak and every live value."""
    from oracle.sim import memory_curve
    seq = OS.step_sequence(kf, kb, reorder, OS.BEFORE if fb else OS.AFTER, OS.BEFORE if bb else OS.AFTER,
                           keep_first=bool(seed % 2))
    rng = np.random.Generator(np.random.Philox(seed))
    big = lambda k: [int(x) for x in rng.integers(0, 2 ** 40, size=k)]   # noqa: E731  (> 2^32: 64-bit sums)
    agf, fuf, agb, fub, grb, rsb = big(kf), big(kf), big(kb), big(kb), big(kb), big(kb)
    if seed % 2 and kf and kb:
        fub[0] = fuf[kf - 1]     # G42: backward bucket 0 binds the last forward bucket's parameters
    ref = memory_curve(seq, lambda ph, b: (agf if ph == 0 else agb)[b], lambda ph, b: (fuf if ph == 0 else fub)[b],
                       lambda b: grb[b], lambda b: rsb[b])
    peak, live = F.simulate_memory(seq, agf, fuf, agb, fub, grb, rsb)
    assert peak == ref["peak"] and live == ref["live"]


def test_memory_model_rejects_bad_input():
    seq = OS.step_sequence(1, 1, True)
    one = [1]
    with pytest.raises(L.FsdpError):
        F.simulate_memory(seq, one, one, [], [], [], [])            # backward bucket out of range
    with pytest.raises(L.FsdpError):
        F.simulate_memory(seq, [-1], one, one, one, one, one)       # negative size
    with pytest.raises(L.FsdpError):
        F.simulate_memory([(0, OS.UNPACK, 0, 0), (0, OS.COMPUTE_F, 0, 0), (0, OS.COMPUTE_F, 0, 0)],
                          one, one, [], [], [], [])                 # freed twice


def test_simulator_spec_traces(golden):
    for ex in golden("spec_examples.json")["sim_traces"]:
        if ex["case"] == "compute_only":
            continue
        seq = OS.forward_sequence(len(ex["ag_ns"]), ex["reorder"], OS.BEFORE)
        dur = [ex["compute_ns"][e[2]] if e[1] == OS.COMPUTE_F else ex["ag_ns"][e[2]] if e[1] == OS.AG else 0
               for e in seq]
        tot, exp, _, _ = F.simulate_schedule(seq, dur)
        assert (tot, exp) == (ex["total_ns"], ex["exposed_ns"]), ex["cite"]


def test_toy_plan_parity():
    ps = toy_mlp()
    params = [(p.dim0, p.row_numel, p.module_id) for p in ps]
    tc = [20000 if p.row_numel > 1 else 0 for p in ps]
    for phase in (FWD, BWD):
        for mode in (PER_PARAM, MANUAL, GREEDY):
            pi = PlanInput(params, 2, tc, (10000, 1000), (10000, 1000), 10**9, mode, phase, param_bytes=4)
            _assert_same(*_both_plans(pi, L.FP32), mode)


def test_one_cublaslt_in_process_whatever_the_import_order():
    """The library loaded before torch must resolve the same cuBLASLt build as
    torch (DT_RPATH over LD_LIBRARY_PATH): two builds in one process broke
    torch's own GEMMs (CUBLAS_STATUS_INVALID_VALUE) in the Llama compute hook."""
    import subprocess
    import sys
    code = ("from paper_2411_00284_b200 import _lib\n"
            "import torch\n"
            "m = open('/proc/self/maps').read()\n"
            "print(sorted({l.split()[-1] for l in m.splitlines() if 'libcublasLt' in l}))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr
    libs = eval(out.stdout.strip().splitlines()[-1])
    assert len(libs) == 1, libs
