"""O6 / O7 / O8 pins: SPEC's cost worked example, additivity; apportionment
examples; Algorithm 1 hand-worked traces; boundary cases; SIZE_CAP against
textbook next-fit partitioning; the independent verifier over fuzzed
instances; brute force over all 2^(P-1) contiguous partitions."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle.brute import contiguous_partitions, verify_greedy
from oracle.cost import comm_time
from oracle.planner import (BWD, FWD, GREEDY, MANUAL, PER_PARAM, SIZE_CAP, PlanInput,
                            bucket_begin, plan)
from workloads import llama, toy_mlp
from workloads.compute_model import apportioned_compute_ns, per_param_compute_ns
from workloads.shapes import ParamSpec


def test_comm_time_spec_examples(golden):
    for ex in golden("spec_examples.json")["comm_time"]:
        assert comm_time(ex["nbytes"], ex["alpha_ns"], ex["beta_fs_per_byte"]) == ex["ns"], ex["cite"]


@given(a=st.integers(0, 10**10), b=st.integers(0, 10**10), alpha=st.integers(0, 10**6),
       beta=st.integers(0, 10**7))
def test_comm_time_additivity(a, b, alpha, beta):
    # one alpha saved per merge, within 1 ns of ceiling rounding
    d = comm_time(a + b, alpha, beta) - (comm_time(a, alpha, beta) + comm_time(b, alpha, beta) - alpha)
    assert -1 <= d <= 0


def test_apportion_examples(golden):
    for ex in golden("spec_examples.json")["apportion"]:
        ps = [ParamSpec("p%d" % i, s, 1, 0) for i, s in enumerate(ex["sizes"])]
        assert apportioned_compute_ns(ps, {0: ex["module_ns"]}) == ex["parts"], ex["cite"]


def test_per_op_compute_model_block_totals():
    # 8B block fwd 0.476 ms at T = 1024 (F 1 PF/s, H 6 TB/s)
    ps = llama("8b", n_layers=1, with_embeddings=False)
    f, b = per_param_compute_ns(ps, 1024)
    assert abs(sum(f) - 476_000) < 1_500
    assert sum(b) == 2 * sum(f)


def _hand_input(phase, ex):
    P = 7
    params = [(1, 500000, i) for i in range(P)]
    return PlanInput(params, 1, [ex["t_c_ns"]] * P, (10000, ex["beta_ag_fs"]),
                     (10000, ex["beta_rs_fs"]), 3_000_000, GREEDY, phase,
                     param_bytes=2, reduce_bytes=4, align=16, mem_bytes=[10**6] * P)


@pytest.mark.parametrize("phase", [FWD, BWD])
def test_alg1_hand_examples(golden, phase):
    ex = golden("alg1_hand_examples.json")["forward" if phase == FWD else "backward"]
    pi = _hand_input(phase, ex)
    buckets, trace = plan(pi)
    pos = {j: k + 1 for k, j in enumerate(pi.order())}   # forward index -> phase label
    assert [[pos[j] for j in b] for b in buckets] == ex["buckets"]
    got = [dict(param=pos[t["param"]], t_lhs=t["t_lhs"], t_rhs=t["t_rhs"], m_lhs=t["m_lhs"],
                accept=t["accept"]) for t in trace]
    assert got == ex["trace"]
    assert verify_greedy(pi, buckets)


def test_boundaries():
    P = 6
    params = [(64, 64, i) for i in range(P)]
    base = dict(params=params, world=4, t_compute_ns=[10**6] * P, ag=(5000, 1000), rs=(5000, 1000))
    for phase in (FWD, BWD):
        # M_max below every M_i -> singletons
        b, _ = plan(PlanInput(mem_max=1, mode=GREEDY, phase=phase, **base))
        assert all(len(x) == 1 for x in b)
        # huge T_c for q_1, M_max = inf -> [{q1}, rest]  (first window is 0, G10)
        tc = [0] * P
        q1 = 0 if phase == FWD else P - 1
        tc[q1] = 10**12
        b, _ = plan(PlanInput(params, 4, tc, (5000, 1000), (5000, 1000), 10**18, GREEDY, phase))
        assert b == [[q1], [j for j in (range(P) if phase == FWD else range(P - 1, -1, -1)) if j != q1]]
        # SIZE_CAP ignores the time test: with M_max = inf everything merges
        b, _ = plan(PlanInput(mem_max=10**18, mode=SIZE_CAP, phase=phase, **base))
        assert len(b) == 1


def _next_fit(sizes, cap):
    """Textbook next-fit sequential partitioning with capacity ``cap``."""
    out, cur, load = [], [], 0
    for i, s in enumerate(sizes):
        if cur and load + s > cap:
            out.append(cur)
            cur, load = [], 0
        cur.append(i)
        load += s
    out.append(cur)
    return out


@given(sizes=st.lists(st.integers(1, 50), min_size=1, max_size=20), cap=st.integers(1, 120))
@settings(max_examples=200, deadline=None)
def test_size_cap_is_next_fit(sizes, cap):
    P = len(sizes)
    pi = PlanInput([(1, 8, i) for i in range(P)], 1, [0] * P, (0, 0), (0, 0), cap, SIZE_CAP, FWD,
                   mem_bytes=sizes)
    b, _ = plan(pi)
    assert b == _next_fit(sizes, cap)


def test_manual_llama_blocks():
    ps = llama("8b")
    params = [(p.dim0, p.row_numel, p.module_id) for p in ps]
    for phase in (FWD, BWD):
        pi = PlanInput(params, 8, [0] * len(ps), (0, 0), (0, 0), 0, MANUAL, phase)
        b, _ = plan(pi)
        assert len(b) == 35  # emb, 32 blocks, norm, output
        sizes = sorted(len(x) for x in b)
        assert sizes == [1, 1, 1] + [9] * 32
        flat = [j for x in b for j in x]
        assert flat == pi.order()
    pi = PlanInput(params, 8, [0] * len(ps), (0, 0), (0, 0), 0, PER_PARAM, FWD)
    b, _ = plan(pi)
    assert bucket_begin(b) == list(range(len(ps) + 1))


inst = st.tuples(
    st.integers(1, 9),                 # P
    st.integers(1, 8),                 # world
    st.integers(0, 2**31),             # seed
    st.sampled_from([FWD, BWD]),
    st.sampled_from([GREEDY, SIZE_CAP]),
)


def _random_input(P, world, seed, phase, mode):
    rng = np.random.Generator(np.random.Philox(seed))
    params = [(int(rng.integers(1, 40)), int(rng.integers(1, 40)), i) for i in range(P)]
    tc = [int(x) for x in rng.integers(0, 20000, size=P)]
    mem = [int(x) for x in rng.integers(1, 5000, size=P)]
    mmax = int(rng.integers(1, 15000))
    ag = (int(rng.integers(0, 5000)), int(rng.integers(0, 200000)))
    rs = (int(rng.integers(0, 5000)), int(rng.integers(0, 200000)))
    return PlanInput(params, world, tc, ag, rs, mmax, mode, phase, mem_bytes=mem)


@given(inst)
@settings(max_examples=1000, deadline=None)
def test_verifier_accepts_every_greedy_plan(x):
    pi = _random_input(*x)
    b, trace = plan(pi)
    assert [j for bb in b for j in bb] == pi.order()
    assert verify_greedy(pi, b)
    assert len(trace) == len(pi.params) - 1
    assert sum(t["accept"] for t in trace) == len(pi.params) - len(b)


@given(inst)
@settings(max_examples=150, deadline=None)
def test_brute_force_unique_greedy_plan(x):
    pi = _random_input(*x)
    b, _ = plan(pi)
    passing = [p for p in contiguous_partitions(pi.order()) if verify_greedy(pi, p)]
    assert passing == [b]


def test_partition_count():
    for n in range(1, 11):
        assert sum(1 for _ in contiguous_partitions(list(range(n)))) == 2 ** (n - 1)


def test_toy_greedy_plan_runs():
    ps = toy_mlp()
    params = [(p.dim0, p.row_numel, p.module_id) for p in ps]
    tc = [20000 if p.row_numel > 1 else 0 for p in ps]
    for phase in (FWD, BWD):
        pi = PlanInput(params, 2, tc, (10000, 1000), (10000, 1000), 10**9, GREEDY, phase,
                       param_bytes=4)
        b, _ = plan(pi)
        assert verify_greedy(pi, b)


def _world3_input(ex, setup):
    params = [(d, r, i) for i, (d, r) in enumerate(setup["params_forward_order"])]
    return PlanInput(params, setup["world"], ex["t_c_ns"], (setup["alpha_ns"], setup["beta_ag_fs"]),
                     (setup["alpha_ns"], setup["beta_rs_fs"]), ex["mem_max"], GREEDY,
                     FWD if ex["phase"] == "fwd" else BWD, param_bytes=setup["param_bytes"],
                     reduce_bytes=setup["reduce_bytes"], align=setup["align"])   # default M_i (G13)


def _labelled(buckets, trace):
    return ([[j + 1 for j in b] for b in buckets],
            [dict(param=t["param"] + 1, t_lhs=t["t_lhs"], t_rhs=t["t_rhs"], m_lhs=t["m_lhs"],
                  accept=t["accept"]) for t in trace])


@pytest.mark.parametrize("case", ["forward_time", "forward_memory", "backward"])
def test_alg1_world3_hand_examples(golden, case):
    """World factor pins (P:222 n = transmitted bytes; P:237 M_ci; G8 / G13):
    hand-worked at N = 3 with uneven dim 0 and the default M_i."""
    g = golden("alg1_world3_examples.json")
    ex = g[case]
    pi = _world3_input(ex, g["setup"])
    assert pi.mem_bytes == [12, 720000, 480000, 720000, 12, 720000]   # N ceil(d/N) R e_p by hand
    buckets, trace = plan(pi)
    got_b, got_t = _labelled(buckets, trace)
    assert got_b == ex["buckets"]
    assert got_t == ex["trace"]
    assert verify_greedy(pi, buckets)


def test_alg1_world3_examples_detect_a_dropped_world_factor(golden, monkeypatch):
    """The examples are sensitive: the oracle with N dropped from n (AG, RS) or
    from the default M_i disagrees with at least one of them."""
    from oracle import planner as OP
    from oracle.cost import comm_time
    from oracle.layout import bucket_layout
    g = golden("alg1_world3_examples.json")

    def all_match():
        out = []
        for case in ("forward_time", "forward_memory", "backward"):
            ex = g[case]
            pi = _world3_input(ex, g["setup"])
            b, t = plan(pi)
            out.append(_labelled(b, t) == (ex["buckets"], ex["trace"]))
        return all(out)

    assert all_match()
    with monkeypatch.context() as m:
        m.setattr(OP.PlanInput, "t_ag", lambda self, mem: comm_time(
            bucket_layout(self.dims(mem), self.world, self.param_bytes, self.align)[1], *self.ag))
        assert not all_match()
    with monkeypatch.context() as m:
        m.setattr(OP.PlanInput, "t_rs", lambda self, mem: comm_time(
            bucket_layout(self.dims(mem), self.world, self.reduce_bytes, self.align)[1], *self.rs))
        assert not all_match()
    orig_init = OP.PlanInput.__init__

    def init_no_n(self, *a, **k):
        orig_init(self, *a, **k)
        self.mem_bytes = [(-(-d // self.world)) * r * self.param_bytes for d, r, _ in self.params]
    with monkeypatch.context() as m:
        m.setattr(OP.PlanInput, "__init__", init_no_n)
        assert not all_match()
