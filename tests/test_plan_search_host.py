"""Host logic of tools/plan_search.py (the simulator-guided plan search, a
planner beyond the paper's Algorithm 1): on a 2-block Llama-3-8B slice the
search returns a contiguous partition of every phase that covers each
parameter once, respects the memory cap, and is never slower -- in the same
two-stream model (fsdp_simulate_schedule) -- than the plan it started from."""
import os
import sys

import pytest

pytest.importorskip("paper_2411_00284_b200._lib", reason="libfsdp_b200.so not built")

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import plan_search as PS  # noqa: E402
from paper_2411_00284_b200 import _lib as L  # noqa: E402
from paper_2411_00284_b200 import harness as H  # noqa: E402
from workloads import llama  # noqa: E402
from workloads.compute_model import per_param_compute_ns  # noqa: E402


@pytest.mark.parametrize("phase", [0, 1])
@pytest.mark.parametrize("mode", [L.PLAN_MANUAL, L.PLAN_GREEDY, L.PLAN_PER_PARAM])
def test_search_never_worse_and_valid(phase, mode):
    specs = llama("8b", n_layers=2)
    P = len(specs)
    tf, tb = per_param_compute_ns(specs, 1024)
    link = (20000, 1215)
    mem = int(6e8)
    fp, bp = H.plans_for(specs, 8, mode, tf, tb, link, link, mem)
    model = PS.PhaseModel(specs, 8, phase, tf if phase == 0 else tb, link, mem)
    flags = L.SCHED_REORDER | (L.SCHED_FWD_AG_BEFORE_WAIT if phase == 0 else 0)
    start = PS.cuts_of(fp if phase == 0 else bp, P, phase)
    t_start = model.time(start, flags)[0]
    cuts, t = PS.search(model, start, flags, budget_s=20)
    assert t <= t_start and t == model.time(cuts, flags)[0]
    assert cuts[0] == 0 and cuts[-1] == P and all(a < b for a, b in zip(cuts, cuts[1:]))
    assert model.feasible(cuts)
    plan = PS.plan_of(cuts, model)
    assert sorted(j for b in plan for j in b) == list(range(P))
    order = list(range(P)) if phase == 0 else list(range(P - 1, -1, -1))
    assert [j for b in plan for j in b] == order          # contiguous, in execution order


@pytest.mark.parametrize("phase", [0, 1])
@pytest.mark.parametrize("mode", [L.PLAN_MANUAL, L.PLAN_GREEDY, L.PLAN_PER_PARAM])
def test_library_search_matches_reference(phase, mode):
    """fsdp_plan_search (C++) == the Python reference in tools/plan_search.py:
    same moves in the same order, same integer cost model -> the same plan and
    the same predicted phase time, both run to convergence."""
    import paper_2411_00284_b200 as F
    specs = llama("8b", n_layers=2)
    P = len(specs)
    tf, tb = per_param_compute_ns(specs, 2048)
    link = (20000, 1215)
    mem = int(6e8)
    fp, bp = H.plans_for(specs, 8, mode, tf, tb, link, link, mem)
    t_c = tf if phase == 0 else tb
    flags = L.SCHED_REORDER | (L.SCHED_FWD_AG_BEFORE_WAIT if phase == 0 else 0)
    model = PS.PhaseModel(specs, 8, phase, t_c, link, mem)
    start = fp if phase == 0 else bp
    cuts, t = PS.search(model, PS.cuts_of(start, P, phase), flags, budget_s=1e9)
    descs = [(s.dim0, s.row_numel, s.module_id) for s in specs]
    plan, t_lib = F.plan_search(descs, 8, t_c, link, link, mem, phase, start, PS.library_cost(flags))
    assert t_lib == t
    assert plan == PS.plan_of(cuts, model)


def test_library_search_rejects_bad_start():
    import paper_2411_00284_b200 as F
    specs = llama("8b", n_layers=1)
    descs = [(s.dim0, s.row_numel, s.module_id) for s in specs]
    tf, _ = per_param_compute_ns(specs, 1024)
    cost = PS.library_cost(L.SCHED_REORDER)
    with pytest.raises(L.FsdpError):    # does not cover every parameter
        F.plan_search(descs, 8, tf, (1, 1), (1, 1), 10 ** 12, L.PHASE_FWD, [[0, 1]], cost)
    with pytest.raises(L.FsdpError):    # start bucket over the memory cap
        F.plan_search(descs, 8, tf, (1, 1), (1, 1), 10, L.PHASE_FWD, [list(range(len(specs)))], cost)


def test_plans_search_covers_every_parameter():
    specs = llama("8b", n_layers=3)
    tf, tb = per_param_compute_ns(specs, 1024)
    f, b = H.plans_search(specs, 8, tf, tb, (20000, 1215), (20000, 1215), int(2e9))
    P = len(specs)
    assert [j for bk in f for j in bk] == list(range(P))
    assert [j for bk in b for j in bk] == list(range(P - 1, -1, -1))
