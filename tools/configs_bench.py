#!/usr/bin/env python
"""Measures the BASELINE.json configs other than the headline one, on 1 GPU
(rank 0 of a simulated world; every kernel at its per-rank size, no peers):

  c0  toy 4-layer MLP, fp32, 2 ranks: PER_PARAM vs GREEDY plan, step latency
  c2  Llama-3-8B Table 5 / Table 6 variants with the compute proxy at T tokens:
      vanilla / +reorder / +bucket / +both / greedy+reorder, 4 placements
  c2w the same at world sizes 2 / 4 / 8 (vanilla, manual+reorder, greedy+reorder)
  c2m the c2 variants with the real Llama-3 layers through the compute hook,
      the greedy plan fed with per-parameter compute times measured on the B200
  c3  Llama-3-70B SIZE_CAP bucket-size sweep 25-500 MB at N = 8
  c4  Llama-3-405B one layer at N = 8: one whole-layer bucket vs per-parameter

    python tools/configs_bench.py [c0 c2 c3 c4] [--out F]

Each line: step ms (CUDA events around K plain steps after warm-up), per-kernel
GB/s from a profiled pass, bucket counts.  With no peers on one GPU the
collectives are absent, so "exposed" is not measured here: the variants differ
by copy-kernel work and launch count (the paper's single-node finding that
bucketing adds copy-in/copy-out).
"""
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_variant(specs, world, mode, flags, t_fwd=None, t_bwd=None, mem_max=0, tokens=0, steps=5, warmup=2,
                link=(20000, 1500), param_dtype=None, nspi=None, predict_link=None, graph=False, model_T=0,
                profile=False):
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    pdt = L.BF16 if param_dtype is None else param_dtype
    ctx = F.Ctx(world, 0)
    if mode == "search":    # fsdp_plan_search (beyond Algorithm 1) from the manual and greedy plans
        fplan, bplan = H.plans_search(specs, world, t_fwd, t_bwd, link, link, mem_max, param_dtype=pdt)
    else:
        fplan, bplan = H.plans_for(specs, world, mode, t_fwd, t_bwd, link, link, mem_max, pdt)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, param_dtype=pdt)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    hook = None
    if model_T:   # the real Llama-3 layers through the compute hook instead of the proxy
        from paper_2411_00284_b200.llama_compute import LlamaCompute
        lc = LlamaCompute(st, model_T)
        hook = lc.hook
    pf = pb = None
    if tokens and t_fwd is not None:
        pf = H.proxy_iters(H.bucket_times(fplan, t_fwd), nspi)
        pb = H.proxy_iters(H.bucket_times(bplan, t_bwd), nspi)

    def loop(extra, n):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        a.record(cs)
        for _ in range(n):
            reps.append(st.step(flags | extra, cs.cuda_stream, ms.cuda_stream, pf, pb, hook=hook))
        b.record(cs)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n, reps

    for _ in range(warmup):
        st.step(flags, cs.cuda_stream, ms.cuda_stream, pf, pb, hook=hook)
    ms_step, _ = loop(0, steps)
    _, reps = loop(L.SCHED_TIMING, steps)
    predicted = emulated = None
    if predict_link is not None:
        # the N-rank step predicted by the library's two-stream model: every
        # compute-stream op at its MEASURED duration on this B200 (copies,
        # proxy compute), every collective at alpha + beta n of its bucket
        # (modelled NVLink; no SM / HBM contention)
        rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, pf, pb, want_log=True, hook=hook)
        tot, exp = H.simulate_n_rank(st, rep["log"], predict_link[0], predict_link[1])
        predicted = dict(total_ms=round(tot / 1e6, 3), exposed_ms=round(exp / 1e6, 3))
        # and MEASURED with emulated collectives (K11): contention included
        em = dict(ag=predict_link[0], rs=predict_link[1], ctas=H.emulation_ctas(world))

        def em_loop(extra, emulate, n):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            for _ in range(n):
                st.step(flags | extra, cs.cuda_stream, ms.cuda_stream, pf, pb, hook=hook, emulate=emulate)
            b.record(cs)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n
        em_loop(0, em, 1)
        e_step = em_loop(0, em, steps)
        e_comp = em_loop(L.SCHED_NO_COMM, None, steps)
        emulated = dict(step_ms=round(e_step, 3), compute_only_ms=round(e_comp, 3),
                        exposed_ms=round(e_step - e_comp, 3))
    measured_tc = None
    if profile:
        # per-bucket compute durations of the timed steps (the paper's profiler,
        # P:219-221): with a per-parameter plan, T_c of every parameter
        rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, pf, pb, want_log=True, hook=hook)
        tf, tb = [0] * len(specs), [0] * len(specs)
        for ph, op, b, _s, ns, _t in rep["log"]:
            if op in (L.OP_COMPUTE_F, L.OP_COMPUTE_B):
                bk = (st.fwd if ph == 0 else st.bwd)[b]
                for j in bk.members:   # a multi-member bucket's time goes to its first member
                    (tf if ph == 0 else tb)[j] += max(ns, 0) if j == bk.members[0] else 0
        measured_tc = (tf, tb)
    graph_ms = None
    if graph and hook is None:
        # the same step as one CUDA-graph launch (fsdp_step_graph): host enqueue cost removed
        sg = st.capture(flags, cs.cuda_stream, ms.cuda_stream, pf, pb)
        for _ in range(3):
            sg.launch(cs.cuda_stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        for _ in range(steps):
            sg.launch(cs.cuda_stream)
        b.record(cs)
        torch.cuda.synchronize()
        graph_ms = a.elapsed_time(b) / steps
        sg.close()
    op_ns = [sum(r["op_ns"][i] for r in reps) for i in range(L.N_OPS)]
    kb = st.kernel_bytes()
    names = {L.OP_PACK_AG: "K1", L.OP_UNPACK: "K3", L.OP_PACK_RS: "K4", L.OP_COPYOUT_RS: "K6"}
    kern = {names[o]: round(kb[o] * steps / (op_ns[o] * 1e-9) / 1e9, 1) for o in kb if kb[o] and op_ns[o] > 0}
    ag_b, rs_b = st.step_bytes()
    res = dict(ms_per_step=round(ms_step, 4), buckets_fwd=len(fplan), buckets_bwd=len(bplan),
               kernel_GBps=kern, launches_per_step=reps[0]["kernel_launches"],
               compute_ms_per_step=round((op_ns[L.OP_COMPUTE_F] + op_ns[L.OP_COMPUTE_B]) / steps / 1e6, 3),
               step_GBps=round((ag_b + rs_b) / (ms_step * 1e-3) / 1e9, 1))
    if predicted:
        res["predicted_N%d" % world] = predicted
    if emulated:
        res["emulated_N%d" % world] = emulated
    # peak FSDP-buffer memory of this variant's op order under the G40 model
    # (the paper's memory column, Tables 5 / 6) and the static pools this
    # library actually holds
    mp, pools = H.predict_memory(st, flags)
    res["memory_model_peak_GiB"] = round(mp / 2 ** 30, 3)
    res["static_pools_GiB"] = round(pools / 2 ** 30, 3)
    if graph_ms is not None:
        res["graph_ms_per_step"] = round(graph_ms, 4)
    if measured_tc is not None:
        res["_measured_tc"] = measured_tc
    del st, loop
    ctx.close()
    gc.collect()
    torch.cuda.empty_cache()
    print("  [mem after variant: %.1f GiB allocated]" % (torch.cuda.memory_allocated() / 2**30), file=sys.stderr)
    return res


def c0():
    from paper_2411_00284_b200 import _lib as L
    from workloads import toy_mlp
    specs = toy_mlp()
    tc = [20000 if p.row_numel > 1 else 0 for p in specs]
    out = {}
    for name, mode in (("per_param", L.PLAN_PER_PARAM), ("greedy", L.PLAN_GREEDY)):
        out[name] = run_variant(specs, 2, mode, L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, tc, tc,
                                mem_max=10**9, link=(10000, 100000), param_dtype=L.FP32, steps=50, warmup=5,
                                graph=True)
    return out


def c2(tokens=(1024, 2048)):
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    specs = llama("8b")
    ctx = F.Ctx(8, 0)
    s = torch.cuda.Stream()
    nspi = H.calibrate_proxy(ctx, s.cuda_stream)
    ctx.close()
    R, FB, BB = L.SCHED_REORDER, L.SCHED_FWD_AG_BEFORE_WAIT, L.SCHED_BWD_AG_BEFORE_WAIT
    out = {"proxy_cal": nspi}
    for T in tokens:
        f, b = per_param_compute_ns(specs, T)
        rows = {}
        variants = [("vanilla", L.PLAN_PER_PARAM, 0), ("+reorder", L.PLAN_PER_PARAM, R | FB),
                    ("+bucket", L.PLAN_MANUAL, 0), ("+reorder&bucket", L.PLAN_MANUAL, R | FB),
                    ("greedy+reorder", L.PLAN_GREEDY, R | FB),
                    ("search+reorder", "search", R | FB),
                    ("place fwd-before/bwd-before", L.PLAN_MANUAL, R | FB | BB),
                    ("place fwd-after/bwd-before", L.PLAN_MANUAL, R | BB),
                    ("place fwd-after/bwd-after", L.PLAN_MANUAL, R)]
        # modelled NVLink 5 at N = 8: 720 GB/s bus bandwidth (80 % of 900) and
        # 20 us base latency -> beta = (7/8) / 720e9 s per full byte = 1215 fs/B
        nvl = (20000, 1215)
        for name, mode, flags in variants:
            rows[name] = run_variant(specs, 8, mode, flags, f, b, mem_max=2 * 10**9, tokens=T, nspi=nspi,
                                     steps=3, warmup=1, link=nvl, predict_link=(nvl, nvl))
        out["T=%d" % T] = rows
    return out


def c2w(worlds=(2, 4, 8), T=1024):
    """configs[2] across world sizes: vanilla vs manual+reorder vs greedy+reorder,
    predicted N-rank exposure at each N (link beta scaled by (N-1)/N)."""
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    specs = llama("8b")
    ctx = F.Ctx(8, 0)
    s = torch.cuda.Stream()
    nspi = H.calibrate_proxy(ctx, s.cuda_stream)
    ctx.close()
    R, FB = L.SCHED_REORDER, L.SCHED_FWD_AG_BEFORE_WAIT
    f, b = per_param_compute_ns(specs, T)
    out = {"tokens_per_gpu": T, "proxy_cal": nspi}
    for w in worlds:
        nvl = (20000, round((w - 1) / w / 720e9 * 1e15))
        rows = {}
        for name, mode, flags in (("vanilla", L.PLAN_PER_PARAM, 0), ("manual+reorder", L.PLAN_MANUAL, R | FB),
                                  ("greedy+reorder", L.PLAN_GREEDY, R | FB)):
            rows[name] = run_variant(specs, w, mode, flags, f, b, mem_max=2 * 10**9, tokens=T, nspi=nspi,
                                     steps=3, warmup=1, link=nvl, predict_link=(nvl, nvl))
        out["N=%d" % w] = rows
    return out


def c2m(tokens=(1024, 4096)):
    """configs[2] with the REAL Llama-3-8B layers (attention, SwiGLU, norms,
    loss; paper_2411_00284_b200/llama_compute.py) through the compute hook:
    per-parameter compute times are first MEASURED with a per-parameter plan
    (the paper's profiler) and fed to Algorithm 1 for the greedy
    plan; then the Table 5 / Table 6 variants, each with its N = 8 exposure
    predicted from its measured compute-stream ops (copies + real compute)."""
    from paper_2411_00284_b200 import _lib as L
    from workloads import llama
    specs = llama("8b")
    R, FB, BB = L.SCHED_REORDER, L.SCHED_FWD_AG_BEFORE_WAIT, L.SCHED_BWD_AG_BEFORE_WAIT
    nvl = (20000, 1215)
    out = {}
    for T in tokens:
        rows = {}
        prof = run_variant(specs, 8, L.PLAN_PER_PARAM, 0, steps=2, warmup=1, link=nvl, predict_link=(nvl, nvl),
                           model_T=T, profile=True)
        f, b = prof.pop("_measured_tc")
        rows["vanilla"] = prof
        rows["measured_compute_ms"] = {"fwd": round(sum(f) / 1e6, 3), "bwd": round(sum(b) / 1e6, 3)}
        for name, mode, flags in (("+reorder", L.PLAN_PER_PARAM, R | FB), ("+bucket", L.PLAN_MANUAL, 0),
                                  ("+reorder&bucket", L.PLAN_MANUAL, R | FB),
                                  ("greedy+reorder (measured T_c)", L.PLAN_GREEDY, R | FB),
                                  ("search+reorder (measured T_c)", "search", R | FB),
                                  ("place fwd-after/bwd-before", L.PLAN_MANUAL, R | BB)):
            rows[name] = run_variant(specs, 8, mode, flags, f, b, mem_max=2 * 10**9, steps=2, warmup=1, link=nvl,
                                     predict_link=(nvl, nvl), model_T=T)
        out["T=%d" % T] = rows
    return out


def c3(caps_mb=(25, 50, 100, 200, 500), T=2048):
    """configs[3]: Llama-3-70B at N = 8, SIZE_CAP bucket-size sweep, with the
    compute proxy at T tokens and the predicted N = 8 step / exposure (same
    model as c2), plus the greedy plan and the per-block plan for reference."""
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns
    specs = llama("70b")
    ctx = F.Ctx(8, 0)
    s = torch.cuda.Stream()
    nspi = H.calibrate_proxy(ctx, s.cuda_stream)
    ctx.close()
    f, b = per_param_compute_ns(specs, T)
    nvl = (20000, 1215)
    RF = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    out = {"tokens_per_gpu": T, "proxy_cal": nspi}
    for m in caps_mb:
        out["size_cap %d MB" % m] = run_variant(specs, 8, L.PLAN_SIZE_CAP, RF, f, b, mem_max=m * 10**6, tokens=T,
                                                nspi=nspi, steps=2, warmup=1, link=nvl, predict_link=(nvl, nvl))
    out["manual (per block)"] = run_variant(specs, 8, L.PLAN_MANUAL, RF, f, b, mem_max=2 * 10**9, tokens=T,
                                            nspi=nspi, steps=2, warmup=1, link=nvl, predict_link=(nvl, nvl))
    out["greedy (M_max 2 GB)"] = run_variant(specs, 8, L.PLAN_GREEDY, RF, f, b, mem_max=2 * 10**9, tokens=T,
                                             nspi=nspi, steps=2, warmup=1, link=nvl, predict_link=(nvl, nvl))
    out["search (M_max 2 GB)"] = run_variant(specs, 8, "search", RF, f, b, mem_max=2 * 10**9, tokens=T,
                                             nspi=nspi, steps=2, warmup=1, link=nvl, predict_link=(nvl, nvl))
    return out


def c4():
    from paper_2411_00284_b200 import _lib as L
    from workloads import llama
    specs = llama("405b", n_layers=1, with_embeddings=False)
    return {"layer_bucket": run_variant(specs, 8, L.PLAN_MANUAL, L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT,
                                        steps=3, warmup=1),
            "per_param": run_variant(specs, 8, L.PLAN_PER_PARAM, L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT,
                                     steps=3, warmup=1)}


def main():
    which = [a for a in sys.argv[1:] if a in ("c0", "c2", "c2w", "c2m", "c3", "c4")] or ["c0", "c2", "c2w", "c3",
                                                                                         "c4"]
    res = {}
    for w in which:
        res[w] = globals()[w]()
        print(w, json.dumps(res[w]), flush=True)
    if "--out" in sys.argv:
        with open(sys.argv[sys.argv.index("--out") + 1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
