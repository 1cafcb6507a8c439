#!/usr/bin/env python
"""Benchmark of the SimpleFSDP hot path on B200 -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the whole hot path for one rank of a Llama-3-8B FSDP
job (BASELINE.json configs[1]: bf16 params, fp32 reduce, per-transformer-block
buckets = MANUAL wrapping, reordered with the Table 6 default placements):
forward all-gathers (pack K1, NCCL AG, unpack K3) and backward re-gathers,
gradient pack (K4), NCCL reduce-scatter, copy-out (K6) for all 35 buckets.

* N = 1 (default): one GPU holds rank 0 of an 8-way job (layout world 8,
  "1 GPU (pack/unpack only)" in BASELINE.json) -- every kernel runs at the
  8-GPU per-rank size; the collectives are absent because there are no peers.
* N > 1 (torchrun): one process per GPU, an NCCL communicator of N ranks,
  real in-place all-gather / reduce-scatter on a high-priority comm stream,
  a calibrated compute proxy per bucket (--tokens, default 1024 tokens/GPU).

value = sum over ranks of the full bucket bytes the step's collectives carry
(forward AG + backward AG in bf16, RS in fp32) / step time, in GB/s.  Inputs
(64.3 GB of bucket traffic per rank-step) are far larger than the 126 MB L2.

Beside the contract keys the line carries (N = 1): `roofline` (dominant
kernel vs the measured HBM peak), `kernels` (per-kernel GB/s), `predicted`
(the N-rank step from measured op durations and alpha + beta n links, with
vanilla / greedy / searched plan variants and the G40 memory peak),
`emulated` (the N-rank step MEASURED with emulated collectives, contention
included), `fused_p2p` (the fused peer-memory path K8 / K9, with its own
`emulated`), `e2e` (host I/O through fsdp_run_schedule), `cpu_baseline`
(the oracle on one host core), `clocks`, `env` and `paper_context`.
"""
import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AG/RS bus GB/s and exposed-comm ms/step, Llama-3-8B shards, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="8b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--plan", default="manual", choices=["manual", "greedy", "per_param", "size_cap", "search"],
                    help="search: fsdp_plan_search (simulator-guided, beyond Algorithm 1) from the manual and "
                         "greedy plans, with the per-op compute model at --tokens (or --predict-tokens)")
    ap.add_argument("--sim-world", type=int, default=8, help="layout world size at N=1")
    ap.add_argument("--plan-file", default=None,
                    help="JSON with plans.fwd / plans.bwd (buckets of forward indices in execution order), e.g. "
                         "from tools/plan_search.py; overrides --plan")
    ap.add_argument("--tokens", type=int, default=None, help="proxy compute tokens/GPU (0 = none)")
    ap.add_argument("--no-reorder", action="store_true")
    ap.add_argument("--grad-slots", type=int, default=2,
                    help="full-gradient slots the backward buckets rotate through (peer-memory path: the backward "
                         "of bucket b waits for the peers' K9 of bucket b - slots)")
    ap.add_argument("--keep-last", action="store_true",
                    help="FSDP_SCHED_KEEP_LAST_GATHERED (G42): the first backward bucket reuses the last forward "
                         "bucket's gathered parameters (no re-gather; FSDP2-style, beyond the paper)")
    ap.add_argument("--fwd-placement", default="before", choices=["before", "after"])
    ap.add_argument("--bwd-placement", default="after", choices=["before", "after"])
    ap.add_argument("--mem-limit", type=float, default=2e9)
    ap.add_argument("--alpha-ns", type=int, default=20000)
    ap.add_argument("--beta-fs", type=int, default=1500)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--proxy-ctas", type=int, default=1)
    ap.add_argument("--proxy-smem", type=int, default=0)
    ap.add_argument("--trace", default=None, help="write a Chrome trace of one profiled step to this path")
    ap.add_argument("--eager", action="store_true",
                    help="time the eager enqueue of every step instead of the CUDA-graph replay (fsdp_step_graph)")
    ap.add_argument("--compute", default="proxy", choices=["proxy", "gemm", "llama"],
                    help="bucket compute: calibrated proxy kernel (--tokens), cuBLASLt linear layers on the "
                         "gathered parameters, or the real Llama-3 layers (attention, SwiGLU, norms, loss) "
                         "through the schedule's compute hook (tokens = --tokens or 1024; eager timing)")
    ap.add_argument("--pg", default="auto", choices=["auto", "nccl", "gloo"],
                    help="torch.distributed backend for host plumbing (auto: nccl, gloo for p2p)")
    ap.add_argument("--same-device", action="store_true",
                    help="TEST ONLY: put every rank on cuda:0 (exercises the multi-process p2p path on one GPU; "
                         "timings are meaningless)")
    ap.add_argument("--predict-tokens", type=int, default=1024,
                    help="N=1: tokens/GPU of the compute proxy for the predicted N-rank exposure (0 = off)")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "p2p"],
                    help="nccl: pack + NCCL + copy-out (the paper's bucketing); p2p: fused peer-memory "
                         "kernels K8/K9 (1 GPU: the 7 peers are simulated as separate buffers)")
    ap.add_argument("--nccl-register", default="none", choices=["none", "local", "symmetric"],
                    help="N > 1 NCCL path: allocate the collective buffers with ncclMemAlloc and register them "
                         "(ncclCommRegister / symmetric ncclCommWindowRegister) for zero-copy NVLS / symmetric "
                         "kernels")
    ap.add_argument("--p2p-max-ctas", type=int, default=-1,
                    help="N > 1 peer-memory path: K8 / K9 grid cap (-1 = harness.emulation_ctas_p2p(N), 0 = full "
                         "GPU)")
    ap.add_argument("--nccl-max-ctas", type=int, default=0,
                    help="N > 1 NCCL path: cap NCCL's CTAs per collective (fsdp_ctx_create_config; 0 = NCCL default)")
    ap.add_argument("--no-variants", action="store_true",
                    help="N=1: skip the predicted exposure of the vanilla and greedy plans")
    ap.add_argument("--ag", default="flat", choices=["flat", "grouped"],
                    help="flat: the paper's bucketing (copy-in, one AG of the flat buffer, copy-out); grouped: one "
                         "NCCL group of per-member AGs straight into the full parameters (FSDP_BUCKET_GROUPED_AG)")
    ap.add_argument("--dist", action="store_true",
                    help="run the torch.distributed / NCCL-communicator path even at --gpus 1 (world 1 with a "
                         "real communicator: checks the N > 1 plumbing on one GPU)")
    ap.add_argument("--no-gemm-comparison", action="store_true",
                    help="N=1: skip the emulated N-rank step with GEMM compute for per-block NCCL vs searched fused "
                         "(two child runs)")
    ap.add_argument("--no-fused-leg", action="store_true",
                    help="N=1 with --collective nccl: skip the extra run of the fused peer-memory mode whose "
                         "summary is reported under 'fused_p2p'")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(r[0]) for r in self.rows if r[0].isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": int(self.rows[0][1]) if self.rows[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# The paper's own numbers (H100, training TPS / peak memory -- it reports no
# bus bandwidth or exposed-comm time): context beside this run, not a target.
PAPER_CONTEXT = {
    "hardware": "H100, 8 per node, NVLink intra-node (P:344); Llama 3.1; TorchTitan; C4",
    "headline_vs_FSDP2_eager": {"peak_memory_reduction": "up to 28.54%", "throughput_gain": "up to 68.67%",
                                "cite": "P:55"},
    "8b_fsdp_vs_FSDP2_eager": {"memory": "-27.72%", "tps": "+7.49%", "gpus": "32/64/128", "cite": "P:414"},
    "table5_1node_tps_mem": {"vanilla": [50976, 67.26], "+reorder": [54544, 68.72], "+bucket": [49168, 69.06],
                             "+reorder&bucket": [52480, 69.08], "cite": "P:556-570 (8B, FSDP only, bs 1)"},
    "table5_8node_tps_mem": {"vanilla": [333440, 56.42], "+reorder": [404032, 57.88], "+bucket": [405632, 58.15],
                             "+reorder&bucket": [428352, 65.74], "cite": "P:556-570"},
    "note": "context only: the paper's metrics are training TPS and peak GiB on H100; this line's are bucket "
            "bytes per second, kernel HBM fractions and exposure predicted / measured on B200",
}


def run_env(torch):
    """GPU / host identity and library versions of this run (SURVEY §8(d)
    protocol step 6)."""
    cpu = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    try:
        nccl = ".".join(str(x) for x in torch.cuda.nccl.version())
    except Exception:
        nccl = None
    return {"gpu": torch.cuda.get_device_name(), "sm_count": torch.cuda.get_device_properties(0).multi_processor_count,
            "torch": torch.__version__, "cuda_runtime": torch.version.cuda, "nccl": nccl,
            "host_cpu": cpu, "host_cpus": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0)),
            "nccl_env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_peak_bf16():
    """Sustained dense bf16 TFLOP/s (MEASURED_PEAKS.json; for a kernel timed
    inside a long step), else the guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except (OSError, KeyError, ValueError):
        return 1400.0


def ncu_traffic(op_name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(op_name)
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------- CPU oracle
class CpuOracleSample:
    """The oracle as it stands, on a bounded sample of the same workload:
    whole 8B-block tensors (attention_norm, wq, wk, wv, wo, ffn_norm) at world
    N -- forward AG (shard + pack all ranks + gather + unpack), the backward
    re-gather, and the bucketed RS (pack every rank, rank-order sum, copy-out).
    Inputs are generated once; run() times one step of the oracle."""

    def __init__(self, world):
        from oracle.layout import bucket_layout
        from workloads import llama
        from workloads.data import grad_tensor, param_tensor
        self.world = world
        specs = [s for s in llama("8b", n_layers=1, with_embeddings=False)
                 if s.name.split(".")[-2] in ("attention_norm", "wq", "wk", "wv", "wo", "ffn_norm")]
        self.params = [param_tensor(s, "bf16", 1 + i) for i, s in enumerate(specs)]
        self.grads = [[grad_tensor(s, "bf16", 2, r) for s in specs] for r in range(world)]
        dims = [(s.dim0, s.row_numel) for s in specs]
        self.bytes = 2 * world * bucket_layout(dims, world, 2, 16)[1] + world * bucket_layout(dims, world, 4, 16)[1]
        n = sum(s.dim0 * s.row_numel for s in specs)
        self.desc = ("oracle (NumPy, 1 thread) on %d tensors / %.1f M params of one Llama-3-8B block at N=%d: "
                     "fwd AG + bwd AG + RS over all %d simulated ranks per step" % (len(specs), n / 1e6, world, world))

    def run(self):
        """Returns (GB/s in the bench's unit, seconds)."""
        from oracle import collectives as OC
        t0 = time.perf_counter()
        OC.bucketed_all_gather(self.params, self.world, 16)     # forward
        OC.bucketed_all_gather(self.params, self.world, 16)     # backward re-gather
        OC.bucketed_reduce_scatter(self.grads, self.world, 16)
        dt = time.perf_counter() - t0
        return self.bytes / dt / 1e9, dt


def run_reference(args, rank):
    if rank != 0:
        return
    world = args.sim_world if args.gpus == 1 else args.gpus
    t0 = time.perf_counter()
    sample = CpuOracleSample(world)
    desc = sample.desc
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(sample.run())
    timed = vals[args.warmup:]
    v = sum(x[0] for x in timed) / len(timed)
    ms = 1e3 * sum(x[1] for x in timed) / len(timed)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": "llama3-8b FSDP rank step sample (see cpu_baseline.sample)",
                       "world": world, "plan": "one bucket of the sampled tensors"},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": desc, "host_cpus": os.cpu_count()},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.perf_counter() - t0, 1)}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def fused_leg(args):
    """bench.py --collective p2p at N = 1 on the same workload (child process)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--collective", "p2p", "--steps", str(args.steps),
           "--warmup", str(args.warmup), "--no-e2e", "--no-cpu-baseline", "--no-fused-leg", "--no-gemm-comparison",
           "--predict-tokens", str(args.predict_tokens), "--plan", args.plan, "--model", args.model, "--sim-world", str(args.sim_world)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    except Exception as e:  # reported, never fatal to the headline
        return {"error": "%s: %s" % (type(e).__name__, str(e)[:200])}
    return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
            "collective": d["config"]["collective"], "kernels": d["kernels"], "roofline": d["roofline"],
            "gpu_launches": d["gpu_launches"], "p2p_wait_timeouts": d["p2p_wait_timeouts"],
            "emulated": d.get("emulated"),
            "how": "bench.py --collective p2p (same workload, same K/W, own process)"}


def gemm_comparison(args):
    """The N = 8 step with real tensor-core compute (cuBLASLt linear layers,
    T = 1024) and emulated collectives, measured for the paper-style design
    (per-block buckets, NCCL + copy kernels) and the B200-native one (searched
    buckets, fused peer-memory kernels K8 / K9) -- child processes."""
    out = {}
    for name, extra in (("per-block + NCCL + copy kernels", ["--plan", "manual", "--collective", "nccl"]),
                        ("searched + fused K8/K9", ["--plan", "search", "--collective", "p2p"])):
        cmd = [sys.executable, os.path.abspath(__file__), "--compute", "gemm", "--tokens", "1024", "--steps",
               str(args.steps), "--warmup", str(args.warmup), "--no-e2e", "--no-cpu-baseline", "--no-fused-leg",
               "--no-variants", "--no-gemm-comparison", "--model", args.model,
               "--sim-world", str(args.sim_world)] + extra
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
            e = d["emulated"]
            out[name] = {"emulated_step_ms": e["step_ms"], "compute_only_ms": e["compute_only_ms"],
                         "exposed_ms": e["exposed_ms"], "buckets": [d["config"]["buckets_fwd"],
                                                                    d["config"]["buckets_bwd"]]}
        except Exception as ex:  # reported, never fatal to the headline
            out[name] = {"error": "%s: %s" % (type(ex).__name__, str(ex)[:200])}
    out["how"] = ("bench.py --compute gemm --tokens 1024 (cuBLASLt bf16 linear layers on the gathered parameters) "
                  "with the N-rank collectives emulated (K11 / paced K8-K9), own processes")
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist

    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns

    assert torch.cuda.is_available(), "bench.py needs a B200"
    if args.same_device:
        local = 0    # test only: every rank on cuda:0 (exercises the multi-process path on one GPU)
    torch.cuda.set_device(local)
    multi = args.gpus > 1 or args.dist
    p2p = args.collective == "p2p"
    pg = args.pg if args.pg != "auto" else ("gloo" if (p2p or args.same_device) else "nccl")
    if multi:
        assert world_env == args.gpus, "launch with torchrun --nproc-per-node %d" % args.gpus
        if pg == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        world = args.gpus
        if p2p:
            ctx = F.Ctx(world, rank, local)   # peer-memory collectives need no NCCL communicator
        else:
            uid = [F.nccl_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            cfg = dict(max_ctas=args.nccl_max_ctas) if args.nccl_max_ctas > 0 else None
            ctx = F.Ctx(world, rank, local, nccl_uid=uid[0], nccl_config=cfg)
    else:
        world = args.sim_world
        ctx = F.Ctx(world, 0, local)   # layout-only: rank 0 of a simulated `world`-way job
    tokens = args.tokens if args.tokens is not None else (1024 if multi else 0)

    specs = llama(args.model, n_layers=args.layers)
    t_fwd, t_bwd = per_param_compute_ns(specs, tokens) if tokens else ([0] * len(specs), [0] * len(specs))
    mode = {"manual": L.PLAN_MANUAL, "greedy": L.PLAN_GREEDY, "per_param": L.PLAN_PER_PARAM,
            "size_cap": L.PLAN_SIZE_CAP, "search": L.PLAN_GREEDY}[args.plan]
    link = (args.alpha_ns, args.beta_fs)
    fplan, bplan = H.plans_for(specs, world, mode, t_fwd, t_bwd, link, link, int(args.mem_limit))
    if args.plan == "search":
        st_tok = tokens or args.predict_tokens or 1024
        sf, sb = per_param_compute_ns(specs, st_tok)
        slink = (20000, round((world - 1) / world / 720e9 * 1e15)) if not multi else link
        fplan, bplan = H.plans_search(specs, world, sf, sb, slink, slink, int(args.mem_limit))
    if args.plan_file:
        with open(args.plan_file) as f:
            pj = json.load(f)["plans"]
        fplan, bplan = pj["fwd"], pj["bwd"]
        flat_f = sorted(j for b in fplan for j in b)
        flat_b = sorted(j for b in bplan for j in b)
        assert flat_f == flat_b == list(range(len(specs))), "plan file does not cover the model's parameters"
    reg = args.nccl_register if (multi and not p2p and args.nccl_register != "none") else None
    st = H.RankState(specs, world, rank if multi else 0, fplan, bplan, ctx, seed=1234 + rank,
                     ipc=multi and p2p, nccl_register=reg, ag_grouped=args.ag == "grouped",
                     grad_slots=args.grad_slots)
    compute = torch.cuda.Stream()
    comm = torch.cuda.Stream(priority=-1)
    cs, ms = compute.cuda_stream, comm.cuda_stream

    pf = pb = None
    if tokens:
        nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
        pf = H.proxy_iters(H.bucket_times(fplan, t_fwd), nspi)
        pb = H.proxy_iters(H.bucket_times(bplan, t_bwd), nspi)
    if p2p:
        if multi:
            def exchange(obj):
                out = [None] * world
                dist.all_gather_object(out, obj)
                return out
            st.setup_p2p_ipc(exchange)
            # N > 1: cap the fused kernels' grid like NCCL's channels so the
            # NVLink-bound K8 / K9 leave the SMs to the compute stream
            st.p2p_max_ctas = args.p2p_max_ctas if args.p2p_max_ctas >= 0 else H.emulation_ctas_p2p(world)
        else:
            st.setup_p2p_simulated(seed=99)
    flags = 0 if args.no_reorder else L.SCHED_REORDER
    if p2p:
        flags |= L.SCHED_P2P
    if args.fwd_placement == "before":
        flags |= L.SCHED_FWD_AG_BEFORE_WAIT
    if args.bwd_placement == "before":
        flags |= L.SCHED_BWD_AG_BEFORE_WAIT
    if args.keep_last:
        flags |= L.SCHED_KEEP_LAST_GATHERED

    gemm = model = None
    if args.compute == "llama":
        # the real model through the compute hook (fsdp_compute_hook): forward
        # / backward of every bucket's layers on the gathered parameters, the
        # weight gradients written where the reduce-scatter reads them
        from paper_2411_00284_b200.llama_compute import LlamaCompute
        model = LlamaCompute(st, tokens or 1024)
        pf = pb = None
    if args.compute == "gemm":
        # linear-layer compute: cuBLASLt bf16 GEMMs on the gathered parameters,
        # the backward writing the gradients the reduce-scatter averages
        gemm = st.setup_gemm(tokens or 1024)
        pf = pb = None

    hook = model.hook if model else None

    def step(extra=0):
        return st.step(flags | extra, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm, hook=hook)

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not multi:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if pg == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    host_enqueue = []

    def timed_loop(extra, n, clocks=None):
        """n steps bracketed by events on the compute stream; max over ranks.
        Also records the host time to enqueue each step (SURVEY §8(d) protocol
        step 5: is the eager step launch-bound?)."""
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        a.record(compute)
        for _ in range(n):
            h0 = time.perf_counter()
            reps.append(step(extra))
            if extra == 0:
                host_enqueue.append(time.perf_counter() - h0)
        b.record(compute)
        barrier()
        return max_over_ranks(a.elapsed_time(b) / n), reps

    for _ in range(args.warmup):
        step()
    # (1) the headline: K plain steps, no instrumentation -- replayed as one
    #     CUDA graph per step (fsdp_step_graph: the library's whole step,
    #     kernels + NCCL collectives + cross-stream events, captured once) unless
    #     --eager (the p2p path replays too: its epochs advance on the device);
    #     the eager enqueue of the same steps is timed beside it
    sg = None
    if not args.eager and model is None:
        sg = st.capture(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm)
        for _ in range(args.warmup):
            sg.launch(cs)
    elif not args.eager:
        # the model's torch ops through the hook: torch captures the whole step
        # (library kernels, collectives and the hook's ops) into one graph
        tg = st.capture_with_torch(flags, compute, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm,
                                   hook=hook)

        class _TorchGraph:
            def launch(self, stream):
                with torch.cuda.stream(compute):
                    tg.replay()

            def close(self):
                pass
        sg = _TorchGraph()
        for _ in range(args.warmup):
            sg.launch(cs)

    def graph_loop(n):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(compute)
        for _ in range(n):
            sg.launch(cs)
        b.record(compute)
        barrier()
        return max_over_ranks(a.elapsed_time(b) / n)

    with ClockSampler(local) as clk:
        if sg is not None:
            ms_step = graph_loop(args.steps)
        else:
            ms_step, _ = timed_loop(0, args.steps)
    ms_eager = timed_loop(0, args.steps)[0] if sg is not None else ms_step
    # (2) the same K steps with a CUDA event pair around every op (per-kernel
    #     device time on the launching stream; synchronises once per step)
    ms_prof, reports = timed_loop(L.SCHED_TIMING, args.steps)
    # NOTE: every step below runs on EVERY rank (a step holds collectives / epoch
    # handshakes); only the reporting is rank 0's
    if args.trace:
        rep_t = st.step(flags | L.SCHED_TIMING, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, want_log=True,
                        gemm=gemm, hook=hook)
        if rank == 0:
            H.chrome_trace(rep_t["log"], args.trace)
    # model check (runs with real collectives): the two-stream simulator fed
    # with THIS run's measured op durations (collectives included) against the
    # measured eager step -- the gap is what the model leaves out (SM / HBM
    # contention between the streams, launch gaps)
    model_check = None
    if multi or p2p:
        rep_m = st.step(flags | L.SCHED_TIMING, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, want_log=True,
                        gemm=gemm, hook=hook)
        tot_m, exp_m, _, _ = F.simulate_schedule(rep_m["log"], [max(e[4], 0) for e in rep_m["log"]])
        model_check = {"simulated_ms": round(tot_m / 1e6, 3), "simulated_exposed_ms": round(exp_m / 1e6, 3),
                       "how": "fsdp_simulate_schedule on one timed step's measured op durations"}
    # (3) compute-stream-only baseline: same ops, no collective, no wait
    step(L.SCHED_NO_COMM)
    ms_compute, _ = timed_loop(L.SCHED_NO_COMM, args.steps)

    if sg is not None:
        sg.close()

    ag_b, rs_b = st.step_bytes()
    ranks = world_env if multi else 1
    value = ranks * (ag_b + rs_b) / (ms_step * 1e-3) / 1e9

    # N = 1 has no peers, so exposure cannot be measured; report the library's
    # two-stream PREDICTION for the N-rank job instead (fsdp_simulate_schedule):
    # every compute-stream op at its duration measured here (copy kernels and
    # the compute proxy at --predict-tokens), every collective at alpha + beta n
    # of modelled NVLink 5 (720 GB/s bus, 20 us); no contention modelled.
    predicted = None
    if not multi and not p2p and (args.predict_tokens or gemm or model):
        beta = round((world - 1) / world / 720e9 * 1e15)
        link = (20000, beta)
        if gemm or model:   # the measured compute of this run is the compute
            ppf = ppb = None
        else:
            ptf, ptb = per_param_compute_ns(specs, args.predict_tokens)
            nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
            ppf = H.proxy_iters(H.bucket_times(fplan, ptf), nspi)
            ppb = H.proxy_iters(H.bucket_times(bplan, ptb), nspi)
        tot, exp = H.predict_exposure(st, flags, cs, ms, ppf, ppb, link, link, args.proxy_ctas, args.proxy_smem,
                                      gemm=gemm, hook=hook)
        predicted = {"world": world,
                     "tokens_per_gpu": gemm["tokens"] if gemm else model.T if model else args.predict_tokens,
                     "compute": ("cuBLASLt linear layers (measured)" if gemm else
                                 "Llama-3 layers through the compute hook (measured)" if model else
                                 "calibrated proxy (per-op model)"),
                     "link_alpha_ns": link[0], "link_beta_fs_per_byte": link[1], "total_ms": round(tot / 1e6, 3),
                     "exposed_ms": round(exp / 1e6, 3), "exposed_comm_ms": round(exp / 1e6, 3),
                     "model": "measured compute-stream ops + alpha/beta NVLink collectives, no contention"}
        # the paper's other metric (Tables 5 / 6): peak memory of the
        # step's FSDP buffers under allocate-on-produce / free-after-use (G40),
        # beside what this library's static two-slot pools hold
        mp, pools = H.predict_memory(st, flags)
        predicted["memory_model_peak_GiB"] = round(mp / 2 ** 30, 3)
        predicted["static_pools_GiB"] = round(pools / 2 ** 30, 3)
        if not gemm and not model and not args.no_variants:
            # the north star's comparison: exposure under the greedy plan (Alg. 1)
            # vs the unbucketed, unreordered baseline, same model, same compute
            variants = {}
            RF = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
            for name, vmode, vflags in (("vanilla (per-param, no reorder)", L.PLAN_PER_PARAM, 0),
                                        ("greedy + reorder", L.PLAN_GREEDY, RF),
                                        ("search + reorder (fsdp_plan_search, beyond the paper)", "search", RF)):
                if vmode == "search":
                    vf, vb = H.plans_search(specs, world, ptf, ptb, link, link, int(args.mem_limit))
                else:
                    vf, vb = H.plans_for(specs, world, vmode, ptf, ptb, link, link, int(args.mem_limit))
                vst = H.RankState(specs, world, 0, vf, vb, ctx, seed=99)
                vpf = H.proxy_iters(H.bucket_times(vf, ptf), nspi)
                vpb = H.proxy_iters(H.bucket_times(vb, ptb), nspi)
                vst.step(vflags, cs, ms, vpf, vpb, args.proxy_ctas, args.proxy_smem)   # warm-up
                vt, ve = H.predict_exposure(vst, vflags, cs, ms, vpf, vpb, link, link, args.proxy_ctas,
                                            args.proxy_smem)
                variants[name] = {"buckets_fwd": len(vf), "buckets_bwd": len(vb),
                                  "total_ms": round(vt / 1e6, 3), "exposed_ms": round(ve / 1e6, 3),
                                  "memory_model_peak_GiB": round(H.predict_memory(vst, vflags)[0] / 2 ** 30, 3)}
                del vst
                gc.collect()
                torch.cuda.empty_cache()
            variants["manual (per-block) + reorder [this run]"] = {
                "buckets_fwd": len(fplan), "buckets_bwd": len(bplan),
                "total_ms": predicted["total_ms"], "exposed_ms": predicted["exposed_ms"],
                "memory_model_peak_GiB": predicted["memory_model_peak_GiB"]}
            predicted["variants"] = variants

    # MEASURED exposure of the N-rank step with emulated collectives (K11,
    # fsdp_comm_emulation): every AG / RS runs on the comm stream with the
    # modelled NVLink duration, 32 CTAs and the HBM traffic a rank sees, so
    # (step - compute-only step) includes the SM / HBM contention the
    # two-stream prediction leaves out.  Timing only (no peers, no real data).
    emulated = None
    if not multi and p2p and (args.predict_tokens or gemm or model):
        # the fused peer-memory path: K8 / K9 against the simulated peers, paced to
        # the modelled link time (fsdp_comm_emulation with FSDP_SCHED_P2P)
        link = (20000, round((world - 1) / world / 720e9 * 1e15))
        ppf = ppb = None
        if not gemm and not model:
            ptf, ptb = per_param_compute_ns(specs, args.predict_tokens)
            nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
            ppf = H.proxy_iters(H.bucket_times(fplan, ptf), nspi)
            ppb = H.proxy_iters(H.bucket_times(bplan, ptb), nspi)
    if not multi and (args.predict_tokens or gemm or model):
        # with --compute gemm / llama the compute is the real tensor-core work, a
        # more faithful co-runner for the collectives than the ALU-bound proxy
        em = dict(ag=link, rs=link,   # 32 CTAs at N = 8 for K11 (16 could not keep up); 57 for paced K8 / K9
                  ctas=H.emulation_ctas_p2p(world) if p2p else H.emulation_ctas(world))

        def em_loop(extra, emulate, n):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(compute)
            for _ in range(n):
                st.step(flags | extra, cs, ms, ppf, ppb, args.proxy_ctas, args.proxy_smem, emulate=emulate,
                        gemm=gemm, hook=hook)
            b.record(compute)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n
        em_loop(0, em, 1)   # warm-up
        em_step = em_loop(0, em, args.steps)
        em_comp = em_loop(L.SCHED_NO_COMM, None, args.steps)
        emulated = {"world": world, "compute": args.compute,
                    "tokens_per_gpu": (gemm["tokens"] if gemm else model.T if model else args.predict_tokens),
                    "link_alpha_ns": link[0],
                    "link_beta_fs_per_byte": link[1], "ctas_per_collective": em["ctas"],
                    "step_ms": round(em_step, 3), "compute_only_ms": round(em_comp, 3),
                    "exposed_ms": round(em_step - em_comp, 3),
                    "predicted_exposed_ms": predicted["exposed_ms"] if predicted else None,
                    "how": ("same plan and compute as `predicted`, collectives emulated on the comm stream "
                            "(kernel K11: modelled duration, enough CTAs for the rank's HBM traffic); measured with "
                            "CUDA events, eager enqueue" if not p2p else
                            "fused peer-memory kernels K8 / K9 against the simulated peers on a grid of that many "
                            "CTAs, each held to the modelled link time (AG: bf16 bucket; RS: the bf16 gradients "
                            "K9 pulls); the run's compute (see `compute`); CUDA events, eager enqueue")}

    # linear-layer compute throughput (cuBLASLt, tensor cores) of the timed steps
    gemm_report = None
    if model:
        ops_ns = sum(r["op_ns"][L.OP_COMPUTE_F] + r["op_ns"][L.OP_COMPUTE_B] for r in reports) / len(reports)
        tf = model.flops / (ops_ns * 1e-9) / 1e12
        peak_tf = measured_peak_bf16()
        gemm_report = {"tokens": model.T, "model": "Llama-3 layers (torch: cuBLAS GEMMs, SDPA causal GQA, RoPE, "
                                                   "RMSNorm, SwiGLU, cross-entropy) via fsdp_compute_hook",
                       "tflops_per_step": round(model.flops / 1e12, 2),
                       "compute_ms_per_step": round(ops_ns / 1e6, 3), "achieved_TFLOPs": round(tf, 1),
                       "peak_TFLOPs": peak_tf, "frac": round(tf / peak_tf, 3),
                       "note": "model FLOPs / device time of the COMPUTE ops (library GEMM / attention kernels)"}
    if gemm:
        ops_ns = sum(r["op_ns"][L.OP_COMPUTE_F] + r["op_ns"][L.OP_COMPUTE_B] for r in reports) / len(reports)
        tf = st.gemm_flops / (ops_ns * 1e-9) / 1e12
        peak_tf = measured_peak_bf16()
        gemm_report = {"tokens": gemm["tokens"], "tflops_per_step": round(st.gemm_flops / 1e12, 2),
                       "compute_ms_per_step": round(ops_ns / 1e6, 3), "achieved_TFLOPs": round(tf, 1),
                       "peak_TFLOPs": peak_tf, "frac": round(tf / peak_tf, 3),
                       "note": "library GEMMs (cuBLASLt), bf16 in/out, fp32 accumulate"}

    # per-op device time from the timed steps' events -> dominant data kernel
    op_ns = [sum(r["op_ns"][i] for r in reports) for i in range(L.N_OPS)]
    op_cnt = [sum(r["op_count"][i] for r in reports) for i in range(L.N_OPS)]
    if p2p:
        k8, k9 = st.p2p_bytes()
        kbytes = {L.OP_AG: k8, L.OP_RS: k9}
        klaunch = {L.OP_AG: len(st.fwd) + len(st.bwd), L.OP_RS: len(st.bwd)}
        names = {L.OP_AG: "fsdp_p2p_allgather_kernel", L.OP_RS: "fsdp_p2p_reduce_scatter_kernel"}
    else:
        kbytes, klaunch = st.kernel_bytes(), st.kernel_launches()
        names = {L.OP_PACK_AG: "fsdp_ag_pack_kernel", L.OP_UNPACK: "fsdp_ag_unpack_kernel",
                 L.OP_PACK_RS: "fsdp_rs_pack_kernel", L.OP_COPYOUT_RS: "fsdp_rs_copyout_kernel"}
    live = [op for op in kbytes if kbytes[op] > 0 and op_ns[op] > 0]
    dom = max(live, key=lambda op: op_ns[op])
    peak, peak_src = measured_peak_hbm()
    achieved = kbytes[dom] * args.steps / (op_ns[dom] * 1e-9) / 1e9
    per_kernel = {names[op]: {"GB/s": round(kbytes[op] * args.steps / (op_ns[op] * 1e-9) / 1e9, 1),
                              "ms_per_step": round(op_ns[op] / args.steps / 1e6, 3),
                              "launches_per_step": klaunch[op],
                              "bytes_per_step": kbytes[op]} for op in live}
    launches = sum(r["kernel_launches"] for r in reports)
    # device time of the collective ops (event pairs on the comm stream); at
    # N = 1 with the NCCL design no collective exists (no peers): null
    coll_ms = None
    if multi or p2p:
        coll_ms = {"ag_ms_per_step": round(op_ns[L.OP_AG] / args.steps / 1e6, 3),
                   "rs_ms_per_step": round(op_ns[L.OP_RS] / args.steps / 1e6, 3)}
    # NCCL's own estimate of this step's collectives (ncclGroupSimulateEnd,
    # its topology-aware model) beside the event-measured collective time
    if coll_ms is not None and not p2p:
        try:
            est = sum(ctx.nccl_estimate_ns(L.OP_AG, world * b.ag_seg) for b in st.fwd + st.bwd)
            est_rs = sum(ctx.nccl_estimate_ns(L.OP_RS, world * b.rs_seg) for b in st.bwd)
            coll_ms["nccl_estimate_ag_ms_per_step"] = round(est / 1e6, 3)
            coll_ms["nccl_estimate_rs_ms_per_step"] = round(est_rs / 1e6, 3)
        except Exception as e:   # reported, never fatal
            coll_ms["nccl_estimate_error"] = str(e)[:200]
    busbw = None
    if multi and op_ns[L.OP_AG] > 0:
        busbw = {"ag": round((world - 1) / world * ag_b * args.steps / (op_ns[L.OP_AG] * 1e-9) / 1e9, 1),
                 "rs": round((world - 1) / world * rs_b * args.steps / (op_ns[L.OP_RS] * 1e-9) / 1e9, 1)}

    # e2e through the public call with HOST buffers: fsdp_run_schedule with
    # fsdp_host_io streams the rank's parameter shards in from pinned host
    # memory and its fp32 gradient shards back out, bucket by bucket,
    # overlapped with the device path; the step ends when the gradients are
    # on the host.
    e2e = None
    if not args.no_e2e:
        h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8, pin_memory=True)
        h_gs = torch.empty(st.gshard_buf.numel(), dtype=torch.uint8, pin_memory=True)
        h_sh.copy_(st.shard_buf)
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        io = st.host_io(h_sh, h_gs, h2d_s.cuda_stream, d2h_s.cuda_stream)
        h2d_bytes = sum(b.ag_seg for b, p in zip(st.fwd, io["fwd_host_shards"]) if p)
        d2h_bytes = sum(b.rs_seg for b, p in zip(st.bwd, io["bwd_host_grads"]) if p)
        st.step(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, io=io, gemm=gemm, hook=hook)   # warm-up
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(compute)
        for _ in range(args.e2e_steps):
            st.step(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, io=io, gemm=gemm, hook=hook)
        x1.record(compute)
        barrier()
        e2e_ms = max_over_ranks(x0.elapsed_time(x1) / args.e2e_steps)
        e2e = {"value": round(ranks * (ag_b + rs_b) / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(h2d_bytes),
               "d2h_bytes_per_step": int(d2h_bytes),
               "how": "fsdp_run_schedule with fsdp_host_io: per-bucket H2D of shards / D2H of grad shards "
                      "from/to pinned host memory inside the call, overlapped with the device path"}
        del h_sh, h_gs

    cpu = None
    if rank == 0 and not multi and not args.no_cpu_baseline:
        sample = CpuOracleSample(world)
        runs = []
        while sum(r[1] for r in runs) < 10.0:     # ~10 s of timed oracle work
            runs.append(sample.run())
        dt = sum(r[1] for r in runs)
        v = len(runs) * sample.bytes / dt / 1e9
        desc = sample.desc + "; %d repetitions" % len(runs)
        cpu = {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc,
               "seconds": round(dt, 2), "host_cpus": os.cpu_count()}

    # the fused peer-memory path (K8/K9) on the same
    # workload, in a child process of its own (separate allocations and
    # timings), summarised beside the headline
    fused = None
    if rank == 0 and not multi and not p2p and not args.no_fused_leg and args.compute == "proxy":
        fused = fused_leg(args)
    gemm_cmp = None
    if rank == 0 and not multi and not p2p and not args.no_gemm_comparison and args.compute == "proxy" \
            and args.model == "8b":
        gemm_cmp = gemm_comparison(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": ("llama3-8b FSDP rank step, %s plan, %s" % (
                    "file:" + os.path.basename(args.plan_file) if args.plan_file else args.plan, "reorder fwd-%s/bwd-%s" % (
                    args.fwd_placement, args.bwd_placement) if not args.no_reorder else "vanilla order")) +
                ((", 1 GPU = rank 0 of a simulated %d-way job (pack/unpack only, no peers)" % world if not p2p else
                  ", 1 GPU = rank 0 of a simulated %d-way job (peers' buffers simulated in local HBM)" % world)
                 if not multi
                 else ", %d ranks over %s%s" % (world, "peer memory (CUDA IPC)" if p2p else "NCCL",
                                               " [TEST: all ranks on one GPU]" if args.same_device else "")),
                "model": "llama3-8b shapes (Table 2; vocab 128256, 8 KV heads)", "layout_world": world,
                "collective": ("NCCL all-gather / reduce-scatter with pack + copy-out kernels" if not p2p else
                               "fused peer-memory kernels K8/K9 over CUDA IPC mappings of the peers" if multi else
                               "fused peer-memory kernels K8/K9 (peers simulated as separate HBM buffers)"),
                "buckets_fwd": len(fplan), "buckets_bwd": len(bplan), "param_dtype": "bf16",
                "reduce_dtype": "fp32", "compute": args.compute,
                "proxy_tokens_per_gpu": tokens if args.compute == "proxy" else 0,
                "compute_tokens_per_gpu": (model.T if model else gemm["tokens"] if gemm else tokens),
                "value_def": "sum over ranks of full AG(fwd)+AG(bwd)+RS bucket bytes per second of step time",
                "bytes_per_rank_step": ag_b + rs_b, "l2": "inputs > L2 (126 MB): 64 GB of bucket traffic per step",
                "parallelism": "fsdp%d" % world if multi else "fsdp1 (simulated %d)" % world,
                "nccl_register": reg or "none", "ag": args.ag},
            # measured exposure: eager step - the same eager step without collectives / waits
            "exposed_comm_ms": round(ms_eager - ms_compute, 3), "compute_stream_ms": round(ms_compute, 3),
            "profiled_ms_per_step": round(ms_prof, 3),
            "predicted": predicted,
            "emulated": emulated,
            "model_check": dict(model_check, measured_eager_ms=round(ms_eager, 3)) if model_check else None,
            "linear_compute": gemm_report,
            "timing": ("eager enqueue" if sg is None else "CUDA-graph replay of the step (fsdp_step_graph)"
                       if model is None else "CUDA-graph replay of the step incl. the hook's torch ops "
                                             "(torch.cuda.graph)"),
            "eager_ms_per_step": round(ms_eager, 3),
            "host_enqueue_ms_per_step": (round(1e3 * sorted(host_enqueue)[len(host_enqueue) // 2], 3)
                                         if host_enqueue else None),
            # the paper's other metric: peak device memory of this rank
            # (torch-allocated buffers: shards, slots, staging; the library's
            # own run tables are a few MB)
            "peak_device_mem_GiB": round(torch.cuda.max_memory_allocated() / 2 ** 30, 2),
            "collectives": coll_ms, "busbw_GBps": busbw, "kernels": per_kernel,
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": ncu_traffic(names[dom]),
                         "traffic_launch_algorithmic_bytes": ncu_traffic(names[dom] + "_algorithmic"),
                         "algorithmic_bytes_per_launch": kbytes[dom] // max(1, klaunch[dom])},
            "zero_copy": st.zero_copy(),
            "p2p_wait_timeouts": int(st.p2p_err.item()) if p2p else None,
            "fused_p2p": fused,
            "emulated_gemm_comparison": gemm_cmp,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
            "env": run_env(torch),
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    ctx_close = getattr(ctx, "close", None)
    st.close_nccl_mem()
    del st
    if ctx_close:
        ctx_close()
    if multi:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
