#!/usr/bin/env python
"""Benchmark of the SimpleFSDP hot path on B200 -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one pass of the whole hot path for one rank of a Llama-3-8B FSDP job
(BASELINE.json configs[1]: bf16 params, fp32 reduce, per-transformer-block
buckets = MANUAL wrapping, reordered with the Table 6 default placements):
the forward all-gathers and backward re-gathers (NCCL AG + copy-out K3, or the
fused peer-memory K8 with --collective p2p), the gradient pack K4 and the
reduce-scatter (NCCL RS, or K9) for all 35 buckets.  No model compute runs in
the headline step (--tokens 0): it times the communication path itself.

value (the headline, whole job):
* N > 1: bus bytes per second summed over the ranks -- per rank (N-1)/N x the
  full bucket bytes of the step's collectives (nccl-tests busbw convention,
  reading G28; AG in bf16, RS in fp32 on the NCCL path / the bf16 gradients K9
  pulls on the peer-memory path) / step time, times N.
* N = 1: there are no peers, so no bus: the GPU holds rank 0 of a simulated
  8-way job (G36) and runs every pack / copy-out kernel at its per-rank size;
  value = the algorithmic HBM bytes of the step's data kernels / step time
  (`value_kind`: "hbm"), reported beside `ms_per_step` and the dominant
  kernel's roofline fraction.

Legs beside the headline (all measured on the device; `predicted` and
`emulated` are labelled models):
* every N: `kernels` (per kernel: in-step event-timed GB/s and the same
  launches back to back in a CUDA graph), `roofline`, `e2e` (host I/O through
  fsdp_run_schedule), `clocks`, `env`;
* N > 1: `parity` (sampled outputs of the step's own buckets checked against
  the CPU oracle: AG bit-exact, RS within G7's bound / bit-exact where it must
  be), `busbw_block` (an isolated 8B-block AG and RS in the nccl-tests
  convention vs 900 GB/s), `alpha_beta` (a size sweep fitted to T = alpha +
  beta n per op at this N), `exposure` (measured exposed-comm ms/step
  at --exposure-tokens for vanilla / per-block + reorder / greedy + reorder
  planned with the fitted alpha, beta), `nccl_info` (NCCL_DEBUG=INFO lines);
* N = 1: `predicted` (the N-rank step from measured op durations + ASSUMED
  alpha / beta links: a model), `fused_p2p` (K8 / K9 against simulated
  peers), `cpu_baseline` (the oracle on the host cores).
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
NVLINK_GBS = 900.0      # NVLink 5 nominal, per direction per GPU (SURVEY §8(d) roofline)
NVLINK_MEASURED_GBS = 770.0   # peer copy per direction measured on this pool (B200_PROFILING.md)
ASSUMED_LINK = (20000, 1215)   # 20 us, (N-1)/N / 720 GB/s at N = 8: used only where nothing was measured


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="8b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--plan", default="manual", choices=["manual", "greedy", "per_param", "size_cap", "search"])
    ap.add_argument("--plan-file", default=None,
                    help="JSON with plans.fwd / plans.bwd (buckets of forward indices in execution order)")
    ap.add_argument("--sim-world", type=int, default=8, help="layout world size at N=1")
    ap.add_argument("--tokens", type=int, default=0, help="compute tokens/GPU inside the headline step (0 = none)")
    ap.add_argument("--no-reorder", action="store_true")
    ap.add_argument("--grad-slots", type=int, default=2)
    ap.add_argument("--keep-last", action="store_true", help="G42 (beyond the paper): no re-gather of the boundary bucket")
    ap.add_argument("--copy-stream", action="store_true",
                    help="FSDP_SCHED_COPY_STREAM: pack / copy-out kernels on a third stream (NCCL path)")
    ap.add_argument("--fwd-placement", default="before", choices=["before", "after"])
    ap.add_argument("--bwd-placement", default="after", choices=["before", "after"])
    ap.add_argument("--mem-limit", type=float, default=2e9)
    ap.add_argument("--alpha-ns", type=int, default=ASSUMED_LINK[0], help="assumed link for planning where none is measured")
    ap.add_argument("--beta-fs", type=int, default=ASSUMED_LINK[1])
    ap.add_argument("--collective", default="nccl", choices=["nccl", "p2p"],
                    help="nccl: pack + NCCL + copy-out (the paper's bucketing); p2p: fused peer-memory K8/K9")
    ap.add_argument("--compute", default="proxy", choices=["proxy", "gemm", "llama"])
    ap.add_argument("--proxy-ctas", type=int, default=1)
    ap.add_argument("--proxy-smem", type=int, default=0)
    ap.add_argument("--eager", action="store_true", help="time the eager enqueue instead of the CUDA-graph replay")
    ap.add_argument("--trace", default=None, help="Chrome trace of one profiled step")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused-leg", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="N>1: skip the busbw sweep / alpha-beta fit")
    ap.add_argument("--exposure-tokens", type=int, default=1024,
                    help="N>1: tokens/GPU of the compute proxy for the measured exposure variants (0 = skip)")
    ap.add_argument("--quick", action="store_true", help="headline only (no parity / sweep / exposure / side legs)")
    ap.add_argument("--predict-tokens", type=int, default=1024, help="N=1: tokens/GPU of the modelled N-rank step")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--emulate", action="store_true",
                    help="N=1: also run the N-rank step with emulated collectives (K11; a model device)")
    ap.add_argument("--no-gemm-comparison", action="store_true", help="(accepted for old scripts; no effect)")
    ap.add_argument("--pg", default="gloo", choices=["gloo"], help="torch.distributed backend of the host plumbing")
    ap.add_argument("--same-device", action="store_true",
                    help="TEST ONLY: every rank on cuda:0 (multi-process p2p path on one GPU; timings meaningless)")
    ap.add_argument("--dist", action="store_true", help="the N>1 code path at --gpus 1 (world 1, real communicator)")
    ap.add_argument("--n-rank-legs-at-world1", action="store_true",
                    help="TEST ONLY (with --dist): also run the N > 1 legs (block busbw, alpha/beta sweep, exposure, "
                         "NVLS) at world 1, to exercise their code with a real communicator on one GPU")
    ap.add_argument("--nccl-register", default="none", choices=["none", "local", "symmetric"])
    ap.add_argument("--p2p-max-ctas", type=int, default=-1)
    ap.add_argument("--p2p-transport", default="ipc", choices=["ipc", "window"],
                    help="N > 1 peer-memory path: peers mapped through CUDA IPC handles, or through NCCL symmetric "
                         "windows (fsdp_window_peer_pointers; the ctx then holds a communicator)")
    ap.add_argument("--nccl-max-ctas", type=int, default=0)
    ap.add_argument("--ag", default="flat", choices=["flat", "grouped"])
    return ap.parse_args(argv)


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
                                          "--format=csv,noheader,nounits", "-lms", "20"],
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
    "table5_1node_tps_mem": {"vanilla": [50976, 67.26], "+reorder": [54544, 68.72], "+bucket": [49168, 69.06],
                             "+reorder&bucket": [52480, 69.08], "cite": "P:556-570 (8B, FSDP only, bs 1)"},
    "table5_8node_tps_mem": {"vanilla": [333440, 56.42], "+reorder": [404032, 57.88], "+bucket": [405632, 58.15],
                             "+reorder&bucket": [428352, 65.74], "cite": "P:556-570"},
    "note": "context only: the paper reports training TPS and peak GiB on H100, no bus bandwidth or exposure",
}


def run_env(torch):
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
            "devices": torch.cuda.device_count(), "torch": torch.__version__, "cuda_runtime": torch.version.cuda,
            "nccl_torch": nccl, "host_cpu": cpu, "host_cpus": os.cpu_count(),
            "affinity_cpus": len(os.sched_getaffinity(0)),
            "nccl_env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_peak_bf16():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except (OSError, KeyError, ValueError):
        return 1400.0


def ncu_traffic(op_name):
    """DRAM bytes per launch of a kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(op_name)
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------- CPU oracle
class CpuOracleSample:
    """The oracle as it stands, on a bounded sample of the same workload:
    whole 8B-block tensors (attention_norm, wq, wk, wv, wo, ffn_norm) at world
    N -- forward AG, the backward re-gather and the bucketed RS over all N
    simulated ranks.  Inputs are generated once; run() times one step.

    Its value is stated in the headline's unit for the same N: bus bytes (N >
    1: N x (N-1)/N x full bucket bytes) or, at N = 1, the algorithmic HBM bytes
    the N ranks' data kernels would move (per rank: K3 2 x valid full bytes
    per gather, K4 6 B per gradient element, K6 8 B per shard element) -- the
    oracle does every rank's work."""

    def __init__(self, world, kind="bus"):
        from oracle.layout import bucket_layout
        from workloads import llama
        from workloads.data import grad_tensor, param_tensor
        self.world, self.kind = world, kind
        specs = [s for s in llama("8b", n_layers=1, with_embeddings=False)
                 if s.name.split(".")[-2] in ("attention_norm", "wq", "wk", "wv", "wo", "ffn_norm")]
        self.params = [param_tensor(s, "bf16", 1 + i) for i, s in enumerate(specs)]
        self.grads = [[grad_tensor(s, "bf16", 2, r) for s in specs] for r in range(world)]
        dims = [(s.dim0, s.row_numel) for s in specs]
        full_bytes = 2 * world * bucket_layout(dims, world, 2, 16)[1] + world * bucket_layout(dims, world, 4, 16)[1]
        n = sum(s.dim0 * s.row_numel for s in specs)
        shard_elems = sum(-(-s.dim0 // world) * s.row_numel for s in specs)
        if kind == "bus":
            self.bytes = world * (world - 1) / world * full_bytes
            how = "N x (N-1)/N x full bucket bytes"
        else:
            self.bytes = world * (2 * 2 * 2 * n + 6 * n + 8 * shard_elems)
            how = "N ranks x the data kernels' algorithmic HBM bytes (K3 x 2, K4, K6)"
        self.desc = ("oracle (NumPy, 1 thread) on %d tensors / %.1f M params of one Llama-3-8B block at N=%d: "
                     "fwd AG + bwd AG + RS over all %d simulated ranks per step; value = %s / time"
                     % (len(specs), n / 1e6, world, world, how))

    def run(self):
        """Returns (GB/s in the headline's unit, seconds)."""
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
    sample = CpuOracleSample(world, "hbm" if args.gpus == 1 else "bus")
    vals = [sample.run() for _ in range(args.warmup + args.steps)]
    timed = vals[args.warmup:]
    v = sum(x[0] for x in timed) / len(timed)
    ms = 1e3 * sum(x[1] for x in timed) / len(timed)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s",
            "value_kind": sample.kind, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "llama3-8b FSDP rank step sample (see cpu_baseline.sample)",
                       "world": world, "plan": "one bucket of the sampled tensors"},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": sample.desc, "host_cpus": os.cpu_count()},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.perf_counter() - t0, 1)}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------- parity (N ranks)
# Verification leg (after the timed region): sampled outputs of the step's own
# buckets, produced by the same library calls, kernels and communicator as the
# step, against the CPU oracle computing those elements.  With the CPU
# baseline this is the only part of bench.py that calls oracle/; the product
# path never does.

def sample_local_rows(c, seed, n=6):
    """Deterministic local row indices in [0, c): the first and last row of
    a chunk plus n - 2 seeded ones (same on every rank)."""
    import numpy as np
    if c <= n:
        return list(range(c))
    rng = np.random.Generator(np.random.Philox(seed))
    mid = sorted(set(int(x) for x in rng.integers(1, c - 1, size=n - 2)))
    return sorted(set([0, c - 1] + mid))


def sample_buckets(n):
    return sorted({0, 1, n // 2, n - 2, n - 1} & set(range(n)))


def expected_ag_rows(d, world, rows, shard_rows_by_rank):
    """Oracle O2 / O4 one element at a time: global row g of the gathered
    parameter = local row g - row_begin_q of the shard of its owner q.
    shard_rows_by_rank[q][t] = rank q's shard row t (bytes).  Returns
    {g: bytes}."""
    from oracle.shard import shard_rows
    out = {}
    for g in rows:
        for q in range(world):
            _, begin, v = shard_rows(d, world, q)
            if begin <= g < begin + v:
                out[g] = shard_rows_by_rank[q][g - begin]
                break
    return out


def expected_rs_rows(d, R, world, rank, local_rows, grad_rows_by_rank):
    """Oracle O5 on the sampled elements: rank `rank`'s gradient-shard rows
    `local_rows` = the rank-order fp32 sum of fl32(widen(g_q) x fl32(1/N))
    over q.  grad_rows_by_rank[q][g] = rank q's bf16 full-gradient row g
    (uint16 [R]).  Built as a small bucket whose chunk of every rank holds the
    sampled rows of that rank's chunk, then oracle.bucketed_reduce_scatter.
    Returns (expected fp32 [n, R], abs-sum scale fp64 [n, R]) for the valid rows."""
    import numpy as np
    from oracle.collectives import bucketed_reduce_scatter, inv_world_f32
    from oracle import bf16 as OB
    c = -(-d // world)
    n = len(local_rows)
    fakes = []
    for q in range(world):
        f = np.zeros((world * n, R), dtype=np.uint16)
        for rp in range(world):
            for i, t in enumerate(local_rows):
                g = rp * c + t
                if g < d:
                    f[rp * n + i] = grad_rows_by_rank[q][g]
        fakes.append([f])
    _, _, shards = bucketed_reduce_scatter(fakes, world, 16)
    exp = shards[rank][0]
    inv = float(inv_world_f32(world))
    scale = np.zeros((n, R), dtype=np.float64)
    for q in range(world):
        scale += np.abs(OB.widen(fakes[q][0][rank * n:(rank + 1) * n]).astype(np.float64)) * inv
    return exp, scale


def rs_tolerance(world, scale):
    """G7: |gpu - oracle| <= 1.01 N 2^-24 sum_r |g_r| / N, element-wise."""
    return 1.01 * world * 2.0 ** -24 * scale


def ag_check(world, rank, members, exchange, acc):
    """Host side of the AG check for one bucket.  members: list of dicts
    {key, d, ep, own: {t: bytes of this rank's shard row t}, got: {g: bytes of
    the gathered row g}}.  Exchanges the shard rows over the host process
    group, compares every gathered row with expected_ag_rows bit for bit and
    adds to acc (elements, mismatches)."""
    allown = exchange({m["key"]: m["own"] for m in members})
    for m in members:
        exp = expected_ag_rows(m["d"], world, sorted(m["got"]), [allown[q][m["key"]] for q in range(world)])
        for g, b in m["got"].items():
            acc["elements"] += len(b) // m["ep"]
            if exp.get(g) != b:
                acc["mismatches"] += 1


def rs_check(world, rank, members, exchange, acc):
    """Host side of the RS check for one bucket.  members: list of dicts {key,
    d, R, loc (sampled local rows), own (those valid on this rank), grads: {g:
    uint16 [R] full-gradient row g of this rank}, got: fp32 [len(own), R] this
    rank's gradient-shard rows}.  Exchanges the gradient rows, computes the
    oracle's rows (expected_rs_rows) and adds to acc (elements, bit mismatches,
    max error / G7 bound)."""
    import numpy as np
    allg = exchange({m["key"]: m["grads"] for m in members})
    for m in members:
        if not m["own"]:
            continue
        exp, scale = expected_rs_rows(m["d"], m["R"], world, rank, m["loc"], [allg[q][m["key"]] for q in range(world)])
        sel = [m["loc"].index(t) for t in m["own"]]
        exp, scale, got = exp[sel], scale[sel], m["got"]
        err = np.abs(got.astype(np.float64) - exp.astype(np.float64))
        tol = rs_tolerance(world, scale)
        acc["elements"] += got.size
        acc["mismatches"] += int(np.count_nonzero(got.view(np.uint32) != exp.view(np.uint32)))
        if got.size:
            acc["max_err_over_bound"] = max(acc["max_err_over_bound"], float(np.max(err / np.maximum(tol, 1e-300))))


def parity_verdict(ag, rs, world, p2p):
    """AG must be bit-exact; the RS bit-exact where the summation order cannot
    matter or is the oracle's (K9 sums in rank order; N <= 2 is one
    commutative add), else within G7's bound."""
    exact_required = p2p or world <= 2
    rs_ok = rs["mismatches"] == 0 if exact_required else rs["max_err_over_bound"] <= 1.0
    ok = ag["mismatches"] == 0 and ag["elements"] > 0 and rs_ok and rs["elements"] > 0
    return bool(ok), ("bit-exact" if exact_required else "G7 bound 1.01 N 2^-24 sum|g|/N")


def parity_leg(st, ctx, cs, ms, p2p, world, rank, exchange, barrier):
    import numpy as np
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    ep = st.ep
    pdt = np.uint16 if ep == 2 else np.uint32

    def rows_of(buf, off, rows, row_bytes, dtype):
        if not rows:
            return np.zeros((0, row_bytes // np.dtype(dtype).itemsize), dtype=dtype)
        idx = torch.tensor(rows, dtype=torch.int64, device=buf.device)
        t = buf[off:off + (max(rows) + 1) * row_bytes].view(-1, row_bytes).index_select(0, idx)
        return t.cpu().numpy().view(dtype)

    ag = {"buckets": [], "elements": 0, "mismatches": 0}
    for k in sample_buckets(len(st.fwd)):
        bk = st.fwd[k]
        barrier()
        if p2p:
            F.p2p_allgather_bucket(ctx, bk, st.ag_peers[k], cs)
        else:
            F.allgather_bucket(ctx, bk, st.ag_st[k % 2].data_ptr(), cs, ms, L.ISSUE | L.WAIT)
        torch.cuda.synchronize()
        slot = st.full_slots[bk.full_slot]
        members = []
        for j, foff in zip(bk.members, bk.full_offs):
            d, R = st.specs[j].dim0, st.specs[j].row_numel
            c = -(-d // world)
            loc = sample_local_rows(c, 1000 + j)
            grows = sorted({q * c + t for q in range(world) for t in loc if q * c + t < d})
            own = [t for t in loc if rank * c + t < d]
            sh = rows_of(st.shard_buf, st.shard_offs[j], own, R * ep, pdt)
            fr = rows_of(slot, foff, grows, R * ep, pdt)
            members.append({"key": j, "d": d, "ep": ep, "own": {t: sh[i].tobytes() for i, t in enumerate(own)},
                            "got": {g: fr[i].tobytes() for i, g in enumerate(grows)}})
        ag_check(world, rank, members, exchange, ag)
        ag["buckets"].append(k)
    rs = {"buckets": [], "elements": 0, "max_err_over_bound": 0.0, "mismatches": 0, "pad_rows": 0, "pad_nonzero": 0}
    for b in sample_buckets(len(st.bwd)):
        bk = st.bwd[b]
        barrier()
        if p2p:
            F.p2p_reduce_scatter_bucket(ctx, bk, st.rs_peers[b], cs)
        else:
            F.reduce_scatter_bucket(ctx, bk, st.rs_st[b % 2].data_ptr(), cs, ms, L.ISSUE | L.WAIT)
        torch.cuda.synchronize()
        gslot = st.grad_slots[bk.grad_slot]
        members = []
        for j, goff in zip(bk.members, bk.grad_offs):
            d, R = st.specs[j].dim0, st.specs[j].row_numel
            c = -(-d // world)
            loc = sample_local_rows(c, 2000 + j)
            grows = sorted({q * c + t for q in range(world) for t in loc if q * c + t < d})
            gr = rows_of(gslot, goff, grows, R * 2, np.uint16)
            own = [t for t in loc if rank * c + t < d]
            members.append({"key": j, "d": d, "R": R, "loc": loc, "own": own,
                            "grads": {g: gr[i].copy() for i, g in enumerate(grows)},
                            "got": rows_of(st.gshard_buf, st.gs_offs[j], own, R * 4, np.float32)})
            # pad rows of this rank's gradient shard (uneven dim 0) are exactly +0.0 (O5)
            pads = [t for t in range(c) if rank * c + t >= d]
            if pads:
                pr = rows_of(st.gshard_buf, st.gs_offs[j], pads, R * 4, np.uint32)
                rs["pad_rows"] += len(pads)
                rs["pad_nonzero"] += int(np.count_nonzero(pr))
        rs_check(world, rank, members, exchange, rs)
        rs["buckets"].append(b)
    barrier()
    ok, required = parity_verdict(ag, rs, world, p2p)
    ok = ok and rs["pad_nonzero"] == 0
    # every rank checked its own outputs: the verdict is all of them
    allr = exchange((ok, ag, rs))
    ok = all(x[0] for x in allr)
    ag = dict(ag, elements=sum(x[1]["elements"] for x in allr), mismatches=sum(x[1]["mismatches"] for x in allr))
    rs = dict(rs, elements=sum(x[2]["elements"] for x in allr), mismatches=sum(x[2]["mismatches"] for x in allr),
              max_err_over_bound=max(x[2]["max_err_over_bound"] for x in allr),
              pad_rows=sum(x[2]["pad_rows"] for x in allr), pad_nonzero=sum(x[2]["pad_nonzero"] for x in allr))
    return {"ok": ok, "ranks_checked": len(allr), "ag": dict(ag, bit_exact=ag["mismatches"] == 0),
            "rs": dict(rs, bit_exact=rs["mismatches"] == 0, required=required),
            "how": ("sampled rows (first / last / seeded) of every member of buckets %s (fwd AG) / %s (bwd RS) of "
                    "the bench's own state, run through the same calls and communicator as the step, compared "
                    "with the CPU oracle (O2/O4 AG, O5 RS) on inputs exchanged over the host process group"
                    % (ag["buckets"], rs["buckets"]))}


# ------------------------------------------------------------ NCCL INFO log
def nccl_log_path(rank):
    return "/tmp/fsdp_bench_nccl.%d.%d.log" % (os.getpid(), rank)


def nccl_info_summary(path, limit=24):
    """The communicator's own account of itself (NCCL_DEBUG=INFO): version,
    ranks / channels, NVLS and P2P transport, tuning choices."""
    keys = ("NCCL version", "nRanks", "NVLS", "nvls", "Channel 00", "channels", "P2P/", "via P2P", "CollNet",
            "Init COMPLETE", "algorithm", "Algo", "proto", "NCCL_")
    try:
        with open(path, errors="ignore") as f:
            lines = [ln.rstrip() for ln in f]
    except OSError:
        return {"lines": [], "note": "no NCCL log (NCCL_DEBUG set by the caller?)"}
    pick = [ln for ln in lines if any(k in ln for k in keys)]
    nvls = [ln for ln in lines if "NVLS" in ln or "nvls" in ln]
    return {"lines": pick[:limit], "n_lines": len(lines), "nvls_lines": nvls[:6],
            "nvls_mentioned": bool(nvls), "file": path}


# ------------------------------------------------------------------ helpers
def fused_leg(args):
    """bench.py --collective p2p at N = 1 on the same workload (child process):
    K8 / K9 against 7 simulated peers' buffers in local HBM."""
    cmd = [sys.executable, os.path.abspath(__file__), "--collective", "p2p", "--steps", str(args.steps),
           "--warmup", str(args.warmup), "--no-e2e", "--no-cpu-baseline", "--no-fused-leg", "--predict-tokens", "0",
           "--plan", args.plan, "--model", args.model, "--sim-world", str(args.sim_world)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    except Exception as e:  # reported, never fatal to the headline
        return {"error": "%s: %s" % (type(e).__name__, str(e)[:200])}
    return {"ms_per_step": d["ms_per_step"], "value": d["value"], "unit": d["unit"], "value_kind": d["value_kind"],
            "kernels": d["kernels"], "roofline": d["roofline"], "gpu_launches": d["gpu_launches"],
            "how": "bench.py --collective p2p (same workload, own process; the 7 peers simulated in local HBM)"}


def kernel_table(st, ctx, names, kbytes, klaunch, op_ns, steps, cs_stream, peak, p2p=False):
    """Per data kernel: (a) in-step, event-timed -- an event pair around every
    launch in the profiled steps (FSDP_SCHED_TIMING), which also counts each
    launch's event / launch latency (~8 us per launch, tools/
    launch_overhead_probe.py); (b) back to back -- this step's launches of
    that kernel alone (fsdp_bucket_launch_kernel, same tables, staging slots
    and order), captured into one CUDA graph, timed with CUDA events around
    three replays on the launching stream.  Peer-memory path: (a) covers the RS op,
    i.e. K9 with the epoch wait / signal kernels around it; (b) K8 / K9 alone
    (fsdp_p2p_*_bucket, same tables and peer rows)."""
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    out = {}
    for op in kbytes:
        if kbytes[op] <= 0 or op_ns.get(op, 0) <= 0:
            continue
        ev_gbs = kbytes[op] * steps / (op_ns[op] * 1e-9) / 1e9
        row = {"GB/s_in_step_event": round(ev_gbs, 1), "frac_in_step_event": round(ev_gbs / peak, 4),
               "ms_per_step_in_step_event": round(op_ns[op] / steps / 1e6, 3),
               "launches_per_step": klaunch[op], "bytes_per_step": kbytes[op]}
        seq = []
        if p2p:
            # K8 / K9 alone (fsdp_p2p_*_bucket: the same tables and peer rows as
            # the step, without its epoch wait / signal kernels)
            if op == L.OP_AG:
                seq = [("ag", bk, st.ag_peers[i]) for i, bk in enumerate(st.fwd + st.bwd)]
            else:
                seq = [("rs", bk, st.rs_peers[i]) for i, bk in enumerate(st.bwd)]
        elif op in (L.OP_PACK_AG, L.OP_UNPACK):
            seq = [(bk, st.ag_st[b % 2]) for bs in (st.fwd, st.bwd) for b, bk in enumerate(bs)]
        elif op in (L.OP_PACK_RS, L.OP_COPYOUT_RS):
            seq = [(bk, st.rs_st[b % 2]) for b, bk in enumerate(st.bwd)]
        try:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            n = 0
            with torch.cuda.graph(g, stream=s):
                for item in seq:
                    if p2p:
                        kind, bk, peers = item
                        (F.p2p_allgather_bucket if kind == "ag" else F.p2p_reduce_scatter_bucket)(
                            ctx, bk, peers, s.cuda_stream)
                        n += 1
                    else:
                        bk, stg = item
                        n += F.bucket_launch_kernel(ctx, bk, op, stg.data_ptr(), s.cuda_stream)
            with torch.cuda.stream(s):
                g.replay()
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                for _ in range(3):
                    g.replay()
            b.record(s)
            b.synchronize()
            ms_b2b = a.elapsed_time(b) / 3
            gbs = kbytes[op] / (ms_b2b * 1e-3) / 1e9
            row.update({"GB/s": round(gbs, 1), "frac": round(gbs / peak, 4), "ms_per_step": round(ms_b2b, 3),
                        "launches_back_to_back": n})
            del g
        except Exception as e:   # reported, never fatal
            row["back_to_back_error"] = str(e)[:200]
        out[names[op]] = row
    return out


# -------------------------------------------------------------------- ours
def main(argv=None):
    args = parse(argv)
    rank = int(os.environ.get("RANK", "0"))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    multi = args.gpus > 1 or args.dist
    p2p = args.collective == "p2p"
    quick = args.quick
    if multi and not p2p:
        # the communicator's own account (version, channels, NVLS, tuning), one file per rank
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS,ENV")   # init-time only: nothing per call
        if "NCCL_DEBUG_FILE" not in os.environ:
            os.environ["NCCL_DEBUG_FILE"] = nccl_log_path(rank)

    import torch
    import torch.distributed as dist

    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads import llama
    from workloads.compute_model import per_param_compute_ns

    assert torch.cuda.is_available(), "bench.py needs a B200"
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    if multi:
        assert world_env == args.gpus, "launch with torchrun --nproc-per-node %d" % args.gpus
        dist.init_process_group("gloo")      # host plumbing only; the data path is the library's
        world = args.gpus
        if p2p and args.p2p_transport == "ipc":
            ctx = F.Ctx(world, rank, local)  # peer-memory collectives need no NCCL communicator
        else:   # NCCL collectives, or NCCL symmetric windows for the peer-memory path
            uid = [F.nccl_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            cfg = dict(max_ctas=args.nccl_max_ctas) if args.nccl_max_ctas > 0 else None
            ctx = F.Ctx(world, rank, local, nccl_uid=uid[0], nccl_config=cfg)
    else:
        world = args.sim_world
        ctx = F.Ctx(world, 0, local)   # layout-only: rank 0 of a simulated `world`-way job
    my_rank = rank if multi else 0

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def barrier():
        torch.cuda.synchronize()
        if multi:
            dist.barrier()

    def max_over_ranks(x):
        if not multi:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    tokens = args.tokens
    specs = llama(args.model, n_layers=args.layers)
    t_fwd, t_bwd = per_param_compute_ns(specs, tokens) if tokens else ([0] * len(specs), [0] * len(specs))
    mode = {"manual": L.PLAN_MANUAL, "greedy": L.PLAN_GREEDY, "per_param": L.PLAN_PER_PARAM,
            "size_cap": L.PLAN_SIZE_CAP, "search": L.PLAN_GREEDY}[args.plan]
    link = (args.alpha_ns, args.beta_fs)
    fplan, bplan = H.plans_for(specs, world, mode, t_fwd, t_bwd, link, link, int(args.mem_limit))
    if args.plan == "search":
        sf, sb = per_param_compute_ns(specs, tokens or 1024)
        fplan, bplan = H.plans_search(specs, world, sf, sb, link, link, int(args.mem_limit))
    if args.plan_file:
        with open(args.plan_file) as f:
            pj = json.load(f)["plans"]
        fplan, bplan = pj["fwd"], pj["bwd"]
        assert sorted(j for b in fplan for j in b) == sorted(j for b in bplan for j in b) == list(range(len(specs)))
    if p2p and not H.same_buckets(fplan, bplan):
        bplan = H.mirror_plan(fplan)     # one shard layout for both phases (peer-memory path)
    reg = args.nccl_register if (multi and not p2p and args.nccl_register != "none") else None
    win = multi and p2p and args.p2p_transport == "window"
    st = H.RankState(specs, world, my_rank, fplan, bplan, ctx, seed=1234 + my_rank, ipc=multi and p2p and not win,
                     nccl_register=reg, ag_grouped=args.ag == "grouped", grad_slots=args.grad_slots, windows=win)
    compute = torch.cuda.Stream()
    comm = torch.cuda.Stream(priority=-1)
    cs, ms = compute.cuda_stream, comm.cuda_stream

    pf = pb = None
    if tokens and args.compute == "proxy":
        nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
        pf = H.proxy_iters(H.bucket_times(fplan, t_fwd), nspi)
        pb = H.proxy_iters(H.bucket_times(bplan, t_bwd), nspi)
    if p2p:
        if multi:
            if win:
                st.setup_p2p_windows()
            else:
                st.setup_p2p_ipc(exchange)
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
    if args.copy_stream and not p2p:
        flags |= L.SCHED_COPY_STREAM

    gemm = model = None
    if args.compute == "llama":
        from paper_2411_00284_b200.llama_compute import LlamaCompute
        model = LlamaCompute(st, tokens or 1024)
    if args.compute == "gemm":
        gemm = st.setup_gemm(tokens or 1024)
    hook = model.hook if model else None

    def step(extra=0):
        return st.step(flags | extra, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm, hook=hook)

    host_enqueue = []

    def timed_loop(extra, n):
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
    # (1) the headline: K plain steps, each replayed as one CUDA graph
    #     (fsdp_step_graph: kernels + collectives + cross-stream events captured
    #     once) unless --eager; the eager enqueue of the same steps beside it
    sg = None
    if not args.eager and model is None:
        sg = st.capture(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm)
    elif not args.eager:
        tg = st.capture_with_torch(flags, compute, ms, pf, pb, args.proxy_ctas, args.proxy_smem, gemm=gemm,
                                   hook=hook)

        class _TorchGraph:
            def launch(self, stream):
                with torch.cuda.stream(compute):
                    tg.replay()

            def close(self):
                pass
        sg = _TorchGraph()
    if sg is not None:
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
        ms_step = graph_loop(args.steps) if sg is not None else timed_loop(0, args.steps)[0]
    st.check_p2p()
    ms_eager = timed_loop(0, args.steps)[0] if sg is not None else ms_step
    # (2) the same K steps with an event pair around every op (per-op device
    #     time on the launching stream; synchronises once per step)
    ms_prof, reports = timed_loop(L.SCHED_TIMING, args.steps)
    if args.trace:
        rep_t = st.step(flags | L.SCHED_TIMING, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, want_log=True,
                        gemm=gemm, hook=hook)
        if rank == 0:
            H.chrome_trace(rep_t["log"], args.trace)
    # (3) compute-stream-only baseline: same ops, no collective, no wait
    step(L.SCHED_NO_COMM)
    ms_compute, _ = timed_loop(L.SCHED_NO_COMM, args.steps)
    st.check_p2p()
    if sg is not None:
        sg.close()

    # ---- headline value
    ag_b, rs_b = st.step_bytes()
    op_ns = {i: sum(r["op_ns"][i] for r in reports) for i in range(L.N_OPS)}
    if p2p:
        k8, k9 = st.p2p_bytes()
        kbytes = {L.OP_AG: k8, L.OP_RS: k9}
        klaunch = {L.OP_AG: len(st.fwd) + len(st.bwd), L.OP_RS: len(st.bwd)}
        names = {L.OP_AG: "fsdp_p2p_allgather_kernel", L.OP_RS: "fsdp_p2p_reduce_scatter_kernel"}
        wire_rs = rs_b // 2      # K9 pulls the bf16 gradients: half the fp32 RS bytes
    else:
        kbytes, klaunch = st.kernel_bytes(), st.kernel_launches()
        names = {L.OP_PACK_AG: "fsdp_ag_pack_kernel", L.OP_UNPACK: "fsdp_ag_unpack_kernel",
                 L.OP_PACK_RS: "fsdp_rs_pack_kernel", L.OP_COPYOUT_RS: "fsdp_rs_copyout_kernel"}
        wire_rs = rs_b
    hbm_bytes = sum(kbytes.values())
    bus_world = world if multi else 1
    bus_bytes_rank = (bus_world - 1) / bus_world * (ag_b + wire_rs)
    if bus_world > 1:
        value = bus_world * bus_bytes_rank / (ms_step * 1e-3) / 1e9
        value_kind = "bus"
        value_def = ("whole-job bus GB/s: N x (N-1)/N x full bucket bytes of the step's collectives (fwd AG + bwd AG "
                     "bf16, RS %s) / step time (nccl-tests busbw convention, G28, summed over ranks)"
                     % ("bf16 gradients pulled by K9" if p2p else "fp32"))
    else:
        value = hbm_bytes / (ms_step * 1e-3) / 1e9
        value_kind = "hbm"
        value_def = ("N = 1 has no peers and no bus: algorithmic HBM bytes of the step's data kernels (%s) / step "
                     "time, rank 0 of a simulated %d-way job" % (", ".join(names[o] for o in kbytes if kbytes[o]),
                                                                world))

    # ---- per-kernel table and the roofline of the dominant kernel
    peak, peak_src = measured_peak_hbm()
    live = [op for op in kbytes if kbytes[op] > 0 and op_ns.get(op, 0) > 0]
    dom = max(live, key=lambda op: op_ns[op])
    achieved = kbytes[dom] * args.steps / (op_ns[dom] * 1e-9) / 1e9
    barrier()
    per_kernel = kernel_table(st, ctx, names, kbytes, klaunch, op_ns, args.steps, cs, peak, p2p=p2p)
    barrier()
    launches = sum(r["kernel_launches"] for r in reports)
    coll_ms = None
    busbw_step = None
    if multi or p2p:
        coll_ms = {"ag_ms_per_step": round(op_ns[L.OP_AG] / args.steps / 1e6, 3),
                   "rs_ms_per_step": round(op_ns[L.OP_RS] / args.steps / 1e6, 3)}
    if multi and world > 1 and op_ns[L.OP_AG] > 0:
        # the step's collectives alone (event pairs on the comm stream), per GPU
        busbw_step = {"ag": round((world - 1) / world * ag_b * args.steps / (op_ns[L.OP_AG] * 1e-9) / 1e9, 1),
                      "rs": round((world - 1) / world * wire_rs * args.steps / (op_ns[L.OP_RS] * 1e-9) / 1e9, 1),
                      "nvlink_GBps": NVLINK_GBS,
                      "how": "(N-1)/N x full bytes / comm-stream event time of the step's AG / RS, per GPU"}

    # ---- N > 1 verification: sampled oracle parity on the step's own buckets
    parity = None
    if multi and not quick and not args.no_parity and args.compute == "proxy":
        parity = parity_leg(st, ctx, cs, ms, p2p, world, my_rank, exchange, barrier)
        st.check_p2p()

    # ---- e2e through the public call with HOST buffers
    e2e = None
    if not args.no_e2e:
        h_sh = torch.empty(st.shard_buf.numel(), dtype=torch.uint8, pin_memory=True)
        h_gs = torch.empty(st.gshard_buf.numel(), dtype=torch.uint8, pin_memory=True)
        h_sh.copy_(st.shard_buf)
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        # async_d2h: a step's gradient D2H overlaps the next step (each bucket's
        # next gradient writer waits for its own D2H; tools/e2e_probe.py: 83 vs
        # 87 ms per step); the timed region ends when the last step's gradients
        # are on the host (an event on the d2h stream)
        io = st.host_io(h_sh, h_gs, h2d_s.cuda_stream, d2h_s.cuda_stream, async_d2h=not p2p)
        h2d_bytes = sum(b.ag_seg for b, p in zip(st.fwd, io["fwd_host_shards"]) if p)
        d2h_bytes = sum(b.rs_seg for b, p in zip(st.bwd, io["bwd_host_grads"]) if p)
        st.step(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, io=io, gemm=gemm, hook=hook)   # warm-up
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xc = torch.cuda.Event()
        x0.record(compute)
        for _ in range(args.e2e_steps):
            st.step(flags, cs, ms, pf, pb, args.proxy_ctas, args.proxy_smem, io=io, gemm=gemm, hook=hook)
        xc.record(compute)
        d2h_s.wait_event(xc)        # after the device work and every gradient D2H
        x1.record(d2h_s)
        barrier()
        st.check_p2p()
        e2e_ms = max_over_ranks(x0.elapsed_time(x1) / args.e2e_steps)
        e2e_val = (bus_world * bus_bytes_rank if bus_world > 1 else hbm_bytes) / (e2e_ms * 1e-3) / 1e9
        e2e = {"value": round(e2e_val, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h_bytes),
               "how": "fsdp_run_schedule with fsdp_host_io: per-bucket H2D of shards / D2H of fp32 grad shards "
                      "from / to pinned host memory inside the call, overlapped with the device path and (async_d2h; "
                      "PCIe floor of these bytes ~76 ms, tools/pcie_probe.py) with the neighbouring steps; timed "
                      "from the first step's start on the compute stream to the last step's gradients on the host; "
                      "value defined as the headline's (%s)" % value_kind}
        del h_sh, h_gs

    zero_copy = st.zero_copy()
    n_fwd, n_bwd = len(fplan), len(bplan)

    # ---- N = 1: the modelled N-rank step (assumed links; labelled a model)
    predicted = None
    if not multi and not p2p and not quick and args.predict_tokens and args.compute == "proxy":
        plink = (ASSUMED_LINK[0], round((world - 1) / world / 720e9 * 1e15))
        ptf, ptb = per_param_compute_ns(specs, args.predict_tokens)
        nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
        ppf = H.proxy_iters(H.bucket_times(fplan, ptf), nspi)
        ppb = H.proxy_iters(H.bucket_times(bplan, ptb), nspi)
        tot, exp = H.predict_exposure(st, flags, cs, ms, ppf, ppb, plink, plink, args.proxy_ctas, args.proxy_smem)
        predicted = {"kind": "MODEL, not a measurement: this rank's measured compute-stream ops + ASSUMED links "
                             "(alpha 20 us, 720 GB/s busbw = 80 % of NVLink 5), no contention",
                     "world": world, "tokens_per_gpu": args.predict_tokens, "link_alpha_ns": plink[0],
                     "link_beta_fs_per_byte": plink[1], "total_ms": round(tot / 1e6, 3),
                     "exposed_ms": round(exp / 1e6, 3)}
        mp, pools = H.predict_memory(st, flags)
        predicted["memory_model_peak_GiB"] = round(mp / 2 ** 30, 3)
        if not args.no_variants:
            variants = {}
            RF = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
            for name, vmode, vflags in (("vanilla (per-param, no reorder)", L.PLAN_PER_PARAM, 0),
                                        ("greedy + reorder (assumed links)", L.PLAN_GREEDY, RF)):
                vf, vb = H.plans_for(specs, world, vmode, ptf, ptb, plink, plink, int(args.mem_limit))
                vst = H.RankState(specs, world, 0, vf, vb, ctx, seed=99)
                vpf = H.proxy_iters(H.bucket_times(vf, ptf), nspi)
                vpb = H.proxy_iters(H.bucket_times(vb, ptb), nspi)
                vst.step(vflags, cs, ms, vpf, vpb, args.proxy_ctas, args.proxy_smem)   # warm-up
                vt, ve = H.predict_exposure(vst, vflags, cs, ms, vpf, vpb, plink, plink, args.proxy_ctas,
                                            args.proxy_smem)
                variants[name] = {"buckets_fwd": len(vf), "buckets_bwd": len(vb), "total_ms": round(vt / 1e6, 3),
                                  "exposed_ms": round(ve / 1e6, 3)}
                del vst
                gc.collect()
                torch.cuda.empty_cache()
            variants["per-block + reorder [this run's plan]"] = {"buckets_fwd": n_fwd, "buckets_bwd": n_bwd,
                                                                "total_ms": predicted["total_ms"],
                                                                "exposed_ms": predicted["exposed_ms"]}
            predicted["variants"] = variants

    emulated = None
    if not multi and not quick and args.emulate and args.compute == "proxy":
        elink = (ASSUMED_LINK[0], round((world - 1) / world / 720e9 * 1e15))
        ptf, ptb = per_param_compute_ns(specs, args.predict_tokens or 1024)
        nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
        epf = H.proxy_iters(H.bucket_times(fplan, ptf), nspi)
        epb = H.proxy_iters(H.bucket_times(bplan, ptb), nspi)
        em = dict(ag=elink, rs=elink, ctas=H.emulation_ctas_p2p(world) if p2p else 64)

        def em_loop(extra, emulate, n):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(compute)
            for _ in range(n):
                st.step(flags | extra, cs, ms, epf, epb, args.proxy_ctas, args.proxy_smem, emulate=emulate)
            b.record(compute)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n
        em_loop(0, em, 1)
        es, ec = em_loop(0, em, args.steps), em_loop(L.SCHED_NO_COMM, None, args.steps)
        emulated = {"kind": "MODEL DEVICE, not a multi-GPU measurement: collectives emulated on one GPU (K11 / "
                            "paced K8-K9) at ASSUMED links (720 GB/s busbw, 20 us)",
                    "world": world, "step_ms": round(es, 3), "compute_only_ms": round(ec, 3),
                    "exposed_ms": round(es - ec, 3)}

    # free the headline state before the N > 1 sweeps / variants
    st.check_p2p()
    if p2p and multi:
        barrier()
        st.close_ipc()
        barrier()                    # every rank closed its mappings of ours
        st.free_ipc()
    st.close_nccl_mem()
    del st
    gc.collect()
    torch.cuda.empty_cache()

    # ---- N > 1: isolated 8B-block busbw, alpha / beta fit, measured exposure
    busbw_block = alpha_beta = exposure = nvls_block = None
    if multi and (world > 1 or args.n_rank_legs_at_world1) and not quick:
        from workloads.shapes import ParamSpec
        kw = dict(p2p=p2p, exchange=exchange, max_over_ranks=max_over_ranks, windows=args.p2p_transport == "window")
        block = [p for p in llama("8b", n_layers=1, with_embeddings=False)]
        barrier()
        r = H.time_bucket_collectives(block, world, my_rank, ctx, cs, ms, reps=20, warmup=5, **kw)
        wire_rs_block = r["rs_bytes"] // 2 if p2p else r["rs_bytes"]
        bb_ag = (world - 1) / world * r["ag_bytes"] / r["ag_ns"]
        bb_rs = (world - 1) / world * wire_rs_block / r["rs_ns"]
        busbw_block = {"ag_GBps": round(bb_ag, 1), "rs_GBps": round(bb_rs, 1),
                       "ag_frac_nvlink": round(bb_ag / NVLINK_GBS, 4), "rs_frac_nvlink": round(bb_rs / NVLINK_GBS, 4),
                       "ag_frac_measured_peer": round(bb_ag / NVLINK_MEASURED_GBS, 4),
                       "rs_frac_measured_peer": round(bb_rs / NVLINK_MEASURED_GBS, 4),
                       "peer_reference_GBps": NVLINK_MEASURED_GBS,
                       "ag_ms": round(r["ag_ns"] / 1e6, 4), "rs_ms": round(r["rs_ns"] / 1e6, 4),
                       "ag_full_bytes": r["ag_bytes"], "rs_full_bytes": r["rs_bytes"],
                       "rs_wire_dtype": "bf16 (K9 pulls the gradients)" if p2p else "fp32",
                       "target_GBps": 0.8 * NVLINK_GBS,
                       "how": "one Llama-3-8B transformer block as one bucket, alone; median of 20 after 5 warm-up, "
                              "CUDA events around the collective on the comm stream, max over ranks; busbw = "
                              "(N-1)/N x full bytes / t (nccl-tests)"}
        if not args.no_sweep:
            rows = []
            for n in [2 ** 13, 2 ** 16, 2 ** 19, 2 ** 22, 2 ** 25, 2 ** 26, 2 ** 27, 2 ** 28, 2 ** 29, 2 ** 30]:
                d = max(world, (n // 2048) // world * world)
                barrier()
                rows.append(H.time_bucket_collectives([ParamSpec("x", d, 1024, 0)], world, my_rank, ctx, cs, ms,
                                                      reps=10, warmup=3, **kw))
            fa, fr = H.fit_link(rows, "ag_bytes", "ag_ns"), H.fit_link(rows, "rs_bytes", "rs_ns")
            alpha_beta = {"ag": {"alpha_ns": fa[0], "beta_fs_per_byte": fa[1]},
                          "rs": {"alpha_ns": fr[0], "beta_fs_per_byte": fr[1]},
                          "source": "measured at this N (fit: alpha = t at 8 KiB; beta = least-squares slope over "
                                    "n >= 64 MiB; n = full bucket bytes, bf16 AG / fp32 RS, G8)",
                          "rows": [{k: (round(v, 1) if isinstance(v, float) else v) for k, v in x.items()}
                                   for x in rows]}
        if args.exposure_tokens:
            exposure = exposure_leg(args, specs, world, my_rank, ctx, cs, ms, compute, p2p, exchange, barrier,
                                    max_over_ranks, alpha_beta)
        nvls_block = nvls_leg(world, my_rank, ctx, exchange, barrier, max_over_ranks)
    elif not multi:
        alpha_beta = {"ag": {"alpha_ns": args.alpha_ns, "beta_fs_per_byte": args.beta_fs},
                      "rs": {"alpha_ns": args.alpha_ns, "beta_fs_per_byte": args.beta_fs},
                      "source": "assumed (N = 1: no collective to measure)"}

    nccl_info = None
    if multi and not p2p and rank == 0 and os.environ.get("NCCL_DEBUG_FILE") == nccl_log_path(rank):
        nccl_info = nccl_info_summary(nccl_log_path(rank))

    cpu = None
    if rank == 0 and not multi and not args.no_cpu_baseline and not quick:
        sample = CpuOracleSample(world, "hbm")
        runs = []
        while sum(r_[1] for r_ in runs) < 10.0:     # ~10 s of timed oracle work
            runs.append(sample.run())
        dt = sum(r_[1] for r_ in runs)
        cpu = {"value": round(len(runs) * sample.bytes / dt / 1e9, 3), "unit": "GB/s", "cores": 1,
               "kind": "oracle", "sample": sample.desc + "; %d repetitions" % len(runs), "seconds": round(dt, 2),
               "host_cpus": os.cpu_count()}

    fused = None
    if rank == 0 and not multi and not p2p and not args.no_fused_leg and not quick and args.compute == "proxy":
        fused = fused_leg(args)

    workload = "llama3-%s FSDP rank step, %s plan, %s, %s" % (
        args.model, "file:" + os.path.basename(args.plan_file) if args.plan_file else args.plan,
        "reorder fwd-%s/bwd-%s" % (args.fwd_placement, args.bwd_placement) if not args.no_reorder else "vanilla order",
        "compute: none (the communication path alone)" if not tokens and args.compute == "proxy"
        else "compute: %s at %d tokens/GPU" % (args.compute, tokens or 1024))
    if not multi:
        workload += ", 1 GPU = rank 0 of a simulated %d-way job (%s)" % (
            world, "peers simulated in local HBM" if p2p else "pack/unpack only, no peers")
    else:
        workload += ", %d ranks over %s%s" % (world, "peer memory (CUDA IPC)" if p2p else "NCCL",
                                             " [TEST: one GPU]" if args.same_device else "")
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "value_kind": value_kind,
            "value_def": value_def, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded N(0, 0.02) bf16 params, N(0, 1e-3) bf16 grads)",
            "config": {
                "workload": workload,
                "shapes": "llama3-%s (Table 2; vocab 128256, 8 KV heads)" % args.model, "layout_world": world,
                "collective": ("NCCL all-gather / reduce-scatter with copy kernels" if not p2p else
                               "fused peer-memory kernels K8/K9"),
                "buckets_fwd": n_fwd, "buckets_bwd": n_bwd, "param_dtype": "bf16", "reduce_dtype": "fp32",
                "compute": args.compute if tokens or args.compute != "proxy" else "none",
                "tokens_per_gpu": tokens, "bus_bytes_per_rank_step": int(bus_bytes_rank),
                "full_bucket_bytes_per_rank_step": ag_b + rs_b, "hbm_algorithmic_bytes_per_step": hbm_bytes,
                "l2": "inputs > L2 (126 MB): every bucket but the 8 KB norms exceeds it",
                "parallelism": "fsdp%d" % world if multi else "fsdp1 (simulated %d)" % world,
                "nccl_register": reg or "none", "ag": args.ag},
            "exposed_comm_ms": round(ms_eager - ms_compute, 3), "compute_stream_ms": round(ms_compute, 3),
            "eager_ms_per_step": round(ms_eager, 3), "profiled_ms_per_step": round(ms_prof, 3),
            "timing": "eager enqueue" if sg is None else "CUDA-graph replay of the step",
            "host_enqueue_ms_per_step": (round(1e3 * sorted(host_enqueue)[len(host_enqueue) // 2], 3)
                                         if host_enqueue else None),
            "collectives": coll_ms, "busbw_step": busbw_step, "busbw_block": busbw_block,
            "alpha_beta": alpha_beta, "exposure": exposure, "parity": parity, "nccl_info": nccl_info,
            "nvls_block": nvls_block,
            "kernels": per_kernel,
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "achieved_how": "algorithmic bytes / in-step event-timed launch duration (conservative: "
                                         "includes each launch's event / launch latency)",
                         "traffic": ncu_traffic(names[dom]),
                         "traffic_launch_algorithmic_bytes": ncu_traffic(names[dom] + "_algorithmic"),
                         "algorithmic_bytes_per_launch": kbytes[dom] // max(1, klaunch[dom])},
            "zero_copy": zero_copy, "predicted": predicted, "emulated": emulated, "fused_p2p": fused,
            "peak_device_mem_GiB": round(torch.cuda.max_memory_allocated() / 2 ** 30, 2),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "p2p_wait_timeouts": 0 if p2p else None,
            "clocks": clk.summary(), "env": run_env(torch), "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if multi:
        dist.destroy_process_group()


def nvls_leg(world, rank, ctx, exchange, barrier, max_over_ranks, reps=20):
    """N > 1: the NVLS reduce-scatter read-out K10 on one Llama-3-8B block
    bucket: every rank packs its bf16 gradients (K4)
    into its unicast mapping of one multicast object over the N GPUs; after a
    barrier K10 reads this rank's segment through the multicast mapping (the
    NVSwitch sums the N copies) into the fp32 gradient shards.  K10 alone is
    timed with events (median of `reps`, max over ranks) -> busbw (N-1)/N x the
    fp32 bucket / t; the result is checked against the oracle on sampled rows
    (rs_check: G7 bound).  {"unavailable": why} where the platform refuses
    multicast objects."""
    import numpy as np
    import torch
    import paper_2411_00284_b200 as F
    from paper_2411_00284_b200 import _lib as L
    from workloads import llama
    specs = llama("8b", n_layers=1, with_embeddings=False)
    descs = [(p.dim0, p.row_numel, 0) for p in specs]
    g = torch.Generator(device="cuda").manual_seed(500 + rank)
    grads = [torch.empty(p.dim0 * p.row_numel, dtype=torch.bfloat16, device="cuda").normal_(0, 1e-3, generator=g)
             for p in specs]
    gsh = [torch.zeros(-(-p.dim0 // world) * p.row_numel, dtype=torch.float32, device="cuda") for p in specs]
    b = F.Bucket(ctx, descs, full_grads=[t.data_ptr() for t in grads], grad_shards=[t.data_ptr() for t in gsh],
                 param_dtype=L.BF16, grad_dtype=L.BF16)
    m, err, route, win_ptr = None, None, None, None

    def agree(local_err):
        """Every rank's error (or None) -> the first one, on every rank: the
        collective steps below stay in lockstep even when one rank fails."""
        errs = [e for e in exchange(local_err) if e]
        return errs[0] if errs else None

    # route 1: a multicast object of our own (cuMulticastCreate, fabric or
    # POSIX-fd handle exchanged by the binding)
    try:
        if rank == 0:
            m = F.Nvls(ctx, b.rs_seg)
    except Exception as e:
        err = "%s: %s" % (type(e).__name__, e)
    handle = exchange(m.handle if m is not None else None)[0]
    err = agree(err)
    if err is None and rank != 0:
        try:
            m = F.Nvls(ctx, b.rs_seg, handle=handle)
        except Exception as e:
            err = "%s: %s" % (type(e).__name__, e)
        err = agree(err)
    elif err is None:
        err = agree(None)
    uc = mc = None
    if err is None:
        barrier()                      # every GPU added before any binding
        try:
            uc, mc, _ = m.bind()
        except Exception as e:
            err = "%s: %s" % (type(e).__name__, e)
        err = agree(err)
    route = "cuMulticast object (fsdp_nvls_*)" if err is None else None
    # route 2 (needs a communicator): NCCL's own multicast mapping of a
    # symmetric window (fsdp_window_multimem_pointer, the NCCL device API)
    has_comm = exchange(bool(getattr(ctx, "has_nccl", False)))
    if err is not None and all(has_comm):
        first_err, err = err, None
        if m is not None:
            m.close()
            m = None
        try:
            win_ptr = F.mem_alloc(ctx, world * b.rs_seg)
        except Exception as e:
            err = "%s: %s" % (type(e).__name__, e)
        err = agree(err)
        if err is None:
            try:
                F.register_buffer(ctx, win_ptr, world * b.rs_seg, L.REG_SYMMETRIC)   # collective
            except Exception as e:
                err = "%s: %s" % (type(e).__name__, e)
            err = agree(err)
        if err is None:
            try:
                uc, mc = win_ptr, F.window_multimem_pointer(ctx, win_ptr)        # collective on first use
            except Exception as e:
                err = "%s: %s" % (type(e).__name__, e)
            err = agree(err)
        if err is None:
            route = "NCCL symmetric window (fsdp_window_multimem_pointer)"
        else:
            err = "own multicast object: %s; NCCL window: %s" % (first_err[:150], err[:150])
    t = None
    members = []
    if err is None:
        barrier()
        s = torch.cuda.Stream()
        try:
            F.reduce_scatter_bucket(ctx, b, uc, s.cuda_stream, 0, L.ISSUE | L.NO_COLLECTIVE)   # K4 into uc
            s.synchronize()
        except Exception as e:
            err = "%s: %s" % (type(e).__name__, e)
        err = agree(err)
    if err is None:
        barrier()                      # every rank packed
        try:
            ts = []
            for _ in range(reps + 3):
                a, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                F.nvls_reduce_scatter_bucket(ctx, b, mc, s.cuda_stream)
                e_.record(s)
                e_.synchronize()
                ts.append(a.elapsed_time(e_) * 1e6)
            t = float(np.median(ts[3:]))
            for j, p in enumerate(specs):
                d, R = p.dim0, p.row_numel
                c = -(-d // world)
                loc = sample_local_rows(c, 3000 + j)
                grows = sorted({q * c + t_ for q in range(world) for t_ in loc if q * c + t_ < d})
                gv = grads[j].view(torch.int16).view(d, R)
                gr = gv[torch.tensor(grows, device="cuda")].cpu().numpy().view(np.uint16)
                own = [t_ for t_ in loc if rank * c + t_ < d]
                got = (gsh[j].view(c, R)[torch.tensor(own, device="cuda")].cpu().numpy() if own
                       else np.zeros((0, R), np.float32))
                members.append({"key": j, "d": d, "R": R, "loc": loc, "own": own,
                                "grads": {g_: gr[i].copy() for i, g_ in enumerate(grows)}, "got": got})
        except Exception as e:
            err = "%s: %s" % (type(e).__name__, e)
        err = agree(err)
    out = None
    if err is None:
        t = max_over_ranks(t)
        barrier()                      # every rank done reading before teardown
        acc = {"elements": 0, "mismatches": 0, "max_err_over_bound": 0.0}
        rs_check(world, rank, members, exchange, acc)
        alla = exchange(acc)           # every rank's own rows
        acc = {"elements": sum(a_["elements"] for a_ in alla), "mismatches": sum(a_["mismatches"] for a_ in alla),
               "max_err_over_bound": max(a_["max_err_over_bound"] for a_ in alla), "ranks_checked": len(alla)}
        full = world * b.rs_seg
        bus = (world - 1) / world * full / t
        out = {"rs_ms": round(t / 1e6, 4), "busbw_GBps": round(bus, 1), "frac_nvlink": round(bus / NVLINK_GBS, 4),
               "frac_measured_peer": round(bus / NVLINK_MEASURED_GBS, 4),
               "rs_full_bytes": full,
               "parity": dict(acc, ok=acc["elements"] > 0 and acc["max_err_over_bound"] <= 1.0,
                              required="G7 bound (the switch's summation order)"),
               "how": "K10 alone (multimem.ld_reduce.add.v4.f32 through the multicast mapping), events, median "
                      "of %d, max over ranks; busbw = (N-1)/N x fp32 bucket bytes / t" % reps}
    barrier()
    if m is not None:
        m.close()
    if win_ptr is not None:
        F.mem_free(ctx, win_ptr)       # deregisters the window (collective: every rank gets here)
    b.close()
    if out is not None:
        out["route"] = route
        return out
    return {"unavailable" if "refused" in err or "multicast" in err or "UNSUPPORTED" in err else "error": err[:300]}


def exposure_leg(args, specs, world, rank, ctx, cs, ms, compute, p2p, exchange, barrier, max_over_ranks, alpha_beta):
    """BASELINE configs[2] at this N, MEASURED: the step with the compute proxy
    at --exposure-tokens tokens/GPU per variant; exposed = step - the same
    step with no collective and no wait (FSDP_SCHED_NO_COMM), both CUDA-graph
    replays timed with events, max over ranks.  Greedy (Algorithm 1) is
    planned with the alpha / beta fitted at this N.  `predicted_exposed_ms` =
    the two-stream model (fsdp_simulate_schedule) from a timed step's
    compute-stream ops + alpha + beta n collectives (the estimate P:600 blames
    for auto-wrap's misses), beside the measurement."""
    import torch
    from paper_2411_00284_b200 import _lib as L
    from paper_2411_00284_b200 import harness as H
    from workloads.compute_model import per_param_compute_ns
    T = args.exposure_tokens
    tf, tb = per_param_compute_ns(specs, T)
    if alpha_beta and "ag" in alpha_beta:
        lag = (alpha_beta["ag"]["alpha_ns"], alpha_beta["ag"]["beta_fs_per_byte"])
        lrs = (alpha_beta["rs"]["alpha_ns"], alpha_beta["rs"]["beta_fs_per_byte"])
        src = "fitted at this N"
    else:
        lag = lrs = ASSUMED_LINK
        src = "assumed (no sweep)"
    nspi = H.calibrate_proxy(ctx, cs, args.proxy_ctas, args.proxy_smem)
    RF = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT
    out = {"tokens_per_gpu": T, "links": {"ag": lag, "rs": lrs, "source": src}, "variants": {}}
    for name, vmode, vflags in (("vanilla (per-param, no reorder)", L.PLAN_PER_PARAM, 0),
                                ("per-block + reorder (manual wrap)", L.PLAN_MANUAL, RF),
                                ("greedy + reorder (Algorithm 1, fitted links)", L.PLAN_GREEDY, RF)):
        vf, vb = H.plans_for(specs, world, vmode, tf, tb, lag, lrs, int(args.mem_limit))
        if p2p and not H.same_buckets(vf, vb):
            vb = H.mirror_plan(vf)           # one shard layout for both phases (peer-memory path)
        win = p2p and args.p2p_transport == "window"
        vst = H.RankState(specs, world, rank, vf, vb, ctx, seed=77 + rank, ipc=p2p and not win, windows=win)
        if win:
            vst.setup_p2p_windows()
        elif p2p:
            vst.setup_p2p_ipc(exchange)
            vst.p2p_max_ctas = args.p2p_max_ctas if args.p2p_max_ctas >= 0 else H.emulation_ctas_p2p(world)
        fl = vflags | (L.SCHED_P2P if p2p else 0)
        vpf = H.proxy_iters(H.bucket_times(vf, tf), nspi)
        vpb = H.proxy_iters(H.bucket_times(vb, tb), nspi)
        res = {"buckets_fwd": len(vf), "buckets_bwd": len(vb)}
        for key, extra in (("step_ms", 0), ("compute_only_ms", L.SCHED_NO_COMM)):
            for _ in range(2):
                vst.step(fl | extra, cs, ms, vpf, vpb, args.proxy_ctas, args.proxy_smem)
            g = vst.capture(fl | extra, cs, ms, vpf, vpb, args.proxy_ctas, args.proxy_smem)
            for _ in range(2):
                g.launch(cs)
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(compute)
            for _ in range(args.steps):
                g.launch(cs)
            b.record(compute)
            barrier()
            res[key] = round(max_over_ranks(a.elapsed_time(b) / args.steps), 3)
            g.close()
        vst.check_p2p()
        res["exposed_ms"] = round(res["step_ms"] - res["compute_only_ms"], 3)
        rep = vst.step(fl | L.SCHED_TIMING, cs, ms, vpf, vpb, args.proxy_ctas, args.proxy_smem, want_log=True)
        ptot, pexp = H.simulate_n_rank(vst, rep["log"], lag, lrs)
        res["predicted_exposed_ms"] = round(max_over_ranks(pexp / 1e6), 3)
        res["predicted_step_ms"] = round(max_over_ranks(ptot / 1e6), 3)
        out["variants"][name] = res
        barrier()
        if p2p:
            vst.close_ipc()
            barrier()                # every rank closed its mappings of ours
            vst.free_ipc()
        vst.close_nccl_mem()
        del vst
        gc.collect()
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
