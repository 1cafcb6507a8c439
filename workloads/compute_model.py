"""Synthetic per-parameter compute times T_ci (ns) -- planner INPUTS.

The paper's profiler runs each compute node on real tensors and records its
CUDA-event time.  There is no model compute on this path, so the
harness supplies T_ci from a per-op roofline model of a Llama block at T
tokens per GPU (reading G25: the paper states only batch size 1,
P:494, so T is swept):

  linear [out, in]   2 T out in / F_eff       (attributed to that weight)
  RMSNorm / embed    2 T d 2 B / H_eff        (attributed to the norm / embedding)
  SDPA (causal)      2 T^2 d / F_eff          (attributed to wv, the last QKV weight)
  SiLU * mul         3 T f 2 B / H_eff        (attributed to w3)
  backward           2 x forward (activation checkpointing off)

Parameterless ops are attributed to the preceding parameter consumer: that is
the compute between that parameter's wait and the next one, which is what a
prefetch overlaps (Table 1, "time to compute the parameters pre-fetched by
i-th AG").  F_eff defaults to 1.0 PFLOP/s and H_eff to 6 TB/s; both are
stated in every report.
"""


def per_param_compute_ns(params, tokens, f_eff=1.0e15, h_eff=6.0e12, dim=None):
    """Returns (t_fwd_ns, t_bwd_ns), lists indexed like ``params``."""
    fwd = []
    T = tokens
    for p in params:
        name = p.name
        if p.row_numel == 1:                       # RMSNorm weight
            t = 2.0 * T * p.dim0 * 2 / h_eff
        elif "embeddings" in name:                 # lookup: read + write T x d bf16
            t = 2.0 * T * p.row_numel * 2 / h_eff
        else:                                      # linear [out, in]
            t = 2.0 * T * p.dim0 * p.row_numel / f_eff
            if name.endswith("wv.weight"):
                d = dim if dim is not None else p.row_numel
                t += 2.0 * T * T * d / f_eff       # causal SDPA
            if name.endswith("w3.weight"):
                t += 3.0 * T * p.dim0 * 2 / h_eff  # SiLU(w1 x) * (w3 x)
        fwd.append(int(round(t * 1e9)))
    return fwd, [2 * t for t in fwd]


def apportioned_compute_ns(params, module_ns):
    """SPEC-mode apportionment: a module's time T_mod split over its
    parameters by element count, floor division with the remainder on the
    module's last parameter so the parts sum to T_mod exactly.
    ``module_ns``: dict module_id -> ns."""
    out = [0] * len(params)
    by_mod = {}
    for i, p in enumerate(params):
        by_mod.setdefault(p.module_id, []).append(i)
    for m, idx in by_mod.items():
        tot = module_ns[m]
        sizes = [params[i].dim0 * params[i].row_numel for i in idx]
        s = sum(sizes)
        acc = 0
        for k, i in enumerate(idx):
            v = tot * sizes[k] // s if k + 1 < len(idx) else tot - acc
            out[i] = v
            acc += v
    return out
