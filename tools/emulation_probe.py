#!/usr/bin/env python
"""How long the emulated collectives (K11) last, alone and under contention:
one Llama-3-8B rank step at N = 8 (per-block buckets), the emulated AG / RS op
times from a FSDP_SCHED_TIMING step in vanilla order (each collective alone)
and reordered (overlapping the copy kernels and, with --tokens, the compute
proxy), against alpha + beta n.  Prints one JSON object."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_00284_b200 as F  # noqa: E402
from paper_2411_00284_b200 import _lib as L  # noqa: E402
from paper_2411_00284_b200 import harness as H  # noqa: E402
from workloads import llama  # noqa: E402
from workloads.compute_model import per_param_compute_ns  # noqa: E402


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    ctas = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16]
    specs = llama("8b")
    world = 8
    link = (20000, 1215)
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=4)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    cal = H.calibrate_proxy(ctx, cs.cuda_stream)
    tf, tb = per_param_compute_ns(specs, T)
    pf, pb = H.proxy_iters(H.bucket_times(fplan, tf), cal), H.proxy_iters(H.bucket_times(bplan, tb), cal)
    want = {"ag": sum(F.comm_time_ns(world * b.ag_seg, link) for b in st.fwd + st.bwd) / 1e6,
            "rs": sum(F.comm_time_ns(world * b.rs_seg, link) for b in st.bwd) / 1e6}
    out = {"tokens": T, "modelled_ms": want, "runs": {}}
    for c in ctas:
        em = dict(ag=link, rs=link, ctas=c)
        for name, flags, p in (("vanilla, no compute", 0, (None, None)),
                               ("reorder, no compute", L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, (None, None)),
                               ("reorder, proxy compute", L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT, (pf, pb))):
            st.step(flags, cs.cuda_stream, ms.cuda_stream, p[0], p[1], emulate=em)
            rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, p[0], p[1], emulate=em)
            out["runs"]["%d CTAs, %s" % (c, name)] = {"ag_ms": round(rep["op_ns"][L.OP_AG] / 1e6, 3),
                                                      "rs_ms": round(rep["op_ns"][L.OP_RS] / 1e6, 3),
                                                      "step_ms": round(rep["step_ns"] / 1e6, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
