#!/usr/bin/env python
"""Where the fused path's emulated N = 8 step goes: per-op device time of one
FSDP_SCHED_TIMING step with paced K8 / K9 (fsdp_comm_emulation) and the
compute proxy at T tokens, against the modelled link time of the collectives
and the compute-only step.  Prints one JSON object."""
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
    world = 8
    specs = llama("8b")
    ctx = F.Ctx(world, 0)
    fplan, bplan = H.plans_for(specs, world, L.PLAN_MANUAL)
    st = H.RankState(specs, world, 0, fplan, bplan, ctx, seed=4)
    st.setup_p2p_simulated(seed=5)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    cal = H.calibrate_proxy(ctx, cs.cuda_stream)
    tf, tb = per_param_compute_ns(specs, T)
    pf, pb = H.proxy_iters(H.bucket_times(fplan, tf), cal), H.proxy_iters(H.bucket_times(bplan, tb), cal)
    link = (20000, 1215)
    out = {"tokens": T, "modelled_link_ms": {
        "ag": sum(F.comm_time_ns(world * b.ag_seg, link) for b in st.fwd + st.bwd) / 1e6,
        "rs": sum(F.comm_time_ns(world * b.rs_seg // 2, link) for b in st.bwd) / 1e6}}
    flags = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT | L.SCHED_P2P
    names = ["PACK_AG", "AG", "WAIT_AG", "UNPACK", "COMPUTE_F", "COMPUTE_B", "PACK_RS", "RS", "WAIT_RS", "COPYOUT_RS"]
    for ctas in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["57", "96", "148"])]:
        em = dict(ag=link, rs=link, ctas=ctas)
        st.step(flags, cs.cuda_stream, ms.cuda_stream, pf, pb, emulate=em)
        rep = st.step(flags | L.SCHED_TIMING, cs.cuda_stream, ms.cuda_stream, pf, pb, emulate=em)
        out["ctas=%d" % ctas] = {"step_ms": round(rep["step_ns"] / 1e6, 3),
                                 "op_ms": {n: round(rep["op_ns"][i] / 1e6, 3) for i, n in enumerate(names)}}
    comp = st.step(flags | L.SCHED_TIMING | L.SCHED_NO_COMM, cs.cuda_stream, ms.cuda_stream, pf, pb)
    out["compute_only"] = {"step_ms": round(comp["step_ns"] / 1e6, 3),
                           "op_ms": {n: round(comp["op_ns"][i] / 1e6, 3) for i, n in enumerate(names)}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
