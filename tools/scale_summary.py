#!/usr/bin/env python
"""Summarise a multi-GPU measurement run (tools/scale_check.sh output,
gpurun_out/scale/bench_<tag>_N<n>.json) as one markdown table per quantity:
parity verdicts, the headline (whole-job bus GB/s), the isolated 8B-block
AG / RS busbw against 900 GB/s nominal and 770 GB/s measured peer bandwidth,
the fitted alpha / beta, the measured exposure of vanilla / per-block / greedy
and the NVLS K10 leg.  Reads only the JSON lines bench.py printed.

    python tools/scale_summary.py [gpurun_out/scale] > profiles/rNN_scale_summary.md
"""
import glob
import json
import os
import re
import sys


def load(d):
    rows = []
    for p in sorted(glob.glob(os.path.join(d, "bench_*_N*.json"))):
        m = re.match(r"bench_(.+)_N(\d+)\.json$", os.path.basename(p))
        if not m:
            continue
        line = None
        with open(p) as f:
            for ln in f:
                ln = ln.strip()
                if ln.startswith("{"):
                    line = ln
        if line:
            try:
                rows.append((m.group(1), int(m.group(2)), json.loads(line)))
            except ValueError:
                pass
    return rows


def fmt(x, nd=1):
    if x is None:
        return "-"
    if isinstance(x, float):
        return ("%%.%df" % nd) % x
    return str(x)


def summary(rows):
    out = ["# Multi-GPU bench summary", ""]
    out += ["| run | N | ms/step | value (GB/s) | kind | parity | AG bit-exact | RS max err / bound | pad rows ok |",
            "|---|---|---|---|---|---|---|---|---|"]
    for tag, n, d in rows:
        par = d.get("parity") or {}
        rs = par.get("rs") or {}
        out.append("| %s | %d | %s | %s | %s | %s | %s | %s | %s |" % (
            tag, n, fmt(d.get("ms_per_step"), 3), fmt(d.get("value")), d.get("value_kind", "-"),
            fmt(par.get("ok")), fmt((par.get("ag") or {}).get("bit_exact")), fmt(rs.get("max_err_over_bound"), 3),
            fmt(rs.get("pad_nonzero") == 0 if "pad_nonzero" in rs else None)))
    out += ["", "| run | N | block AG busbw | block RS busbw | frac of 900 (AG / RS) | frac of 770 (AG / RS) |",
            "|---|---|---|---|---|---|"]
    for tag, n, d in rows:
        bb = d.get("busbw_block") or {}
        if not bb:
            continue
        out.append("| %s | %d | %s | %s | %s / %s | %s / %s |" % (
            tag, n, fmt(bb.get("ag_GBps")), fmt(bb.get("rs_GBps")), fmt(bb.get("ag_frac_nvlink"), 3),
            fmt(bb.get("rs_frac_nvlink"), 3), fmt(bb.get("ag_frac_measured_peer"), 3),
            fmt(bb.get("rs_frac_measured_peer"), 3)))
    out += ["", "| run | N | AG alpha ns | AG beta fs/B | RS alpha ns | RS beta fs/B |", "|---|---|---|---|---|---|"]
    for tag, n, d in rows:
        ab = d.get("alpha_beta") or {}
        if "ag" not in ab or not str(ab.get("source", "")).startswith("measured"):
            continue
        out.append("| %s | %d | %s | %s | %s | %s |" % (tag, n, ab["ag"]["alpha_ns"], ab["ag"]["beta_fs_per_byte"],
                                                       ab["rs"]["alpha_ns"], ab["rs"]["beta_fs_per_byte"]))
    out += ["", "| run | N | variant | buckets fwd / bwd | step ms | compute-only ms | exposed ms | predicted exposed ms |",
            "|---|---|---|---|---|---|---|---|"]
    for tag, n, d in rows:
        ex = d.get("exposure") or {}
        for name, v in (ex.get("variants") or {}).items():
            out.append("| %s | %d | %s | %s / %s | %s | %s | %s | %s |" % (
                tag, n, name, v.get("buckets_fwd"), v.get("buckets_bwd"), fmt(v.get("step_ms"), 3),
                fmt(v.get("compute_only_ms"), 3), fmt(v.get("exposed_ms"), 3), fmt(v.get("predicted_exposed_ms"), 3)))
    out += ["", "| run | N | NVLS K10 |", "|---|---|---|"]
    for tag, n, d in rows:
        nv = d.get("nvls_block")
        if nv is None:
            continue
        if "busbw_GBps" in nv:
            txt = "%s GB/s busbw (%s of 900), parity %s, route: %s" % (
                fmt(nv["busbw_GBps"]), fmt(nv.get("frac_nvlink"), 3), fmt((nv.get("parity") or {}).get("ok")),
                nv.get("route", "-"))
        else:
            txt = "unavailable: %s" % (nv.get("unavailable") or nv.get("error"))
        out.append("| %s | %d | %s |" % (tag, n, txt.replace("|", "/")))
    return "\n".join(out) + "\n"


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else os.path.join("gpurun_out", "scale")
    sys.stdout.write(summary(load(d)))


if __name__ == "__main__":
    main()
