#!/usr/bin/env python
"""PCIe floor of bench.py's e2e leg (measurement tool, not the product path).

Copies the e2e step's bytes between pinned host memory and the device with
cudaMemcpyAsync (torch copy_), events on the copy streams: the 2.0 GB of
bf16 shards H2D alone, the 4.0 GB of fp32 gradient shards D2H alone, and both
at once on two streams (full duplex).  In 109 MB pieces like the per-bucket
copies of fsdp_host_io.  Prints one JSON object.
"""
import json

import torch

H2D_BYTES, D2H_BYTES, PIECE = 2007565312, 4015130624, 109056000


def pieces(total):
    out, o = [], 0
    while o < total:
        out.append((o, min(PIECE, total - o)))
        o += PIECE
    return out


def main():
    hs = torch.empty(H2D_BYTES, dtype=torch.uint8).pin_memory()
    hg = torch.empty(D2H_BYTES, dtype=torch.uint8).pin_memory()
    ds = torch.empty(H2D_BYTES, dtype=torch.uint8, device="cuda")
    dg = torch.empty(D2H_BYTES, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            for o, n in pieces(H2D_BYTES):
                ds[o:o + n].copy_(hs[o:o + n], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            for o, n in pieces(D2H_BYTES):
                hg[o:o + n].copy_(dg[o:o + n], non_blocking=True)

    def timed(fns):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(torch.cuda.current_stream())
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for f in fns:
            f()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record(torch.cuda.current_stream())
        b.synchronize()
        return a.elapsed_time(b)

    out = {}
    for name, fns, nbytes in (("h2d_2.0GB", [h2d], H2D_BYTES), ("d2h_4.0GB", [d2h], D2H_BYTES),
                              ("both", [h2d, d2h], H2D_BYTES + D2H_BYTES)):
        timed(fns)
        ms = min(timed(fns) for _ in range(3))
        out[name] = {"ms": round(ms, 2), "GB/s": round(nbytes / ms / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
