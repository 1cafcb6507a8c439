"""O2 -- per-parameter dim-0 sharding (test infrastructure; see oracle/__init__.py).

P:69  "partitioned per the number of devices ... Each device only holds one of
       the partitions";
P:133 "SimpleFSDP shards the parameters as DTensors" -- Shard(0), i.e. dim 0.

Reading G1 (uneven split): ceil chunking as torch.chunk / DTensor Shard(0):
c = ceil(d / N) rows per rank; rank r owns rows [r*c, r*c + v_r) with
v_r = clamp(d - r*c, 0, c); its local buffer has c rows, the missing
(c - v_r) rows are padding filled with +0 (G3).  Tail ranks may own 0 rows.
"""
import numpy as np


def shard_rows(d, world, rank):
    """Return (c, row_begin, valid_rows) for a dim-0 size ``d``.

    row_begin is r*c clamped to d so that it is always a valid slice start.
    """
    if world < 1 or not (0 <= rank < world) or d < 1:
        raise ValueError("bad shard arguments")
    c = -(-d // world)
    v = max(0, min(d - rank * c, c))
    return c, min(rank * c, d), v


def shard(p, world, rank):
    """Local padded shard of ``p`` ([d, ...]) held by ``rank``: shape [c, ...]."""
    p = np.asarray(p)
    d = p.shape[0]
    c, begin, v = shard_rows(d, world, rank)
    out = np.zeros((c,) + p.shape[1:], dtype=p.dtype)
    out[:v] = p[begin:begin + v]
    return out
