"""O4 / O5 -- bucketed all-gather and reduce-scatter(avg) over N simulated ranks
(test infrastructure; see oracle/__init__.py).

All-gather bucketing: the member shards are flattened and concatenated
into one buffer (copy-in), one all-gather AG12 gathers every rank's buffer, and
after the wait Wa12 the data are "copy[ied] out ... based on their original
tensor size" (copy-out).

Reduce-scatter bucketing: each gradient is split "into chunks based on
world size"; chunk q of every member goes to rank q's segment ("concatenates");
one reduce-scatter RS12 then "average[s] the buffer data gathered from other
devices" and the gradients "are read out from RS12".  Averaging with
``Partial(reduce_op="avg")`` in ``reduce_dtype``: the gradient
is widened to fp32 and pre-scaled by fl32(1/N) before the sum (reading G6), and
the sum is taken in rank order ((in_0 + in_1) + in_2) + ... (reading G7).

Arrays: a parameter / gradient is a 2-D NumPy array [d, R] of dtype uint16
(bf16 bit patterns) or float32.  Buffers are uint8 byte arrays (AG) or float32
element arrays (RS input/output), so that every byte of padding is explicit.
"""
import numpy as np

from . import bf16
from .layout import bucket_layout
from .shard import shard, shard_rows


def _as_bytes(a):
    return np.ascontiguousarray(a).reshape(-1).view(np.uint8)


def ag_pack(shards, world, rank, align=16):
    """Copy-in: rank ``rank``'s AG segment (uint8, seg bytes) for one bucket.

    ``shards``: this rank's local padded shards [c_j, R_j] of the members in
    forward order.  Pad bytes are zero (G3).
    """
    e = shards[0].dtype.itemsize
    # O3 layout; it needs d_j only through c_j, the shard's row count, and
    # ceil((c_j * world) / world) == c_j.
    offs, seg = bucket_layout([(s.shape[0] * world, s.shape[1]) for s in shards],
                              world, e, align)
    buf = np.zeros(seg, dtype=np.uint8)
    for s, o in zip(shards, offs):
        b = _as_bytes(s)
        buf[o:o + b.size] = b
    return buf


def all_gather(segments):
    """The collective: every rank receives the concatenation of all segments."""
    return np.concatenate(segments)


def ag_unpack(gathered, dims, world, dtype, align=16):
    """Copy-out: full parameters [d_j, R_j] from the gathered buffer.

    For member j and source rank q, the first v_{j,q} rows of rank q's chunk
    (padding rows dropped) become rows [q c_j, q c_j + v_{j,q}) of the full
    parameter.  ``dims`` is the list of (d_j, R_j) in forward order.
    """
    dtype = np.dtype(dtype)
    e = dtype.itemsize
    offs, seg = bucket_layout(dims, world, e, align)
    assert gathered.size == world * seg
    fulls = []
    for (d, r), o in zip(dims, offs):
        full = np.zeros((d, r), dtype=dtype)
        for q in range(world):
            c, begin, v = shard_rows(d, world, q)
            lo = q * seg + o
            chunk = gathered[lo:lo + v * r * e].view(dtype).reshape(v, r)
            full[begin:begin + v] = chunk
        fulls.append(full)
    return fulls


def bucketed_all_gather(params, world, align=16):
    """shard -> per-rank copy-in -> all-gather -> copy-out, for one bucket.

    Returns (gathered_buffer, fulls).  ``params`` are the full [d_j, R_j]
    arrays in forward order; every rank ends with the same gathered buffer.
    """
    segs = [ag_pack([shard(p, world, q) for p in params], world, q, align)
            for q in range(world)]
    g = all_gather(segs)
    dims = [p.shape for p in params]
    return g, ag_unpack(g, dims, world, params[0].dtype, align)


def mixed_precision_all_gather(masters, world, align=16):
    """All-gather of fp32 master weights in param_dtype = bf16 ("the
    parameters are cast to param_dtype" before they are used).  Step order as
    in the paper's fp32-sharded / bf16-communicated setting: each rank holds
    shard(master) in fp32, casts its shard to bf16 (round to nearest even),
    copies it in, and the bucket is gathered and copied out in bf16.

    ``masters``: full fp32 [d_j, R_j] master parameters in forward order.
    Returns (gathered_buffer, fulls) like ``bucketed_all_gather``.
    """
    segs = []
    for q in range(world):
        local = [bf16.narrow(shard(m, world, q)) for m in masters]
        segs.append(ag_pack(local, world, q, align))
    g = all_gather(segs)
    dims = [m.shape for m in masters]
    return g, ag_unpack(g, dims, world, np.uint16, align)


def _to_f32(g):
    if g.dtype == np.uint16:
        return bf16.widen(g)
    if g.dtype == np.float32:
        return g
    raise TypeError("gradients are bf16 (uint16 bits) or float32")


def inv_world_f32(world):
    """fl32(1/N): the correctly rounded fp32 value of 1/N."""
    return np.float32(1.0) / np.float32(world)


def rs_pack(grads, world, align=16):
    """RS copy-in of one rank's full gradients, fused with the cast to
    ``reduce_dtype`` = fp32 and the 1/N pre-scale of the average.

    Returns the float32 buffer of N * seg' / 4 elements: for each member j
    and destination rank q, rows [q c_j, q c_j + v_{j,q}) of g_j, widened and
    multiplied by fl32(1/N), at element (q seg' + off'_j)/4; everything else
    (padding rows, alignment gaps) is +0.0.
    """
    dims = [g.shape for g in grads]
    offs, seg = bucket_layout(dims, world, 4, align)
    inv = inv_world_f32(world)
    out = np.zeros(world * seg // 4, dtype=np.float32)
    for g, (d, r), o in zip(grads, dims, offs):
        gf = _to_f32(g)
        for q in range(world):
            c, begin, v = shard_rows(d, world, q)
            lo = (q * seg + o) // 4
            out[lo:lo + v * r] = (gf[begin:begin + v].reshape(-1) * inv).astype(np.float32)
    return out


def reduce_scatter(inputs, world):
    """The collective: rank q receives slot q of the rank-order fp32 sum."""
    n = inputs[0].size
    assert n % world == 0
    seg = n // world
    outs = []
    for q in range(world):
        acc = inputs[0][q * seg:(q + 1) * seg].copy()
        for r in range(1, world):
            acc = (acc + inputs[r][q * seg:(q + 1) * seg]).astype(np.float32)
        outs.append(acc)
    return outs


def rs_copyout(rs_out, dims, world, align=16):
    """Read-out of the sharded gradients [c_j, R_j] (fp32) from the RS output."""
    offs, seg = bucket_layout(dims, world, 4, align)
    assert rs_out.size * 4 == seg
    res = []
    for (d, r), o in zip(dims, offs):
        c = -(-d // world)
        res.append(rs_out[o // 4:o // 4 + c * r].reshape(c, r).copy())
    return res


def rs_copyout_bf16(rs_out, dims, world, align=16):
    """Read-out into bf16 gradient shards (reading G41; the north star's
    "1 bf16 ulp after cast"): the fp32 RS result (reduce_dtype) is
    rounded once, RNE, to bf16 bit patterns (O1 narrow)."""
    return [bf16.narrow(x) for x in rs_copyout(rs_out, dims, world, align)]


def accumulate_grad_shards(existing, new):
    """Gradient accumulation over micro-batches: the
    gradient shards read out of this reduce-scatter are added to the shards
    already held, one fp32 addition per element: existing + new."""
    return [(e + n).astype(np.float32) for e, n in zip(existing, new)]


def bucketed_reduce_scatter(grads_per_rank, world, align=16):
    """Full pipeline for one bucket.  ``grads_per_rank[r]`` is rank r's list
    of full gradients.  Returns (packed inputs, RS outputs, grad shards per
    rank)."""
    ins = [rs_pack(g, world, align) for g in grads_per_rank]
    outs = reduce_scatter(ins, world)
    dims = [g.shape for g in grads_per_rank[0]]
    shards = [rs_copyout(o, dims, world, align) for o in outs]
    return ins, outs, shards
