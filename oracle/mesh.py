"""O11 -- 2-D DP x TP composition (test infrastructure; see oracle/__init__.py).

P:315: "a model parameter can be initialized as a 2D DTensor, doubly sharded on
both Data Parallel (DP) and Tensor Parallel (TP) dimensions. During
computation, it is first redistributed (via an all-gather) on the DP sub-mesh,
and then represented as a sharded DTensor on the TP sub-mesh".

A parameter p [d, R] is split along its TP axis (0: rows, 1: columns) into tp
equal blocks; TP rank t holds block t, and FSDP shards that TP-local tensor
along its dim 0 over the DP sub-mesh (O2).  The DP all-gather (O4) therefore
returns the TP-local block, and the DP reduce-scatter (O5) averages TP-local
gradients over the DP ranks of one TP index.
"""
import numpy as np

from .collectives import bucketed_all_gather, bucketed_reduce_scatter
from .shard import shard


def tp_slice(p, tp, t, axis):
    """Block t of p along `axis` (0 or 1; None: the whole, replicated)."""
    if axis is None or tp == 1:
        return np.ascontiguousarray(p)
    n = p.shape[axis]
    assert n % tp == 0, "TP split needs divisibility"
    b = n // tp
    blk = p[t * b:(t + 1) * b] if axis == 0 else p[:, t * b:(t + 1) * b]
    return np.ascontiguousarray(blk)


def shard_2d(p, dp, tp, r, t, axis):
    """What DP rank r of TP index t stores: shard(tp_slice(p), dp, r)."""
    return shard(tp_slice(p, tp, t, axis), dp, r)


def dp_all_gather(params, axes, dp, tp, t, align=16):
    """The DP-sub-mesh all-gather of one bucket for TP index t: returns the
    TP-local blocks (gathered buffer, fulls) exactly as O4 on them."""
    return bucketed_all_gather([tp_slice(p, tp, t, a) for p, a in zip(params, axes)], dp, align)


def dp_reduce_scatter(grads_per_dp_rank, axes, dp, tp, t, align=16):
    """DP-sub-mesh reduce-scatter(avg) for TP index t: grads_per_dp_rank[r] are
    DP rank r's FULL gradients; each is cut to its TP block first."""
    local = [[tp_slice(g, tp, t, a) for g, a in zip(gs, axes)] for gs in grads_per_dp_rank]
    return bucketed_reduce_scatter(local, dp, align)
