"""O11 pins (2-D DP x TP): TP blocks tile the parameter; the DP
all-gather of 2-D shards returns the TP block; the reduce-scatter over the DP
sub-mesh of TP blocks equals the TP block of the full-mesh average where the
average is exact; DP = 1 and TP = 1 reduce to plain slicing / plain FSDP."""
import numpy as np
from hypothesis import given, settings, strategies as st

from oracle.collectives import bucketed_all_gather, bucketed_reduce_scatter
from oracle.mesh import dp_all_gather, dp_reduce_scatter, shard_2d, tp_slice
from oracle.shard import shard
from workloads import llama
from workloads.shapes import tp_axis, tp_local


def _rand(shape, seed, dtype=np.uint16):
    rng = np.random.Generator(np.random.Philox(seed))
    if dtype == np.uint16:
        return rng.integers(0, 65536, size=shape).astype(np.uint16)
    return rng.standard_normal(shape, dtype=np.float32)


@given(d=st.integers(1, 12), r=st.integers(1, 12), tp=st.sampled_from([1, 2, 4]), axis=st.sampled_from([0, 1, None]),
       seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_tp_blocks_tile_the_parameter(d, r, tp, axis, seed):
    d, r = d * tp, r * tp
    p = _rand((d, r), seed)
    blocks = [tp_slice(p, tp, t, axis) for t in range(tp)]
    if axis is None:
        assert all(np.array_equal(b, p) for b in blocks)
    else:
        assert np.array_equal(np.concatenate(blocks, axis=axis), p)


@given(dp=st.integers(1, 6), tp=st.sampled_from([1, 2, 4]), seed=st.integers(0, 2**31))
@settings(max_examples=60, deadline=None)
def test_dp_all_gather_returns_the_tp_block(dp, tp, seed):
    shapes = [(3 * tp, 5 * tp), (7 * tp, 2 * tp), (4 * tp, 1 * tp)]
    axes = [0, 1, None]
    params = [_rand(s, seed + i) for i, s in enumerate(shapes)]
    for t in range(tp):
        _, fulls = dp_all_gather(params, axes, dp, tp, t)
        for p, a, f in zip(params, axes, fulls):
            assert np.array_equal(f, tp_slice(p, tp, t, a))
            # what every DP rank stored is that block's FSDP shard
            for r in range(dp):
                assert np.array_equal(shard_2d(p, dp, tp, r, t, a), shard(f, dp, r))


def test_dp_reduce_scatter_of_exact_data_is_tp_block_of_mean():
    # exactly representable gradients, DP = 4: the DP average of the TP block
    # is the TP block of the average, bit for bit
    dp, tp = 4, 2
    shapes = [(8, 6), (6, 4)]
    axes = [0, 1]
    rng = np.random.Generator(np.random.Philox(3))
    g = [[(rng.integers(-64, 65, size=s).astype(np.float32) * np.float32(2 ** -6)) for s in shapes]
         for _ in range(dp)]
    for t in range(tp):
        _, _, shards = dp_reduce_scatter(g, axes, dp, tp, t)
        for j, (s, a) in enumerate(zip(shapes, axes)):
            mean = sum(gr[j].astype(np.float64) for gr in g) / dp
            blk = tp_slice(mean.astype(np.float32), tp, t, a)
            for r in range(dp):
                assert np.array_equal(shards[r][j].view(np.uint32), shard(blk, dp, r).view(np.uint32))


def test_degenerate_meshes():
    p = [_rand((6, 4), 1)]
    # TP = 1: plain FSDP
    assert np.array_equal(dp_all_gather(p, [0], 3, 1, 0)[0], bucketed_all_gather(p, 3)[0])
    # DP = 1: the gather is the TP block itself
    assert np.array_equal(dp_all_gather(p, [1], 1, 2, 1)[1][0], p[0][:, 2:])
    g = [[_rand((6, 4), 2, np.float32)]]
    assert all(np.array_equal(a, b) for a, b in zip(dp_reduce_scatter(g, [None], 1, 2, 0)[2][0],
                                                      bucketed_reduce_scatter(g, 1)[2][0]))


def test_llama_tp_local_shapes():
    specs = llama("8b", n_layers=1)
    loc = tp_local(specs, 4)
    by = {p.name: p for p in loc}
    assert by["layers.0.attention.wq.weight"][1:3] == (1024, 4096)
    assert by["layers.0.attention.wo.weight"][1:3] == (4096, 1024)
    assert by["layers.0.attention_norm.weight"][1:3] == (4096, 1)
    assert by["tok_embeddings.weight"][1:3] == (128256 // 4, 4096)
    assert sum(p.dim0 * p.row_numel for p in loc) < sum(p.dim0 * p.row_numel for p in specs)
    assert tp_axis(by["layers.0.ffn_norm.weight"]) is None
