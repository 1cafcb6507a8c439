"""O4 / O5 pins.

AG: the BASELINE.json invariant all_gather(shard(p)) == p, bit-exact; zero
padding in the raw gathered buffer; a bucket changes no bits versus
per-parameter gathers.
RS: the invariant reduce_scatter(g_0..g_{N-1}) == shard(sum_r g_r / N) checked
(a) bit-exactly where the exact result is representable: N = 2 (one IEEE add
of two halved values = the correctly rounded (a + b) / 2) and exact-representable
data at N = 2^k, computed independently in float64 then rounded once;
(b) otherwise within the proven fp32 error bound of an fp64 reference.
"""
import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import bf16
from oracle.collectives import (all_gather, ag_pack, bucketed_all_gather,
                                bucketed_reduce_scatter, rs_pack)
from oracle.layout import bucket_layout
from oracle.shard import shard, shard_rows
from workloads import toy_mlp, llama
from workloads.data import param_tensor, grad_tensor, EDGE_BF16_BITS

dims_st = st.lists(st.tuples(st.integers(1, 60), st.integers(1, 17)), min_size=1, max_size=8)


def _rand_params(dims, dtype, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    if dtype == np.uint16:
        return [rng.integers(0, 65536, size=(d, r)).astype(np.uint16) for d, r in dims]
    return [rng.standard_normal((d, r), dtype=np.float32) for d, r in dims]


@given(dims=dims_st, world=st.integers(1, 8), a=st.sampled_from([1, 16]),
       dt=st.sampled_from([np.uint16, np.float32]), seed=st.integers(0, 2**31))
@settings(max_examples=200, deadline=None)
def test_allgather_of_shards_is_identity(dims, world, a, dt, seed):
    params = _rand_params(dims, dt, seed)
    g, fulls = bucketed_all_gather(params, world, a)
    for p, f in zip(params, fulls):
        assert f.dtype == p.dtype and np.array_equal(f.view(np.uint8), p.view(np.uint8))
    # the raw gathered buffer: every byte outside the shard data is zero
    e = np.dtype(dt).itemsize
    offs, seg = bucket_layout(dims, world, e, a)
    mask = np.zeros(g.size, dtype=bool)
    for q in range(world):
        for (d, r), o in zip(dims, offs):
            c, begin, v = shard_rows(d, world, q)
            lo = q * seg + o
            mask[lo:lo + v * r * e] = True
    assert np.all(g[~mask] == 0)  # pad rows and alignment gaps


@given(dims=dims_st, world=st.integers(1, 8), seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_gathered_segments_hold_rank_shards(dims, world, seed):
    params = _rand_params(dims, np.uint16, seed)
    g, _ = bucketed_all_gather(params, world, 16)
    offs, seg = bucket_layout(dims, world, 2, 16)
    for q in range(world):
        for p, o in zip(params, offs):
            s = shard(p, world, q).reshape(-1).view(np.uint8)
            assert np.array_equal(g[q * seg + o: q * seg + o + s.size], s)


@given(dims=dims_st, world=st.integers(1, 8), seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_bucketing_changes_no_bits(dims, world, seed):
    params = _rand_params(dims, np.uint16, seed)
    _, fulls = bucketed_all_gather(params, world, 16)
    for p, f in zip(params, fulls):
        _, single = bucketed_all_gather([p], world, 16)
        assert np.array_equal(single[0], f)


@given(dims=dims_st, world=st.integers(1, 8), a=st.sampled_from([1, 16]), seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_mixed_precision_allgather_is_rne_cast(dims, world, a, seed):
    """P:302 master weights: gathered full params == the fp32 masters rounded
    to bf16, the rounding taken by torch's CPU cast (an independent library
    routine); zero bytes outside shard data as for bf16 params."""
    import torch
    from oracle.collectives import mixed_precision_all_gather
    masters = _rand_params(dims, np.float32, seed)
    g, fulls = mixed_precision_all_gather(masters, world, a)
    for m, f in zip(masters, fulls):
        ref = torch.from_numpy(m).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        assert f.dtype == np.uint16 and np.array_equal(f, ref)
    offs, seg = bucket_layout(dims, world, 2, a)
    assert g.size == world * seg


def test_mixed_precision_allgather_of_bf16_values_is_identity():
    # a master that holds bf16-representable values gathers to those bf16 bits
    dims = [(13, 7), (5, 16), (1, 3)]
    rng = np.random.Generator(np.random.Philox(5))
    bits16 = [rng.integers(0, 65536, size=d).astype(np.uint16) for d in dims]
    bits16 = [np.where((b & 0x7F80) == 0x7F80, b & 0x807F, b) for b in bits16]  # drop inf/NaN
    masters = [bf16.widen(b) for b in bits16]
    for w in (1, 2, 3, 8):
        _, fulls = mixed_precision_all_gather_ref(masters, w)
        for b, f in zip(bits16, fulls):
            assert np.array_equal(f, b)


def mixed_precision_all_gather_ref(masters, world):
    from oracle.collectives import mixed_precision_all_gather
    return mixed_precision_all_gather(masters, world, 16)


def test_pack_writes_own_segment_only():
    ps = toy_mlp()
    params = [param_tensor(p, "f32", 11 + i) for i, p in enumerate(ps)]
    segs = [ag_pack([shard(p, 2, q) for p in params], 2, q) for q in range(2)]
    g = all_gather(segs)
    assert g.size == 2 * segs[0].size


def _fp64_avg(grads_per_rank, j, world):
    return sum(bf16.widen(g[j]).astype(np.float64) if g[j].dtype == np.uint16 else
               g[j].astype(np.float64) for g in grads_per_rank) / world


def _check_rs(grads_per_rank, world, align, exact):
    ins, outs, shards = bucketed_reduce_scatter(grads_per_rank, world, align)
    dims = [g.shape for g in grads_per_rank[0]]
    for j, (d, r) in enumerate(dims):
        ref = _fp64_avg(grads_per_rank, j, world)
        absum = sum(np.abs(bf16.widen(g[j]) if g[j].dtype == np.uint16 else g[j]).astype(np.float64)
                    for g in grads_per_rank) / world
        for q in range(world):
            got = shards[q][j]
            want = shard(ref, world, q)
            c, _, v = shard_rows(d, world, q)
            assert np.all(got[v:].view(np.uint32) == 0)  # pads exactly +0.0
            if exact:
                assert np.array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32))
            else:
                bound = 1.01 * world * 2.0 ** -24 * shard(absum, world, q) + 1e-45
                assert np.all(np.abs(got.astype(np.float64) - want) <= bound)
                assert np.all(bound <= 1e-6 * shard(absum, world, q) + 1e-45)


@given(dims=dims_st, seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_rs_bit_exact_at_two_ranks(dims, seed):
    # fl(a/2 + b/2) == fl((a+b)/2): a single rounding of the exact mean
    rng = np.random.Generator(np.random.Philox(seed))
    g = [[(rng.standard_normal((d, r), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
          for d, r in dims] for _ in range(2)]
    _check_rs(g, 2, 16, exact=True)


@given(dims=dims_st, k=st.integers(0, 3), seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_rs_bit_exact_on_exact_data(dims, k, seed):
    world = 2 ** k
    rng = np.random.Generator(np.random.Philox(seed))
    g = [[(((rng.integers(-256, 257, size=(d, r)).astype(np.float32) * np.float32(2 ** -8))
            .view(np.uint32)) >> 16).astype(np.uint16) for d, r in dims] for _ in range(world)]
    _check_rs(g, world, 16, exact=True)


@given(dims=dims_st, world=st.integers(1, 8), a=st.sampled_from([1, 16]), seed=st.integers(0, 2**31),
       f32=st.booleans())
@settings(max_examples=150, deadline=None)
def test_rs_within_fp32_bound(dims, world, a, seed, f32):
    rng = np.random.Generator(np.random.Philox(seed))
    if f32:
        g = [[rng.standard_normal((d, r), dtype=np.float32) for d, r in dims] for _ in range(world)]
    else:
        g = [[(rng.standard_normal((d, r), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
              for d, r in dims] for _ in range(world)]
    _check_rs(g, world, a, exact=False)


def test_rs_pack_widens_and_scales_exactly():
    # widen is exact and x * 2^-k is exact for normal x: the packed buffer is
    # the bf16 value / N exactly (checked in float64), pads +0.0
    g = [EDGE_BF16_BITS.reshape(-1, 1)[[0, 1, 5, 6, 9, 10, 11]]]
    out = rs_pack(g, world=4, align=16)
    offs, seg = bucket_layout([g[0].shape], 4, 4, 16)
    vals = bf16.widen(g[0].reshape(-1)).astype(np.float64) / 4
    flat = []
    for q in range(4):
        c, begin, v = shard_rows(7, 4, q)
        flat += list(out[(q * seg + offs[0]) // 4:(q * seg + offs[0]) // 4 + v])
    assert np.array_equal(np.array(flat, dtype=np.float32).view(np.uint32),
                          vals.astype(np.float32).view(np.uint32))


def test_llama_block_rs_sample():
    # one 8B block, rows sampled: full rank-order sum within the fp32 bound at N = 8
    ps = llama("8b", n_layers=1, with_embeddings=False)
    small = [type(p)(p.name, p.dim0, min(p.row_numel, 8), p.module_id) for p in ps]
    g = [[grad_tensor(p, "bf16", 5, r) for p in small] for r in range(8)]
    _check_rs(g, 8, 16, exact=False)


@given(dims=dims_st, seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_accumulate_is_correctly_rounded_sum(dims, seed):
    # fp32 a + b, against the exact sum rounded once: the float64 sum of two
    # fp32 values rounded to fp32 (53 >= 2*24 + 2 bits: double rounding is
    # innocuous for addition)
    from oracle.collectives import accumulate_grad_shards
    rng = np.random.Generator(np.random.Philox(seed))
    a = [(rng.standard_normal((d, r)) * 10.0 ** rng.integers(-30, 30)).astype(np.float32) for d, r in dims]
    b = [rng.standard_normal((d, r), dtype=np.float32) for d, r in dims]
    for x, y, z in zip(a, b, accumulate_grad_shards(a, b)):
        want = (x.astype(np.float64) + y.astype(np.float64)).astype(np.float32)
        assert np.array_equal(z.view(np.uint32), want.view(np.uint32))


def test_accumulated_micro_batches_equal_exact_mean_sum():
    # k micro-batches of exactly representable gradients at N = 4: the
    # accumulated shards equal sum_m mean_r g_{m,r}, computed in float64
    from oracle.collectives import accumulate_grad_shards
    dims, world = [(37, 5), (8, 16), (3, 1)], 4
    rng = np.random.Generator(np.random.Philox(11))
    acc = None
    total = [np.zeros(d) for d in dims]
    for m in range(5):
        g = [[(rng.integers(-256, 257, size=d).astype(np.float32) * np.float32(2 ** -8)) for d in dims]
             for _ in range(world)]
        _, _, shards = bucketed_reduce_scatter(g, world)
        acc = shards if acc is None else [accumulate_grad_shards(a, s) for a, s in zip(acc, shards)]
        for j in range(len(dims)):
            total[j] += sum(g[r][j].astype(np.float64) for r in range(world)) / world
    for q in range(world):
        for j, (d, r) in enumerate(dims):
            want = shard(total[j].astype(np.float32), world, q)
            assert np.array_equal(acc[q][j].view(np.uint32), want.view(np.uint32))


# ---------------------------------------------------- bf16 gradient shards (G41)
def test_rs_bf16_shards_hand_ties():
    """N = 2, one element: the fp32 mean is exact, the bf16 cast is one RNE
    rounding.  (1.0 + 1.0078125) / 2 = 1 + 2^-8 lies halfway between bf16
    1.0 (0x3F80, even) and 1.0078125 (0x3F81): -> 0x3F80.
    (1.0078125 + 1.015625) / 2 = 1 + 3 * 2^-8 lies halfway between 0x3F81 and
    0x3F82 (even): -> 0x3F82.  1.0 and 3.0 -> 2.0 exactly (0x4000)."""
    from oracle.collectives import rs_copyout_bf16
    for a, b, want in ((0x3F80, 0x3F81, 0x3F80), (0x3F81, 0x3F82, 0x3F82), (0x3F80, 0x4040, 0x4000)):
        g = [[np.array([[a]], dtype=np.uint16)], [np.array([[b]], dtype=np.uint16)]]
        _, outs, _ = bucketed_reduce_scatter(g, 2, 16)
        got = [rs_copyout_bf16(o, [(1, 1)], 2, 16) for o in outs]
        assert int(got[0][0][0, 0]) == want      # rank 0 owns the only row
        assert got[1][0].shape == (1, 1) and int(got[1][0][0, 0]) == 0   # rank 1: one pad row, +0


@given(dims=dims_st, k=st.integers(0, 3), seed=st.integers(0, 2**31))
@settings(max_examples=100, deadline=None)
def test_rs_bf16_shards_are_one_rounding_of_the_exact_mean(dims, k, seed):
    """Exact-representable data at N = 2^k: the fp32 RS result is the exact
    mean, so the bf16 shard must be the exact mean correctly rounded to bf16
    (torch's float -> bfloat16 conversion of the fp64 mean, a library routine)."""
    import torch
    from oracle.collectives import rs_copyout_bf16
    world = 2 ** k
    rng = np.random.Generator(np.random.Philox(seed))
    ks = [[rng.integers(-256, 257, size=(d, r)) for d, r in dims] for _ in range(world)]
    g = [[(((x.astype(np.float32) * np.float32(2 ** -8)).view(np.uint32)) >> 16).astype(np.uint16) for x in kr]
         for kr in ks]
    _, outs, _ = bucketed_reduce_scatter(g, world, 16)
    for q in range(world):
        got = rs_copyout_bf16(outs[q], dims, world, 16)
        for j, (d, r) in enumerate(dims):
            mean = sum(ks[rr][j].astype(np.float64) for rr in range(world)) * 2.0 ** -8 / world
            want = torch.from_numpy(shard(mean, world, q)).to(torch.float32).to(torch.bfloat16).view(torch.int16)
            assert np.array_equal(got[j].view(np.int16), want.numpy())
