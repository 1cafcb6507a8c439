"""O2 / O3 pins: sharding against torch.chunk (library routine), the invariant
concat_r(shard_r[:v_r]) == p, SPEC worked examples; layout invariants and
the A = 1 special case that reduces to np.concatenate."""
import numpy as np
import torch
from hypothesis import given, settings, strategies as st

from oracle.layout import bucket_layout
from oracle.shard import shard, shard_rows
from oracle.collectives import ag_pack


@given(d=st.integers(1, 300), r=st.integers(1, 5), world=st.integers(1, 9))
@settings(max_examples=300, deadline=None)
def test_shard_matches_torch_chunk_and_reassembles(d, r, world):
    p = np.arange(d * r, dtype=np.int64).reshape(d, r)
    chunks = list(torch.chunk(torch.from_numpy(p), world, dim=0))
    chunks += [torch.empty(0, r, dtype=torch.int64)] * (world - len(chunks))
    vs = []
    for q in range(world):
        c, begin, v = shard_rows(d, world, q)
        s = shard(p, world, q)
        assert s.shape == (c, r)
        assert np.array_equal(s[:v], chunks[q].numpy())
        assert np.all(s[v:] == 0)
        vs.append(v)
    assert sum(vs) == d
    assert all(a >= b for a, b in zip(vs, vs[1:]))  # non-increasing
    assert np.array_equal(np.concatenate([shard(p, world, q)[:vs[q]] for q in range(world)]), p)


def test_shard_zero_row_rank():
    # 13 rows over 8 ranks: c = 2 -> valid rows 2,2,2,2,2,2,1,0 (torch.chunk gives 7 chunks)
    assert [shard_rows(13, 8, q)[2] for q in range(8)] == [2, 2, 2, 2, 2, 2, 1, 0]
    assert len(torch.chunk(torch.zeros(13), 8)) == 7


def test_spec_sharded_bytes(golden):
    for ex in golden("spec_examples.json")["sharded_param_bytes"]:
        c, _, _ = shard_rows(ex["numel"], ex["world"], 0)
        assert c * ex["elem_bytes"] == ex["bytes"], ex["cite"]


@given(dims=st.lists(st.tuples(st.integers(1, 200), st.integers(1, 70)), min_size=1, max_size=12),
       world=st.integers(1, 8), e=st.sampled_from([2, 4]), a=st.sampled_from([1, 4, 16, 128]))
@settings(max_examples=300, deadline=None)
def test_layout_invariants(dims, world, e, a):
    offs, seg = bucket_layout(dims, world, e, a)
    sizes = [-(-d // world) * r * e for d, r in dims]
    assert offs[0] == 0
    assert all(o % a == 0 for o in offs) and seg % a == 0
    for k in range(len(dims)):
        end = offs[k + 1] if k + 1 < len(dims) else seg
        assert offs[k] + sizes[k] <= end < offs[k] + sizes[k] + a  # minimal gap
    assert seg >= sum(sizes)
    if a == 1:
        assert seg == sum(sizes)  # byte conservation, tight packing


def test_pack_align1_is_concatenate():
    rng = np.random.Generator(np.random.Philox(3))
    shards = [rng.integers(0, 65535, size=(c, r)).astype(np.uint16) for c, r in [(3, 5), (1, 1), (7, 3)]]
    buf = ag_pack(shards, world=1, rank=0, align=1)
    assert np.array_equal(buf, np.concatenate([s.reshape(-1) for s in shards]).view(np.uint8))
