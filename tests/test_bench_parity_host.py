"""CPU tests of bench.py's N > 1 verification leg (the host side of its
sampled oracle parity), so that the first multi-GPU run's `parity` field can be
trusted:

* the element-wise expectations it builds (expected_ag_rows: O2/O4 one row at
  a time; expected_rs_rows: O5 on a small bucket of the sampled rows) equal the
  oracle's full-size all-gather / reduce-scatter at those rows, for uneven
  dim 0 and zero-row ranks;
* over a real world-2/3 gloo process group, ag_check / rs_check exchange each
  rank's rows and accept correct results, flag a single flipped bit, accept a
  reordered fp32 sum within G7's bound only where bit-exactness is not
  required (NCCL at N > 2), and reject it where it is (K9, or N <= 2).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench as B
from oracle import bf16 as OB
from oracle.collectives import bucketed_all_gather, bucketed_reduce_scatter
from oracle.shard import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def _bf16(rng, shape, std):
    return OB.narrow(rng.normal(0.0, std, size=shape).astype(np.float32))


@pytest.mark.parametrize("d,R,world", [(13, 5, 8), (71, 33, 2), (10, 4, 3), (4096, 3, 8), (7, 1, 3)])
def test_expected_ag_rows_equal_the_oracle_gather(d, R, world):
    p = _bf16(_rng(d * R), (d, R), 0.02)
    _, full = bucketed_all_gather([p], world, 16)
    c = -(-d // world)
    loc = B.sample_local_rows(c, 5)
    rows = sorted({q * c + t for q in range(world) for t in loc if q * c + t < d})
    by_rank = [{t: shard(p, world, q)[t].tobytes() for t in loc} for q in range(world)]
    exp = B.expected_ag_rows(d, world, rows, by_rank)
    assert sorted(exp) == rows
    for g in rows:
        assert exp[g] == full[0][g].tobytes()


@pytest.mark.parametrize("d,R,world", [(13, 5, 8), (71, 33, 2), (10, 4, 3), (300, 7, 5), (7, 1, 3)])
def test_expected_rs_rows_equal_the_oracle_reduce_scatter(d, R, world):
    rng = _rng(d + R + world)
    grads = [_bf16(rng, (d, R), 1e-3) for _ in range(world)]
    _, _, shards = bucketed_reduce_scatter([[g] for g in grads], world, 16)
    c = -(-d // world)
    loc = B.sample_local_rows(c, 9)
    for rank in range(world):
        own = [t for t in loc if rank * c + t < d]
        if not own:
            continue
        rows = {g: None for q in range(world) for t in loc for g in [q * c + t] if g < d}
        by_rank = [{g: grads[q][g] for g in rows} for q in range(world)]
        exp, scale = B.expected_rs_rows(d, R, world, rank, loc, by_rank)
        sel = [loc.index(t) for t in own]
        assert np.array_equal(exp[sel].view(np.uint32), shards[rank][0][own].view(np.uint32))
        assert np.all(scale >= 0)


def test_sample_rows_cover_chunk_ends():
    assert B.sample_local_rows(3, 1) == [0, 1, 2]
    r = B.sample_local_rows(1000, 1)
    assert r[0] == 0 and r[-1] == 999 and len(r) <= 6 and r == sorted(set(r))
    assert B.sample_buckets(35) == [0, 1, 17, 33, 34] and B.sample_buckets(1) == [0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _members(world, rank, params, grads, corrupt_ag, order):
    """Fabricate what parity_leg reads on a rank from oracle-computed results:
    gathered rows (optionally one flipped bit) and gradient-shard rows summed in
    `order` ('rank' = the oracle's order, 'reverse' = another valid order)."""
    ag, rs = [], []
    for key, p in enumerate(params):
        d, R = p.shape
        c = -(-d // world)
        loc = B.sample_local_rows(c, 100 + key)
        grows = sorted({q * c + t for q in range(world) for t in loc if q * c + t < d})
        own = [t for t in loc if rank * c + t < d]
        got = {g: p[g].tobytes() for g in grows}
        if corrupt_ag and key == 0 and grows:
            row = p[grows[-1]].copy()
            row[0] ^= 1
            got[grows[-1]] = row.tobytes()
        ag.append({"key": key, "d": d, "ep": 2, "own": {t: shard(p, world, rank)[t].tobytes() for t in own},
                   "got": got})
        inv = np.float32(1.0) / np.float32(world)
        qs = list(range(world)) if order == "rank" else list(range(world - 1, -1, -1))
        out = np.zeros((len(own), R), dtype=np.float32)
        for i, t in enumerate(own):
            acc = None
            for q in qs:
                v = (OB.widen(grads[q][key][rank * c + t]) * inv).astype(np.float32)
                acc = v if acc is None else (acc + v).astype(np.float32)
            out[i] = acc
        rs.append({"key": key, "d": d, "R": R, "loc": loc, "own": own,
                   "grads": {g: grads[rank][key][g].copy() for g in grows}, "got": out})
    return ag, rs


def _check_worker(rank, world, port, errq, case, p2p, want_ok):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)

        def exchange(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
        rng = _rng(7)
        shapes = [(13, 5), (4096, 1), (10, 33), (7, 64)]
        params = [_bf16(rng, s, 0.02) for s in shapes]
        # large-magnitude, mixed-sign gradients so that summation order changes bits
        grads = [[_bf16(_rng(100 * q + k), s, 1.0) for k, s in enumerate(shapes)] for q in range(world)]
        ag_m, rs_m = _members(world, rank, params, grads, case == "flip_ag", "reverse" if case == "reorder" else "rank")
        ag = {"elements": 0, "mismatches": 0}
        rs = {"elements": 0, "mismatches": 0, "max_err_over_bound": 0.0}
        B.ag_check(world, rank, ag_m, exchange, ag)
        B.rs_check(world, rank, rs_m, exchange, rs)
        ok, _ = B.parity_verdict(ag, rs, world, p2p)
        oks = exchange(ok)
        assert all(o == want_ok for o in oks), (case, oks, ag, rs)
        if case == "reorder":
            assert rs["max_err_over_bound"] <= 1.0
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        errq.put("rank %d: %s\n%s" % (rank, e, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world,case,p2p,want_ok", [
    (2, "correct", False, True),
    (3, "correct", True, True),
    (3, "flip_ag", False, False),
    (3, "reorder", False, True),    # NCCL at N = 3: another order is fine within G7
    (3, "reorder", True, False),    # K9 must reproduce the oracle's rank order bit for bit
])
def test_parity_checks_over_gloo(world, case, p2p, want_ok):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_check_worker, args=(r, world, port, errq, case, p2p, want_ok)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]


def test_mirror_plan_for_the_peer_memory_path():
    """The peer-memory path keeps one shard layout, so when Algorithm 1's two
    phase plans differ the backward re-gathers the forward's buckets, in the
    backward execution order (parameters in reverse)."""
    from paper_2411_00284_b200 import harness as H
    fwd = [[0], [1, 2], [3, 4, 5], [6]]
    bwd = [[6, 5], [4, 3, 2], [1, 0]]
    assert not H.same_buckets(fwd, bwd)
    m = H.mirror_plan(fwd)
    assert m == [[6], [5, 4, 3], [2, 1], [0]]
    assert H.same_buckets(fwd, m)
    assert [j for b in m for j in b] == list(range(6, -1, -1))
