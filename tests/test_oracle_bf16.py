"""O1 pins: the oracle's bf16 codec against an independent library (ml_dtypes)
and torch's CPU cast -- special cases that reduce to a library routine."""
import ml_dtypes
import numpy as np
import torch

from oracle import bf16
from workloads.data import EDGE_F32_BITS


def _ml_narrow(f32):
    return np.asarray(f32, dtype=np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)


def test_widen_exhaustive():
    u = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = bf16.widen(u)
    ref = u.view(ml_dtypes.bfloat16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))


def test_narrow_ties_every_exponent():
    # every bf16 high half with the low half at each rounding boundary
    hi = np.arange(65536, dtype=np.uint32) << np.uint32(16)
    lows = np.array([0x0000, 0x0001, 0x7FFF, 0x8000, 0x8001, 0xFFFF], dtype=np.uint32)
    bits = (hi[:, None] | lows[None, :]).reshape(-1)
    f = bits.view(np.float32)
    keep = ~np.isnan(f)
    assert np.array_equal(bf16.narrow(f[keep]), _ml_narrow(f[keep]))


def test_narrow_random_sample_vs_ml_dtypes_and_torch():
    rng = np.random.Generator(np.random.Philox(7))
    bits = rng.integers(0, 2**32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    f = bits.view(np.float32)
    keep = ~np.isnan(f)
    ours = bf16.narrow(f[keep])
    assert np.array_equal(ours, _ml_narrow(f[keep]))
    t = torch.from_numpy(f[keep].copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, t)


def test_narrow_edges():
    f = EDGE_F32_BITS.view(np.float32)
    out = bf16.narrow(f)
    nan = np.isnan(f)
    # NaN -> some quiet NaN (class compare, G27)
    assert np.all(np.isnan(bf16.widen(out[nan])))
    assert np.array_equal(out[~nan], _ml_narrow(f[~nan]))
    # 0x7F7FFFFF (fp32 max) rounds up to +inf in bf16
    assert bf16.narrow(np.array([0x7F7FFFFF], np.uint32).view(np.float32))[0] == 0x7F80
    # signed zeros survive
    assert bf16.narrow(np.array([-0.0], np.float32))[0] == 0x8000
