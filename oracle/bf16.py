"""O1 -- bf16 codec (test infrastructure; see oracle/__init__.py).

Mixed precision: parameters travel in ``param_dtype`` (bf16)
and gradients are reduced in ``reduce_dtype`` (fp32).  bf16 values are held as
``uint16`` bit patterns so that comparisons are bit comparisons.

widen  : bf16 -> fp32 is exact: the bf16 pattern is the high half of the fp32
         pattern.
narrow : fp32 -> bf16 round-to-nearest-even on the bit pattern
         (u + 0x7FFF + ((u >> 16) & 1)) >> 16; NaN maps to a quiet NaN whose
         payload is unspecified (G27: NaNs are compared by class).
"""
import numpy as np


def widen(u16):
    """bf16 bit patterns (uint16) -> float32, exact."""
    u16 = np.asarray(u16, dtype=np.uint16)
    return (u16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def narrow(f32):
    """float32 -> bf16 bit patterns (uint16), round to nearest, ties to even."""
    f32 = np.asarray(f32, dtype=np.float32)
    u = f32.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    nan = np.isnan(f32)
    if nan.any():
        sign = ((u >> np.uint64(16)) & np.uint64(0x8000)).astype(np.uint16)
        r = np.where(nan, sign | np.uint16(0x7FC0), r).astype(np.uint16)
    return r
