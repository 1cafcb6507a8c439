"""The 1-bf16-ulp comparator the bf16 gradient-shard parity uses (G41), pinned
against the bf16 number line (ml_dtypes.nextafter)."""
import ml_dtypes
import numpy as np

from tests.gpu_util import bf16_ulp_distance


def test_ulp_distance_on_the_bf16_number_line():
    bf = ml_dtypes.bfloat16
    xs = np.array([0.0, -0.0, 1.0, -1.0, 3.5e-40, 1e38, -2.5], dtype=np.float32).astype(bf)
    up = np.nextafter(xs, np.array(np.inf, dtype=bf))
    assert np.all(bf16_ulp_distance(xs.view(np.uint16), up.view(np.uint16)) == 1)
    assert np.all(bf16_ulp_distance(xs.view(np.uint16), xs.view(np.uint16)) == 0)
    # +0 / -0 are the same point; the smallest subnormals of either sign are 2 apart
    assert bf16_ulp_distance(np.uint16(0x0000), np.uint16(0x8000)) == 0
    assert bf16_ulp_distance(np.uint16(0x0001), np.uint16(0x8001)) == 2
    # 1.0 -> 2.0 spans the 128 mantissa steps of one binade
    assert bf16_ulp_distance(np.uint16(0x3F80), np.uint16(0x4000)) == 128
