"""Host helpers of the measurement harness (no GPU): the compute proxy's
affine calibration model and the CTA counts of the emulated collectives."""
import pytest

pytest.importorskip("paper_2411_00284_b200._lib", reason="libfsdp_b200.so not built")

from paper_2411_00284_b200 import harness as H  # noqa: E402


def test_proxy_iters_affine_model():
    # (ns per iteration, fixed ns): the fixed part comes off long ops; short ops keep half their time
    assert H.proxy_iters([0, 1000, 100000], (2.0, 10000.0)) == [0, 250, 45000]
    # a plain ns-per-iteration (the old ratio model) still works
    assert H.proxy_iters([4000], 4.0) == [1000]


def test_emulation_cta_counts():
    # enough CTAs (~29 GB/s each) for the RS's HBM traffic at the modelled bus rate
    assert [H.emulation_ctas(n) for n in (1, 2, 4, 8)] == [32, 75, 42, 32]
    # paced K8 / K9: 2 x the bucket of local HBM traffic within the link time
    assert H.emulation_ctas_p2p(8) == 57
    assert H.emulation_ctas_p2p(2) == 100
    assert all(32 <= H.emulation_ctas(n) <= 148 and 32 <= H.emulation_ctas_p2p(n) <= 148 for n in range(1, 17))
