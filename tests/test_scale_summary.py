"""CPU check of tools/scale_summary.py (the table maker for the first
multi-GPU run): it reads bench.py's N > 1 JSON line keys."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import scale_summary as S  # noqa: E402


def test_summary_tables(tmp_path):
    line = {"ms_per_step": 60.1, "value": 5000.0, "value_kind": "bus",
            "parity": {"ok": True, "ag": {"bit_exact": True}, "rs": {"max_err_over_bound": 0.2, "pad_nonzero": 0}},
            "busbw_block": {"ag_GBps": 700.0, "rs_GBps": 690.0, "ag_frac_nvlink": 0.778, "rs_frac_nvlink": 0.767,
                            "ag_frac_measured_peer": 0.909, "rs_frac_measured_peer": 0.896},
            "alpha_beta": {"ag": {"alpha_ns": 15000, "beta_fs_per_byte": 1300},
                           "rs": {"alpha_ns": 16000, "beta_fs_per_byte": 1350}, "source": "measured at this N"},
            "exposure": {"variants": {"vanilla": {"buckets_fwd": 291, "buckets_bwd": 291, "step_ms": 150.0,
                                                  "compute_only_ms": 60.0, "exposed_ms": 90.0,
                                                  "predicted_exposed_ms": 85.0}}},
            "nvls_block": {"unavailable": "multicast object refused"}}
    (tmp_path / "bench_flat_N8.json").write_text("noise\n" + json.dumps(line) + "\n")
    rows = S.load(str(tmp_path))
    assert len(rows) == 1 and rows[0][:2] == ("flat", 8)
    md = S.summary(rows)
    assert "| flat | 8 | 60.100 | 5000.0 | bus | True | True | 0.200 | True |" in md
    assert "| flat | 8 | 15000 | 1300 | 16000 | 1350 |" in md
    assert "| flat | 8 | vanilla | 291 / 291 | 150.000 | 60.000 | 90.000 | 85.000 |" in md
    assert "unavailable: multicast object refused" in md
