"""CPU: the measurement models bench.py reports next to the timings (no GPU):
the SURVEY §8(d) algorithmic-byte model per launch and the L2 request model
(DESIGN §4), checked against hand-computed values for the C4 / C5 shapes."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

E4, N4 = 114_228_325, 232_965


def test_gathered_rows_per_kernel():
    # GAT 8x8: V (256 B) + el (32 B) in fwd / pass A; dO + records (128 B) in pass B
    assert bench.gathered_rows("fwd", "gat", 8, 8) == [256, 32]
    assert bench.gathered_rows("bwd_rows", "gat", 8, 8) == [256, 32]
    assert bench.gathered_rows("bwd_cols", "gat", 8, 8) == [256, 128]
    # GT 8x16: V + Q (512 B each); pass B dO + K + records
    assert bench.gathered_rows("fwd", "gt", 8, 16) == [512, 512]
    assert bench.gathered_rows("bwd_cols", "gt", 8, 16) == [512, 512, 128]


def test_l2_request_model_c4():
    a, b = 2.48, 1.02  # ps per 128 B line / per 32 B sector (probe fit, profiles/README.md)
    # fwd: V = 2 lines + 8 sectors, el = 1 line + 1 sector
    want = E4 * (3 * a + 9 * b) * 1e-9
    assert bench.l2_request_model_ms("fwd", "gat", 8, 8, E4, a, b) == pytest.approx(want)
    assert want == pytest.approx(1.90, abs=0.01)
    # pass B: dO 2 lines + 8 sectors, record 1 line + 4 sectors
    want_b = E4 * (3 * a + 12 * b) * 1e-9
    assert bench.l2_request_model_ms("bwd_cols", "gat", 8, 8, E4, a, b) == pytest.approx(want_b)


def test_algorithmic_bytes_c4():
    # SURVEY §8(d) gather model (DESIGN §4 table): 33.4 / 33.5 / 44.5 GB per launch
    got = {k: bench.algorithmic_bytes(k, "gat", N4, E4, 8, 8) / 1e9
           for k in ("fwd", "bwd_rows", "bwd_cols")}
    assert got["fwd"] == pytest.approx(33.4, abs=0.1)
    assert got["bwd_rows"] == pytest.approx(33.5, abs=0.1)
    assert got["bwd_cols"] == pytest.approx(44.5, abs=0.1)


def test_layer_form_models():
    """GAT layer form (GF_FLAG_LOGITS_FROM_V): no el gather in fwd / pass A."""
    assert bench.gathered_rows("fwd", "gat", 8, 8, from_v=True) == [256]
    assert bench.gathered_rows("bwd_rows", "gat", 8, 8, from_v=True) == [256]
    assert bench.gathered_rows("bwd_cols", "gat", 8, 8, from_v=True) == [256, 128]
    full = bench.algorithmic_bytes("fwd", "gat", N4, E4, 8, 8)
    lay = bench.algorithmic_bytes("fwd", "gat", N4, E4, 8, 8, from_v=True)
    assert full - lay == 4 * E4 * 8 - 4 * N4 * (64 - 8)  # el per edge gone; own V row per node
