"""Engine vs oracle at the benchmark configurations' shapes, every output
compared (oracle/compare.full_parity: findings, warnings, per-category / union sums, the
eliminable set, the overlap flag, attribution rows), both RT modes.

  C3  stencil time loop (1 target device, round trip per iteration): 10k iterations =
      30,004 events -- every hashed transfer lands in one device queue, RT strict walks it
  C4  allocation-heavy (UA / UT / RA populated; 65,536-hash palette -> long equal-hash runs
      that take the segmented fix-up's long-run path), 200k and 1M events
  C2  1M-event cycle trace with code locations (attribution over many buckets)
Reference semantics: detectors.py:85-326, prep.py:45-96, estimator.py:51-151, report.py:44-95.
"""
import pytest

from oracle import analysis_ref as R
from oracle.compare import full_parity

pytestmark = pytest.mark.gpu


def _check(cols, strict):
    """Both savings paths: separate (b2l_savings_compute) and fused into the analyze call
    (B2L_ANALYZE_WITH_SAVINGS, categories fed in as the detector chains finish)."""
    from paper_2601_12713_b200 import analyze_columns, savings_columns
    cf = analyze_columns(cols, strict=strict)
    sv = savings_columns(cols, cf)
    rf = R.analyze_cols(cols, strict=strict)
    assert full_parity(cols, cf, sv, rf=rf) == []
    cf2 = analyze_columns(cols, strict=strict, with_savings=True)
    assert cf2._handle.ptr.contents.internal  # the fused results ride on the findings
    sv2 = savings_columns(cols, cf2)
    assert full_parity(cols, cf2, sv2, rf=rf) == []
    return cf, rf


@pytest.mark.parametrize("strict", [False, True])
def test_c3_stencil_vs_oracle(cuda, strict):
    from paper_2601_12713_b200.synth import c3_trace, with_locations
    cols = with_locations(c3_trace(10_000), n_locs=6, seed=3)
    cf, rf = _check(cols, strict)
    assert cf.counts()["RT"] == 10_000


@pytest.mark.parametrize("strict", [False, True])
def test_c4_alloc_heavy_200k_vs_oracle(cuda, strict):
    from paper_2601_12713_b200.synth import c4_trace, with_locations
    cols = with_locations(c4_trace(200_000, seed=4), seed=4)
    cf, rf = _check(cols, strict)
    c = cf.counts()
    assert c["UA"] > 0 and c["UT"] > 0 and c["RA"] > 0 and c["DD"] > 0 and c["RT"] > 0


def test_c4_alloc_heavy_1m_vs_oracle(cuda):
    from paper_2601_12713_b200.synth import c4_trace, with_locations
    cols = with_locations(c4_trace(1_000_000, seed=14), seed=14)
    _check(cols, False)


def test_c2_1m_with_locations_vs_oracle(cuda):
    from paper_2601_12713_b200.synth import c2_trace, with_locations
    cols = with_locations(c2_trace(1_000_000, seed=2), seed=2)
    _check(cols, False)


def test_c4_device_resident_matches_host(cuda):
    """The same trace from device-resident columns (the bench path) and from host columns."""
    from paper_2601_12713_b200 import analyze_columns, savings_columns
    from paper_2601_12713_b200.analysis import DeviceColumns
    from paper_2601_12713_b200.synth import c4_trace, with_locations
    cols = with_locations(c4_trace(300_000, seed=24), seed=24)
    d = DeviceColumns(cols, cuda)
    cf = analyze_columns(d)
    sv = savings_columns(d, cf)
    assert full_parity(cols, cf, sv) == []
    cf = analyze_columns(d, with_savings=True)
    assert full_parity(cols, cf, savings_columns(d, cf)) == []
    assert full_parity(cols, cf, savings_columns(d, cf)) == []  # second call: computed again
