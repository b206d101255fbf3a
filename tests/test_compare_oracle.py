"""The checker itself (oracle/compare.py): oracle-derived columnar findings compare equal,
and a perturbed result is reported (CPU only)."""
import numpy as np

from oracle import analysis_ref as R
from oracle.compare import SYNTH_IDX, full_parity
from paper_2601_12713_b200.analysis import ColumnarFindings
from paper_2601_12713_b200.synth import c4_trace, with_locations


def _columnar(rf, n):
    u32 = lambda x: np.array(x, dtype=np.uint32)  # noqa: E731
    off = lambda gs: np.cumsum([0] + [len(g) for g in gs]).astype(np.uint64)  # noqa: E731
    dd = [m for *_, m in rf.dd]
    rt = [t for *_, t in rf.rt]
    ra = [p for *_, p in rf.ra]
    return ColumnarFindings(
        n_events=n, dd_offsets=off(dd), dd_members=u32([i for m in dd for i in m]), rt_offsets=off(rt),
        rt_tx=u32([a for t in rt for a, _ in t]), rt_rx=u32([b for t in rt for _, b in t]),
        pair_alloc=u32([a for a, _ in rf.pairs]),
        pair_delete=u32([SYNTH_IDX if d == R.SYNTH else d for _, d in rf.pairs]), synthetic_end_ns=rf.synthetic_end,
        warn_index=u32(rf.warnings), ra_offsets=off(ra), ra_pairs=u32([p for g in ra for p in g]),
        ua_pairs=u32(rf.ua), ut_events=u32(rf.ut))


def test_checker_accepts_oracle_and_flags_perturbations():
    cols = with_locations(c4_trace(20_000, seed=9), seed=9)
    rf = R.analyze_cols(cols)
    cf = _columnar(rf, cols.n)
    assert full_parity(cols, cf, None, rf=rf) == []
    cf.ut_events = cf.ut_events[:-1]
    assert any(m.startswith("ut:") for m in full_parity(cols, cf, None, rf=rf))
    cf = _columnar(rf, cols.n)
    cf.rt_rx = cf.rt_rx.copy()
    cf.rt_rx[0] += 1
    assert any(m.startswith("rt:") for m in full_parity(cols, cf, None, rf=rf))
