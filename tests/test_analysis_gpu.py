"""GPU parity of the trace-analysis engine (b2l_analyze / b2l_savings_compute
through the C ABI) against the reference's golden outputs and the oracle."""
import numpy as np
import pytest

from oracle import analysis_ref as R
from tests._cases import (canon_columnar, canon_findings_objects, canon_oracle, canon_ref_json, cases,
                          trace_from_json)
from tests._gen import cycle_trace_columns, nasty_trace

pytestmark = pytest.mark.gpu


def _attr_rows(rows):
    return [[r.category, [r.location.codeptr, r.location.file, r.location.line], r.occurrence_count, r.total_ns,
             r.total_bytes, repr(r.pct_of_wall)] for r in rows]


def test_golden_cases_drop_in(cuda):
    from paper_2601_12713_b200 import InvalidTrace, analyze, attribute, estimate
    for case in cases():
        tr = trace_from_json(case["trace"])
        if "violations" in case:
            with pytest.raises(InvalidTrace) as ei:
                analyze(tr)
            got = [[v.rule, v.message, v.seq] for v in ei.value.violations]
            assert got == case["violations"], case["name"]
            continue
        warns = []
        f = analyze(tr, warn=warns.append)
        assert canon_findings_objects(f) == canon_ref_json(case["findings"]), case["name"]
        assert [[w.seq, w.reason] for w in warns] == case["warnings"], case["name"]
        fs = analyze(tr, strict_pseudocode=True)
        assert canon_findings_objects(fs) == canon_ref_json(case["findings_strict"]), case["name"]
        s = estimate(tr, f)
        e = case["estimate"]
        assert s.per_category_ns == e["per_category_ns"], case["name"]
        assert (s.union_ns, s.wall_time_ns) == (e["union_ns"], e["wall_time_ns"]), case["name"]
        assert repr(s.predicted_speedup) == e["predicted_speedup"], case["name"]
        assert sorted(s.eliminable_seqs) == e["eliminable_seqs"], case["name"]
        assert list(s.warnings) == e["warnings"], case["name"]
        assert _attr_rows(attribute(tr, f)) == case["attribute"], case["name"]


def test_engine_matches_oracle_on_nasty_traces(cuda):
    from paper_2601_12713_b200 import analyze_columns, savings_columns
    from paper_2601_12713_b200.columns import to_columns
    for seed in range(1500):
        tr = nasty_trace(seed)
        cols = to_columns(tr)
        if R.validate_cols(cols):
            continue
        for strict in (False, True):
            cf = analyze_columns(cols, strict=strict)
            rf = R.analyze_cols(cols, strict=strict)
            assert canon_columnar(cf, cols) == canon_oracle(rf, cols), (seed, strict)
            assert cf.warn_index.tolist() == rf.warnings, seed
        sv = savings_columns(cols, cf)
        est = R.estimate_cols(cols, rf, tr.wall_time_ns)
        assert sv.per_category_ns == est["per_category_ns"], seed
        assert sorted(sv.union_index.tolist()) == est["eliminable"], seed


def test_columnar_c2_shaped_trace_vs_oracle(cuda):
    from oracle.compare import full_parity
    from paper_2601_12713_b200 import analyze_columns, savings_columns
    from paper_2601_12713_b200.synth import with_locations
    cols = with_locations(cycle_trace_columns(200_000, seed=5))
    cf = analyze_columns(cols)
    sv = savings_columns(cols, cf)
    assert full_parity(cols, cf, sv) == []
    assert cf.counts()["DD"] > 0 and cf.counts()["RT"] > 0 and cf.counts()["RA"] > 0


def test_invalid_events_flagged_in_order(cuda):
    from paper_2601_12713_b200 import InvalidTrace, analyze
    from paper_2601_12713_b200 import types as T
    ev = [T.TraceEvent(5, T.EventKind.TRANSFER, 10, 5, 0, 9, 0, 0, 8, 0),
          T.TraceEvent(4, T.EventKind.ALLOC, 3, 4, 0, 1, 0, 0, 0, 0, T.CodeLocation(1, "x.c", None))]
    with pytest.raises(InvalidTrace) as ei:
        analyze(T.Trace(1, 2, 0, None, ev))
    got = [(v.rule, v.message, v.seq) for v in ei.value.violations]
    assert got == [("interval", "start_ns 10 > end_ns 5", 5), ("device", "dst_device=9 out of range [0,2)", 5),
                   ("transfer", "non-empty transfer has no content hash", 5),
                   ("alloc", "allocation of zero bytes", 4), ("alloc", "allocation with null device address", 4),
                   ("location", "file present but line missing", 4),
                   ("order", "events not sorted by (start_ns, seq)", 4),
                   ("order", "seq values not strictly increasing", 4)]


def test_unrepresentable_values_rejected_with_reference_messages(cuda):
    from paper_2601_12713_b200 import InvalidTrace, analyze
    from paper_2601_12713_b200 import types as T
    e = T.TraceEvent(0, T.EventKind.ALLOC, 0, 1, 0, 1, 0, 0xD00, -1, 0)
    with pytest.raises(InvalidTrace) as ei:
        analyze(T.Trace(1, 2, 0, None, [e]))
    assert [(v.rule, v.seq) for v in ei.value.violations] == [("field-range", 0), ("alloc", 0)]


def test_foreign_findings_mismatch(cuda):
    from paper_2601_12713_b200 import FindingsTraceMismatch, analyze, estimate
    from paper_2601_12713_b200 import types as T
    tr = nasty_trace(3)
    f = analyze(tr)
    other = T.Trace(1, tr.num_devices_total, tr.host_device, None, tr.events[:1])
    if f.unused_transfers or f.duplicates:
        with pytest.raises(FindingsTraceMismatch):
            estimate(other, f)


def test_analyze_many_pipelined_matches_single_calls(cuda):
    """analyze_many (upload of trace k+1 overlapped with the analysis of trace k) gives, per
    trace and in order, exactly the single-call results."""
    from oracle.compare import full_parity
    from paper_2601_12713_b200 import analyze_many
    from paper_2601_12713_b200.analysis import pinned_columns
    from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace
    traces = [pinned_columns(c2_trace(20_000, seed=5)), c4_trace(30_000, seed=6), c3_trace(500),
              pinned_columns(c2_trace(5, seed=1))]
    got = list(analyze_many(traces))
    assert len(got) == len(traces)
    for cols, (cf, sv) in zip(traces, got):
        assert full_parity(cols, cf, sv) == []
    # later calls reuse the device's copy stream: a second call, and two generators interleaved
    g1, g2 = analyze_many(traces[::-1]), analyze_many(traces)
    for a, b, ca, cb in zip(g1, g2, traces[::-1], traces):
        assert full_parity(ca, *a) == [] and full_parity(cb, *b) == []


def test_fused_savings_packed_records_and_fallback(cuda):
    """Fused analyze + savings (B2L_ANALYZE_WITH_SAVINGS): attribution reads the front pass's
    packed per-event records; a duration >= 2^40 ns cannot be packed and takes the column gathers."""
    from oracle.compare import full_parity
    from paper_2601_12713_b200 import analyze_columns, savings_columns
    from paper_2601_12713_b200.columns import to_columns
    checked = huge = 0
    for seed in range(300):
        cols = to_columns(nasty_trace(seed))
        if R.validate_cols(cols):
            continue
        cf = analyze_columns(cols, with_savings=True)
        assert full_parity(cols, cf, savings_columns(cols, cf)) == [], seed
        checked += 1
        if seed % 10 == 0 and cols.end_ns.size:
            cols.end_ns[cols.end_ns.size // 2] += np.uint64(1 << 41)  # one very long event
            if R.validate_cols(cols):
                continue
            cf = analyze_columns(cols, with_savings=True)
            assert full_parity(cols, cf, savings_columns(cols, cf)) == [], ("huge", seed)
            huge += 1
    assert checked > 100 and huge > 5
