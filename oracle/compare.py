"""Full engine-vs-oracle comparison -- TEST INFRASTRUCTURE ONLY (the checker).

Compares everything the reference's analyze / estimate / attribute produce
(detectors.py:274-326, estimator.py:51-151, report.py:44-95) between the
engine's columnar results (paper_2601_12713_b200.analysis.ColumnarFindings /
ColumnarSavings, index-based) and the oracle restatement (analysis_ref):

  findings   DD groups + members, RT groups + trips, alloc/delete pairs (incl.
             synthetic deletes), RA groups, UA pairs, UT events -- all in the
             reference's orders
  warnings   unmatched deletes, chronological (prep.py:73-76)
  estimate   per-category eliminable ns, union ns, the eliminable event set,
             the overlap flag (estimator.py:51-58)
  attribute  rows (category, first member, count, total_ns, total_bytes) in
             report order (-total_ns, location key)

Used by tests/ and by bench.py's `verified` flag (outside timed regions).
"""
from __future__ import annotations

from . import analysis_ref as R

SYNTH_IDX = 0xFFFFFFFF


def _engine_findings(cf):
    off, mem = cf.dd_offsets.tolist(), cf.dd_members.tolist()
    dd = [mem[off[g]:off[g + 1]] for g in range(len(off) - 1)]
    off, tx, rx = cf.rt_offsets.tolist(), cf.rt_tx.tolist(), cf.rt_rx.tolist()
    rt = [list(zip(tx[off[g]:off[g + 1]], rx[off[g]:off[g + 1]])) for g in range(len(off) - 1)]
    pairs = [(a, R.SYNTH if d == SYNTH_IDX else d) for a, d in zip(cf.pair_alloc.tolist(), cf.pair_delete.tolist())]
    off, rp = cf.ra_offsets.tolist(), cf.ra_pairs.tolist()
    ra = [rp[off[g]:off[g + 1]] for g in range(len(off) - 1)]
    return dict(dd=dd, rt=rt, pairs=pairs, ra=ra, ua=cf.ua_pairs.tolist(), ut=cf.ut_events.tolist(),
                warnings=cf.warn_index.tolist())


def _oracle_findings(rf):
    return dict(dd=[list(m) for _, _, m in rf.dd], rt=[[tuple(t) for t in tr] for *_, tr in rf.rt],
                pairs=[tuple(p) for p in rf.pairs], ra=[list(ps) for *_, ps in rf.ra], ua=list(rf.ua),
                ut=list(rf.ut), warnings=list(rf.warnings))


def engine_attribute_rows(cols, sv):
    """ColumnarSavings attribution arrays -> report.py:73-95 rows (category, first member event,
    count, total_ns, total_bytes), sorted per category by (-total_ns, location key)."""
    rows = []
    for c, cat in enumerate(R.CATEGORIES):
        cr = []
        for b in range(sv.attr_count.shape[1]):
            cnt = int(sv.attr_count[c, b])
            if not cnt:
                continue
            first = int(sv.attr_first[c, b]) & 0xFFFFFFFF
            cr.append((cat, first, cnt, sv.attr_ns[c][b], sv.attr_bytes[c][b], cols.bucket_keys[b]))
        cr.sort(key=lambda r: (-r[3], r[5]))
        rows.extend(r[:5] for r in cr)
    return rows


def full_parity(cols, cf, sv, rf=None, strict=False):
    """List of mismatch descriptions (empty = engine equals the oracle on every output)."""
    if rf is None:
        rf = R.analyze_cols(cols, strict=strict)
    bad = []
    e, o = _engine_findings(cf), _oracle_findings(rf)
    for k in ("dd", "rt", "pairs", "ra", "ua", "ut", "warnings"):
        if e[k] != o[k]:
            n = next((i for i, (a, b) in enumerate(zip(e[k], o[k])) if a != b), min(len(e[k]), len(o[k])))
            bad.append(f"{k}: engine {len(e[k])} vs oracle {len(o[k])} entries, first difference at {n}")
    if sv is None:
        return bad
    est = R.estimate_cols(cols, rf, cols.wall_time_ns)
    if sv.per_category_ns != est["per_category_ns"]:
        bad.append(f"per_category_ns: {sv.per_category_ns} vs {est['per_category_ns']}")
    union_raw = sum(int(cols.end_ns[i]) - int(cols.start_ns[i]) for i in est["eliminable"])
    if sv.union_ns != union_raw:
        bad.append(f"union_ns: {sv.union_ns} vs {union_raw}")
    if sorted(sv.union_index.tolist()) != est["eliminable"]:
        bad.append("eliminable set differs")
    ov = any(w.startswith("trace contains overlapping") for w in est["warnings"])
    if bool(sv.has_overlaps) != ov:
        bad.append(f"has_overlaps: {sv.has_overlaps} vs {ov}")
    want = [r[:5] for r in R.attribute_cols(cols, rf, cols.wall_time_ns)]
    got = engine_attribute_rows(cols, sv)
    if got != want:
        bad.append(f"attribute rows differ ({len(got)} vs {len(want)})")
    return bad
