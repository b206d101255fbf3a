"""Columnar findings -> report, no per-event Python objects.

The reference CLI (cli.py:126-165) materialises Findings, filters them by
--min-bytes (cli.py:112-123), then estimate() / attribute() / render_*().  Here
the filter works on the engine's index arrays, the integer sums come from
b2l_savings_compute, and the two renderers below produce the reference's text and
JSON reports (report.py:98-213) from those aggregates -- byte-identical output
(tests/golden/report_cases.json.gz holds the reference's own reports).
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .analysis import CATEGORIES, INFINITE_SPEEDUP, ColumnarFindings, savings_columns

TITLES = (("DD", "Duplicate Target Data Transfer"), ("RT", "Round-Trip Target Data Transfer"),
          ("RA", "Repeated Device Memory Allocation"), ("UA", "Unused Device Memory Allocation"),
          ("UT", "Unused Data Transfer"))
REPORT_VERSION = 1


def filter_min_bytes(cols, cf: ColumnarFindings, min_bytes: int) -> ColumnarFindings:
    """cli.py:112-123 on index arrays: DD groups whose first member moved < min_bytes and RT
    trips whose send moved < min_bytes are dropped (empty RT groups with them)."""
    if min_bytes <= 1:
        return cf
    nb = cols.bytes
    off = cf.dd_offsets.astype(np.int64)
    keep = nb[cf.dd_members[off[:-1]]] >= min_bytes if off.size > 1 else np.zeros(0, bool)
    sizes = np.diff(off)[keep]
    dd_mem = np.concatenate([cf.dd_members[a:b] for a, b in zip(off[:-1][keep], off[1:][keep])]) if sizes.size \
        else np.zeros(0, np.uint32)
    dd_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    roff = cf.rt_offsets.astype(np.int64)
    tkeep = nb[cf.rt_tx] >= min_bytes
    grp = np.repeat(np.arange(roff.size - 1), np.diff(roff)) if roff.size > 1 else np.zeros(0, np.int64)
    kept_per_group = np.bincount(grp[tkeep], minlength=roff.size - 1) if roff.size > 1 else np.zeros(0, np.int64)
    rt_off = np.concatenate([[0], np.cumsum(kept_per_group[kept_per_group > 0])]).astype(np.uint64)
    return ColumnarFindings(n_events=cf.n_events, dd_offsets=dd_off, dd_members=dd_mem.astype(np.uint32),
                            rt_offsets=rt_off, rt_tx=cf.rt_tx[tkeep], rt_rx=cf.rt_rx[tkeep],
                            pair_alloc=cf.pair_alloc, pair_delete=cf.pair_delete,
                            synthetic_end_ns=cf.synthetic_end_ns, warn_index=cf.warn_index,
                            ra_offsets=cf.ra_offsets, ra_pairs=cf.ra_pairs, ua_pairs=cf.ua_pairs,
                            ut_events=cf.ut_events)


@dataclass
class Row:
    category: str
    loc: tuple          # (codeptr, file, line)
    count: int
    total_ns: int
    total_bytes: int
    pct: float


@dataclass
class Report:
    wall: int
    per_category_ns: dict
    union_ns: int
    speedup: float
    warnings: tuple
    rows: list
    counts: dict
    eliminable: int
    num_devices: int
    host_device: int
    events: int


def build_report(cols, cf: ColumnarFindings) -> Report:
    """estimator.py:61-151 + report.py:73-95 from the device aggregates."""
    sv = savings_columns(cols, cf)
    if cols.wall_time_ns is not None:
        wall = cols.wall_time_ns
    else:
        wall = (sv.max_end_ns - sv.min_start_ns) if cols.n else 0
    warnings, union = [], sv.union_ns
    if union > wall:
        warnings.append(f"eliminable time {union} ns exceeds wall time {wall} ns; clamped to wall time")
        union = wall
    if union == 0:
        speed = 1.0
    elif union == wall:
        warnings.append("eliminable time equals wall time; predicted speedup is unbounded")
        speed = INFINITE_SPEEDUP
    else:
        speed = wall / (wall - union)
    if sv.has_overlaps:
        warnings.append("trace contains overlapping event intervals; savings assume serialized "
                        "operations and may be unreliable")
    rows = []
    for c, cat in enumerate(CATEGORIES):
        cr = []
        for b in np.nonzero(sv.attr_count[c])[0].tolist():
            ev = int(sv.attr_first[c, b]) & 0xFFFFFFFF
            loc = cols.locs[int(cols.loc[ev])]
            tot = sv.attr_ns[c][b]
            cr.append(Row(cat, loc, int(sv.attr_count[c, b]), tot, sv.attr_bytes[c][b], (tot / wall) if wall else 0.0))
        cr.sort(key=lambda r: (-r.total_ns, _key(r.loc)))
        rows.extend(cr)
    return Report(wall=wall, per_category_ns=sv.per_category_ns, union_ns=union, speedup=speed,
                  warnings=tuple(warnings), rows=rows, counts=cf.counts(), eliminable=int(sv.union_index.size),
                  num_devices=cols.num_devices_total, host_device=cols.host_device, events=cols.n)


def _key(loc):
    cp, f, ln = loc
    return (0, f, ln or 0) if f is not None else (1, "", cp)


def _where(loc) -> str:
    cp, f, ln = loc
    if f is not None:
        return f"{f}:{ln}"
    return f"0x{cp:x}" if cp else "<unknown>"


def render_text(rep: Report, color: bool = False) -> str:
    b0, b1 = ("\033[1m", "\033[0m") if color else ("", "")
    out = []
    for cat, title in TITLES:
        out.append(f"{b0}=== {title} Analysis ==={b1}")
        rows = [r for r in rep.rows if r.category == cat]
        if rows:
            out.append(f"{'time(%)':>8}  {'time(ns)':>14}  {'count':>8}  {'bytes':>14}  location")
            out.extend(f"{f'{r.pct * 100:.2f}%':>8}  {r.total_ns:>14}  {r.count:>8}  {r.total_bytes:>14}  "
                       f"{_where(r.loc)}" for r in rows)
        else:
            out.append("(none detected)")
        out.append("")
    out.append(f"{b0}=== Summary ==={b1}")
    out.append(f"{'wall time (ns):':<28}{rep.wall}")
    for cat, _ in TITLES:
        n = sum(1 for r in rep.rows if r.category == cat)
        out.append(f"{f'{cat} eliminable (ns):':<28}{rep.per_category_ns[cat]}  ({n} locations)")
    out.append(f"{'union eliminable (ns):':<28}{rep.union_ns}")
    sp = "inf" if rep.speedup == INFINITE_SPEEDUP else f"{rep.speedup:.4f}x"
    out.append(f"{'predicted speedup:':<28}{sp}")
    out.extend(f"warning: {w}" for w in rep.warnings)
    out.append("")
    return "\n".join(out)


def render_json(rep: Report) -> str:
    def issue(r):
        cp, f, ln = r.loc
        return {"location": {"codeptr": cp, "file": f, "line": ln, "display": _where(r.loc)},
                "occurrence_count": r.count, "total_ns": r.total_ns, "total_bytes": r.total_bytes,
                "pct_of_wall": r.pct}
    doc = {
        "report_version": REPORT_VERSION,
        "trace": {"num_devices": rep.num_devices, "host_device": rep.host_device, "events": rep.events,
                  "wall_time_ns": rep.wall},
        "issues": {cat: [issue(r) for r in rep.rows if r.category == cat] for cat, _ in TITLES},
        "finding_counts": dict(rep.counts),
        "savings": {"per_category_ns": {cat: rep.per_category_ns[cat] for cat, _ in TITLES},
                    "union_ns": rep.union_ns, "wall_time_ns": rep.wall,
                    "predicted_speedup": None if rep.speedup == INFINITE_SPEEDUP else rep.speedup,
                    "eliminable_event_count": rep.eliminable, "warnings": list(rep.warnings)},
    }
    return json.dumps(doc, indent=2) + "\n"
