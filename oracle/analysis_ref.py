"""Trace-analysis oracle -- TEST INFRASTRUCTURE ONLY (the checker, never shipped).

A sequential CPU restatement of the reference analyzer, written over the SoA
columns the engine consumes (paper_2601_12713_b200.columns.Columns) and
producing the same columnar result shape as the engine (event / pair indices),
so GPU results can be compared element by element.

Followed reference code (paths under /root/reference/pkg/src/dmlens/):
  validate_cols          model.py:125-200
  analyze_cols           detectors.py:274-326 (partition 287-318)
  _pairs                 prep.py:45-96
  _dd                    detectors.py:85-103
  _rt                    detectors.py:106-167 (default + strict_pseudocode)
  _ra                    detectors.py:170-191
  _ua                    detectors.py:194-216 (+ prep.sort_by_device 99-115)
  _ut                    detectors.py:232-271
  estimate_cols          estimator.py:51-151 (integer parts; float tail identical)
  attribute_cols         report.py:44-95

Pinned against the reference: tests/golden/analysis_cases.json holds traces
and the reference's own findings / estimate / attribute outputs
(tests/golden/make_golden.py), and test_analysis_oracle.py additionally
compares against the live reference on thousands of random traces when the
checkout is present.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

TRANSFER, ALLOC, DELETE, KERNEL = 0, 1, 2, 3
U64_MAX = 2**64 - 1
CATEGORIES = ("DD", "RT", "RA", "UA", "UT")
SYNTH = -1


@dataclass
class RefFindings:
    violations: list = field(default_factory=list)   # (rule, message, seq)
    dd: list = field(default_factory=list)           # [(hash, dst, [event idx...])]
    rt: list = field(default_factory=list)           # [(hash, src, dst, [(tx, rx)...])]
    pairs: list = field(default_factory=list)        # [(alloc idx, delete idx | SYNTH)] alloc order
    synthetic_end: int = 0
    warnings: list = field(default_factory=list)     # unmatched delete event indices
    ra: list = field(default_factory=list)           # [(src_addr, dev, bytes, [pair idx...])]
    ua: list = field(default_factory=list)           # [pair idx]
    ut: list = field(default_factory=list)           # [event idx]


def _ints(c):
    L = lambda a: [int(x) for x in a]  # noqa: E731
    return dict(seq=L(c.seq), start=L(c.start_ns), end=L(c.end_ns), src=L(c.src_device), dst=L(c.dst_device),
                kind=L(c.kind), sa=L(c.src_addr), da=L(c.dst_addr), nb=L(c.bytes), h=L(c.hash), loc=L(c.loc))


def validate_cols(c, wall_time_ns=None):
    """model.py:125-200 over columns (u64 range is guaranteed by the column types)."""
    v = []
    ndev, host = c.num_devices_total, c.host_device
    if ndev < 1:
        v.append(("header", f"num_devices_total={ndev} must be positive", None))
    if not 0 <= host < max(ndev, 1):
        v.append(("header", f"host_device={host} out of range", None))
    d = _ints(c)
    lf = [int(x) for x in c.loc_flags]
    prev_start, prev_seq = -1, -1
    for i in range(c.n):
        s, t0, t1, src, dst, k = d["seq"][i], d["start"][i], d["end"][i], d["src"][i], d["dst"][i], d["kind"][i]
        if t0 > t1:
            v.append(("interval", f"start_ns {t0} > end_ns {t1}", s))
        if not 0 <= src < ndev:
            v.append(("device", f"src_device={src} out of range [0,{ndev})", s))
        if not 0 <= dst < ndev:
            v.append(("device", f"dst_device={dst} out of range [0,{ndev})", s))
        if k == TRANSFER and d["nb"][i] > 0 and d["h"][i] == 0:
            v.append(("transfer", "non-empty transfer has no content hash", s))
        elif k == ALLOC:
            if d["nb"][i] <= 0:
                v.append(("alloc", "allocation of zero bytes", s))
            if d["da"][i] == 0:
                v.append(("alloc", "allocation with null device address", s))
        elif k == DELETE and d["da"][i] == 0:
            v.append(("delete", "deletion with null device address", s))
        elif k == KERNEL and src != dst:
            v.append(("kernel", "kernel src_device must equal dst_device", s))
        fl = lf[d["loc"][i]]
        if fl & 1:
            v.append(("location", "file present but line missing", s))
        if fl & 2:
            v.append(("location", f"line={c.locs[d['loc'][i]][2]} must be positive", s))
        if t0 < prev_start or (t0 == prev_start and s < prev_seq):
            v.append(("order", "events not sorted by (start_ns, seq)", s))
        if s <= prev_seq:
            v.append(("order", "seq values not strictly increasing", s))
        prev_start, prev_seq = t0, s
    return v


def _pairs(d, data_ops):
    """prep.py:45-96: LIFO per (dst_device, dst_addr); synthetic delete at max end."""
    live, pairs, warns, max_end = {}, [], [], 0
    for i in data_ops:
        max_end = max(max_end, d["end"][i])
        k = d["kind"][i]
        key = (d["dst"][i], d["da"][i])
        if k == ALLOC:
            live.setdefault(key, []).append(i)
        elif k == DELETE:
            st = live.get(key)
            if st:
                pairs.append((st.pop(), i))
            else:
                warns.append(i)
    for st in live.values():
        for a in st:
            pairs.append((a, SYNTH))
    pairs.sort(key=lambda p: p[0])  # (alloc.start, alloc.seq) == alloc index order in a valid trace
    return pairs, warns, max_end


def _dd(d, hashed):
    groups = {}
    for i in hashed:
        groups.setdefault((d["h"][i], d["dst"][i]), []).append(i)
    out = [(k[0], k[1], m) for k, m in groups.items() if len(m) >= 2]
    out.sort(key=lambda g: (d["start"][g[2][0]], g[0], g[1]))
    return out


def _rt(d, hashed, strict):
    queues = {}
    for i in hashed:
        queues.setdefault((d["h"][i], d["dst"][i]), deque()).append(i)
    trips = {}
    for tx in hashed:
        q = queues.get((d["h"][tx], d["src"][tx]))
        if not q:
            continue
        if strict:
            rx = q[0]
        else:
            while q and q[0] <= tx:  # (start, seq) order == index order
                q.popleft()
            if not q:
                continue
            rx = q.popleft()
        trips.setdefault((d["h"][tx], d["src"][tx], d["dst"][tx]), []).append((tx, rx))
        if strict:
            own = queues.get((d["h"][tx], d["dst"][tx]))
            if own:
                own.popleft()
    out = [(k[0], k[1], k[2], t) for k, t in trips.items()]
    out.sort(key=lambda g: (d["start"][g[3][0][0]], g[0], g[1], g[2]))
    return out


def _ra(d, pairs):
    groups = {}
    for pi, (a, _) in enumerate(pairs):
        groups.setdefault((d["sa"][a], d["dst"][a], d["nb"][a]), []).append(pi)
    out = [(k[0], k[1], k[2], m) for k, m in groups.items() if len(m) >= 2]
    out.sort(key=lambda g: (d["start"][pairs[g[3][0]][0]], g[0], g[1], g[2]))
    return out


def _by_device(d, idx, ndev):
    out = [[] for _ in range(max(ndev, 0))]
    for i in idx:
        out[d["dst"][i]].append(i)
    return out


def _ua(d, kernels, pairs, target_pairs, ndev, synth_end):
    dk = _by_device(d, kernels, ndev)
    per = [[] for _ in range(max(ndev, 0))]
    for pi in target_pairs:
        per[d["dst"][pairs[pi][0]]].append(pi)
    unused = []
    for dev in range(ndev):
        K, c = dk[dev], 0
        for pi in per[dev]:
            a, dl = pairs[pi]
            while c < len(K) and d["end"][K[c]] < d["start"][a]:
                c += 1
            del_end = synth_end if dl == SYNTH else d["end"][dl]
            if c == len(K) or d["start"][K[c]] > del_end:
                unused.append(pi)
    unused.sort(key=lambda pi: pairs[pi][0])
    return unused


def _ut(d, kernels, tt, ndev):
    dk, dt = _by_device(d, kernels, ndev), _by_device(d, tt, ndev)
    unused = []
    for dev in range(ndev):
        K, c, cand = dk[dev], 0, {}
        for x in dt[dev]:
            while c < len(K) and d["end"][K[c]] < d["start"][x]:
                c += 1
                cand.clear()
            if c == len(K):
                unused.append(x)
            elif d["start"][K[c]] > d["start"][x]:
                p = cand.get(d["sa"][x])
                if p is not None:
                    unused.append(p)
                cand[d["sa"][x]] = x
            else:
                cand.clear()
    unused.sort()
    return unused


def analyze_cols(c, strict=False, synth_end=None) -> RefFindings:
    """detectors.py:274-326 over columns (assumes validate_cols() was empty).  ``synth_end``
    overrides the synthetic-delete time (prep.py:61-62) -- used for shards of a trace."""
    d = _ints(c)
    host, ndev = c.host_device, c.num_devices_total
    hashed, tt, data_ops, tk = [], [], [], []
    for i in range(c.n):
        k = d["kind"][i]
        if k == TRANSFER:
            data_ops.append(i)
            if d["nb"][i] > 0 and d["h"][i] != 0:
                hashed.append(i)
            if d["dst"][i] != host:
                tt.append(i)
        elif k in (ALLOC, DELETE):
            data_ops.append(i)
        elif k == KERNEL and d["dst"][i] != host:
            tk.append(i)
    pairs, warns, local_end = _pairs(d, data_ops)
    if synth_end is None:
        synth_end = local_end
    target_pairs = [pi for pi, (a, _) in enumerate(pairs) if d["dst"][a] != host]
    return RefFindings(dd=_dd(d, hashed), rt=_rt(d, hashed, strict), pairs=pairs, synthetic_end=synth_end,
                       warnings=warns, ra=_ra(d, pairs), ua=_ua(d, tk, pairs, target_pairs, ndev, synth_end),
                       ut=_ut(d, tk, tt, ndev))


def category_members(f: RefFindings):
    """estimator.py:77-113 per-category eliminable event sets (indices; synthetic deletes skipped)."""
    cats = {c: set() for c in CATEGORIES}
    for _, _, m in f.dd:
        cats["DD"].update(m[1:])
    for *_, trips in f.rt:
        cats["RT"].update(rx for _, rx in trips)

    def add(bucket, pi):
        a, dl = f.pairs[pi]
        bucket.add(a)
        if dl != SYNTH:
            bucket.add(dl)
    for *_, ps in f.ra:
        for pi in ps[1:]:
            add(cats["RA"], pi)
    for pi in f.ua:
        add(cats["UA"], pi)
    cats["UT"].update(f.ut)
    return cats


def estimate_cols(c, f: RefFindings, wall_time_ns=None):
    """estimator.py:61-151 -> dict with the SavingsEstimate fields (eliminable as event indices)."""
    d = _ints(c)
    cats = category_members(f)
    dur = lambda i: d["end"][i] - d["start"][i]  # noqa: E731
    per = {k: sum(dur(i) for i in s) for k, s in cats.items()}
    union = set().union(*cats.values())
    union_ns = sum(dur(i) for i in union)
    if wall_time_ns is not None:
        wall = wall_time_ns
    elif c.n == 0:
        wall = 0
    else:
        wall = max(d["end"]) - min(d["start"])
    warnings = []
    if union_ns > wall:
        warnings.append(f"eliminable time {union_ns} ns exceeds wall time {wall} ns; clamped to wall time")
        union_ns = wall
    if union_ns < 0:
        warnings.append("negative eliminable time clamped to 0")
        union_ns = 0
    if union_ns == 0:
        speed = 1.0
    elif union_ns == wall:
        warnings.append("eliminable time equals wall time; predicted speedup is unbounded")
        speed = float("inf")
    else:
        speed = wall / (wall - union_ns)
    frontier, overl = -1, False
    for i in range(c.n):
        if d["start"][i] < frontier:
            overl = True
            break
        frontier = max(frontier, d["end"][i])
    if overl:
        warnings.append("trace contains overlapping event intervals; savings assume serialized "
                        "operations and may be unreliable")
    return dict(per_category_ns=per, union_ns=union_ns, wall_time_ns=wall, predicted_speedup=speed,
                eliminable=sorted(union), warnings=tuple(warnings))


def attribute_cols(c, f: RefFindings, wall_time_ns=None):
    """report.py:44-95 -> rows (category, first member event index, count, total_ns, total_bytes, pct)."""
    d = _ints(c)
    bucket = [int(c.loc_bucket[d["loc"][i]]) for i in range(c.n)]
    if wall_time_ns is not None:
        wall = wall_time_ns
    elif c.n == 0:
        wall = 0
    else:
        wall = max(d["end"]) - min(d["start"])
    seqs = {c_: [] for c_ in CATEGORIES}
    for _, _, m in f.dd:
        seqs["DD"].extend(m)
    for *_, trips in f.rt:
        for tx, rx in trips:
            seqs["RT"] += [tx, rx]

    def pair_events(pi):
        a, dl = f.pairs[pi]
        return [a] if dl == SYNTH else [a, dl]
    for *_, ps in f.ra:
        for pi in ps:
            seqs["RA"] += pair_events(pi)
    for pi in f.ua:
        seqs["UA"] += pair_events(pi)
    seqs["UT"] = list(f.ut)
    rows = []
    for cat in CATEGORIES:
        b = {}
        for i in seqs[cat]:
            b.setdefault(bucket[i], []).append(i)
        cr = []
        for bk, mem in b.items():
            tot = sum(d["end"][i] - d["start"][i] for i in mem)
            cr.append((cat, mem[0], len(mem), tot, sum(d["nb"][i] for i in mem),
                       (tot / wall) if wall else 0.0, c.bucket_keys[bk]))
        cr.sort(key=lambda r: (-r[3], r[6]))
        rows.extend(r[:6] for r in cr)
    return rows
