"""Shared helpers: golden analysis cases -> traces / columns, and a canonical
(seq-based) form of findings so engine, oracle and reference compare equal."""
import gzip
import json
import os

from paper_2601_12713_b200 import types as T
from paper_2601_12713_b200.columns import to_columns

HERE = os.path.dirname(os.path.abspath(__file__))
_CASES = None


def cases():
    global _CASES
    if _CASES is None:
        with gzip.open(os.path.join(HERE, "golden", "analysis_cases.json.gz"), "rt") as f:
            _CASES = json.load(f)
    return _CASES


def trace_from_json(tj, types=T):
    evs = [types.TraceEvent(seq=e[0], kind=types.EventKind(e[1]), start_ns=e[2], end_ns=e[3], src_device=e[4],
                            dst_device=e[5], src_addr=e[6], dst_addr=e[7], bytes=e[8], hash=int(e[9]),
                            loc=types.CodeLocation(codeptr=e[10], file=e[11], line=e[12]))
           for e in tj["events"]]
    return types.Trace(version=tj["version"], num_devices_total=tj["num_devices_total"],
                       host_device=tj["host_device"], wall_time_ns=tj["wall_time_ns"], events=evs)


def canon_ref_json(fj):
    """Fixture findings JSON -> canonical tuples."""
    pj = lambda p: (p[0], p[1], bool(p[2]))  # noqa: E731
    return {
        "dd": [(int(h), d, list(m)) for h, d, m in fj["dd"]],
        "rt": [(int(h), s, d, [tuple(t) for t in tr]) for h, s, d, tr in fj["rt"]],
        "ra": [(a, d, b, [pj(p) for p in ps]) for a, d, b, ps in fj["ra"]],
        "ua": [pj(p) for p in fj["ua"]],
        "ut": list(fj["ut"]),
    }


def canon_findings_objects(f):
    """Findings objects (dmlens's or ours) -> canonical tuples."""
    pj = lambda p: (p.alloc_event.seq, p.delete_event.seq, bool(p.synthetic_delete))  # noqa: E731
    return {
        "dd": [(g.hash, g.dest_device, [e.seq for e in g.events]) for g in f.duplicates],
        "rt": [(g.hash, g.src_device, g.dest_device, [(a.seq, b.seq) for a, b in g.trips]) for g in f.round_trips],
        "ra": [(g.host_addr, g.tgt_device, g.bytes, [pj(p) for p in g.pairs]) for g in f.repeated_allocs],
        "ua": [pj(p) for p in f.unused_allocs],
        "ut": [e.seq for e in f.unused_transfers],
    }


def canon_oracle(rf, cols):
    """oracle RefFindings (indices) -> canonical tuples."""
    seq = [int(x) for x in cols.seq]

    def pj(pi):
        a, d = rf.pairs[pi]
        return (seq[a], seq[a] if d < 0 else seq[d], d < 0)
    return {
        "dd": [(h, d, [seq[i] for i in m]) for h, d, m in rf.dd],
        "rt": [(h, s, d, [(seq[a], seq[b]) for a, b in tr]) for h, s, d, tr in rf.rt],
        "ra": [(a, d, b, [pj(pi) for pi in ps]) for a, d, b, ps in rf.ra],
        "ua": [pj(pi) for pi in rf.ua],
        "ut": [seq[i] for i in rf.ut],
    }


def columns_of(case):
    return to_columns(trace_from_json(case["trace"]))


def canon_columnar(cf, cols):
    """engine ColumnarFindings (indices) -> canonical tuples."""
    seq = [int(x) for x in cols.seq]
    h = [int(x) for x in cols.hash]
    src = [int(x) for x in cols.src_device]
    dst = [int(x) for x in cols.dst_device]
    sa = [int(x) for x in cols.src_addr]
    nb = [int(x) for x in cols.bytes]
    pa, pd = cf.pair_alloc.tolist(), cf.pair_delete.tolist()

    def pj(r):
        a, d = pa[r], pd[r]
        return (seq[a], seq[a] if d == 0xFFFFFFFF else seq[d], d == 0xFFFFFFFF)
    off, mem = cf.dd_offsets.tolist(), cf.dd_members.tolist()
    dd = [(h[mem[off[g]]], dst[mem[off[g]]], [seq[i] for i in mem[off[g]:off[g + 1]]]) for g in range(len(off) - 1)]
    off, tx, rx = cf.rt_offsets.tolist(), cf.rt_tx.tolist(), cf.rt_rx.tolist()
    rt = [(h[tx[off[g]]], src[tx[off[g]]], dst[tx[off[g]]], [(seq[tx[t]], seq[rx[t]]) for t in range(off[g], off[g + 1])])
          for g in range(len(off) - 1)]
    off, rp = cf.ra_offsets.tolist(), cf.ra_pairs.tolist()
    ra = [(sa[pa[rp[off[g]]]], dst[pa[rp[off[g]]]], nb[pa[rp[off[g]]]], [pj(r) for r in rp[off[g]:off[g + 1]]])
          for g in range(len(off) - 1)]
    return {"dd": dd, "rt": rt, "ra": ra, "ua": [pj(r) for r in cf.ua_pairs.tolist()],
            "ut": [seq[i] for i in cf.ut_events.tolist()]}
