"""Generates the committed golden fixtures from the UNMODIFIED reference.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
The fixtures travel with the repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("DMLENS_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from dmlens.hashing import hash_bytes  # noqa: E402  (the reference's own implementation)

from oracle.hash_ref import payload  # noqa: E402  (deterministic payload bytes only)

# frozen cross-language vectors of the reference (pkg/shim/test/hash64.test.ts:8-24)
TS_VECTORS = [
    ("00", 13822439871872589623), ("ff", 12844647536454529852), ("61", 2714998891557577425),
    ("616263", 16769191619139763278), ("6162636465666768", 2402220733500462054),
    ("616263646566676869", 11245955420054164285),
    ("000102030405060708090a0b0c0d0e0f", 13029654848220864353),
    ("aa" * 7, 17947520978646933045), ("55" * 63, 4886044645629322746),
    (bytes(range(256)).hex(), 5613354006569079831),
    (bytes(i % 251 for i in range(1024)).hex(), 11562279238887807506),
    ("00" * 32, 9077827906869418884),
]


def hash_fixture():
    out = {"ts_vectors": [], "stability": None, "by_length": {}, "large": []}
    for hexp, want in TS_VECTORS:
        got = hash_bytes(bytes.fromhex(hexp))
        assert got == want, (hexp, got, want)
        out["ts_vectors"].append([hexp, str(want)])
    stab = bytes(range(256)) * 4096
    out["stability"] = {"expr": "bytes(range(256)) * 4096", "digest": str(hash_bytes(stab))}
    seed = 7
    out["by_length"] = {"seed": seed, "content_id": "length", "lengths": "1..4096",
                        "digests": [str(hash_bytes(payload(n, seed, n))) for n in range(1, 4097)]}
    for i, n in enumerate([1024, 4097, 65536, 131077, 262144, 1048576, 1048573]):
        out["large"].append({"len": n, "seed": 11, "content_id": 1000 + i,
                             "digest": str(hash_bytes(payload(n, 11, 1000 + i)))})
    return out


if __name__ == "__main__" and not set(sys.argv) & {"--analysis", "--standalone", "--ingest", "--reports", "--serialize"}:
    with open(os.path.join(HERE, "hash_vectors.json"), "w") as f:
        json.dump(hash_fixture(), f, indent=0)
    print("wrote hash_vectors.json")


# ----------------------------------------------------------------------------- analysis
def _trace_json(tr):
    return {"version": tr.version, "num_devices_total": tr.num_devices_total, "host_device": tr.host_device,
            "wall_time_ns": tr.wall_time_ns,
            "events": [[e.seq, e.kind.value, e.start_ns, e.end_ns, e.src_device, e.dst_device, e.src_addr,
                        e.dst_addr, e.bytes, str(e.hash), e.loc.codeptr, e.loc.file, e.loc.line]
                       for e in tr.events]}


def _pair_json(p):
    return [p.alloc_event.seq, p.delete_event.seq, p.synthetic_delete]


def _findings_json(f):
    return {
        "dd": [[str(g.hash), g.dest_device, [e.seq for e in g.events]] for g in f.duplicates],
        "rt": [[str(g.hash), g.src_device, g.dest_device, [[a.seq, b.seq] for a, b in g.trips]]
               for g in f.round_trips],
        "ra": [[g.host_addr, g.tgt_device, g.bytes, [_pair_json(p) for p in g.pairs]] for g in f.repeated_allocs],
        "ua": [_pair_json(p) for p in f.unused_allocs],
        "ut": [e.seq for e in f.unused_transfers],
    }


def _case(name, tr):
    from dmlens import analyze, attribute, estimate
    from dmlens.detectors import InvalidTrace
    from dmlens.prep import get_alloc_delete_pairs
    from dmlens.model import EventKind
    case = {"name": name, "trace": _trace_json(tr)}
    try:
        warns = []
        f = analyze(tr, warn=warns.append)
    except InvalidTrace as exc:
        case["violations"] = [[v.rule, v.message, v.seq] for v in exc.violations]
        return case
    case["warnings"] = [[w.seq, w.reason] for w in warns]
    case["findings"] = _findings_json(f)
    case["findings_strict"] = _findings_json(analyze(tr, strict_pseudocode=True))
    data_ops = [e for e in tr.events if e.kind is not EventKind.KERNEL]
    case["pairs"] = [_pair_json(p) for p in get_alloc_delete_pairs(data_ops)]
    s = estimate(tr, f)
    case["estimate"] = {"per_category_ns": s.per_category_ns, "union_ns": s.union_ns,
                        "wall_time_ns": s.wall_time_ns, "predicted_speedup": repr(s.predicted_speedup),
                        "eliminable_seqs": sorted(s.eliminable_seqs), "warnings": list(s.warnings)}
    case["attribute"] = [[r.category, [r.location.codeptr, r.location.file, r.location.line], r.occurrence_count,
                          r.total_ns, r.total_bytes, repr(r.pct_of_wall)] for r in attribute(tr, f)]
    return case


def analysis_fixture():
    import importlib.util
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REF), "tests",
                                                                               "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from dmlens.synth import PATTERNS, PatternSpec, generate, generate_scale
    from dmlens.model import CodeLocation, EventKind, Trace, TraceEvent
    cases = []
    for seed in range(300):
        cases.append(_case(f"random_trace({seed})", conf.random_trace(seed)))
    for seed in range(1000, 1012):
        cases.append(_case(f"random_trace({seed}, 2000, 6)", conf.random_trace(seed, max_events=2000,
                                                                                 max_devices=6)))
    for pat in PATTERNS:
        for n, nd in ((1, 2), (3, 3), (5, 4)):
            tr, _ = generate(PatternSpec(pattern=pat, n_iterations=n, n_devices=nd, seed=n * 7 + nd))
            cases.append(_case(f"synth({pat},{n},{nd})", tr))
    cases.append(_case("generate_scale(20000,1,3)", generate_scale(20000, seed=1, n_devices=3)))
    # invalid traces (model.py:125-200 messages)
    mk = conf.make_event
    bad = [
        ("inverted", [mk(0, EventKind.TRANSFER, 10, 5, hash=1, nbytes=8)]),
        ("hashless", [mk(0, EventKind.TRANSFER, 0, 5, nbytes=8, hash=0)]),
        ("alloc0", [mk(0, EventKind.ALLOC, 0, 5, nbytes=0, dst_addr=0)]),
        ("delete0", [mk(0, EventKind.DELETE, 0, 5, dst_addr=0)]),
        ("kernel", [mk(0, EventKind.KERNEL, 0, 5, src=0, dst=1)]),
        ("device", [mk(0, EventKind.TRANSFER, 0, 5, src=7, dst=-1, nbytes=0)]),
        ("unsorted", [mk(0, EventKind.KERNEL, 10, 15, src=1, dst=1), mk(1, EventKind.KERNEL, 5, 6, src=1, dst=1)]),
        ("seqdup", [mk(3, EventKind.KERNEL, 0, 1, src=1, dst=1), mk(3, EventKind.KERNEL, 0, 1, src=1, dst=1),
                    mk(2, EventKind.KERNEL, 0, 1, src=1, dst=1)]),
        ("loc", [mk(0, EventKind.KERNEL, 0, 1, src=1, dst=1, file="a.c"),
                 mk(1, EventKind.KERNEL, 0, 1, src=1, dst=1, codeptr=5, file="b.c", line=0),
                 mk(2, EventKind.KERNEL, 0, 1, src=1, dst=1, line=-3)]),
    ]
    for name, evs in bad:
        cases.append(_case("invalid:" + name, Trace(1, 2, 0, None, evs)))
    cases.append(_case("invalid:header", Trace(1, 0, 3, None, [])))
    return cases


if __name__ == "__main__" and "--analysis" in sys.argv:
    import gzip
    with gzip.open(os.path.join(HERE, "analysis_cases.json.gz"), "wt") as f:
        json.dump(analysis_fixture(), f)
    print("wrote analysis_cases.json.gz")


# ----------------------------------------------------------------------------- standalone detectors
def standalone_fixture():
    import importlib.util
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REF), "tests",
                                                                               "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from dmlens.detectors import (find_duplicate_transfers, find_repeated_allocs, find_round_trips,
                                  find_unused_allocs, find_unused_transfers)
    from dmlens.model import EventKind
    from dmlens.prep import get_alloc_delete_pairs, sort_by_device
    out = []
    for seed in range(3000, 3080):
        tr = conf.random_trace(seed)
        ev, host, nd = tr.events, tr.host_device, tr.num_devices_total
        transfers = [e for e in ev if e.kind is EventKind.TRANSFER]
        data_ops = [e for e in ev if e.kind is not EventKind.KERNEL]
        kernels = [e for e in ev if e.kind is EventKind.KERNEL]
        tk = [e for e in kernels if e.dst_device != host]
        tt = [e for e in transfers if e.dst_device != host]
        warns = []
        c = {"seed": seed, "trace": _trace_json(tr),
             # raw lists: every transfer (hash 0 / zero-byte included), every kernel (host included)
             "dd_raw": _findings_json_part_dd(find_duplicate_transfers(transfers)),
             "rt_raw": _findings_json_part_rt(find_round_trips(transfers)),
             "rt_raw_strict": _findings_json_part_rt(find_round_trips(transfers, strict_pseudocode=True)),
             "pairs": [_pair_json(p) for p in get_alloc_delete_pairs(data_ops, warn=warns.append)],
             "ra": [[g.host_addr, g.tgt_device, g.bytes, [_pair_json(p) for p in g.pairs]]
                    for g in find_repeated_allocs(data_ops)],
             "ua_all_kernels": [_pair_json(p) for p in find_unused_allocs(kernels, data_ops, nd)],
             "ut_all": [e.seq for e in find_unused_transfers(kernels, transfers, nd)],
             "ut_target": [e.seq for e in find_unused_transfers(tk, tt, nd)],
             "by_device_dst": [[e.seq for e in lst] for lst in sort_by_device(ev, nd, key="dst")],
             "by_device_src": [[e.seq for e in lst] for lst in sort_by_device(ev, nd, key="src")]}
        c["warnings"] = [w.seq for w in warns]
        out.append(c)
    return out


def _findings_json_part_dd(groups):
    return [[str(g.hash), g.dest_device, [e.seq for e in g.events]] for g in groups]


def _findings_json_part_rt(groups):
    return [[str(g.hash), g.src_device, g.dest_device, [[a.seq, b.seq] for a, b in g.trips]] for g in groups]


if __name__ == "__main__" and "--standalone" in sys.argv:
    import gzip
    with gzip.open(os.path.join(HERE, "standalone_cases.json.gz"), "wt") as f:
        json.dump(standalone_fixture(), f)
    print("wrote standalone_cases.json.gz")


# ----------------------------------------------------------------------------- NDJSON ingest
def ingest_fixture():
    import importlib.util
    import random as _r
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REF), "tests",
                                                                               "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from dmlens.traceio import parse_trace, serialize_trace
    H = '{"dmlens":1,"num_devices":2,"host_device":0,"wall_time_ns":100}'
    E = ('{"seq":0,"kind":"transfer","t0":0,"t1":10,"src_dev":0,"dst_dev":1,'
         '"src_addr":1,"dst_addr":2,"bytes":8,"hash":7,"codeptr":0}')
    texts = []
    for seed in range(40):
        tr = conf.random_trace(seed)
        lines = serialize_trace(tr).decode().split("\n")
        body = lines[1:-1]
        _r.Random(seed).shuffle(body)  # any order in the file; parse re-sorts by (t0, seq)
        texts.append(("random%d" % seed, "\n".join([lines[0]] + body) + "\n"))
    odd = [
        ("crlf-comments-blank", "# c\r\n\r\n" + H + "\r\n\r\n# x\r\n" + E + "\r\n"),
        ("spaces-unicode-escape", H + "\n" + E.replace('"codeptr":0', ' "codeptr" : 0 , "file":"k\\u00e9rnel\\n.c","line":3 ')),
        ("unknown-nested", H + "\n" + E.replace('"codeptr":0', '"codeptr":0,"extra":{"a":[1,2.5,{"b":null}],"c":"x"}')),
        ("duplicate-key-last-wins", H + "\n" + E.replace('"hash":7', '"hash":5,"hash":7')),
        ("minus-zero", H + "\n" + E.replace('"bytes":8', '"bytes":-0')),
        ("float-in-unknown", H + "\n" + E.replace('"codeptr":0', '"codeptr":0,"ratio":1.5e3')),
        ("nbsp-stripped", " " + H + "\n" + E),
        ("line-huge", H + "\n" + E.replace('"codeptr":0', '"codeptr":0,"file":"a.c","line":%d' % (2**70))),
        ("null-file-line", H + "\n" + E.replace('"codeptr":0', '"codeptr":0,"file":null,"line":null')),
        ("no-wall", '{"dmlens":1,"num_devices":3,"host_device":1}\n' + E.replace('"dst_dev":1', '"dst_dev":2')),
        ("header-true-version", '{"dmlens":true,"num_devices":2,"host_device":0}\n'),
        ("bad-json-trailing", H + "\n" + E + " x\n"),
        ("bad-leading-zero", H + "\n" + E.replace('"bytes":8', '"bytes":08')),
        ("nan-value", H + "\n" + E.replace('"hash":7', '"hash":NaN')),
        ("control-char", H + "\n" + E.replace('"codeptr":0', '"codeptr":0,"file":"a\tb","line":1')),
        ("kind-escaped", H + "\n" + E.replace('"transfer"', '"transf\\u0065r"')),
        ("second-header", H + "\n" + H + "\n"),
        ("array-record", H + "\n[1,2,3]\n"),
        ("device-huge", H + "\n" + E.replace('"dst_dev":1', '"dst_dev":%d' % (2**40))),
    ]
    mut = [
        ("missing-seq", lambda o: o.pop("seq")), ("kind-warp", lambda o: o.update(kind="warp")),
        ("inverted", lambda o: o.update(t0=50, t1=5)), ("neg-bytes", lambda o: o.update(bytes=-4)),
        ("big-bytes", lambda o: o.update(bytes=2**64)), ("str-hash", lambda o: o.update(hash="abc")),
        ("float-hash", lambda o: o.update(hash=1.5)), ("bool-hash", lambda o: o.update(hash=True)),
        ("file-no-line", lambda o: o.update(file="a.c")), ("file-int", lambda o: o.update(file=9, line=1)),
        ("line-zero", lambda o: o.update(file="a.c", line=0)), ("kind-int", lambda o: o.update(kind=3)),
    ]
    for name, m in mut:
        o = json.loads(E)
        m(o)
        texts.append(("mut-" + name, H + "\n" + json.dumps(o)))
    corpus = [
        ("empty-file", ""), ("comment-only", "# nothing here\n"), ("event-before-header", E + "\n"),
        ("bad-version", '{"dmlens":3,"num_devices":2,"host_device":0}\n'), ("header-not-json", '{"dmlens":1,,}\n'),
        ("event-not-json", H + "\n{not json}\n"), ("event-not-object", H + "\n42\n"),
        ("hashless-transfer", H + "\n" + E.replace('"hash":7', '"hash":0') + "\n"),
        ("duplicate-seq", H + "\n" + E + "\n" + E.replace('"t0":0,"t1":10', '"t0":20,"t1":30') + "\n"),
        ("bad-host-device", '{"dmlens":1,"num_devices":2,"host_device":5}\n'),
    ]
    out = []
    for name, text in texts + odd + corpus:
        rec = {"name": name, "text": text}
        try:
            tr = parse_trace(text)
            rec["trace"] = _trace_json(tr)
        except Exception as exc:  # noqa: BLE001 - record the reference's exact exception
            rec["error"] = [type(exc).__name__, str(exc)]
        out.append(rec)
    return out


if __name__ == "__main__" and "--ingest" in sys.argv:
    with open(os.path.join(HERE, "ingest_cases.json"), "w") as f:
        json.dump(ingest_fixture(), f)
    print("wrote ingest_cases.json")


# ----------------------------------------------------------------------------- reports (CLI path)
def report_fixture():
    import importlib.util
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REF), "tests",
                                                                               "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from dmlens.cli import _filter_min_bytes
    from dmlens import analyze, attribute, estimate, render_json, render_text
    from dmlens.synth import PATTERNS, PatternSpec, generate
    from dmlens.traceio import serialize_trace
    traces = [("listing1", generate(PatternSpec(pattern="listing1"))[0])]
    for pat in PATTERNS:
        traces.append((f"synth-{pat}", generate(PatternSpec(pattern=pat, n_iterations=3, n_devices=3, seed=5))[0]))
    for seed in range(20):
        tr = conf.random_trace(seed)
        if tr.wall_time_ns is None:
            tr.wall_time_ns = tr.wall_time()
        traces.append((f"random{seed}", tr))
    out = []
    for name, tr in traces:
        f = analyze(tr)
        for mb in (0, 64, 4096):
            rep = _filter_min_bytes(f, mb)
            s = estimate(tr, rep)
            iss = attribute(tr, rep)
            out.append({"name": name, "min_bytes": mb, "ndjson": serialize_trace(tr).decode(),
                        "text": render_text(tr, rep, s, iss), "json": render_json(tr, rep, s, iss)})
    return out


if __name__ == "__main__" and "--reports" in sys.argv:
    import gzip
    with gzip.open(os.path.join(HERE, "report_cases.json.gz"), "wt") as f:
        json.dump(report_fixture(), f)
    print("wrote report_cases.json.gz")


# ----------------------------------------------------------------------------- serialize_trace
def serialize_fixture():
    """traceio.serialize_trace (traceio.py:193-237) outputs of the unmodified reference: random
    traces, synth patterns, location edge cases (non-ASCII / escaped / surrogate file names,
    line without file), and the invalid traces it refuses."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REF), "tests",
                                                                               "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from dmlens.model import EventKind, Trace
    from dmlens.synth import PATTERNS, PatternSpec, generate
    from dmlens.traceio import InvalidTrace, serialize_trace
    cases = []

    def add(name, tr):
        c = {"name": name, "trace": _trace_json(tr)}
        try:
            c["text"] = serialize_trace(tr).decode("utf-8")
        except InvalidTrace as exc:
            c["error"] = [type(exc).__name__, str(exc), [[v.rule, v.message, v.seq] for v in exc.violations]]
        cases.append(c)
    for seed in range(40):
        tr = conf.random_trace(seed)
        if seed % 2 == 0 and tr.wall_time_ns is None:
            tr.wall_time_ns = tr.wall_time()
        add(f"random_trace({seed})", tr)
    for pat in PATTERNS:
        tr, _ = generate(PatternSpec(pattern=pat, n_iterations=3, n_devices=3, seed=5))
        add(f"synth({pat})", tr)
    mk = conf.make_event
    evs = [mk(0, EventKind.KERNEL, 0, 1, src=1, dst=1, codeptr=7, file="café.c", line=3),
           mk(1, EventKind.KERNEL, 1, 2, src=1, dst=1, codeptr=8, file='q"uo\\te\n\t.c', line=4),
           mk(2, EventKind.KERNEL, 2, 3, src=1, dst=1, codeptr=9, file="\U0001F600\ud800x\x00y", line=5),
           mk(3, EventKind.KERNEL, 3, 4, src=1, dst=1, codeptr=2**64 - 1, line=6),
           mk(4, EventKind.TRANSFER, 4, 9, src=0, dst=1, nbytes=2**64 - 1, hash=2**64 - 1, src_addr=2**64 - 1,
              dst_addr=1)]
    add("locations", Trace(1, 2, 0, 2**64 - 1, evs))
    add("empty", Trace(1, 3, 0, None, []))
    add("invalid:host", Trace(1, 2, 9, None, []))
    add("invalid:version", Trace(2, 2, 0, None, []))
    add("invalid:inverted", Trace(1, 2, 0, None, [mk(0, EventKind.TRANSFER, 10, 5, hash=1, nbytes=8)]))
    return cases


if __name__ == "__main__" and "--serialize" in sys.argv:
    import gzip
    with gzip.open(os.path.join(HERE, "serialize_cases.json.gz"), "wt") as f:
        json.dump(serialize_fixture(), f)
    print("wrote serialize_cases.json.gz")
