"""Native NDJSON ingest vs the reference's parse_trace outputs (golden).
CPU: the C++ parser's columns / rejection points and the exact-path errors.
GPU: the full parse_trace drop-in (GPU sort + validation) on every fixture."""
import json
import os

import numpy as np
import pytest

from paper_2601_12713_b200 import ingest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "ingest_cases.json")))


def _events_json(cols_or_none):
    return cols_or_none


def test_native_parser_columns_match_reference_order_free():
    accepted = 0
    for c in CASES:
        got = ingest._native(c["text"].encode("utf-8"), threads=3)
        if isinstance(got, ingest._Unvouched):
            continue
        accepted += 1
        assert "trace" in c or c["error"][0] == "InvariantViolation", c["name"]
        if "trace" not in c:
            continue
        header, cols, locs = got
        tj = c["trace"]
        assert header[1:3] == (tj["num_devices_total"], tj["host_device"]), c["name"]
        order = np.lexsort((cols["seq"], cols["start_ns"]))
        rows = []
        for i in order.tolist():
            cp, f, ln = locs[int(cols["loc"][i])]
            rows.append([int(cols["seq"][i]), ingest._KINDS[int(cols["kind"][i])], int(cols["start_ns"][i]),
                         int(cols["end_ns"][i]), int(cols["src_device"][i]), int(cols["dst_device"][i]),
                         int(cols["src_addr"][i]), int(cols["dst_addr"][i]), int(cols["bytes"][i]),
                         str(int(cols["hash"][i])), cp, f, ln])
        assert rows == tj["events"], c["name"]
    assert accepted >= 45  # every serialized random trace and the plain odd cases take the native path


def test_native_parser_multithreaded_large_input():
    lines = ['{"dmlens":1,"num_devices":3,"host_device":0}']
    for i in range(200_000):
        lines.append('{"seq":%d,"kind":"kernel","t0":%d,"t1":%d,"src_dev":1,"dst_dev":1,"src_addr":0,'
                     '"dst_addr":0,"bytes":0,"hash":0,"codeptr":%d}' % (i, 10 * i, 10 * i + 5, i % 7))
    raw = ("\n".join(lines) + "\n").encode()
    header, cols, locs = ingest._native(raw, threads=8)
    assert cols["seq"].size == 200_000 and np.array_equal(cols["seq"], np.arange(200_000, dtype=np.uint64))
    assert len(locs) == 7
    bad = raw.replace(b'"seq":123456,', b'"seq":123456,,')
    from paper_2601_12713_b200 import _lib
    got = ingest._native(bad, threads=8)
    assert isinstance(got, ingest._Unvouched) and got.lines == [123456 + 2] and got.header_line == 1
    del _lib


def test_exact_path_errors_match_reference():
    for c in CASES:
        if "error" not in c or c["error"][0] == "InvariantViolation":
            continue
        with pytest.raises(ingest.TraceIOError) as ei:
            ingest._parse_exact(c["text"])
        assert [type(ei.value).__name__, str(ei.value)] == c["error"], c["name"]


@pytest.mark.gpu
def test_parse_trace_drop_in_matches_reference(cuda):
    from tests._cases import trace_from_json
    for c in CASES:
        if "error" in c:
            with pytest.raises(ingest.TraceIOError) as ei:
                ingest.parse_trace(c["text"])
            assert [type(ei.value).__name__, str(ei.value)] == c["error"], c["name"]
        else:
            got = ingest.parse_trace(c["text"])
            want = trace_from_json(c["trace"])
            assert got.events == want.events and got.wall_time_ns == want.wall_time_ns, c["name"]
            assert (got.num_devices_total, got.host_device) == (want.num_devices_total, want.host_device)
            cols = ingest.parse_trace_columns(c["text"])
            assert [int(x) for x in cols.seq] == [e.seq for e in want.events], c["name"]


def test_canonical_fast_path_equals_general_scanner():
    """Lines in the capture agents' canonical shape take the allocation-free fast path; every
    edge around it (20-digit / leading-zero numbers, escapes, non-ASCII files, reordered keys,
    whitespace, inverted intervals) must give exactly what the general scanner gives."""
    import subprocess
    import sys
    head = '{"dmlens":1,"num_devices":3,"host_device":0}'
    ev = ('{"seq":%s,"kind":"%s","t0":%s,"t1":%s,"src_dev":1,"dst_dev":2,"src_addr":0,"dst_addr":%s,'
          '"bytes":%s,"hash":%s,"codeptr":%s%s}')
    rows = [ev % (i, k, t0, t1, da, nb, h, cp, extra) for i, (k, t0, t1, da, nb, h, cp, extra) in enumerate([
        ("kernel", 0, 0, 0, 0, 0, 0, ""),
        ("transfer", 5, 9, 7, 12, 18446744073709551615, 1, ""),          # 20-digit hash: general path
        ("alloc", 10, 10, 4096, 8, 0, 99999999999999999, ',"file":"a.c","line":3'),
        ("delete", 11, 12, 4096, 0, 0, 7, ',"file":"dir/x y.c","line":9223372036854775807'),
        ("transfer", 13, 14, 1, 2, 3, 4, ',"file":"\\u00e9.c","line":1'),  # escape: general path
        ("transfer", 15, 16, 1, 2, 3, 4, ',"file":"café.c","line":2'),  # non-ASCII: general path
        ("kernel", 17, 18, 0, 0, 0, 10, ""),
    ])]
    rows.append('{"kind":"kernel","seq":7,"t0":19,"t1":20,"src_dev":1,"dst_dev":1,"src_addr":0,"dst_addr":0,'
                '"bytes":0,"hash":0,"codeptr":1}')                       # reordered keys
    rows.append('{"seq":8, "kind":"kernel","t0":21,"t1":22,"src_dev":1,"dst_dev":1,"src_addr":0,"dst_addr":0,'
                '"bytes":0,"hash":0,"codeptr":1}')                       # whitespace
    good = "\n".join([head] + rows) + "\n"
    bad_variants = [
        good.replace('"seq":0,', '"seq":00,'),                           # leading zero: invalid JSON
        good.replace('"t0":17,"t1":18', '"t0":18,"t1":17'),               # inverted interval
        good.replace('"codeptr":10}', '"codeptr":10,"line":0}'),          # line 0
        good.replace('"hash":3,', '"hash":3.0,'),                          # float
    ]
    code = ("import sys, json, pickle; sys.path.insert(0, %r); from paper_2601_12713_b200 import ingest; "
            "inp = pickle.loads(sys.stdin.buffer.read()); out = []\n"
            "for t in inp:\n"
            "    r = ingest._native(t.encode(), threads=2)\n"
            "    out.append(('U', r.lines) if isinstance(r, ingest._Unvouched) else "
            "(r[0], {k: v.tolist() for k, v in r[1].items()}, r[2]))\n"
            "sys.stdout.buffer.write(pickle.dumps(out))") % os.path.dirname(HERE)
    import pickle
    inputs = pickle.dumps([good] + bad_variants)
    res = {}
    for general in (False, True):
        env = dict(os.environ)
        if general:
            env["B2L_INGEST_GENERAL_ONLY"] = "1"
        p = subprocess.run([sys.executable, "-c", code], input=inputs, capture_output=True, env=env, check=True)
        res[general] = pickle.loads(p.stdout)
    assert res[False] == res[True]
    assert res[False][0][0] != "U" and all(r[0] == "U" for r in res[False][1:])


def _rows(got):
    header, cols, locs = got
    order = np.lexsort((cols["seq"], cols["start_ns"]))
    rows = []
    for i in order.tolist():
        cp, f, ln = locs[int(cols["loc"][i])]
        rows.append([int(cols["seq"][i]), ingest._KINDS[int(cols["kind"][i])], int(cols["start_ns"][i]),
                     int(cols["end_ns"][i]), int(cols["src_device"][i]), int(cols["dst_device"][i]),
                     int(cols["src_addr"][i]), int(cols["dst_addr"][i]), int(cols["bytes"][i]),
                     str(int(cols["hash"][i])), cp, f, ln])
    return header, rows


def test_unvouched_lines_checked_one_by_one_match_reference(monkeypatch):
    """Every golden input through the native parser + per-line checks: the reference's exception
    for bad input, the reference's records for good input -- and never a whole-input Python parse."""
    def no_whole_parse(*a, **k):
        raise AssertionError("whole-input Python parse")
    monkeypatch.setattr(ingest, "_parse_exact", no_whole_parse)
    for c in CASES:
        raw = c["text"].encode("utf-8")
        if "error" in c and c["error"][0] != "InvariantViolation":
            with pytest.raises(ingest.TraceIOError) as ei:
                ingest._native_checked(raw, 3, None)
            assert [type(ei.value).__name__, str(ei.value)] == c["error"], c["name"]
            continue
        try:
            got = ingest._native_checked(raw, 3, None)
        except ingest._Unrepresentable:  # only a line number beyond the i64 location column
            assert any(e[12] is not None and e[12] > 2**63 - 1 for e in c["trace"]["events"]), c["name"]
            continue
        if "trace" in c:
            header, rows = _rows(got)
            assert header[1:3] == (c["trace"]["num_devices_total"], c["trace"]["host_device"]), c["name"]
            assert rows == c["trace"]["events"], c["name"]


def test_unusual_but_valid_lines_patched_not_reparsed(monkeypatch):
    monkeypatch.setattr(ingest, "_parse_exact", lambda *a, **k: (_ for _ in ()).throw(AssertionError("whole")))
    ev = ('{"seq":%d,"kind":"kernel","t0":%d,"t1":%d,"src_dev":1,"dst_dev":1,"src_addr":0,"dst_addr":0,'
          '"bytes":0,"hash":0,"codeptr":5%s}')
    lines = ["\u00a0", "# comment", '{"dmlens":1.0,"num_devices":2,"host_device":0,"note":[1,2.5]}']
    lines += [ev % (i, i, i + 1, "") for i in range(3000)]
    lines[100] = "\u2003" + lines[100] + "\u3000"                      # Unicode whitespace around a record
    lines[200] = "\u00a0# a comment after Unicode whitespace"
    lines[300] = ev % (297, 297, 298, ',"extra":1.5e3')                 # float in an unknown field
    lines[400] = ev % (397, 397, 398, ',"file":"a\\u0000b.c","line":4')  # NUL in a file name
    lines[500] = ev % (497, 497, 498, ',"file":"\\ud800x","line":2')     # lone surrogate in a file name
    lines[600] = ev % (597, 597, 598, ',"file":null,"line":7')         # explicit null file
    raw = ("\n".join(lines) + "\n").encode("utf-8")
    header, cols, locs = ingest._native_checked(raw, 4, None)
    assert header[:3] == (1, 2, 0) and cols["seq"].size == 2999
    by_seq = {int(q): locs[int(l)] for q, l in zip(cols["seq"], cols["loc"])}
    assert by_seq[397] == (5, "a\x00b.c", 4) and by_seq[497] == (5, "\ud800x", 2) and by_seq[597] == (5, None, 7)
    bad = raw.replace(b'"seq":2000,', b'"seq":-1,')
    with pytest.raises(ingest.MalformedRecord) as ei:
        ingest._native_checked(bad, 4, None)
    assert str(ei.value) == 'line 2004: field "seq"=-1 outside 64-bit unsigned range'
