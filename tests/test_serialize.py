"""serialize_trace drop-in (traceio.py:193-246): the native writer against the reference's own
bytes (tests/golden/serialize_cases.json.gz, made by make_golden.py --serialize).
CPU: the writer on the fixtures' columns (no validation).  GPU: the full drop-in
(validation first, InvalidTrace for the traces the reference refuses), and round trips."""
import gzip
import json
import os

import numpy as np
import pytest

from paper_2601_12713_b200 import ingest
from paper_2601_12713_b200.columns import to_columns
from tests._cases import trace_from_json

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(gzip.open(os.path.join(HERE, "golden", "serialize_cases.json.gz"), "rt"))


def test_native_writer_matches_reference_bytes():
    n = 0
    for c in CASES:
        if "text" not in c:
            continue
        tr = trace_from_json(c["trace"])
        got = ingest.serialize_columns(to_columns(tr), version=tr.version, threads=3, validate=False)
        assert got == c["text"].encode("utf-8"), c["name"]
        n += 1
    assert n >= 45


def test_native_writer_threads_and_large_values():
    from paper_2601_12713_b200.columns import columns_from_arrays
    k = 300_000
    seq = np.arange(k, dtype=np.uint64) + np.uint64(2**64 - k)
    c = columns_from_arrays(3, 0, seq, seq, seq, np.ones(k, np.int32), np.ones(k, np.int32),
                            np.full(k, 3, np.uint8), seq, seq, seq, seq, wall_time_ns=7)
    a = ingest.serialize_columns(c, threads=1, validate=False)
    b = ingest.serialize_columns(c, threads=8, validate=False)
    assert a == b and a.count(b"\n") == k + 1
    want = ('{"seq":%d,"kind":"kernel","t0":%d,"t1":%d,"src_dev":1,"dst_dev":1,"src_addr":%d,"dst_addr":%d,'
            '"bytes":%d,"hash":%d,"codeptr":0}' % ((2**64 - 1,) * 7))
    assert a.split(b"\n")[-2].decode() == want


@pytest.mark.gpu
def test_serialize_trace_drop_in(cuda):
    for c in CASES:
        tr = trace_from_json(c["trace"])
        if "error" in c:
            with pytest.raises(ingest.InvalidTrace) as ei:
                ingest.serialize_trace(tr)
            assert [type(ei.value).__name__, str(ei.value)] == c["error"][:2], c["name"]
            assert [[v.rule, v.message, v.seq] for v in ei.value.violations] == c["error"][2], c["name"]
        else:
            data = ingest.serialize_trace(tr)
            assert data == c["text"].encode("utf-8"), c["name"]
            back = ingest.parse_trace(data)  # parse(serialize(t)) == t  (test_traceio.py:160-184)
            lossless = all(e.loc.file is not None or e.loc.line is None for e in tr.events)  # a bare line is dropped
            if tr.wall_time_ns is not None and lossless:  # parse derives a wall time when the header has none
                assert back.events == tr.events and back.wall_time_ns == tr.wall_time_ns, c["name"]
                assert ingest.serialize_trace(back) == data, c["name"]
