"""Columnar report path: NDJSON -> native ingest -> GPU analysis ->
--min-bytes on index arrays -> device sums -> text / JSON reports, byte-identical to
the reference CLI's reports (tests/golden/report_cases.json.gz)."""
import gzip
import json
import os

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    with gzip.open(os.path.join(HERE, "golden", "report_cases.json.gz"), "rt") as f:
        return json.load(f)


def test_cli_reports_byte_identical(cuda, tmp_path, capsys):
    from paper_2601_12713_b200.__main__ import main
    os.environ["DMLENS_COLOR"] = "never"
    for c in _cases():
        p = tmp_path / f"{c['name']}.ndjson"
        p.write_text(c["ndjson"])
        assert main(["analyze", str(p), "--min-bytes", str(c["min_bytes"]), "-q"]) == 0
        assert capsys.readouterr().out == c["text"], (c["name"], c["min_bytes"])
        assert main(["analyze", str(p), "--min-bytes", str(c["min_bytes"]), "-q", "--json"]) == 0
        assert capsys.readouterr().out == c["json"], (c["name"], c["min_bytes"])


def test_cli_input_errors_exit_1(cuda, tmp_path, capsys):
    from paper_2601_12713_b200.__main__ import main
    p = tmp_path / "bad.ndjson"
    p.write_text('{"dmlens":3,"num_devices":2,"host_device":0}\n')
    assert main(["analyze", str(p)]) == 1
    assert "UnsupportedVersion" in capsys.readouterr().err
    assert main(["analyze", str(tmp_path / "missing.ndjson")]) == 1


def test_cli_event_violations_match_parse_trace(cuda, tmp_path, capsys):
    """The CLI validates events in its analysis run (one engine call); the error must be the
    one parse_trace raises for the same input."""
    from paper_2601_12713_b200 import ingest
    from paper_2601_12713_b200.__main__ import main
    text = ('{"dmlens":1,"num_devices":3,"host_device":0}\n'
            '{"seq":0,"kind":"transfer","t0":1,"t1":2,"src_dev":0,"dst_dev":1,"src_addr":1,"dst_addr":2,'
            '"bytes":64,"hash":0,"codeptr":1}\n'
            '{"seq":1,"kind":"kernel","t0":3,"t1":4,"src_dev":1,"dst_dev":2,"src_addr":0,"dst_addr":0,'
            '"bytes":0,"hash":0,"codeptr":1}\n'
            '{"seq":2,"kind":"alloc","t0":5,"t1":6,"src_dev":0,"dst_dev":7,"src_addr":1,"dst_addr":0,'
            '"bytes":0,"hash":0,"codeptr":1}\n')
    p = tmp_path / "viol.ndjson"
    p.write_text(text)
    with pytest.raises(ingest.TraceIOError) as ei:
        ingest.parse_trace_columns(text.encode())
    assert main(["analyze", str(p)]) == 1
    assert capsys.readouterr().err.strip() == f"dmlens: error: {type(ei.value).__name__}: {ei.value}"
