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
