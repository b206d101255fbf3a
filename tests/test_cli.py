"""Command-line surface of the drop-in (`dmlens` cli.py:41-93): argument forms only --
the reports themselves are pinned byte-for-byte in test_reports_gpu.py."""
import pytest

from paper_2601_12713_b200.__main__ import main


def test_version(capsys):
    assert main(["version"]) == 0
    assert capsys.readouterr().out == "dmlens 0.1.0\n"


def test_oracle_flag_rejected_explicitly(capsys, tmp_path):
    assert main(["analyze", str(tmp_path / "t.trace"), "--oracle"]) == 2
    assert "--oracle" in capsys.readouterr().err


def test_audit_needs_payload_dir(capsys, tmp_path):
    assert main(["audit", str(tmp_path / "t.trace")]) == 2
    assert "--payload-dir" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["option", "positional"])
def test_audit_payload_dir_forms(capsys, tmp_path, form):
    from oracle.hash_ref import fold64_c  # checker: the digest the trace records
    p1, p2 = bytes(range(40)), bytes(range(1, 41))
    lines = ['{"dmlens":1,"num_devices":2,"host_device":0,"wall_time_ns":100}']
    for seq, p in enumerate((p1, p1, p2)):
        lines.append('{"seq":%d,"kind":"transfer","t0":%d,"t1":%d,"src_dev":0,"dst_dev":1,"src_addr":4096,'
                     '"dst_addr":8192,"bytes":%d,"hash":%d,"codeptr":0}' % (seq, 10 * seq, 10 * seq + 5, len(p),
                                                                          fold64_c(p)))
    trace = tmp_path / "t.trace"
    trace.write_text("\n".join(lines) + "\n")
    d = tmp_path / "payloads"
    d.mkdir()
    for seq, p in enumerate((p1, p1, p2)):
        (d / f"{seq}.bin").write_bytes(p)
    argv = ["audit", str(trace), "--payload-dir", str(d)] if form == "option" else ["audit", str(trace), str(d)]
    assert main(argv) == 0
    assert capsys.readouterr().out == "collision_count: 0\n"
