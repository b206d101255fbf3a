"""CPU: the analysis oracle (oracle/analysis_ref.py) against the reference's
own outputs -- the committed golden cases, and the live reference on
thousands of random traces when the checkout is present."""
import pytest

from oracle import analysis_ref as R
from tests._cases import canon_oracle, canon_ref_json, cases, columns_of, trace_from_json


def _check_case(case):
    cols = columns_of(case)
    viol = R.validate_cols(cols)
    if "violations" in case:
        assert [list(v) for v in viol] == case["violations"], case["name"]
        return
    assert viol == [], case["name"]
    for key, strict in (("findings", False), ("findings_strict", True)):
        rf = R.analyze_cols(cols, strict=strict)
        assert canon_oracle(rf, cols) == canon_ref_json(case[key]), (case["name"], key)
    rf = R.analyze_cols(cols)
    seq = [int(x) for x in cols.seq]
    assert [[seq[i], "delete without a live allocation at this device address"] for i in rf.warnings] == \
        case["warnings"]
    est = R.estimate_cols(cols, rf, cols.wall_time_ns)
    e = case["estimate"]
    assert est["per_category_ns"] == e["per_category_ns"]
    assert est["union_ns"] == e["union_ns"] and est["wall_time_ns"] == e["wall_time_ns"]
    assert repr(est["predicted_speedup"]) == e["predicted_speedup"]
    assert sorted(seq[i] for i in est["eliminable"]) == e["eliminable_seqs"]
    assert list(est["warnings"]) == e["warnings"]
    rows = R.attribute_cols(cols, rf, cols.wall_time_ns)
    got = [[r[0], list(cols.locs[int(cols.loc[r[1]])]), r[2], r[3], r[4], repr(r[5])] for r in rows]
    assert got == case["attribute"], case["name"]


def test_oracle_matches_golden_cases():
    cs = cases()
    assert len(cs) > 300
    for case in cs:
        _check_case(case)


@pytest.mark.slow
def test_oracle_matches_live_reference_random_traces():
    from tests.conftest import REFERENCE_SRC, import_reference
    dmlens = import_reference()
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(os.path.dirname(REFERENCE_SRC),
                                                                               "tests", "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    from paper_2601_12713_b200.columns import to_columns
    from tests._cases import canon_findings_objects
    for seed in range(300, 3300):
        tr = conf.random_trace(seed)
        cols = to_columns(tr)
        for strict in (False, True):
            want = canon_findings_objects(dmlens.analyze(tr, strict_pseudocode=strict))
            assert canon_oracle(R.analyze_cols(cols, strict=strict), cols) == want, (seed, strict)
