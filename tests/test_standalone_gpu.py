"""GPU parity of the standalone detector entry points (find_*, get_alloc_delete_pairs,
sort_by_device, validate) against outputs of the reference's own functions."""
import gzip
import json
import os

import pytest

from tests._cases import cases, trace_from_json

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _standalone_cases():
    with gzip.open(os.path.join(HERE, "golden", "standalone_cases.json.gz"), "rt") as f:
        return json.load(f)


def _pj(p):
    return [p.alloc_event.seq, p.delete_event.seq, p.synthetic_delete]


def test_standalone_detectors_match_reference(cuda):
    import paper_2601_12713_b200 as b
    from paper_2601_12713_b200.types import EventKind
    for c in _standalone_cases():
        tr = trace_from_json(c["trace"])
        ev, host, nd = tr.events, tr.host_device, tr.num_devices_total
        transfers = [e for e in ev if e.kind is EventKind.TRANSFER]
        data_ops = [e for e in ev if e.kind is not EventKind.KERNEL]
        kernels = [e for e in ev if e.kind is EventKind.KERNEL]
        tk = [e for e in kernels if e.dst_device != host]
        tt = [e for e in transfers if e.dst_device != host]
        name = c["seed"]
        assert [[str(g.hash), g.dest_device, [e.seq for e in g.events]]
                for g in b.find_duplicate_transfers(transfers)] == c["dd_raw"], name
        for key, strict in (("rt_raw", False), ("rt_raw_strict", True)):
            assert [[str(g.hash), g.src_device, g.dest_device, [[x.seq, y.seq] for x, y in g.trips]]
                    for g in b.find_round_trips(transfers, strict_pseudocode=strict)] == c[key], (name, key)
        warns = []
        assert [_pj(p) for p in b.get_alloc_delete_pairs(data_ops, warn=warns.append)] == c["pairs"], name
        assert [w.seq for w in warns] == c["warnings"], name
        assert [[g.host_addr, g.tgt_device, g.bytes, [_pj(p) for p in g.pairs]]
                for g in b.find_repeated_allocs(data_ops)] == c["ra"], name
        assert [_pj(p) for p in b.find_unused_allocs(kernels, data_ops, nd)] == c["ua_all_kernels"], name
        assert [e.seq for e in b.find_unused_transfers(kernels, transfers, nd)] == c["ut_all"], name
        assert [e.seq for e in b.find_unused_transfers(tk, tt, nd)] == c["ut_target"], name
        assert [[e.seq for e in lst] for lst in b.sort_by_device(ev, nd, key="dst")] == c["by_device_dst"], name
        assert [[e.seq for e in lst] for lst in b.sort_by_device(ev, nd, key="src")] == c["by_device_src"], name


def test_validate_matches_reference(cuda):
    import paper_2601_12713_b200 as b
    for case in cases():
        tr = trace_from_json(case["trace"])
        got = [[v.rule, v.message, v.seq] for v in b.validate(tr)]
        assert got == case.get("violations", []), case["name"]


def test_sort_by_device_out_of_range(cuda):
    import paper_2601_12713_b200 as b
    from paper_2601_12713_b200 import types as T
    e = T.TraceEvent(4, T.EventKind.KERNEL, 0, 1, 0, 5, 0, 0, 0, 0)
    with pytest.raises(b.DeviceOutOfRange):
        b.sort_by_device([e], 2)
