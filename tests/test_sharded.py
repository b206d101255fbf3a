"""Multi-rank (key-range sharded) analysis: G-way results must equal the
single-shard results exactly.  CPU: ranks as threads and as gloo processes
(world_size 2) with the oracle as the per-shard analyzer; GPU: ranks as
threads sharing one B200 with the engine."""
import os

import numpy as np
import pytest

from oracle import analysis_ref as R
from paper_2601_12713_b200 import sharded
from paper_2601_12713_b200.columns import to_columns
from tests._cases import canon_columnar, canon_oracle
from tests._gen import nasty_trace
from tests._oracle_analyzer import oracle_analyzer


def _valid_traces(k, seed0=0):
    out, s = [], seed0
    while len(out) < k:
        c = to_columns(nasty_trace(s, max_events=120))
        s += 1
        if c.n and not R.validate_cols(c):
            out.append(c)
    return out


@pytest.mark.parametrize("g", [2, 3, 4])
def test_local_ranks_with_oracle_match_single(g):
    for c in _valid_traces(60, seed0=g * 1000):
        for strict in (False, True):
            got = sharded.run_local(c, g, strict=strict, analyzer=oracle_analyzer)
            want = R.analyze_cols(c, strict=strict)
            assert canon_columnar(got, c) == canon_oracle(want, c)
            assert got.warn_index.tolist() == want.warnings
            assert got.synthetic_end_ns == want.synthetic_end


def _spread(cols, g):
    """(pairing records, UT records) per rank."""
    (ad, o_ad), (tt, o_tt) = sharded.device_owners(cols, g)
    return np.bincount(o_ad[ad], minlength=g), np.bincount(o_tt[tt], minlength=g)


@pytest.mark.parametrize("g", [2, 3, 4])
def test_one_and_four_device_traces_spread_over_ranks(g):
    """Traces with ONE target device (C2 cycles on one device; C3) and four (C4): the G-way
    findings equal the single-shard ones, and device-keyed work spreads over the ranks by
    (device, address) key rather than by device.  A key is indivisible: C2 cycles reuse one
    device address per device (one pairing key per device) and C3 has one host array in flight
    (one UT key), so only the keys that exist spread."""
    from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace
    balanced = lambda x: x.min() > 0.5 * x.mean()  # noqa: E731
    every = lambda x: x.min() > 0  # noqa: E731
    none = lambda x: True  # noqa: E731
    for c, ok_pairs, ok_ut in ((c2_trace(3000, n_targets=1, seed=8, n_host_vars=256), none, balanced),
                               (c4_trace(3000, seed=5, n_host_vars=64, palette=128), balanced, balanced),
                               (c2_trace(3000, n_targets=2 * g, seed=9), every, balanced),
                               (c3_trace(400, array_bytes=1 << 16), none, none)):
        pairs, ut = _spread(c, g)
        assert ok_pairs(pairs), pairs
        assert ok_ut(ut), ut
        for strict in (False, True):
            got = sharded.run_local(c, g, strict=strict, analyzer=oracle_analyzer)
            want = R.analyze_cols(c, strict=strict)
            assert canon_columnar(got, c) == canon_oracle(want, c)
            assert got.warn_index.tolist() == want.warnings


def test_routing_keys_match_the_kernels():
    """route_mix / route_owner restate b2l_analyze.cu's routing (fixed vectors)."""
    a = np.array([0, 1, 0xFFFFFFFFFFFFFFFF, 0xD000], np.uint64)
    b = np.array([0, 7, 3, 0x1234], np.uint64)
    key = sharded.route_mix(a, b)
    assert key.dtype == np.uint64
    # splitmix64(0) is the well-known first output of the generator seeded with 0
    assert int(sharded.route_splitmix(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    assert sharded.route_owner(key, 1).tolist() == [0, 0, 0, 0]
    assert all(0 <= o < 8 for o in sharded.route_owner(key, 8).tolist())


def test_local_ranks_report_invalid_shard():
    c = _valid_traces(1, seed0=77)[0]
    c.start_ns = c.start_ns.copy()
    c.start_ns[c.n // 2] = 0 if c.start_ns[c.n // 2 - 1] > 0 else c.start_ns[c.n // 2]
    if not R.validate_cols(c):
        pytest.skip("mutation kept the trace valid")
    with pytest.raises(sharded.EngineInvalid):
        sharded.run_local(c, 2, analyzer=oracle_analyzer)


def _gloo_worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.TorchComm()
        ok = True
        for c in _valid_traces(25, seed0=500):
            shard, base = sharded.split(c, world)[rank]
            got = sharded.analyze_sharded(shard, base, comm, analyzer=oracle_analyzer)
            if rank == 0:
                ok &= canon_columnar(got, c) == canon_oracle(R.analyze_cols(c), c)
        if rank == 0:
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2(tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "result.txt"
    mp.spawn(_gloo_worker, args=(2, port, str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 4])
def test_local_ranks_engine_on_gpu(cuda, g):
    from paper_2601_12713_b200 import analyze_columns
    from paper_2601_12713_b200.synth import c2_trace, c4_trace
    cases = _valid_traces(40, seed0=9000 + g) + [c2_trace(100_000, seed=3), c4_trace(100_000, seed=5)]
    for c in cases:
        for strict in (False, True):
            got = sharded.run_local(c, g, strict=strict)
            want = analyze_columns(c, strict=strict)
            assert canon_columnar(got, c) == canon_columnar(want, c)
            assert got.warn_index.tolist() == want.warn_index.tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 3, 4])
def test_device_resident_ranks_on_gpu(cuda, g):
    """The device-resident pipeline (b2l_shard_route / all-to-all of device rows /
    b2l_shard_unpack / engine on device sub-traces) equals the single-GPU engine."""
    from paper_2601_12713_b200 import analyze_columns
    from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace
    cases = _valid_traces(40, seed0=7000 + g) + [c2_trace(100_000, seed=3), c4_trace(100_000, seed=5),
                                                 c2_trace(30_000, n_targets=1, seed=6, n_host_vars=512),
                                                 c3_trace(2000, array_bytes=1 << 16)]
    for c in cases:
        for strict in (False, True):
            got = sharded.run_local_device(c, g, strict=strict)
            want = analyze_columns(c, strict=strict)
            assert canon_columnar(got, c) == canon_columnar(want, c)
            assert got.warn_index.tolist() == want.warn_index.tolist()
            assert got.synthetic_end_ns == want.synthetic_end_ns


@pytest.mark.gpu
def test_device_resident_invalid_shard_reports_global_indices(cuda):
    from paper_2601_12713_b200.analysis import EngineInvalid
    c = _valid_traces(1, seed0=77)[0]
    c.start_ns = c.start_ns.copy()
    c.start_ns[c.n // 2] = 0 if c.start_ns[c.n // 2 - 1] > 0 else c.start_ns[c.n // 2]
    if not R.validate_cols(c):
        pytest.skip("mutation kept the trace valid")
    with pytest.raises(EngineInvalid) as ei:
        sharded.run_local_device(c, 2)
    with pytest.raises(EngineInvalid) as ej:
        sharded.run_local(c, 2)
    assert ei.value.bad_index.tolist() == ej.value.bad_index.tolist()
    assert ei.value.bad_rules.tolist() == ej.value.bad_rules.tolist()


def _gloo_engine_worker(rank, world, port, result_path):
    """Two processes on one GPU: TorchComm over gloo for the exchange, the CUDA engine per shard."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_12713_b200 import analyze_columns
        from paper_2601_12713_b200.synth import c2_trace, c4_trace
        comm = sharded.TorchComm()
        ok = True
        from paper_2601_12713_b200.analysis import DeviceColumns
        for c in _valid_traces(10, seed0=700) + [c2_trace(50_000, seed=7), c4_trace(50_000, seed=8)]:
            shard, base = sharded.split(c, world)[rank]
            got = sharded.analyze_sharded(shard, base, comm)
            got_dev = sharded.analyze_sharded_device(DeviceColumns(shard), base, comm)
            if rank == 0:
                want = canon_columnar(analyze_columns(c), c)
                ok &= canon_columnar(got, c) == want
                ok &= canon_columnar(got_dev, c) == want
        if rank == 0:
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_two_processes_engine_on_gpu(cuda, tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "result.txt"
    mp.spawn(_gloo_engine_worker, args=(2, port, str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"


def _findings_sample(rank):
    rng = np.random.default_rng(rank)
    out = {"dd": (np.arange(4, dtype=np.int64), rng.integers(0, 99, 3), rng.integers(0, 2**63, 3, dtype=np.uint64)
                  | np.uint64(2**63), rng.integers(0, 2**63, 3, dtype=np.uint64), np.array([-1, 2, 7], np.int32),
                  np.zeros(0, np.int64)),
           "warn": np.array([rank, 5], np.int64), "ut": np.zeros(0, np.int64)}
    if rank:
        out["pairs"] = (np.arange(3, dtype=np.int64), np.array([-1, 2, 3], np.int64))
    return out


def _same_findings(a, b):
    if sorted(a) != sorted(b):
        return False
    for k in a:
        x, y = (a[k], b[k]) if isinstance(a[k], tuple) else ((a[k],), (b[k],))
        if not isinstance(b[k], type(a[k])) or len(x) != len(y):
            return False
        if any(p.dtype != q.dtype or not np.array_equal(p, q) for p, q in zip(x, y)):
            return False
    return True


def test_findings_wire_format_roundtrip():
    for r in (0, 1):
        f = _findings_sample(r)
        assert _same_findings(f, sharded._unpack_findings(sharded._pack_findings(f)))
    assert sharded._unpack_findings(sharded._pack_findings({})) == {}


def _gloo_gather_worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = sharded.TorchComm().gather0_findings(_findings_sample(rank))
        if rank == 0:
            ok = len(got) == world and all(_same_findings(_findings_sample(r), got[r]) for r in range(world))
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


def test_gloo_findings_gather_world_size_2(tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "result.txt"
    mp.spawn(_gloo_gather_worker, args=(2, port, str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"
