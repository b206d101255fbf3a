"""Capture agent (SPEC.md "ompt-shim"): the behaviours the reference's capture tests pin
(pkg/shim/test/capture.test.ts) on the native agent, plus the B200 part -- payloads hashed on
the GPU from their device copies -- and the OMPT tool glue driven by a fake runtime.
Kernel / alloc / delete capture needs no GPU; anything that hashes is marked gpu."""
import ctypes
import json
import os

import numpy as np
import pytest

from paper_2601_12713_b200.capture import CaptureShim

HOST_RUNTIME_ID = 4  # runtimes number the host above the targets (capture.test.ts:10)


def new_shim(**kw):
    t = [0]

    def clock():
        t[0] += 100
        return t[0]
    return CaptureShim(HOST_RUNTIME_ID, clock=clock, **kw)


def lines(text):
    return [json.loads(x) for x in text.rstrip("\n").split("\n")]


def events(shim, wall=None):
    return lines(shim.finalize(wall))[1:]


# ---------------------------------------------------------------- target (kernel) capture
def test_pairs_begin_end_into_one_kernel_event():
    shim = new_shim()
    shim.on_target_begin(1, 0, codeptr=0x400100, time_ns=10)
    shim.on_target_end(1, 0, time_ns=60)
    ev = events(shim)
    assert len(ev) == 1
    assert {k: ev[0][k] for k in ("kind", "t0", "t1", "src_dev", "dst_dev", "codeptr")} == {
        "kind": "kernel", "t0": 10, "t1": 60, "src_dev": 1, "dst_dev": 1, "codeptr": 0x400100}


def test_one_event_per_region():
    shim = new_shim()
    for i in range(2):
        shim.on_target_begin(i, 0, time_ns=i * 100)
        shim.on_target_end(i, 0, time_ns=i * 100 + 50)
    assert sum(e["kind"] == "kernel" for e in events(shim)) == 2


def test_unmatched_ends_counted():
    shim = new_shim()
    shim.on_target_end(99, 0, time_ns=5)
    assert events(shim) == []
    assert shim.warnings.unmatched_ends == 1


def test_ops_open_at_finalize_reported():
    shim = new_shim()
    shim.on_target_begin(1, 0, time_ns=5)
    shim.finalize()
    assert shim.warnings.unfinished_at_exit == 1


# ---------------------------------------------------------------- data ops without payloads
def test_unreadable_transfer_recorded_opaque():
    shim = new_shim()
    shim.on_data_op_begin(3, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=0x1000, dest_addr=0xd000,
                          bytes=512, time_ns=10)
    shim.on_data_op_end(3, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=20)
    ev = events(shim)
    assert ev[0]["hash"] == 0 and ev[0]["bytes"] == 0
    assert shim.warnings.hash_skipped == 1


def test_alloc_delete_share_the_device_address():
    shim = new_shim()
    shim.on_data_op_begin(4, "alloc", HOST_RUNTIME_ID, 0, src_addr=0x1000, dest_addr=0xd000, bytes=64, time_ns=0)
    shim.on_data_op_end(4, "alloc", HOST_RUNTIME_ID, 0, time_ns=10)
    shim.on_data_op_begin(5, "delete", HOST_RUNTIME_ID, 0, dest_addr=0xd000, time_ns=20)
    shim.on_data_op_end(5, "delete", HOST_RUNTIME_ID, 0, time_ns=30)
    ev = events(shim)
    assert [e["kind"] for e in ev] == ["alloc", "delete"]
    assert ev[0]["dst_addr"] == 0xd000 and ev[1]["dst_addr"] == 0xd000 and ev[0]["bytes"] == 64


def test_malformed_ops_dropped_and_counted():
    shim = new_shim()
    shim.on_data_op_begin(6, "alloc", HOST_RUNTIME_ID, 0, dest_addr=0, bytes=64, time_ns=0)
    shim.on_data_op_begin(7, "delete", HOST_RUNTIME_ID, 0, dest_addr=0, time_ns=5)
    assert events(shim) == []
    assert shim.warnings.dropped_malformed == 2


# ---------------------------------------------------------------- sequence numbers and merging
def test_seqs_unique_and_increasing_in_t0_arrival_order():
    shim = new_shim()
    for i in range(30):  # interleaved ops from three threads, overlapping in time
        shim.on_target_begin(i, 0, thread_id=i % 3, time_ns=1000 - i * 10)
        shim.on_target_end(i, 0, thread_id=i % 3, time_ns=2000 + i)
    ev = events(shim)
    assert len(ev) == 30 and len({e["seq"] for e in ev}) == 30
    for a, b in zip(ev, ev[1:]):
        assert b["t0"] >= a["t0"] and b["seq"] > a["seq"]


def test_device_ids_normalised_with_host_at_slot_0():
    shim = new_shim()
    assert shim.device_slot(HOST_RUNTIME_ID) == 0
    assert shim.device_slot(2) == 1
    assert shim.device_slot(0) == 2
    assert shim.device_slot(2) == 1
    shim.on_target_begin(1, 2, time_ns=0)
    shim.on_target_end(1, 2, time_ns=1)
    header = lines(shim.finalize())[0]
    assert header["num_devices"] == 3 and header["host_device"] == 0


def test_wall_time_from_last_end_unless_given():
    shim = new_shim()
    shim.on_target_begin(1, 0, time_ns=10)
    shim.on_target_end(1, 0, time_ns=470)
    assert lines(shim.finalize())[0]["wall_time_ns"] == 470
    assert lines(shim.finalize(9999))[0]["wall_time_ns"] == 9999


def test_output_path_required(monkeypatch, tmp_path):
    from paper_2601_12713_b200.errors import EngineError
    monkeypatch.delenv("DMLENS_OUT", raising=False)
    shim = new_shim()
    with pytest.raises(EngineError, match="DMLENS_OUT"):
        shim.write_trace()


@pytest.mark.gpu
def test_trace_parses_with_the_reference_format(cuda, tmp_path):
    """The merged output satisfies the trace-model invariants (SPEC ompt-shim): our ingest,
    which accepts exactly what traceio.parse_trace accepts, parses and validates it."""
    from paper_2601_12713_b200 import ingest
    shim = new_shim(out_path=str(tmp_path / "t.ndjson"))
    t = 0
    for i in range(20):
        shim.on_data_op_begin(100 + i, "alloc", HOST_RUNTIME_ID, i % 2, src_addr=0x1000 + i, dest_addr=0xd000 + i,
                              bytes=64, thread_id=i % 3, time_ns=t)
        shim.on_data_op_end(100 + i, "alloc", HOST_RUNTIME_ID, i % 2, thread_id=i % 3, time_ns=t + 5)
        shim.on_target_begin(i, i % 2, thread_id=i % 3, time_ns=t + 10)
        shim.on_target_end(i, i % 2, thread_id=i % 3, time_ns=t + 20)
        shim.on_data_op_begin(200 + i, "delete", HOST_RUNTIME_ID, i % 2, dest_addr=0xd000 + i, thread_id=i % 3,
                              time_ns=t + 30)
        shim.on_data_op_end(200 + i, "delete", HOST_RUNTIME_ID, i % 2, thread_id=i % 3, time_ns=t + 35)
        t += 7  # overlapping ops across threads
    path = shim.write_trace()
    cols = ingest.parse_trace_columns(open(path, "rb").read())
    assert cols.n == 60 and cols.num_devices_total == 3


# ---------------------------------------------------------------- payloads hashed on the GPU
@pytest.mark.gpu
def test_h2d_host_payload_hashed_at_begin(cuda):
    from oracle.hash_ref import fold64_c as hash_bytes  # the checker, not the engine
    shim = new_shim()
    payload = bytes([1, 2, 3, 4, 5, 6, 7, 8])
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=0x1000, dest_addr=0xd000, bytes=8,
                          host_buffer=payload, time_ns=10)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=20)
    ev = events(shim)[0]
    assert {k: ev[k] for k in ("kind", "t0", "t1", "src_dev", "dst_dev", "bytes")} == {
        "kind": "transfer", "t0": 10, "t1": 20, "src_dev": 0, "dst_dev": 1, "bytes": 8}
    assert ev["hash"] == hash_bytes(payload)


@pytest.mark.gpu
def test_h2d_landed_device_copy_hashed_at_end(cuda):
    import torch

    from oracle.hash_ref import fold64_c as hash_bytes  # the checker, not the engine
    shim = new_shim()
    payload = np.arange(4099, dtype=np.uint8).tobytes()  # ragged length
    dev = torch.empty(len(payload), dtype=torch.uint8, device=cuda)
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=0x1000, dest_addr=dev.data_ptr(),
                          bytes=len(payload), time_ns=10)
    dev.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))  # the runtime's copy lands
    torch.cuda.synchronize()
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=20, device_buffer=dev)
    dev.fill_(0)  # the program's next kernel overwrites it: the digest was taken in the callback
    assert events(shim)[0]["hash"] == hash_bytes(payload)


@pytest.mark.gpu
def test_d2h_device_source_hashed_at_end(cuda):
    import torch

    from oracle.hash_ref import fold64_c as hash_bytes  # the checker, not the engine
    shim = new_shim()
    src = torch.full((4,), 9, dtype=torch.uint8, device=cuda)
    shim.on_data_op_begin(2, "transfer_from_device", 0, HOST_RUNTIME_ID, src_addr=src.data_ptr(), dest_addr=0x1000,
                          bytes=4, time_ns=10)
    shim.on_data_op_end(2, "transfer_from_device", 0, HOST_RUNTIME_ID, time_ns=30, device_buffer=src)
    ev = events(shim)[0]
    assert ev["hash"] == hash_bytes(bytes([9, 9, 9, 9])) and ev["bytes"] == 4


@pytest.mark.gpu
def test_d2h_landed_host_buffer_hashed_at_end(cuda):
    from oracle.hash_ref import fold64_c as hash_bytes  # the checker, not the engine
    shim = new_shim()
    shim.on_data_op_begin(2, "transfer_from_device", 0, HOST_RUNTIME_ID, src_addr=0xd000, dest_addr=0x1000,
                          bytes=4, time_ns=10)
    shim.on_data_op_end(2, "transfer_from_device", 0, HOST_RUNTIME_ID, time_ns=30, host_buffer=bytes([9] * 4))
    assert events(shim)[0]["hash"] == hash_bytes(bytes([9] * 4))


@pytest.mark.gpu
def test_full_64_bit_hash_as_bare_integer(cuda):
    shim = new_shim()
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=1, dest_addr=2, bytes=1,
                          host_buffer=bytes.fromhex("ff"), time_ns=0)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=1)
    line = shim.finalize().split("\n")[1]
    assert '"hash":12844647536454529852' in line and '"hash":"' not in line


@pytest.mark.gpu
def test_wire_field_names(cuda):
    shim = new_shim()
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=0x1000, dest_addr=0xd000, bytes=16,
                          host_buffer=bytes(range(16)), codeptr=0x400200, time_ns=10)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=42)
    header, ev = lines(shim.finalize())
    assert header == {"dmlens": 1, "num_devices": 2, "host_device": 0, "wall_time_ns": 42}
    assert list(ev) == ["seq", "kind", "t0", "t1", "src_dev", "dst_dev", "src_addr", "dst_addr", "bytes", "hash",
                        "codeptr"]


@pytest.mark.gpu
def test_trace_and_audit_sidecars_written(cuda, tmp_path):
    import torch
    shim = new_shim(out_path=str(tmp_path / "out.trace"), audit_dir=str(tmp_path / "payloads"))
    dev = torch.full((8,), 7, dtype=torch.uint8, device=cuda)
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=1, dest_addr=dev.data_ptr(),
                          bytes=8, time_ns=0)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=5, device_buffer=dev)
    dev.fill_(255)  # later reuse: the sidecar is a snapshot
    assert shim.write_trace() == str(tmp_path / "out.trace")
    assert '"kind":"transfer"' in open(tmp_path / "out.trace").read()
    assert os.listdir(tmp_path / "payloads") == ["0.bin"]
    assert open(tmp_path / "payloads" / "0.bin", "rb").read() == bytes([7] * 8)


@pytest.mark.gpu
def test_unhashable_device_buffer_still_emitted_opaque(cuda):
    """A hashing failure (here: a 'device' pointer that is plain host memory) never drops the
    transfer: it is emitted opaque and counted, as capture.ts:212-217 records an unreadable one."""
    shim = new_shim()
    host = np.full(64, 3, dtype=np.uint8)
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=1, dest_addr=0xd000, bytes=64,
                          time_ns=0)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=5,
                        device_buffer=int(host.ctypes.data))
    evs = events(shim)
    assert len(evs) == 1 and evs[0]["kind"] == "transfer"
    assert evs[0]["bytes"] == 0 and evs[0]["hash"] == 0
    assert shim.warnings.hash_skipped == 1


@pytest.mark.gpu
def test_large_device_payload_goes_through_k2(cuda):
    import torch

    from oracle.hash_ref import fold64_c
    shim = new_shim()
    n = (32 << 20) + 13
    dev = torch.randint(0, 256, (n,), dtype=torch.uint8, device=cuda)
    shim.on_data_op_begin(1, "transfer_to_device", HOST_RUNTIME_ID, 0, src_addr=1, dest_addr=dev.data_ptr(),
                          bytes=n, time_ns=0)
    shim.on_data_op_end(1, "transfer_to_device", HOST_RUNTIME_ID, 0, time_ns=5, device_buffer=dev)
    assert events(shim)[0]["hash"] == fold64_c(dev.cpu().numpy().tobytes())


# ---------------------------------------------------------------- the OMPT tool, fake runtime
class _Data(ctypes.Union):
    _fields_ = [("value", ctypes.c_uint64), ("ptr", ctypes.c_void_p)]


_TARGET_EMI = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.POINTER(_Data), ctypes.c_void_p)
_DATA_OP_EMI = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_size_t, ctypes.c_void_p)
_INIT = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(_Data))
_FINI = ctypes.CFUNCTYPE(None, ctypes.POINTER(_Data))


class _StartResult(ctypes.Structure):
    _fields_ = [("initialize", ctypes.c_void_p), ("finalize", ctypes.c_void_p), ("tool_data", _Data)]


@pytest.mark.gpu
def test_ompt_tool_with_a_fake_runtime(cuda, tmp_path, monkeypatch):
    """ompt_start_tool -> initialize registers the two EMI callbacks through ompt_set_callback;
    a program's map(to:) / target / map(from:) sequence through them yields a valid trace whose
    transfer digests equal the oracle fold of the payloads (hashed from the device copies)."""
    import torch

    from oracle.hash_ref import fold64_c as hash_bytes  # the checker, not the engine
    from paper_2601_12713_b200 import _build, ingest
    monkeypatch.setenv("DMLENS_OUT", str(tmp_path / "omp.trace"))
    tool = ctypes.CDLL(_build.OMPT_LIB)
    tool.ompt_start_tool.restype = ctypes.POINTER(_StartResult)
    res = tool.ompt_start_tool(51, b"fake-runtime").contents
    callbacks = {}
    SETCB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.c_void_p)
    set_cb = SETCB(lambda ev, fn: callbacks.__setitem__(ev, fn) or 5)  # ompt_set_always
    LOOKUP = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_char_p)
    lookup = LOOKUP(lambda name: ctypes.cast(set_cb, ctypes.c_void_p).value if name == b"ompt_set_callback" else None)
    host_dev, target = 1, 0
    assert _INIT(res.initialize)(ctypes.cast(lookup, ctypes.c_void_p), host_dev, ctypes.byref(res.tool_data)) == 1
    assert set(callbacks) == {33, 34}
    target_emi, data_op = _TARGET_EMI(callbacks[33]), _DATA_OP_EMI(callbacks[34])

    payload = np.frombuffer(np.random.default_rng(3).bytes(40000), dtype=np.uint8).copy()
    dev = torch.empty(payload.size, dtype=torch.uint8, device=cuda)
    op = ctypes.c_uint64(0)
    tdata = _Data()
    BEGIN, END = 1, 2
    # alloc, map(to:) (the copy lands between begin and end), target region, map(from:), delete
    data_op(BEGIN, None, None, ctypes.byref(op), 1, payload.ctypes.data, host_dev, dev.data_ptr(), target,
            payload.size, 0x401000)
    data_op(END, None, None, ctypes.byref(op), 1, payload.ctypes.data, host_dev, dev.data_ptr(), target,
            payload.size, 0x401000)
    data_op(BEGIN, None, None, ctypes.byref(op), 2, payload.ctypes.data, host_dev, dev.data_ptr(), target,
            payload.size, 0x401010)
    dev.copy_(torch.from_numpy(payload))
    torch.cuda.synchronize()
    data_op(END, None, None, ctypes.byref(op), 2, payload.ctypes.data, host_dev, dev.data_ptr(), target,
            payload.size, 0x401010)
    target_emi(1, BEGIN, target, None, None, ctypes.byref(tdata), 0x401020)
    dev[:8].fill_(42)  # the kernel writes
    torch.cuda.synchronize()
    target_emi(1, END, target, None, None, ctypes.byref(tdata), 0x401020)
    out = np.zeros_like(payload)
    data_op(BEGIN, None, None, ctypes.byref(op), 3, dev.data_ptr(), target, out.ctypes.data, host_dev,
            payload.size, 0x401030)
    out[:] = dev.cpu().numpy()
    data_op(END, None, None, ctypes.byref(op), 3, dev.data_ptr(), target, out.ctypes.data, host_dev,
            payload.size, 0x401030)
    data_op(BEGIN, None, None, ctypes.byref(op), 4, None, host_dev, dev.data_ptr(), target, 0, 0x401040)
    data_op(END, None, None, ctypes.byref(op), 4, None, host_dev, dev.data_ptr(), target, 0, 0x401040)
    _FINI(res.finalize)(ctypes.byref(res.tool_data))

    text = open(tmp_path / "omp.trace").read()
    ev = lines(text)[1:]
    assert [e["kind"] for e in ev] == ["alloc", "transfer", "kernel", "transfer", "delete"]
    assert ev[1]["hash"] == hash_bytes(payload.tobytes())
    assert ev[3]["hash"] == hash_bytes(out.tobytes()) != ev[1]["hash"]
    assert ev[1]["dst_dev"] == ev[2]["dst_dev"] == 1 and ev[1]["src_dev"] == 0
    cols = ingest.parse_trace_columns(text.encode())
    assert cols.n == 5
