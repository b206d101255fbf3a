timeout 600 python - <<'PY'
import time, sys, os, ctypes
sys.path.insert(0, ".")
from paper_2601_12713_b200 import ingest, _lib
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(1_000_000)
kinds = ["transfer", "alloc", "delete", "kernel"]
lines = ['{"dmlens":1,"num_devices":%d,"host_device":%d,"wall_time_ns":%d}' % (c.num_devices_total, c.host_device, c.wall_time_ns or 0)]
for i in range(c.n):
    lines.append('{"seq":%d,"kind":"%s","t0":%d,"t1":%d,"src_dev":%d,"dst_dev":%d,"src_addr":%d,"dst_addr":%d,"bytes":%d,"hash":%d,"codeptr":%d}' % (c.seq[i], kinds[c.kind[i]], c.start_ns[i], c.end_ns[i], c.src_device[i], c.dst_device[i], c.src_addr[i], c.dst_addr[i], c.bytes[i], c.hash[i], 4096 + (i % 7)))
raw = ("\n".join(lines) + "\n").encode()
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)), "bytes", len(raw))
L = _lib.lib()
L.b2l_ingest_ndjson.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.POINTER(ingest._Ingest))]
L.b2l_ingest_free.argtypes = [ctypes.POINTER(ingest._Ingest)]
for th in (1, 4, 16, len(os.sched_getaffinity(0))):
    best = 1e9
    for _ in range(3):
        out = ctypes.POINTER(ingest._Ingest)()
        t = time.perf_counter(); L.b2l_ingest_ndjson(raw, len(raw), th, ctypes.byref(out)); best = min(best, time.perf_counter() - t)
        L.b2l_ingest_free(out)
    print(f"threads={th} native parse {best*1e3:.1f} ms  {1e6/best/1e6:.1f} M ev/s", flush=True)
for _ in range(3):
    t = time.perf_counter(); cols = ingest.parse_trace_columns(raw); dt = time.perf_counter() - t
    print(f"parse_trace_columns (parse + GPU sort/validate) {dt*1e3:.1f} ms  {cols.n/dt/1e6:.1f} M ev/s", flush=True)
PY
