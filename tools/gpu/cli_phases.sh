timeout 300 python - <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(1_000_000)
kinds = ["transfer", "alloc", "delete", "kernel"]
with open("/tmp/c2_1m.ndjson", "w") as f:
    f.write('{"dmlens":1,"num_devices":%d,"host_device":%d,"wall_time_ns":%d}\n' % (c.num_devices_total, c.host_device, c.wall_time_ns or 0))
    for i in range(c.n):
        f.write('{"seq":%d,"kind":"%s","t0":%d,"t1":%d,"src_dev":%d,"dst_dev":%d,"src_addr":%d,"dst_addr":%d,"bytes":%d,"hash":%d,"codeptr":%d}\n' % (c.seq[i], kinds[c.kind[i]], c.start_ns[i], c.end_ns[i], c.src_device[i], c.dst_device[i], c.src_addr[i], c.dst_addr[i], c.bytes[i], c.hash[i], 4096 + (i % 7)))
PY
timeout 300 python - <<'PY'
import time
t0 = time.perf_counter()
import sys; sys.path.insert(0, ".")
import paper_2601_12713_b200 as b
from paper_2601_12713_b200 import _lib
t1 = time.perf_counter()
print("device count", _lib.device_count())
t2 = time.perf_counter()
from paper_2601_12713_b200.__main__ import _load
cols = _load("/tmp/c2_1m.ndjson")
t3 = time.perf_counter()
from paper_2601_12713_b200.analysis import analyze_columns
from paper_2601_12713_b200.reporting import build_report, render_text
cf = analyze_columns(cols)
t4 = time.perf_counter()
rep = build_report(cols, cf)
t5 = time.perf_counter()
txt = render_text(rep, color=False)
t6 = time.perf_counter()
print(f"import {t1-t0:.3f}  cuda-init {t2-t1:.3f}  load(read+parse+sort+validate) {t3-t2:.3f}  analyze {t4-t3:.3f}  report {t5-t4:.3f}  render {t6-t5:.3f}")
PY

t() { local label=$1; shift; local s=$(date +%s.%N); "$@" > /dev/null; local e=$(date +%s.%N); echo "$label wall $(python -c "print(round($e-$s,2))") s"; }
for i in 1 2; do t "cli analyze" python -m paper_2601_12713_b200 analyze /tmp/c2_1m.ndjson; done
timeout 600 python -m pytest tests/test_reports_gpu.py -q 2>&1 | tail -1
