# End to end: the CLI on a 1M-event C2 NDJSON -- ours vs the unmodified reference (baseline/_ref)
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
ls -la /tmp/c2_1m.ndjson
t() { local label=$1; shift; local out=$1; shift; local s=$(date +%s.%N); "$@" > "$out"; local rc=$?; local e=$(date +%s.%N); echo "$label rc=$rc wall $(python -c "print(round($e-$s,2))") s"; }
for i in 1 2; do t ours /tmp/ours.txt python -m paper_2601_12713_b200 analyze /tmp/c2_1m.ndjson; done
t "ours --json" /tmp/ours.json python -m paper_2601_12713_b200 analyze --json /tmp/c2_1m.ndjson
PYTHONPATH=baseline/_ref t reference /tmp/ref.txt timeout 1200 python baseline/_ref/bin/dmlens analyze /tmp/c2_1m.ndjson
PYTHONPATH=baseline/_ref t "reference --json" /tmp/ref.json timeout 1200 python baseline/_ref/bin/dmlens analyze --json /tmp/c2_1m.ndjson
cmp /tmp/ours.txt /tmp/ref.txt && echo "text reports byte-identical"
cmp /tmp/ours.json /tmp/ref.json && echo "json reports byte-identical"
head -12 /tmp/ours.txt
