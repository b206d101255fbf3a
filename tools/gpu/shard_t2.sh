B2L_SHARD_TRACE=1 timeout 600 python - <<'PY'
import time, sys
sys.path.insert(0, ".")
from paper_2601_12713_b200 import sharded
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(2_000_000, seed=5)
for it in range(3):
    t = time.perf_counter()
    sharded.run_local_device(c, 2)
    print("total", (time.perf_counter() - t) * 1e3, "ms", flush=True)
PY
