timeout 900 python -m pytest tests/test_sharded.py -q -x 2>&1 | grep -E "^E  |passed|failed" | head -20
timeout 600 python - <<'PY'
import time, sys
sys.path.insert(0, ".")
from paper_2601_12713_b200 import sharded
from paper_2601_12713_b200.synth import c2_trace
for n in (2_000_000, 8_000_000):
    c = c2_trace(n, seed=5)
    for g in (2, 4, 8):
        sharded.run_local_device(c, g)
        t = time.perf_counter()
        for _ in range(3):
            sharded.run_local_device(c, g)
        dt = (time.perf_counter() - t) / 3
        print(f"n={n} G={g} run_local_device {dt*1e3:.1f} ms  {n/dt/1e6:.1f} M ev/s (all ranks share one GPU)", flush=True)
PY
bash tools/gpu/shard_t2.sh 2>&1 | tail -9
