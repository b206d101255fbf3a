for n in 1000000 10000000; do timeout 300 python tools/time_analysis.py --device --config c2 --n $n --iters 3 2>&1 | head -3; done
timeout 300 python - <<'PY'
import time, sys, os, subprocess
sys.path.insert(0, ".")
t0 = time.perf_counter()
import paper_2601_12713_b200 as b
from paper_2601_12713_b200 import _lib
_lib.lib()
t1 = time.perf_counter()
import torch; torch.cuda.init(); torch.zeros(1, device="cuda")
t2 = time.perf_counter()
print(f"import {1e3*(t1-t0):.0f} ms, cuda init {1e3*(t2-t1):.0f} ms")
PY
