timeout 600 python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d['analysis']; print('bench no-cpu', a['value'], a['e2e']['value'])"
timeout 600 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.analysis import pinned_columns
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(1_000_000)
big = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True); del big
p = pinned_columns(c)
import numpy as np
for _ in range(3): savings_columns(p, analyze_columns(p))
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20): savings_columns(p, analyze_columns(p))
torch.cuda.synchronize(); print("after 16GB pinned churn: %.3f ms/step" % ((time.perf_counter() - t) / 20 * 1e3))
PY
