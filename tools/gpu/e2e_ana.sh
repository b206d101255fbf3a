# analysis e2e (host pinned columns) per-iteration times and where they go, C2 1M
timeout 600 python - <<'PY'
import sys, time, cProfile, pstats, io, os
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.analysis import pinned_columns, DeviceColumns
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(1_000_000)
d = DeviceColumns(c)
p = pinned_columns(c)
for name, cols in (("device", d), ("pinned", p)):
    ts = []
    for i in range(12):
        torch.cuda.synchronize(); t = time.perf_counter()
        cf = analyze_columns(cols); t1 = time.perf_counter()
        savings_columns(cols, cf); torch.cuda.synchronize(); t2 = time.perf_counter()
        ts.append((round((t1 - t) * 1e3, 3), round((t2 - t1) * 1e3, 3)))
    print(name, ts, flush=True)
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    savings_columns(p, analyze_columns(p))
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(12); print(s.getvalue()[:3000])
PY
B2L_TRACE=1 timeout 300 python - <<'PY' 2>&1 | tail -24
import sys; sys.path.insert(0, ".")
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.analysis import pinned_columns
from paper_2601_12713_b200.synth import c2_trace
p = pinned_columns(c2_trace(1_000_000))
for _ in range(3):
    savings_columns(p, analyze_columns(p))
PY
