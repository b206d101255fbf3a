# small-trace (C1-sized, 10k events) analysis latency: wall per call, phase trace, Python profile
timeout 600 python - <<'PY'
import sys, time, cProfile, pstats, io
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.analysis import DeviceColumns
from paper_2601_12713_b200.synth import c2_trace
c = c2_trace(10_000, seed=1)
dc = DeviceColumns(c)
for _ in range(5):
    savings_columns(dc, analyze_columns(dc))
ts = []
for _ in range(20):
    torch.cuda.synchronize(); t = time.perf_counter()
    cf = analyze_columns(dc); t1 = time.perf_counter(); savings_columns(dc, cf); t2 = time.perf_counter()
    ts.append((round((t1 - t) * 1e3, 3), round((t2 - t1) * 1e3, 3)))
print(ts)
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    savings_columns(dc, analyze_columns(dc))
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14); print(s.getvalue()[:3500])
PY
B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --config c2 --n 10000 --iters 4 2>&1 | tail -24
