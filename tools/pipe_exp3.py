"""Interference between a large host->device upload and the analysis (results D2H, kernels)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, pinned_columns, savings_columns
from paper_2601_12713_b200.synth import c2_trace
c = pinned_columns(c2_trace(1_000_000))
dev = torch.device("cuda")
d = DeviceColumns(c, dev)
big = torch.empty(400 << 20, dtype=torch.uint8, pin_memory=True)
dbig = torch.empty(400 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
for _ in range(3): savings_columns(d, analyze_columns(d, with_savings=True))
def run(label, bg):
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(s):
            dbig.copy_(big, non_blocking=True)  # ~7.5 ms of H2D
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        savings_columns(d, analyze_columns(d, with_savings=True))
        ts.append(1e3 * (time.perf_counter() - t))
    torch.cuda.synchronize()
    print(label, [round(x, 3) for x in ts])
run("analysis alone            ", False)
run("analysis beside a 400MB H2D", True)
# d2h rate while H2D runs
h = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
dd = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
s2 = torch.cuda.Stream()
for bg in (False, True):
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(s):
            dbig.copy_(big, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s2):
        e0.record(s2); h.copy_(dd, non_blocking=True); e1.record(s2)
    torch.cuda.synchronize()
    print("64MB D2H", "beside H2D" if bg else "alone", round(e0.elapsed_time(e1), 3), "ms")
