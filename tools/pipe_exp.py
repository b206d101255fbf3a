import sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, analyze_many, pinned_columns, savings_columns
from paper_2601_12713_b200.synth import c2_trace
c = pinned_columns(c2_trace(1_000_000))
dev = torch.device("cuda")
s = torch.cuda.Stream()
def up():
    d = DeviceColumns(c, dev, stream=s)
    d.ready.synchronize()
    return d
for _ in range(3): up()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): up()
print("upload only ms", (time.perf_counter() - t) / 10 * 1e3)
d = up()
for _ in range(3): savings_columns(d, analyze_columns(d, with_savings=True))
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): savings_columns(d, analyze_columns(d, with_savings=True))
torch.cuda.synchronize(); print("analyze only ms", (time.perf_counter() - t) / 10 * 1e3)
for _ in analyze_many([c] * 3): pass
torch.cuda.synchronize(); t = time.perf_counter()
marks = [t]
for _ in analyze_many([c] * 20): marks.append(time.perf_counter())
torch.cuda.synchronize(); print("analyze_many ms", (time.perf_counter() - t) / 20 * 1e3, [round(1e3*(y-x),2) for x,y in zip(marks, marks[1:])])
# upload concurrently with analysis, without Python thread: queue 10 uploads then analyze 10 times
torch.cuda.synchronize(); t = time.perf_counter()
ds = [DeviceColumns(c, dev, stream=s) for _ in range(10)]
t1 = time.perf_counter()
for x in ds:
    savings_columns(d, analyze_columns(d, with_savings=True))
torch.cuda.synchronize(); print("10 uploads queued (%.2f ms host) + 10 analyses: ms/step" % ((t1 - t) * 1e3), (time.perf_counter() - t) / 10 * 1e3)
