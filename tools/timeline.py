"""Warm GPU timeline of one analyze+savings step (torch.profiler / CUPTI sees libb2l's kernels):
per-kernel warm durations, streams, GPU-busy time vs the step's wall time, and the idle gaps.
  python tools/timeline.py --config c2 --n 1000000 [--json out.json]"""
import argparse
import json
import sys
import time
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2601_12713_b200 import analyze_columns, savings_columns  # noqa: E402
from paper_2601_12713_b200.analysis import DeviceColumns  # noqa: E402
from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--json", default=None)
ap.add_argument("--host", action="store_true", help="host columns (e2e) instead of device-resident")
ap.add_argument("--streams", action="store_true", help="print every op per stream")
ap.add_argument("--many", type=int, default=0, help="profile analyze_many over this many copies of the trace")
ap.add_argument("--bg-h2d", action="store_true", help="a 400 MB host->device copy runs beside the analysis")
a = ap.parse_args()
gen = {"c2": lambda: c2_trace(a.n), "c3": lambda: c3_trace(max(1, a.n // 3)), "c4": lambda: c4_trace(a.n)}[a.config]
c = gen()
cols = c if a.host else DeviceColumns(c)
if a.host:
    from paper_2601_12713_b200.analysis import pinned_columns
    cols = pinned_columns(c)
for _ in range(5):
    savings_columns(cols, analyze_columns(cols, with_savings=True))
torch.cuda.synchronize()
if a.many:
    from paper_2601_12713_b200.analysis import analyze_many, pinned_columns
    pc = pinned_columns(c)
    for _ in analyze_many([pc] * 3):
        pass
if a.bg_h2d:
    big = torch.empty(400 << 20, dtype=torch.uint8, pin_memory=True)
    dbig = torch.empty(400 << 20, dtype=torch.uint8, device="cuda")
    bgs = torch.cuda.Stream()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    if a.bg_h2d:
        with torch.cuda.stream(bgs):
            dbig.copy_(big, non_blocking=True)
    t0 = time.perf_counter()
    if a.many:
        marks = [time.perf_counter()]
        for _ in analyze_many([pc] * a.many):
            marks.append(time.perf_counter())
        print("analyze_many step ms:", [round(1e3 * (y - x), 3) for x, y in zip(marks, marks[1:])])
        t1 = time.perf_counter()
    else:
        cf = analyze_columns(cols, with_savings=True)
        t1 = time.perf_counter()
        savings_columns(cols, cf)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = []
for e in evs:
    kern.append((e.time_range.start, e.time_range.end, e.name))
kern.sort()
if not kern:
    print("no CUDA activity recorded")
    sys.exit(0)
start, end = kern[0][0], max(k[1] for k in kern)
# union of busy intervals
busy, cur_s, cur_e = 0, None, None
for s_, e_, _ in kern:
    if cur_e is None or s_ > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
busy += cur_e - cur_s
agg = defaultdict(lambda: [0, 0.0])
for s_, e_, nm in kern:
    k = nm.replace("void ", "")[:70]
    agg[k][0] += 1
    agg[k][1] += e_ - s_
tot = sum(v[1] for v in agg.values())
print(f"{a.config} n={c.n}: wall analyze {1e3 * (t1 - t0):.3f} ms + savings {1e3 * (t2 - t1):.3f} ms; GPU span "
      f"{(end - start) / 1e3:.3f} ms, busy (union) {busy / 1e3:.3f} ms, kernel sum {tot / 1e3:.3f} ms, "
      f"{len(kern)} activities")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{us:9.1f} us {n:4d}x  {k}")
# per-stream view from the chrome trace (kernel/memcpy "args.stream")
import os
import tempfile
tmp = os.path.join(tempfile.gettempdir(), "b2l_tl.json")
prof.export_chrome_trace(tmp)
tr = json.load(open(tmp))
per = defaultdict(list)
for e in tr.get("traceEvents", []):
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e:
        per[e.get("args", {}).get("stream")].append((e["ts"], e["dur"], e["name"][:50]))
t00 = min(x[0] for v in per.values() for x in v)
for st, v in sorted(per.items(), key=lambda kv: -sum(x[1] for x in kv[1])):
    v.sort()
    span = v[-1][0] + v[-1][1] - v[0][0]
    print(f"stream {st}: {len(v)} ops, busy {sum(x[1] for x in v):.1f} us, span {span:.1f} us "
          f"[{v[0][0] - t00:.1f} .. {v[-1][0] + v[-1][1] - t00:.1f}]")
if a.streams:
    for st, v in per.items():
        print(f"--- stream {st}")
        for ts, dur, nm in v:
            print(f"  {ts - t00:9.1f} {dur:7.1f}  {nm}")
if a.json:
    json.dump({"config": a.config, "n": c.n, "wall_ms": 1e3 * (t2 - t0), "gpu_span_ms": (end - start) / 1e3,
               "busy_ms": busy / 1e3, "kernel_sum_ms": tot / 1e3, "activities": len(kern),
               "kernels": [[k, n, us] for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])],
               "timeline": [[(s_ - start) / 1e3, (e_ - s_) / 1e3, nm[:60]] for s_, e_, nm in kern]},
              open(a.json, "w"))
