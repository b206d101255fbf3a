"""Times the analysis pipeline on synthetic configs (used under ncu for launch lists).
Prints every iteration, then the median of the second half (steady state)."""
import argparse
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2601_12713_b200 import analyze_columns, savings_columns  # noqa: E402
from paper_2601_12713_b200.analysis import DeviceColumns  # noqa: E402
from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--device", action="store_true")
a = ap.parse_args()
gen = {"c2": lambda: c2_trace(a.n), "c3": lambda: c3_trace(max(1, a.n // 3)), "c4": lambda: c4_trace(a.n)}[a.config]
c = gen()
cols = DeviceColumns(c) if a.device else c
an, sv_t = [], []
for i in range(a.iters):
    t = time.perf_counter()
    cf = analyze_columns(cols, with_savings=True)
    t1 = time.perf_counter()
    sv = savings_columns(cols, cf)
    t2 = time.perf_counter()
    an.append(t1 - t)
    sv_t.append(t2 - t1)
    print(f"{a.config} n={c.n} analyze {1e3*(t1-t):.2f} ms  savings {1e3*(t2-t1):.2f} ms  "
          f"{c.n/(t2-t)/1e6:.1f} M ev/s", cf.counts())
h = a.iters // 2
ma, ms = statistics.median(an[h:]), statistics.median(sv_t[h:])
print(f"MEDIAN {a.config} n={c.n} analyze {1e3*ma:.3f} ms  savings {1e3*ms:.3f} ms  {c.n/(ma+ms)/1e6:.1f} M ev/s")
