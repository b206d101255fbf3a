import sys, time
sys.path.insert(0, '.')
from tests._gen import cycle_trace_columns
from paper_2601_12713_b200 import analyze_columns, savings_columns
c = cycle_trace_columns(1_000_000, seed=2)
for i in range(4):
    t = time.perf_counter(); cf = analyze_columns(c); t1 = time.perf_counter(); sv = savings_columns(c, cf); t2 = time.perf_counter()
    print(f"analyze {1e3*(t1-t):.2f} ms  savings {1e3*(t2-t1):.2f} ms", cf.counts())
