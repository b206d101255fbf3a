"""Per-step times of analyze_many (the e2e headline loop) -- which steps are slow, and when."""
import gc, sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200.analysis import analyze_columns, analyze_many, pinned_columns, savings_columns
from paper_2601_12713_b200.synth import c2_trace
cols = pinned_columns(c2_trace(1_000_000))
for _ in range(3):
    savings_columns(cols, analyze_columns(cols, with_savings=True))
for _ in analyze_many([cols] * 3):
    pass
gc.collect(); gc.disable()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); marks = []
    for cf, _ in analyze_many([cols] * 40):
        marks.append(time.perf_counter())
    st = [1e3 * (b - a) for a, b in zip([t0] + marks[:-1], marks)]
    slow = [(i, round(x, 2)) for i, x in enumerate(st) if x > 3]
    print(f"rep {rep}: total {1e3*(marks[-1]-t0):.1f} ms, median {sorted(st)[20]:.3f}, slow steps {slow}", flush=True)
