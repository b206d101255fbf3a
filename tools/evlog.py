"""Host-vs-GPU timeline of one warm analyze call (B2L_TRACE=ev marks, no synchronisation):
  B2L_TRACE=ev python tools/evlog.py --config c2 --n 1000000"""
import argparse
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2601_12713_b200 import analyze_columns  # noqa: E402
from paper_2601_12713_b200.analysis import DeviceColumns  # noqa: E402
from paper_2601_12713_b200.synth import c2_trace, c4_trace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--iters", type=int, default=6)
a = ap.parse_args()
assert os.environ.get("B2L_TRACE") == "ev"
from paper_2601_12713_b200.synth import c3_trace  # noqa: E402
c = {"c2": c2_trace, "c3": c3_trace, "c4": c4_trace}[a.config](a.n)
cols = DeviceColumns(c)
for i in range(a.iters):
    if i == a.iters - 1:
        sys.stderr.write("=== last call\n")
        sys.stderr.flush()
    analyze_columns(cols, with_savings=True)
torch.cuda.synchronize()
