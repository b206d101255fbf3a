# the device-resident sharded pipeline (G ranks as threads sharing the GPU) vs the single-GPU engine
timeout 1500 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
from oracle import analysis_ref as R
from paper_2601_12713_b200 import analyze_columns, sharded
from paper_2601_12713_b200.columns import to_columns
from tests._gen import nasty_trace
from tests._cases import canon_columnar
t = time.time(); bad = 0; done = 0
for seed in range(30000, 30600):
    cols = to_columns(nasty_trace(seed, max_events=2000))
    if R.validate_cols(cols) or cols.n == 0:
        continue
    g = 2 + seed % 3
    for strict in (False, True):
        got = sharded.run_local_device(cols, g, strict=strict)
        want = analyze_columns(cols, strict=strict)
        if canon_columnar(got, cols) != canon_columnar(want, cols) or got.warn_index.tolist() != want.warn_index.tolist():
            bad += 1
            print("SHARD MISMATCH", seed, g, strict, flush=True)
    done += 1
print(f"sharded sweep: {done} valid traces x 2 modes, G=2..4, {bad} mismatches, {time.time()-t:.0f} s")
PY
