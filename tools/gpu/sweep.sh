# broad engine-vs-oracle sweep (beyond the test suite's 1,500 seeds): small and multi-tile nasty traces
timeout 1500 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
from oracle import analysis_ref as R
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.columns import to_columns
from tests._gen import nasty_trace
from tests._cases import canon_columnar, canon_oracle
t = time.time(); bad = 0; done = 0
for lo, hi, mx in ((1500, 9500, 300), (20000, 21200, 4000)):
    for seed in range(lo, hi):
        tr = nasty_trace(seed, max_events=mx)
        cols = to_columns(tr)
        if R.validate_cols(cols):
            continue
        for strict in (False, True):
            cf = analyze_columns(cols, strict=strict)
            rf = R.analyze_cols(cols, strict=strict)
            if canon_columnar(cf, cols) != canon_oracle(rf, cols) or cf.warn_index.tolist() != rf.warnings:
                bad += 1
                print("MISMATCH", seed, strict, flush=True)
        sv = savings_columns(cols, cf)
        est = R.estimate_cols(cols, rf, tr.wall_time_ns)
        if sv.per_category_ns != est["per_category_ns"] or sorted(sv.union_index.tolist()) != est["eliminable"]:
            bad += 1
            print("SAVINGS MISMATCH", seed, flush=True)
        done += 1
print(f"sweep: {done} valid traces x 2 modes, {bad} mismatches, {time.time()-t:.0f} s")
PY
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
