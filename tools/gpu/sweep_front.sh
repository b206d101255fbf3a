# single-pass front sweep: multi-tile nasty traces (up to 30k events = 8 front tiles, so the tiles'
# look-back carries counts and start ranks) vs the oracle in both RT modes, and the same traces
# with injected violations (bad event set vs the oracle's validate)
timeout -k 10 1500 python - <<'PY'
import sys, time
import numpy as np
sys.path.insert(0, ".")
from oracle import analysis_ref as R
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.analysis import EngineInvalid
from paper_2601_12713_b200.columns import to_columns
from tests._gen import nasty_trace
from tests._cases import canon_columnar, canon_oracle
t = time.time(); bad = 0; done = 0; inv = 0
for seed in range(30000, 30120):
    tr = nasty_trace(seed, max_events=30000)
    cols = to_columns(tr)
    if R.validate_cols(cols):
        continue
    for strict in (False, True):
        cf = analyze_columns(cols, strict=strict)
        rf = R.analyze_cols(cols, strict=strict)
        if canon_columnar(cf, cols) != canon_oracle(rf, cols) or cf.warn_index.tolist() != rf.warnings:
            bad += 1
            print("MISMATCH", seed, strict, cols.n, flush=True)
    sv = savings_columns(cols, cf)
    est = R.estimate_cols(cols, rf, tr.wall_time_ns)
    if sv.per_category_ns != est["per_category_ns"] or sorted(sv.union_index.tolist()) != est["eliminable"]:
        bad += 1
        print("SAVINGS MISMATCH", seed, flush=True)
    done += 1
    # injected violations: end < start on a few events, a transfer without a hash
    rng = np.random.default_rng(seed)
    c2 = to_columns(tr)
    k = rng.choice(cols.n, size=min(5, cols.n), replace=False)
    for i in k:
        if c2.start_ns[i] > 0:
            c2.end_ns[i] = c2.start_ns[i] - 1
    tx = np.nonzero((c2.kind == 0) & (c2.bytes > 0))[0]
    if tx.size:
        c2.hash[tx[rng.integers(0, tx.size)]] = 0
    want = {int(x[2]) for x in R.validate_cols(c2) if x[2] is not None}
    try:
        analyze_columns(c2)
        got = set()
    except EngineInvalid as e:
        got = {int(c2.seq[j]) for j in np.asarray(e.bad_index)}
    if got != want:
        bad += 1
        print("VALIDATION MISMATCH", seed, sorted(want)[:5], sorted(got)[:5], flush=True)
    inv += 1
print(f"front sweep: {done} valid multi-tile traces x 2 modes + savings, {inv} corrupted traces, {bad} mismatches, {time.time()-t:.0f} s")
PY
