"""Test-only shard analyzer built on the CPU oracle (same interface as
paper_2601_12713_b200.sharded.engine_analyzer), so the multi-rank partition /
exchange / merge logic can be checked on CPU (gloo) without a GPU."""
import numpy as np

from oracle import analysis_ref as R
from paper_2601_12713_b200.analysis import (FLAG_SKIP_ALLOC, FLAG_SKIP_DDRT, FLAG_VALIDATE_ONLY, ColumnarFindings,
                                            EngineInvalid)

SYN = 0xFFFFFFFF


def oracle_analyzer(cols, flags=0, synthetic_end_ns=None, strict=False):
    if flags & FLAG_VALIDATE_ONLY:
        v = R.validate_cols(cols)
        if v:
            seq_to_i = {int(q): i for i, q in enumerate(cols.seq)}
            bad = sorted({seq_to_i[s] for _, _, s in v if s is not None})
            raise EngineInvalid(np.array(bad, np.uint32), np.ones(len(bad), np.uint32))
        return None
    rf = R.analyze_cols(cols, strict=strict, synth_end=synthetic_end_ns)
    return to_columnar(rf, cols.n, skip_ddrt=bool(flags & FLAG_SKIP_DDRT), skip_alloc=bool(flags & FLAG_SKIP_ALLOC))


def to_columnar(rf, n, skip_ddrt=False, skip_alloc=False):
    u32 = lambda a: np.array(a, dtype=np.uint32)  # noqa: E731

    def groups(gs, pick):
        off, mem = [0], []
        for g in gs:
            mem.extend(pick(g))
            off.append(len(mem))
        return np.array(off, np.uint64), mem
    dd_off, dd_mem = groups([] if skip_ddrt else rf.dd, lambda g: g[2])
    rt_off, trips = groups([] if skip_ddrt else rf.rt, lambda g: g[3])
    pairs = [] if skip_alloc else rf.pairs
    ra_off, ra_mem = groups([] if skip_alloc else rf.ra, lambda g: g[3])
    return ColumnarFindings(
        n_events=n, dd_offsets=dd_off, dd_members=u32(dd_mem), rt_offsets=rt_off,
        rt_tx=u32([t for t, _ in trips]), rt_rx=u32([r for _, r in trips]),
        pair_alloc=u32([a for a, _ in pairs]), pair_delete=u32([SYN if d < 0 else d for _, d in pairs]),
        synthetic_end_ns=rf.synthetic_end, warn_index=u32([] if skip_alloc else rf.warnings),
        ra_offsets=ra_off, ra_pairs=u32(ra_mem), ua_pairs=u32([] if skip_alloc else rf.ua),
        ut_events=u32([] if skip_alloc else rf.ut))
