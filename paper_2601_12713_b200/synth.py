"""Synthetic workloads of the benchmark configurations, generated
directly as columns (no Python objects) so 10^6-10^8-event traces are cheap.

  c2_trace   "1M-event trace with 25% duplicate transfers": [ALLOC, H2D, KERNEL, D2H,
             DELETE] cycles over 8 target devices; 25% of H2D payloads repeat an earlier
             one (duplicates); 30% of kernels leave the array unchanged, so the D2H
             returns the H2D content (round trips); host variables from a 4,096 pool
             (repeated allocations).
  c3_trace   "stencil time loop": 1 target device, arrays A and B; per iteration
             D2H(A, new content), KERNEL, H2D(A, same bytes) -> a round trip per step.
  c4_trace   "allocation-heavy": 4 target devices, 4,096 host variables, allocation
             sizes log-uniform in [4 B, 64 MiB], 20% alloc/delete pairs in kernel-free
             gaps (unused allocations), 10% of H2D overwritten before a kernel (unused
             transfers), hashes from a 65,536-entry palette.
Timing follows the reference generator's defaults (synth.py:52-54: 2 ns/byte
transfers, 400 ns allocs, 10 us kernels), strictly serial (no overlaps).
"""
from __future__ import annotations

import numpy as np

from .columns import columns_from_arrays

TRANSFER, ALLOC, DELETE, KERNEL = 0, 1, 2, 3
HOST = 0
_M = np.uint64(0x9E3779B97F4A7C15)


def _mix(x):
    """splitmix64 finaliser on a uint64 array (content -> 64-bit hash stand-in, never 0)."""
    x = np.asarray(x, dtype=np.uint64) + _M
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    x = x ^ (x >> np.uint64(31))
    return np.where(x == 0, np.uint64(1), x)


def _serial_times(dur):
    start = np.zeros(dur.size, dtype=np.uint64)
    if dur.size:
        np.cumsum(dur[:-1], out=start[1:])
    return start, start + dur


def c2_trace(n_events=1_000_000, n_targets=8, seed=2, dup_frac=0.25, unmodified_frac=0.3, n_host_vars=4096,
             payload=40_000):
    rng = np.random.default_rng(seed)
    ncyc = n_events // 5
    n = ncyc * 5
    state = np.tile(np.arange(5, dtype=np.int64), ncyc)
    dev = (np.arange(ncyc) % n_targets + 1).astype(np.int32)
    d = np.repeat(dev, 5)
    kind = np.array([ALLOC, TRANSFER, KERNEL, TRANSFER, DELETE], dtype=np.uint8)[state]
    dur = np.array([400, 2 * payload, 10_000, 2 * payload, 400], dtype=np.uint64)[state]
    start, end = _serial_times(dur)
    src = np.where((state == 2) | (state == 3), d, HOST).astype(np.int32)
    dst = np.where(state == 3, HOST, d).astype(np.int32)
    hvar = rng.integers(0, n_host_vars, ncyc)
    haddr = np.repeat((0x7F0000000000 + hvar * 0x100000).astype(np.uint64), 5)
    daddr = np.repeat((0xD00000000000 + dev.astype(np.uint64) * np.uint64(0x1000000)), 5)
    zero = np.uint64(0)
    src_addr = np.select([state <= 1, state == 3], [haddr, daddr], zero).astype(np.uint64)
    dst_addr = np.select([state == 3, state == 2], [haddr, zero], daddr).astype(np.uint64)
    nbytes = np.where(state == 0, np.uint64(payload), np.where((state == 1) | (state == 3), np.uint64(payload),
                                                               zero)).astype(np.uint64)
    content = np.arange(ncyc, dtype=np.uint64) + np.uint64(1)
    dup = rng.random(ncyc) < dup_frac
    if ncyc:
        dup[0] = False
    idx = np.nonzero(dup)[0]
    content[idx] = content[(rng.random(idx.size) * idx).astype(np.int64)]
    h_in = _mix(content)
    h_back = np.where(rng.random(ncyc) < unmodified_frac, h_in, _mix(content + np.uint64(1 << 62)))
    hashv = np.zeros(n, dtype=np.uint64)
    hashv[state == 1] = h_in
    hashv[state == 3] = h_back
    seq = np.arange(n, dtype=np.uint64)
    return columns_from_arrays(n_targets + 1, HOST, seq, start, end, src, dst, kind, src_addr, dst_addr, nbytes,
                               hashv, wall_time_ns=int(end[-1]) if n else 0)


def c3_trace(iterations=10_000, array_bytes=268_435_456, seed=3):
    """2 allocs, iterations x [D2H A (new content), KERNEL, H2D A (same bytes)], 2 deletes."""
    it = iterations
    n = 4 + 3 * it
    kind = np.empty(n, dtype=np.uint8)
    kind[:2] = ALLOC
    kind[2:2 + 3 * it] = np.tile(np.array([TRANSFER, KERNEL, TRANSFER], dtype=np.uint8), it)
    kind[-2:] = DELETE
    step = np.tile(np.arange(3), it)
    dur = np.empty(n, dtype=np.uint64)
    dur[:2] = 400
    dur[-2:] = 400
    dur[2:2 + 3 * it] = np.array([2 * array_bytes, 10_000, 2 * array_bytes], dtype=np.uint64)[step]
    start, end = _serial_times(dur)
    A_h, B_h, A_d, B_d = 0x7F0000000000, 0x7F0010000000, 0xD00000000000, 0xD00010000000
    src = np.zeros(n, dtype=np.int32)
    dst = np.ones(n, dtype=np.int32)
    body = slice(2, 2 + 3 * it)
    src[body] = np.where(step == 2, 0, 1)
    dst[body] = np.where(step == 0, 0, 1)
    src_addr = np.zeros(n, dtype=np.uint64)
    dst_addr = np.zeros(n, dtype=np.uint64)
    src_addr[0], dst_addr[0], src_addr[1], dst_addr[1] = A_h, A_d, B_h, B_d
    src_addr[body] = np.select([step == 0, step == 2], [np.uint64(A_d), np.uint64(A_h)], np.uint64(0))
    dst_addr[body] = np.select([step == 0, step == 2], [np.uint64(A_h), np.uint64(A_d)], np.uint64(0))
    dst_addr[-2], dst_addr[-1] = A_d, B_d
    dst[-2:] = 1
    src[-2:] = 0
    src[:2] = 0
    nbytes = np.zeros(n, dtype=np.uint64)
    nbytes[:2] = array_bytes
    nbytes[body] = np.where(step == 1, np.uint64(0), np.uint64(array_bytes))
    content = _mix(np.arange(it, dtype=np.uint64) + np.uint64(seed << 40))
    hashv = np.zeros(n, dtype=np.uint64)
    hashv[body] = np.where(step == 1, np.uint64(0), np.repeat(content, 3))
    seq = np.arange(n, dtype=np.uint64)
    return columns_from_arrays(2, HOST, seq, start, end, src, dst, kind, src_addr, dst_addr, nbytes, hashv,
                               wall_time_ns=int(end[-1]))


def c4_trace(n_events=10_000_000, n_targets=4, seed=4, n_host_vars=4096, palette=65_536, ua_frac=0.2,
             ut_frac=0.1):
    """Cycle mix: normal [A, H2D, K, D2H, D], unused-alloc [A, D] (kernel-free gap), and
    overwritten [A, H2D, H2D', K, D2H, D] (first H2D unused)."""
    rng = np.random.default_rng(seed)
    # choose cycle types until the event budget is met
    est = n_events // 4 + 16
    kinds = rng.random(est)
    ctype = np.where(kinds < ua_frac, 1, np.where(kinds < ua_frac + ut_frac, 2, 0))
    clen = np.array([5, 2, 6])[ctype]
    cum = np.cumsum(clen)
    ncyc = int(np.searchsorted(cum, n_events, side="right"))
    ctype, clen = ctype[:ncyc], clen[:ncyc]
    n = int(clen.sum())
    cyc_of = np.repeat(np.arange(ncyc), clen)
    first = np.zeros(ncyc, dtype=np.int64)
    if ncyc:
        first[1:] = np.cumsum(clen)[:-1]
    pos = np.arange(n) - first[cyc_of]
    ct = ctype[cyc_of]
    # role per event: 0 alloc, 1 h2d, 2 kernel, 3 d2h, 4 delete, 5 overwriting h2d
    role_tab = {0: [0, 1, 2, 3, 4], 1: [0, 4], 2: [0, 1, 5, 2, 3, 4]}
    role = np.empty(n, dtype=np.int64)
    for t, r in role_tab.items():
        m = ct == t
        role[m] = np.array(r)[pos[m]]
    dev = (rng.integers(0, n_targets, ncyc) + 1).astype(np.int32)
    d = dev[cyc_of]
    var_size = np.exp(rng.uniform(np.log(4), np.log(64 << 20), n_host_vars)).astype(np.uint64)
    hvar = rng.integers(0, n_host_vars, ncyc)
    sz = var_size[hvar][cyc_of]  # a host variable always maps the same size (repeated allocations)
    kind = np.array([ALLOC, TRANSFER, KERNEL, TRANSFER, DELETE, TRANSFER], dtype=np.uint8)[role]
    xfer = (role == 1) | (role == 3) | (role == 5)
    dur = np.where(role == 2, np.uint64(10_000), np.where(xfer, np.uint64(2) * sz, np.uint64(400))).astype(np.uint64)
    start, end = _serial_times(dur)
    src = np.where((role == 2) | (role == 3), d, HOST).astype(np.int32)
    dst = np.where(role == 3, HOST, d).astype(np.int32)
    haddr = (0x7F0000000000 + hvar.astype(np.uint64) * np.uint64(0x100000))[cyc_of]
    daddr = (np.uint64(0xD00000000000) + (np.arange(ncyc, dtype=np.uint64) % np.uint64(1 << 16)) *
             np.uint64(0x10000))[cyc_of]
    zero = np.uint64(0)
    src_addr = np.select([(role <= 1) | (role == 5), role == 3], [haddr, daddr], zero).astype(np.uint64)
    dst_addr = np.select([role == 3, role == 2], [haddr, zero], daddr).astype(np.uint64)
    nbytes = np.where((role == 0) | xfer, sz, zero).astype(np.uint64)
    pal = _mix(np.arange(palette, dtype=np.uint64) + np.uint64(seed << 48))
    hashv = np.where(xfer, pal[rng.integers(0, palette, n)], zero).astype(np.uint64)
    seq = np.arange(n, dtype=np.uint64)
    return columns_from_arrays(n_targets + 1, HOST, seq, start, end, src, dst, kind, src_addr, dst_addr, nbytes, hashv,
                               wall_time_ns=int(end[-1]) if n else 0)


def with_locations(cols, n_locs=24, seed=0):
    """The same trace with events spread over ``n_locs`` code locations (codeptrs, some with
    file/line, several sharing one (file, line) -- report.py:67-70 buckets them together), so
    the attribution rows of estimate/attribute are non-trivial at config scale."""
    import dataclasses

    from .columns import loc_key
    rng = np.random.default_rng(seed + 7)
    locs = []
    for j in range(n_locs):
        f = None if j % 3 == 0 else f"kern{j % 5}.c"
        locs.append((0x400000 + 0x40 * j, f, (10 + j % 4) if f else None))
    keys, bucket_of, ids = [], [], {}
    for cp, f, ln in locs:
        k = loc_key(cp, f, ln)
        if k not in ids:
            ids[k] = len(keys)
            keys.append(k)
        bucket_of.append(ids[k])
    loc = rng.integers(0, n_locs, cols.n).astype(np.uint32)
    return dataclasses.replace(cols, loc=loc, loc_flags=np.zeros(n_locs, np.uint8),
                               loc_bucket=np.array(bucket_of, np.uint32), n_buckets=len(keys), bucket_keys=keys,
                               locs=locs)
