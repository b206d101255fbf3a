"""Test-side trace generators (no reference needed, so they run on the GPU box):
an adversarial small-trace generator in the spirit of the reference's
conftest.random_trace (overlaps, equal starts, self transfers, unmatched
deletes, host-slot kernels, tiny hash / address pools), and a columnar
large-trace generator."""
import random

import numpy as np

from paper_2601_12713_b200 import types as T
from paper_2601_12713_b200.columns import columns_from_arrays


def nasty_trace(seed, max_events=300, max_devices=5):
    rng = random.Random(seed * 7919 + 13)
    ndev = rng.randint(2, max_devices)
    host = rng.randrange(ndev)
    n = rng.randint(0, max_events)
    hashes = [rng.randint(1, 2**64 - 1) for _ in range(rng.randint(1, 5))] + [2**64 - 1]
    addrs = [0x1000 * i for i in range(1, rng.randint(2, 6))]
    daddrs = [0xD000 + 0x100 * i for i in range(1, rng.randint(2, 6))]
    locs = [(0, None, None), (0x400100, None, None), (0x400200, "a.c", 3), (0x400300, "a.c", 3), (7, "b.c", 9)]
    raw, t = [], 0
    for _ in range(n):
        t += rng.choice([0, 0, 1, 5, 20, 60])
        dur = rng.randint(0, 80)
        r = rng.random()
        lc = rng.choice(locs)
        if r < 0.45:
            nb = rng.choice([0, 8, 64, 4096, 2**40])
            h = rng.choice(hashes) if nb else rng.choice([0, rng.choice(hashes)])
            raw.append(("transfer", t, t + dur, rng.randrange(ndev), rng.randrange(ndev), rng.choice(addrs),
                        rng.choice(daddrs), nb, h, lc))
        elif r < 0.63:
            raw.append(("alloc", t, t + dur, host, rng.randrange(ndev), rng.choice(addrs), rng.choice(daddrs),
                        rng.choice([8, 64, 256]), 0, lc))
        elif r < 0.82:
            raw.append(("delete", t, t + dur, host, rng.randrange(ndev), 0, rng.choice(daddrs), 0, 0, lc))
        else:
            d = rng.randrange(ndev)
            raw.append(("kernel", t, t + dur, d, d, 0, 0, 0, 0, lc))
    evs = [T.TraceEvent(seq=3 * i + 1, kind=T.EventKind(k), start_ns=a, end_ns=b, src_device=s, dst_device=d,
                        src_addr=sa, dst_addr=da, bytes=nb, hash=h, loc=T.CodeLocation(*lc))
           for i, (k, a, b, s, d, sa, da, nb, h, lc) in enumerate(raw)]
    wall = None if rng.random() < 0.4 else (max((e.end_ns for e in evs), default=0) + rng.choice([0, 5]))
    return T.Trace(version=1, num_devices_total=ndev, host_device=host, wall_time_ns=wall, events=evs)


def cycle_trace_columns(n_events, n_targets=8, seed=2, dup_frac=0.25, n_host_addrs=4096, payload=40000):
    """C2-shaped columnar trace: [ALLOC, H2D, KERNEL, D2H, DELETE] cycles rotating over the
    target devices (device 0 = host), H2D content repeated with probability dup_frac."""
    rng = np.random.default_rng(seed)
    ncyc = n_events // 5
    n = ncyc * 5
    cyc = np.arange(ncyc)
    dev = (cyc % n_targets + 1).astype(np.int32)
    state = np.tile(np.arange(5), ncyc)
    kind = np.array([1, 0, 3, 0, 2], dtype=np.uint8)[state]
    dur = np.array([300, 2 * payload, 10000, 2 * payload, 300], dtype=np.uint64)[state]
    start = np.zeros(n, dtype=np.uint64)
    start[1:] = np.cumsum(dur)[:-1]
    end = start + dur
    d = np.repeat(dev, 5)
    src = np.where((state == 3) | (state == 2), d, 0).astype(np.int32)
    dst = np.where((state == 3), 0, d).astype(np.int32)
    haddr = (0x7F0000000000 + (rng.integers(0, n_host_addrs, ncyc) * 0x100000)).astype(np.uint64)
    daddr = (0xD00000000000 + dev.astype(np.uint64) * 0x1000000).astype(np.uint64)
    h = np.repeat(haddr, 5)
    dv = np.repeat(daddr, 5)
    src_addr = np.where(state == 0, h, np.where(state == 1, h, np.where(state == 3, dv, 0))).astype(np.uint64)
    dst_addr = np.where(state == 3, h, np.where(state == 2, 0, dv)).astype(np.uint64)
    nbytes = np.where((state <= 1) | (state == 3), payload, 0).astype(np.uint64)
    content = np.arange(ncyc, dtype=np.uint64) + 1
    dup = rng.random(ncyc) < dup_frac
    dup[0] = False
    idx = np.nonzero(dup)[0]
    content[idx] = content[(rng.random(idx.size) * idx).astype(np.int64)]
    hh = (content * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    back = (np.arange(ncyc, dtype=np.uint64) + np.uint64(1 << 40)) * np.uint64(0xBF58476D1CE4E5B9) | np.uint64(1)
    hashv = np.zeros(n, dtype=np.uint64)
    hashv[state == 1] = hh
    unmodified = rng.random(ncyc) < 0.3  # kernel left the array unchanged: D2H returns the H2D content
    hashv[state == 3] = np.where(unmodified, hh, back)
    seq = np.arange(n, dtype=np.uint64)
    return columns_from_arrays(n_targets + 1, 0, seq, start, end, src, dst, kind, src_addr, dst_addr, nbytes, hashv,
                               wall_time_ns=int(end[-1]) if n else 0)
