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


def cycle_trace_columns(n_events, seed=2, **kw):
    from paper_2601_12713_b200.synth import c2_trace
    return c2_trace(n_events, seed=seed, **kw)
