#!/usr/bin/env python3
"""Per-config measurements beyond bench.py's headline line,
one JSON object per line, for profiles/.  Single GPU.

  C1  4,000 buffers, log-uniform 1 KiB - 1 MiB (0.6 GB), hashed (K1, longest first);
      10k-event trace analysed
  C3  256 MiB stencil arrays hashed one at a time with the whole GPU (K2), K buffers;
      30k-event stencil trace analysed
  C4  10M-event allocation-heavy trace analysed
  C5s 100M-event C2-style trace analysed on ONE GPU (the single-GPU slice of C5)
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_12713_b200 import _lib, analyze_columns, hash_device, savings_columns  # noqa: E402
from paper_2601_12713_b200.analysis import DeviceColumns  # noqa: E402
from paper_2601_12713_b200.hashing import hash_large  # noqa: E402
from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace  # noqa: E402


def fill(slab, offs, lens, cids, seed):
    s = torch.cuda.current_stream()
    _lib.check(_lib.lib().b2l_fill_payloads(slab.data_ptr(), offs.data_ptr(), lens.data_ptr(), cids.data_ptr(),
                                            offs.numel(), seed, s.cuda_stream))


def time_device(fn, iters):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters


def time_wall(fn, iters):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / iters


def analysis_line(name, cols, iters=5):
    dc = DeviceColumns(cols)
    holder = {}

    def step():
        holder["cf"] = analyze_columns(dc)
        savings_columns(dc, holder["cf"])
    for _ in range(3):  # same object lifetimes as the timed loop: the pinned result slabs are warm
        step()
    dt = time_wall(step, iters)
    return {"config": name, "metric": "M trace events/s analysed", "events": cols.n,
            "value": round(cols.n / dt / 1e6, 2), "ms_per_step": round(dt * 1e3, 3),
            "counts": holder["cf"].counts()}


def c1(args):
    dev = torch.device("cuda")
    rng = np.random.default_rng(1)
    n = 4000
    lens = np.exp(rng.uniform(np.log(1024), np.log(1 << 20), n)).astype(np.int64)
    offs = np.zeros(n, np.int64)
    offs[1:] = np.cumsum((lens + 255) // 256 * 256)[:-1]
    total = int(offs[-1] + lens[-1])
    slab = torch.empty(total, dtype=torch.uint8, device=dev)
    o_d, l_d = torch.from_numpy(offs).to(dev), torch.from_numpy(lens).to(dev)
    fill(slab, o_d, l_d, torch.arange(n, device=dev), 1)
    ptrs = o_d + slab.data_ptr()
    order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    for _ in range(3):
        hash_device(ptrs, l_d, out, order=order)
    dt = time_device(lambda: hash_device(ptrs, l_d, out, order=order), 20)
    nbytes = int(lens.sum())
    chain_floor = int(lens.max()) / 8 * 10 / 1.965e9  # ~10 cycles per word on the longest serial chain
    print(json.dumps({"config": "C1", "metric": "GB/s hashed", "buffers": n, "bytes": nbytes,
                      "value": round(nbytes / dt / 1e9, 2), "ms_per_step": round(dt * 1e3, 4),
                      "note": f"bound by the longest buffer's serial chain (~{chain_floor * 1e3:.2f} ms for "
                              f"{int(lens.max())} B); HBM floor {nbytes / 6.5e12 * 1e3:.3f} ms"}), flush=True)
    print(json.dumps(analysis_line("C1", c2_trace(10_000, seed=1))), flush=True)


def c3(args):
    dev = torch.device("cuda")
    size = 256 << 20
    k = args.c3_buffers
    slab = torch.empty(size * k, dtype=torch.uint8, device=dev)
    offs = torch.arange(k, dtype=torch.int64, device=dev) * size
    fill(slab, offs, torch.full((k,), size, dtype=torch.int64, device=dev), torch.arange(k, device=dev), 3)
    out = torch.empty(k, dtype=torch.int64, device=dev)

    def step():
        for i in range(k):
            hash_large(slab.data_ptr() + i * size, size, out.data_ptr() + 8 * i)
    step()
    dt = time_device(step, 3)
    print(json.dumps({"config": "C3", "metric": "GB/s hashed", "buffers": k, "buffer_bytes": size,
                      "value": round(k * size / dt / 1e9, 2), "ms_per_buffer": round(dt / k * 1e3, 3),
                      "kernel": "k_hash_planes (K2, whole GPU per buffer)",
                      "serial_chain_reference": "one 256 MiB buffer on a single chain: ~0.17 s (~1.5 GB/s)"}),
          flush=True)
    print(json.dumps(analysis_line("C3", c3_trace(10_000))), flush=True)


def c4(args):
    print(json.dumps(analysis_line("C4", c4_trace(10_000_000), iters=3)), flush=True)


def c5s(args):
    print(json.dumps(analysis_line("C5-single-GPU-slice", c2_trace(args.c5_events, seed=5), iters=2)), flush=True)


def ingest_cfg(args):
    """NDJSON -> validated columns (native parser + GPU sort/validate) on the C2 1M-event trace."""
    from paper_2601_12713_b200.ingest import parse_trace_columns
    c = c2_trace(1_000_000, seed=2)
    kinds = ["transfer", "alloc", "delete", "kernel"]
    L = lambda a: a.tolist()  # noqa: E731
    lines = ['{"dmlens":1,"num_devices":%d,"host_device":%d}' % (c.num_devices_total, c.host_device)]
    for q, k, a, b, s_, d, sa, da, nb, h in zip(L(c.seq), L(c.kind), L(c.start_ns), L(c.end_ns), L(c.src_device),
                                                 L(c.dst_device), L(c.src_addr), L(c.dst_addr), L(c.bytes),
                                                 L(c.hash)):
        lines.append('{"seq":%d,"kind":"%s","t0":%d,"t1":%d,"src_dev":%d,"dst_dev":%d,"src_addr":%d,'
                     '"dst_addr":%d,"bytes":%d,"hash":%d,"codeptr":0}' % (q, kinds[k], a, b, s_, d, sa, da, nb, h))
    raw = ("\n".join(lines) + "\n").encode()
    parse_trace_columns(raw)
    t = time.perf_counter()
    for _ in range(3):
        cols = parse_trace_columns(raw)
    dt = (time.perf_counter() - t) / 3
    print(json.dumps({"config": "ingest-C2", "metric": "M events/s parsed (NDJSON -> sorted, validated columns)",
                      "events": cols.n, "bytes": len(raw), "value": round(cols.n / dt / 1e6, 2),
                      "ms_per_step": round(dt * 1e3, 1), "threads": min(32, os.cpu_count() or 1)}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c4,c5s,ingest")
    ap.add_argument("--c3-buffers", type=int, default=8)
    ap.add_argument("--c5-events", type=int, default=100_000_000)
    a = ap.parse_args()
    for c in a.configs.split(","):
        globals()["ingest_cfg" if c == "ingest" else c](a)
