#!/usr/bin/env python3
"""Benchmark of the B200 hot path.

Metric (BASELINE.json): "GB/s of mapped bytes hashed; M trace events/s analysed".
Workload (one per GPU -> weak scaling):
  400,000 buffers x 40,000 B = 16.0 GB of payload per GPU, 25 % byte-identical
  duplicates (counter-based splitmix64 payloads generated on the device, not timed).
A step = one b2l_hash_batch launch over the whole batch (inputs resident in HBM,
16 GB >> 126 MB L2, so no flush is needed).  `e2e` = the same batch through the
host-buffer C-ABI call b2l_hash_host from pinned host memory (H2D copies and the
digest D2H inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun each rank hashes its own C2 batch; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import gc
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BUFS = 400_000
BUF_BYTES = 40_000
DUP_FRAC = 0.25
SEED = 2
METRIC = "GB/s of mapped bytes hashed; M trace events/s analysed"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-bufs", type=int, default=N_BUFS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the 10M-event analysis lines")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--n-events", type=int, default=N_EVENTS)
    ap.add_argument("--no-analysis", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("B2L_BENCH_BACKEND") == "gloo":  # path check with ranks sharing GPUs (not a measurement)
        import torch
        local %= max(1, torch.cuda.device_count())
    return rank, world, local


def content_ids(n, rank):
    import numpy as np
    rng = np.random.default_rng(SEED * 1000 + rank)
    cids = np.arange(n, dtype=np.int64) + rank * n
    dup = rng.random(n) < DUP_FRAC
    dup[0] = False
    # a duplicate repeats the content of an EARLIER buffer (byte copy)
    idx = np.nonzero(dup)[0]
    cids[idx] = cids[(rng.random(idx.size) * idx).astype(np.int64)]
    return cids


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of k_hash_seq from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "hash_ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch")
    return None


def analysis_traffic(n_events, peak=None):
    """DRAM bytes per analyze+savings step from the committed ncu capture of the same workload,
    and the top kernels' own DRAM rates (bytes each moved / its cold ncu duration)."""
    p = os.path.join(ROOT, "profiles", f"analysis_traffic_c2_{n_events}.json")
    if os.path.exists(p):
        d = json.load(open(p))
        top = []
        for k in d.get("kernels", [])[:6]:
            gbs = k["dram_bytes"] / (k["time_us"] * 1e-6) / 1e9 if k["time_us"] else 0.0
            l2 = k.get("l2_bytes", 0.0) / (k["time_us"] * 1e-6) / 1e9 if k["time_us"] else 0.0
            top.append({"kernel": k["kernel"].replace("void ", "")[:60], "launches": k["launches"],
                        "us": round(k["time_us"], 1), "dram_gbs": round(gbs, 1), "l2_gbs": round(l2, 1),
                        "dram_frac": round(gbs / peak, 3) if peak else None})
        return d.get("dram_bytes_per_step"), d.get("launches_per_step"), top
    return None, None, []


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import hash_ref  # checker + CPU baseline only
    from paper_2601_12713_b200 import _lib, hash_device
    from paper_2601_12713_b200.hashing import hash_host_arrays

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n = args.n_bufs
    total = n * BUF_BYTES
    cids = content_ids(n, rank)
    offs = torch.arange(n, dtype=torch.int64, device=dev) * BUF_BYTES
    lens = torch.full((n,), BUF_BYTES, dtype=torch.int64, device=dev)
    slab = torch.empty(total, dtype=torch.uint8, device=dev)
    cid_d = torch.from_numpy(cids).to(dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(_lib.lib().b2l_fill_payloads(slab.data_ptr(), offs.data_ptr(), lens.data_ptr(), cid_d.data_ptr(),
                                            n, SEED, stream.cuda_stream), "fill")
    ptrs = offs + slab.data_ptr()
    out = torch.empty(n, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        hash_device(ptrs, lens, out, stream=stream)
    torch.cuda.synchronize()

    # correctness spot check against the C oracle (64 buffers incl. duplicates)
    sample = np.unique(np.concatenate([np.arange(0, n, max(1, n // 48)), np.nonzero(cids != np.arange(n) + rank * n)[0][:16]]))
    host = {int(i): slab[int(i) * BUF_BYTES:(int(i) + 1) * BUF_BYTES].cpu().numpy() for i in sample}
    got = out.cpu().numpy().view(np.uint64)
    verified = all(int(got[i]) == hash_ref.fold64_c(host[int(i)].tobytes()) for i in sample)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = args._clock
    if True:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for a, b in evs:
            a.record(stream)
            hash_device(ptrs, lens, out, stream=stream)
            b.record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    ms_per_step = elapsed_max / args.steps
    value = world * total * args.steps / (elapsed_max / 1e3) / 1e9

    # ---------------- e2e through the host-buffer C ABI (pinned host memory)
    e2e = None
    if not args.no_e2e:
        hslab = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        hslab.copy_(slab)
        hbase = hslab.data_ptr()
        hptrs = (np.arange(n, dtype=np.uint64) * np.uint64(BUF_BYTES)) + np.uint64(hbase)
        hlens = np.full(n, BUF_BYTES, dtype=np.uint64)
        hout = np.zeros(n, dtype=np.uint64)
        hash_host_arrays(hptrs, hlens, hout)  # warm-up (ring allocation)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            hash_host_arrays(hptrs, hlens, hout)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.barrier()
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_ok = bool(np.array_equal(hout, got))
        e2e = {"value": world * total * e2e_steps / float(dt.item()) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": total + 16 * n, "d2h_bytes_per_step": 8 * n,
               "api": "b2l_hash_host (pinned host buffers, double-buffered device ring)",
               "steps": e2e_steps, "digests_match_device_path": e2e_ok}
        del hslab

    # ---------------- CPU baseline: oracle C port, all host threads, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        hcopy = slab[: min(total, 4_000_000_000)].cpu().numpy()
        nb = hcopy.size // BUF_BYTES
        hp = np.arange(nb, dtype=np.uint64) * np.uint64(BUF_BYTES) + np.uint64(hcopy.ctypes.data)
        hl = np.full(nb, BUF_BYTES, dtype=np.uint64)
        done, t0 = 0, time.perf_counter()
        chunk = max(threads * 64, 1024)
        while time.perf_counter() - t0 < args.cpu_seconds and done < nb:
            k = min(chunk, nb - done)
            hash_ref.fold64_c_batch(hp[done:done + k], hl[done:done + k], threads=threads)
            done += k
        dt = time.perf_counter() - t0
        cpu = {"value": done * BUF_BYTES / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{done} of the {n} C2 buffers ({done * BUF_BYTES / 1e9:.2f} GB), oracle/hash_fold64.c "
                         f"with {threads} pthreads, {dt:.1f} s"}

    peak, peak_src = peaks()
    kern_ms = statistics.mean(launch_ms)
    achieved = total / (kern_ms / 1e3) / 1e9
    traffic = ncu_traffic() if n == N_BUFS else None  # the committed capture is of the default batch
    rec = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"C2: {n:,} x {BUF_BYTES:,} B buffers per GPU ({total / 1e9:.1f} GB), 25% "
                               "duplicates, hashed with the reference FNV-1a/fmix64 fold",
                   "n_buffers_per_gpu": n, "buffer_bytes": BUF_BYTES, "bytes_per_gpu": total,
                   "l2": f"inputs ({total / 1e9:.1f} GB) larger than the 126 MB L2, no flush",
                   "parallelism": f"shard{world}"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel": "k_hash_coop<2,512,2> (b2l_hash_batch default variant)", "algorithmic_bytes_per_launch": total},
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": args.steps, "verified": bool(verified),
        "impl": "ours",
    }
    return rec


# ----------------------------------------------------------------------------- analysis (C2 1M-event trace)
N_EVENTS = 1_000_000
EVENT_BYTES = 64  # algorithmic bytes per event: one read of the packed row


def run_analysis_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, pinned_columns, savings_columns
    from paper_2601_12713_b200.synth import c2_trace

    dev = torch.device("cuda", local)
    if world > 1:
        return run_analysis_sharded(args, rank, world, local)
    cols = c2_trace(args.n_events, seed=SEED + rank)
    dcols = DeviceColumns(cols, dev)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        cf = analyze_columns(dcols)
        savings_columns(dcols, cf)
    verified = None
    if rank == 0 and not args.no_cpu:
        from oracle import analysis_ref as R  # checker only
        t0 = time.perf_counter()
        rf = R.analyze_cols(cols)
        cpu_dt = time.perf_counter() - t0
        est = R.estimate_cols(cols, rf, cols.wall_time_ns)
        sv = savings_columns(dcols, cf)
        verified = bool(
            [len(rf.dd), len(rf.rt), len(rf.ra), len(rf.ua), len(rf.ut)] == list(cf.counts().values())
            and [i for g in rf.dd for i in g[2]] == cf.dd_members.tolist()
            and [t for g in rf.rt for t, _ in g[3]] == cf.rt_tx.tolist()
            and [r for g in rf.rt for _, r in g[3]] == cf.rt_rx.tolist()
            and [p for g in rf.ra for p in g[3]] == cf.ra_pairs.tolist()
            and sv.per_category_ns == est["per_category_ns"])
    else:
        cpu_dt = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cf = analyze_columns(dcols)
        savings_columns(dcols, cf)
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    step_s = float(dt.item()) / args.steps
    value = world * cols.n / step_s / 1e6
    # e2e: host columns in (page-locked host memory), host findings + sums out
    # (a 1M-event step is ~3 ms: 30 steps, with Python's cyclic GC paused, so one host hiccup
    # does not swing the number)
    e2e_steps = max(1, min(args.steps, 30))
    cols = pinned_columns(cols)
    for _ in range(3):  # warm-up with the timed loop's object lifetimes (previous findings alive)
        cfh = analyze_columns(cols)
        savings_columns(cols, cfh)
    gc.collect()
    gc.disable()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    marks = []
    for _ in range(e2e_steps):
        cfh = analyze_columns(cols)
        savings_columns(cols, cfh)
        marks.append(time.perf_counter())
    torch.cuda.synchronize()
    de = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    gc.enable()
    e2e_step_ms = sorted(1e3 * (b - a) for a, b in zip([t0] + marks[:-1], marks))
    if world > 1:
        dist.all_reduce(de, op=dist.ReduceOp.MAX)
    h2d = sum(getattr(cols, f).nbytes for f in DeviceColumns.FIELDS)
    d2h = sum(a.nbytes for a in (cfh.dd_offsets, cfh.dd_members, cfh.rt_offsets, cfh.rt_tx, cfh.rt_rx,
                                 cfh.pair_alloc, cfh.pair_delete, cfh.warn_index, cfh.ra_offsets, cfh.ra_pairs,
                                 cfh.ua_pairs, cfh.ut_events))
    peak, peak_src = peaks()
    achieved = cols.n * EVENT_BYTES / step_s / 1e9
    traffic, launches, top = analysis_traffic(cols.n, peak)
    out = {
        "metric": "M trace events/s analysed", "value": round(value, 3), "unit": "M events/s",
        "ms_per_step": round(step_s * 1e3, 3), "steps": args.steps,
        "config": {"workload": f"C2 trace: {cols.n} events ([ALLOC,H2D,KERNEL,D2H,DELETE] x 8 target devices, "
                               f"25% duplicate H2D content, 30% unmodified D2H), validate + 5 detectors + "
                               f"estimate/attribute sums, columns resident in HBM", "events_per_gpu": cols.n},
        "counts": cf.counts(),
        "timing": "host-synchronous C-ABI call (b2l_analyze + b2l_savings_compute), perf_counter bracketed by "
                  "cuda synchronize, max over ranks",
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 5), "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_step": cols.n * EVENT_BYTES,
                     "traffic_note": "ncu dram bytes summed over every kernel of one analyze+savings step "
                                     "(profiles/analysis_traffic_c2_<n>.json); the pipeline moves traffic/64 B "
                                     "per event across its sort/scan passes",
                     "traffic_gbs_over_step": round(traffic / step_s / 1e9, 1) if traffic else None,
                     "kernel_launches_per_step": launches,
                     "top_kernels_ncu": top},
        "e2e": {"value": round(world * cols.n * e2e_steps / float(de.item()) / 1e6, 3), "unit": "M events/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "step_ms_min_median_max": [round(e2e_step_ms[0], 3), round(e2e_step_ms[len(e2e_step_ms) // 2], 3),
                                           round(e2e_step_ms[-1], 3)],
                "api": "b2l_analyze + b2l_savings_compute on host numpy columns in page-locked memory"},
        "verified": verified,
    }
    if cpu_dt is not None:
        out["cpu_baseline"] = {"value": round(cols.n / cpu_dt / 1e6, 4), "unit": "M events/s", "cores": 1,
                               "kind": "port", "sample": f"the full {cols.n}-event C2 trace through "
                                                         f"oracle/analysis_ref.analyze_cols (1 thread)"}
    if not args.no_large:
        out["larger_traces"] = [_analysis_at(c2_trace, n, dev) for n in (10_000_000,)] + \
            [_analysis_at(_c4, 10_000_000, dev)]
    return out


def _c4(n, seed=4):
    from paper_2601_12713_b200.synth import c4_trace
    return c4_trace(n, seed=seed)


def _analysis_at(gen, n, dev, iters=8):
    """The same device-resident step on a larger trace (throughput rather than launch latency)."""
    import statistics

    import torch

    from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, savings_columns
    cols = gen(n, seed=SEED + 10)
    d = DeviceColumns(cols, dev)
    times = []
    for _ in range(iters):
        torch.cuda.synchronize()
        t = time.perf_counter()
        savings_columns(d, analyze_columns(d))
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    step = statistics.median(times[iters // 2:])
    name = "C4" if gen is _c4 else "C2"
    return {"workload": f"{name} trace, {cols.n} events, columns resident in HBM", "value": round(cols.n / step / 1e6, 1),
            "unit": "M events/s", "ms_per_step": round(step * 1e3, 3),
            "timing": f"median of the last {iters - iters // 2} of {iters} steps"}


def run_analysis_sharded(args, rank, world, local):
    """N>1: one global C2 trace of world x n_events events, seq-range sharded over the ranks,
    analysed with the key-range sharded pipeline (one NCCL all-to-all + final gather)."""
    import torch
    import torch.distributed as dist

    from paper_2601_12713_b200 import sharded
    from paper_2601_12713_b200.synth import c2_trace

    from paper_2601_12713_b200.analysis import DeviceColumns
    cols = c2_trace(args.n_events * world, seed=SEED)
    shard, base = sharded.split(cols, world)[rank]
    dshard = DeviceColumns(shard, torch.device("cuda", local))  # the rank's seq-range shard, resident in HBM
    comm = sharded.TorchComm()
    for _ in range(args.warmup):
        sharded.analyze_sharded_device(dshard, base, comm)
    steps = max(1, min(args.steps, 10))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = sharded.analyze_sharded_device(dshard, base, comm)
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=torch.device("cuda", local))
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    step_s = float(dt.item()) / steps
    # the same pipeline up to per-rank findings (global indices, key-range distributed), i.e.
    # without the gather + rank-0 merge into the reference's global orders
    dist.barrier()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(steps):
        sharded.analyze_sharded_device(dshard, base, comm, gather=False)
    torch.cuda.synchronize()
    dl = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=torch.device("cuda", local))
    dist.all_reduce(dl, op=dist.ReduceOp.MAX)
    dist_s = float(dl.item()) / steps
    out = {"metric": "M trace events/s analysed", "value": round(cols.n / step_s / 1e6, 3), "unit": "M events/s",
           "ms_per_step": round(step_s * 1e3, 3), "steps": steps,
           "config": {"workload": f"C2 trace of {cols.n} events ({args.n_events} per GPU), seq-range shards, "
                                  f"key-range sharded analysis (hash range / device owner): device-resident "
                                  f"routing, one NCCL all-to-all of event rows, engine per sub-trace, findings "
                                  f"gathered and merged on rank 0",
                      "events_total": cols.n},
           "timing": "wall clock around analyze_sharded_device, max over ranks",
           "distributed": {"value": round(cols.n / dist_s / 1e6, 3), "unit": "M events/s",
                           "ms_per_step": round(dist_s * 1e3, 3),
                           "note": "same pipeline, findings left on their key-range ranks (no gather / merge)"}}
    if rank == 0 and res is not None:
        out["counts"] = res.counts()
    return out


# ----------------------------------------------------------------------------- reference arm
_REF_STATE = {}


def _ref_worker_init(ref_path, per_worker, seed):
    sys.path.insert(0, ref_path)
    from dmlens.hashing import hash_bytes  # the unmodified reference
    from oracle import hash_ref  # payload bytes only (input generation, not timed)
    _REF_STATE["hash"] = hash_bytes
    _REF_STATE["payloads"] = [hash_ref.payload(BUF_BYTES, seed, os.getpid() * 10007 + i) for i in range(per_worker)]


def _ref_worker_step(_):
    hb = _REF_STATE["hash"]
    t0 = time.perf_counter()
    for p in _REF_STATE["payloads"]:
        hb(p)
    return time.perf_counter() - t0, len(_REF_STATE["payloads"]) * BUF_BYTES


def run_reference(args, rank, world):
    import multiprocessing as mp

    if rank != 0:
        return None
    ref_path = os.path.join(ROOT, "baseline", "_ref")
    kind = "reference"
    if not os.path.isdir(os.path.join(ref_path, "dmlens")):
        return {"impl": "reference", "unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    per_worker = 400  # 16 MB per worker per step (~0.5 s at the reference's ~33 MB/s/core)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_worker_init, initargs=(ref_path, per_worker, SEED)) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_worker_step, range(cores))
        t0 = time.perf_counter()
        total = 0
        for _ in range(args.steps):
            res = pool.map(_ref_worker_step, range(cores))
            total += sum(b for _, b in res)
        dt = time.perf_counter() - t0
    value = total / dt / 1e9
    analysis = None if args.no_analysis else run_analysis_reference(args, ref_path)
    sample = (f"each step: {cores} processes x {per_worker} C2 buffers of {BUF_BYTES} B "
              f"({cores * per_worker * BUF_BYTES / 1e9:.2f} GB) through dmlens.hashing.hash_bytes "
              f"(unmodified reference from baseline/_ref)")
    return {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C2: 400,000 x 40,000 B buffers per GPU (16.0 GB), 25% duplicates, hashed with "
                               "the reference FNV-1a/fmix64 fold", "parallelism": "host processes"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "analysis": analysis,
    }


def run_analysis_reference(args, ref_path, sample_events=200_000):
    """dmlens.analyze + estimate + attribute (unmodified reference) on a bounded sample of the C2 trace."""
    sys.path.insert(0, ref_path)
    from dmlens import analyze, attribute, estimate
    from dmlens.model import CodeLocation, EventKind, Trace, TraceEvent

    from paper_2601_12713_b200.synth import c2_trace  # input generation only (not timed)
    cols = c2_trace(min(args.n_events, sample_events), seed=SEED)
    kinds = [EventKind.TRANSFER, EventKind.ALLOC, EventKind.DELETE, EventKind.KERNEL]
    loc = CodeLocation()
    L = lambda a: a.tolist()  # noqa: E731
    ev = [TraceEvent(q, kinds[k], a, b, s_, d, sa, da, nb, h, loc) for q, k, a, b, s_, d, sa, da, nb, h in zip(
        L(cols.seq), L(cols.kind), L(cols.start_ns), L(cols.end_ns), L(cols.src_device), L(cols.dst_device),
        L(cols.src_addr), L(cols.dst_addr), L(cols.bytes), L(cols.hash))]
    tr = Trace(1, cols.num_devices_total, cols.host_device, cols.wall_time_ns, ev)
    steps = max(1, min(args.steps, 3))
    f = analyze(tr)
    t0 = time.perf_counter()
    for _ in range(steps):
        f = analyze(tr)
        estimate(tr, f)
        attribute(tr, f)
    dt = (time.perf_counter() - t0) / steps
    v = round(cols.n / dt / 1e6, 4)
    return {"metric": "M trace events/s analysed", "value": v, "unit": "M events/s", "ms_per_step": round(dt * 1e3, 1),
            "cpu_baseline": {"value": v, "unit": "M events/s", "cores": 1, "kind": "reference",
                             "sample": f"first {cols.n} events of the C2 trace as dmlens objects; analyze + "
                                       f"estimate + attribute, {steps} steps (single-threaded by design)"},
            "e2e": {"value": v, "unit": "M events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        rec = run_reference(args, rank, world)
        if rec is not None:
            print(json.dumps(rec), flush=True)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        if os.environ.get("B2L_BENCH_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    with ClockSampler(local) as clk:
        args._clock = clk
        rec = run_ours(args, rank, world, local)
        if not args.no_analysis:
            try:
                rec["analysis"] = run_analysis_ours(args, rank, world, local)
            except Exception as exc:  # the hash line above stands on its own
                rec["analysis"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    rec["clocks"] = clk.summary()
    rec["clocks"]["window"] = "sampled every 100 ms across both legs (warm-up + timed regions)"
    if rank == 0:
        print(json.dumps(rec), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
