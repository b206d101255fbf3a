#!/usr/bin/env python3
"""Benchmark of the B200 hot path.

Metric (BASELINE.json): "GB/s of mapped bytes hashed; M trace events/s analysed".

Headline line (one per GPU -> weak scaling):
  400,000 buffers x 40,000 B = 16.0 GB of payload per GPU, 25 % byte-identical
  duplicates (counter-based splitmix64 payloads generated on the device, not timed).
  A step = one b2l_hash_batch launch over the whole batch (inputs resident in HBM,
  16 GB >> 126 MB L2, so no flush is needed); at N > 1 the step also gathers every
  rank's digests to rank 0 (multigpu.gather_digests, one NCCL call).  `e2e` = the same
  batch through the host-buffer C-ABI call b2l_hash_host from pinned host memory (H2D
  copies and the digest D2H inside the timed region).
Nested lines: `analysis` (C2 1M-event trace: validate + 5 detectors + estimate/attribute
sums, verified against the oracle on every output) and `configs` (C1, C3, C4, C5 slice:
SURVEY 8(d) / BASELINE.md 4), each with its CPU baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun each rank hashes its own C2 batch; rank 0 prints one JSON line.
`--impl reference` times the unmodified reference (baseline/_ref: dmlens) on the host
cores on the same configs (same `config` objects).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
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
N_EVENTS = 1_000_000
EVENT_BYTES = 64  # algorithmic bytes per event: one read of the packed row
METRIC = "GB/s of mapped bytes hashed; M trace events/s analysed"
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
C1_BUFS, C1_SEED = 4000, 1
C3_BUF_BYTES, C3_BUFS, C3_SEED = 256 << 20, 16, 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-bufs", type=int, default=N_BUFS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the 10M/100M-event analysis lines")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C4/C5 config lines")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--n-events", type=int, default=N_EVENTS)
    ap.add_argument("--c5-events", type=int, default=100_000_000)
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


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------- configs (shared by both arms)
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


def hash_config(n, world):
    total = n * BUF_BYTES
    return {"workload": f"C2: {n:,} x {BUF_BYTES:,} B buffers per GPU ({total / 1e9:.1f} GB), 25% duplicates, "
                        "hashed with the reference FNV-1a/fmix64 fold",
            "n_buffers_per_gpu": n, "buffer_bytes": BUF_BYTES, "bytes_per_gpu": total, "seed": SEED,
            "l2": f"inputs ({total / 1e9:.1f} GB) larger than the 126 MB L2, no flush",
            "parallelism": f"shard{world}"}


def analysis_config(n):
    return {"workload": f"C2 trace: {n} events ([ALLOC,H2D,KERNEL,D2H,DELETE] x 8 target devices, 25% duplicate "
                        "H2D content, 30% unmodified D2H), validate + 5 detectors + estimate/attribute sums",
            "events_per_gpu": n, "seed": SEED}


def c1_lens():
    import numpy as np
    rng = np.random.default_rng(C1_SEED)
    return np.exp(rng.uniform(np.log(1024), np.log(1 << 20), C1_BUFS)).astype(np.int64)


CONFIGS = {
    "C1-hash": {"workload": "C1: 4,000 buffers, log-uniform 1 KiB - 1 MiB (seed 1), hashed longest first",
                "metric": "GB/s hashed"},
    "C1-analysis": {"workload": "C1: 10,000-event trace (C2 cycles, seed 1): validate + 5 detectors + sums",
                    "metric": "M trace events/s analysed"},
    "C3-hash": {"workload": f"C3: {C3_BUFS} stencil arrays of 256 MiB (seed 3), hashed in one call (K2: the whole "
                            "GPU folds one buffer)", "metric": "GB/s hashed"},
    "C3-analysis": {"workload": "C3: stencil time loop, 10,000 iterations x [D2H A, KERNEL, H2D A] (30,004 events)",
                    "metric": "M trace events/s analysed"},
    "C4-analysis": {"workload": "C4: allocation-heavy trace, 1,000,000 events (4 target devices, 4,096 host "
                                "variables, 4 B - 64 MiB, 20% unused allocs, 10% overwritten H2D, 65,536-hash "
                                "palette)", "metric": "M trace events/s analysed"},
    "C4-10M-analysis": {"workload": "C4: allocation-heavy trace, 10,000,000 events", "metric":
                        "M trace events/s analysed"},
    "C5-slice-analysis": {"workload": "C5 single-GPU slice: C2-style trace of 100,000,000 events on ONE B200",
                          "metric": "M trace events/s analysed"},
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name="hash_ncu_summary.json"):
    """dram bytes per launch of the hash kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", name)
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


# ----------------------------------------------------------------------------- helpers (ours)
def _fill(slab, offs, lens, cids, seed):
    import torch

    from paper_2601_12713_b200 import _lib
    s = torch.cuda.current_stream(slab.device)
    _lib.check(_lib.lib().b2l_fill_payloads(slab.data_ptr(), offs.data_ptr(), lens.data_ptr(), cids.data_ptr(),
                                            offs.numel(), seed, s.cuda_stream), "fill")


def _time_events(fn, iters, stream):
    """Device time per call (CUDA events on the launch stream) and per-call launch times."""
    import torch
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for a, b in evs:
        a.record(stream)
        fn()
        b.record(stream)
    b0.record(stream)
    torch.cuda.synchronize()
    return a0.elapsed_time(b0) / 1e3 / iters, [a.elapsed_time(b) / 1e3 for a, b in evs]


def _wall(fn, iters):
    import torch
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / iters


def _roofline(achieved, peak, peak_src, **extra):
    d = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
         "frac": round(achieved / peak, 5), "peak_source": peak_src}
    d.update(extra)
    return d


def _cpu_hash_port(ptrs, lens, seconds, label):
    """The oracle's C restatement of _fold64 on every host core over (a prefix of) the buffers."""
    import numpy as np

    from oracle import hash_ref  # CPU baseline only
    threads = host_cores()
    done, nbytes, t0 = 0, 0, time.perf_counter()
    chunk = max(threads * 4, 64)
    while done < len(ptrs) and (done == 0 or time.perf_counter() - t0 < seconds):
        k = min(chunk, len(ptrs) - done)
        hash_ref.fold64_c_batch(ptrs[done:done + k], lens[done:done + k], threads=threads)
        nbytes += int(np.asarray(lens[done:done + k], dtype=np.uint64).sum())
        done += k
    dt = time.perf_counter() - t0
    return {"value": round(nbytes / dt / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{done} of {len(ptrs)} {label} buffers ({nbytes / 1e9:.2f} GB), oracle/hash_fold64.c with "
                      f"{threads} pthreads, {dt:.1f} s", "cpu_model": cpu_model()}


# ----------------------------------------------------------------------------- ours: C2 hash (headline)
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import hash_ref  # checker + CPU baseline only
    from paper_2601_12713_b200 import hash_device, multigpu, sharded
    from paper_2601_12713_b200.hashing import hash_host_arrays

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n = args.n_bufs
    total = n * BUF_BYTES
    cids = content_ids(n, rank)
    offs = torch.arange(n, dtype=torch.int64, device=dev) * BUF_BYTES
    lens = torch.full((n,), BUF_BYTES, dtype=torch.int64, device=dev)
    slab = torch.empty(total, dtype=torch.uint8, device=dev)
    _fill(slab, offs, lens, torch.from_numpy(cids).to(dev), SEED)
    ptrs = offs + slab.data_ptr()
    out = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    comm = sharded.TorchComm(dev) if world > 1 else None
    gidx = torch.arange(n, dtype=torch.int64, device=dev) + rank * n  # global buffer ids of this rank
    torch.cuda.synchronize()

    def step():
        hash_device(ptrs, lens, out, stream=stream)
        if comm is not None:  # every rank's digests to rank 0, in global order
            multigpu.gather_digests(out, gidx, world * n, comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # correctness spot check against the C oracle (64 buffers incl. duplicates)
    sample = np.unique(np.concatenate([np.arange(0, n, max(1, n // 48)),
                                       np.nonzero(cids != np.arange(n) + rank * n)[0][:16]]))
    host = {int(i): slab[int(i) * BUF_BYTES:(int(i) + 1) * BUF_BYTES].cpu().numpy() for i in sample}
    got = out.cpu().numpy().view(np.uint64)
    verified = all(int(got[i]) == hash_ref.fold64_c(host[int(i)].tobytes()) for i in sample)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for a, b in evs:
        a.record(stream)
        hash_device(ptrs, lens, out, stream=stream)
        b.record(stream)
        if comm is not None:
            multigpu.gather_digests(out, gidx, world * n, comm)
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
        hptrs = (np.arange(n, dtype=np.uint64) * np.uint64(BUF_BYTES)) + np.uint64(hslab.data_ptr())
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
        e2e = {"value": round(world * total * e2e_steps / float(dt.item()) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": total + 16 * n, "d2h_bytes_per_step": 8 * n,
               "api": "b2l_hash_host (pinned host buffers, double-buffered device ring)",
               "steps": e2e_steps, "digests_match_device_path": bool(np.array_equal(hout, got))}
        del hslab

    # ---------------- CPU baseline: oracle C port, all host threads, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        hcopy = slab[: min(total, 4_000_000_000)].cpu().numpy()
        nb = hcopy.size // BUF_BYTES
        hp = np.arange(nb, dtype=np.uint64) * np.uint64(BUF_BYTES) + np.uint64(hcopy.ctypes.data)
        cpu = _cpu_hash_port(hp, np.full(nb, BUF_BYTES, dtype=np.uint64), args.cpu_seconds, "C2")
        del hcopy

    peak, peak_src = peaks()
    kern_s = statistics.mean(launch_ms) / 1e3
    rec = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": hash_config(n, world),
        "roofline": _roofline(total / kern_s / 1e9, peak, peak_src,
                              traffic=ncu_traffic() if n == N_BUFS else None,
                              kernel="k_hash_coop<2,512,2> (b2l_hash_batch default variant)",
                              algorithmic_bytes_per_launch=total,
                              timing="CUDA events around each launch on its stream, mean over the timed steps"),
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": args.steps, "verified": bool(verified),
        "impl": "ours",
    }
    if world > 1:
        rec["step"] = (f"b2l_hash_batch over the rank's {total / 1e9:.1f} GB + gather of every rank's digests to "
                       f"rank 0 (NCCL)")
    del slab
    torch.cuda.empty_cache()
    return rec


# ----------------------------------------------------------------------------- ours: analysis
def _verify(cols, cf, sv, strict=False):
    from oracle.compare import full_parity  # the checker (outside timed regions)
    bad = full_parity(cols, cf, sv, strict=strict)
    return not bad, bad[:3]


def _ref_analysis_cpu(cols, label):
    """The unmodified reference (baseline/_ref dmlens) on these exact events: analyze + estimate +
    attribute, one core, one step."""
    if not os.path.isdir(os.path.join(REF_PATH, "dmlens")):
        return None
    dt, n = _time_reference_analysis(cols, steps=1)
    v = round(n / dt / 1e6, 4)
    return {"value": v, "unit": "M events/s", "cores": 1, "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"the full {n}-event {label} trace as dmlens objects: analyze + estimate + attribute "
                      f"(unmodified reference from baseline/_ref, single-threaded by design), {dt:.1f} s"}


def _analysis_e2e(cols, steps):
    """Host columns in (page-locked), host findings + sums out, through the public API:
    analyze_many (each trace's upload overlapped with the previous trace's analysis) -- the
    headline -- and, beside it, one synchronous analyze_columns + savings_columns call per step."""
    import torch

    from paper_2601_12713_b200.analysis import (DeviceColumns, analyze_columns, analyze_many, pinned_columns,
                                                savings_columns)
    cols = pinned_columns(cols)
    for _ in range(3):  # warm-up with the timed loop's object lifetimes (previous findings alive)
        cfh = analyze_columns(cols, with_savings=True)
        savings_columns(cols, cfh)
    for _ in analyze_many([cols] * 3):
        pass
    gc.collect()
    gc.disable()
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        marks = []
        for cfh, _ in analyze_many([cols] * steps):
            marks.append(time.perf_counter())
        torch.cuda.synchronize()
        de = time.perf_counter() - t0
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(steps):
            cfs = analyze_columns(cols, with_savings=True)
            savings_columns(cols, cfs)
        torch.cuda.synchronize()
        ds = time.perf_counter() - t1
    finally:
        gc.enable()
    steps_raw = [1e3 * (b - a) for a, b in zip([t0] + marks[:-1], marks)]
    slowest = max(range(len(steps_raw)), key=steps_raw.__getitem__)
    step_ms = sorted(steps_raw)
    h2d = sum(getattr(cols, f).nbytes for f in DeviceColumns.FIELDS)
    d2h = sum(a.nbytes for a in (cfh.dd_offsets, cfh.dd_members, cfh.rt_offsets, cfh.rt_tx, cfh.rt_rx,
                                 cfh.pair_alloc, cfh.pair_delete, cfh.warn_index, cfh.ra_offsets, cfh.ra_pairs,
                                 cfh.ua_pairs, cfh.ut_events))
    return {"value": round(cols.n * steps / de / 1e6, 3), "unit": "M events/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "step_ms_min_median_max": [round(step_ms[0], 3), round(step_ms[len(step_ms) // 2], 3),
                                       round(step_ms[-1], 3)],
            "slowest_step": slowest,
            "api": "analyze_many over page-locked host columns: each step uploads its trace (overlapped with "
                   "the previous step's analysis on a copy stream), analyses it with the fused savings and reads "
                   "findings + sums back",
            "single_call": {"value": round(cols.n * steps / ds / 1e6, 3), "unit": "M events/s",
                            "api": "analyze_columns + savings_columns, one synchronous call pair per step"}}


def _analysis_device(cols, dev, iters, warm=3):
    """Device-resident columns: median step (wall clock bracketed by synchronize) and the findings."""
    import torch

    from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, savings_columns
    d = DeviceColumns(cols, dev)
    hold = {}

    def step():
        hold["cf"] = analyze_columns(d, with_savings=True)
        hold["sv"] = savings_columns(d, hold["cf"])
    for _ in range(warm):
        step()
    times = []
    for _ in range(iters):
        torch.cuda.synchronize()
        t = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    return statistics.median(times), hold["cf"], hold["sv"], d


def run_analysis_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns, savings_columns
    from paper_2601_12713_b200.synth import c2_trace

    dev = torch.device("cuda", local)
    if world > 1:
        return run_analysis_sharded(args, rank, world, local)
    cols = c2_trace(args.n_events, seed=SEED + rank)
    dcols = DeviceColumns(cols, dev)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        cf = analyze_columns(dcols, with_savings=True)
        sv = savings_columns(dcols, cf)
    verified, why = _verify(cols, cf, sv)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cf = analyze_columns(dcols, with_savings=True)
        savings_columns(dcols, cf)
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    step_s = float(dt.item()) / args.steps
    value = world * cols.n / step_s / 1e6
    # ~0.5 s of pipelined steps: a host-bound loop on a shared host sees the odd scheduling stall
    # (one 147 ms step in a 30-step window cut a measured 705 M events/s to 162); the window is
    # long enough that one stall moves the throughput by a few per cent, not by 4x
    e2e = _analysis_e2e(cols, max(args.steps, int(0.5e3 / max(step_s * 1e3 * 2, 0.05))))
    peak, peak_src = peaks()
    traffic, launches, top = analysis_traffic(cols.n, peak)
    out = {
        "metric": "M trace events/s analysed", "value": round(value, 3), "unit": "M events/s",
        "ms_per_step": round(step_s * 1e3, 3), "steps": args.steps, "config": analysis_config(cols.n),
        "counts": cf.counts(),
        "timing": "host-synchronous C-ABI call (b2l_analyze + b2l_savings_compute) on columns resident in HBM, "
                  "perf_counter bracketed by cuda synchronize",
        "roofline": _roofline(cols.n * EVENT_BYTES / step_s / 1e9, peak, peak_src, traffic=traffic,
                              algorithmic_bytes_per_step=cols.n * EVENT_BYTES,
                              traffic_note="ncu dram bytes summed over every kernel of one analyze+savings step "
                                           "(profiles/analysis_traffic_c2_<n>.json)",
                              traffic_gbs_over_step=round(traffic / step_s / 1e9, 1) if traffic else None,
                              kernel_launches_per_step=launches, top_kernels_ncu=top),
        "e2e": e2e, "verified": verified,
        "verified_scope": "findings (DD/RT/pairs/RA/UA/UT), warnings, per-category and union ns, eliminable set, "
                          "overlap flag, attribution rows -- all vs oracle/analysis_ref (oracle/compare.full_parity)",
    }
    if why:
        out["verify_mismatch"] = why
    if rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = _ref_analysis_cpu(cols, "C2") or _oracle_analysis_cpu(cols, "C2")
    return out


def _oracle_analysis_cpu(cols, label):
    from oracle import analysis_ref as R
    t0 = time.perf_counter()
    rf = R.analyze_cols(cols)
    R.estimate_cols(cols, rf, cols.wall_time_ns)
    R.attribute_cols(cols, rf, cols.wall_time_ns)
    dt = time.perf_counter() - t0
    return {"value": round(cols.n / dt / 1e6, 4), "unit": "M events/s", "cores": 1, "kind": "port",
            "sample": f"the full {cols.n}-event {label} trace through oracle/analysis_ref (1 thread)"}


# ----------------------------------------------------------------------------- ours: configs C1, C3, C4, C5
def run_configs_ours(args, dev):
    out = []
    for fn in (_c1_hash, _c1_analysis, _c3_hash, _c3_analysis, _c4_analysis, _c4_10m, _c5_slice):
        if args.no_large and fn in (_c4_10m, _c5_slice):
            continue
        try:
            out.append(fn(args, dev))
        except Exception as exc:  # one config failing does not take the others down
            out.append({"name": fn.__name__, "error": f"{type(exc).__name__}: {exc}"[:300]})
        import torch
        torch.cuda.empty_cache()
    return out


def _line(name, value, unit, ms, **kw):
    d = {"name": name, "metric": CONFIGS[name]["metric"], "value": round(value, 3), "unit": unit,
         "ms_per_step": round(ms, 4), "config": {"workload": CONFIGS[name]["workload"]}}
    d.update(kw)
    return d


def _c1_hash(args, dev):
    import numpy as np
    import torch

    from oracle import hash_ref
    from paper_2601_12713_b200 import hash_device
    from paper_2601_12713_b200.hashing import hash_host_arrays
    lens = c1_lens()
    n = lens.size
    offs = np.zeros(n, np.int64)
    offs[1:] = np.cumsum((lens + 255) // 256 * 256)[:-1]
    total = int(offs[-1] + lens[-1])
    slab = torch.empty(total, dtype=torch.uint8, device=dev)
    o_d, l_d = torch.from_numpy(offs).to(dev), torch.from_numpy(lens).to(dev)
    _fill(slab, o_d, l_d, torch.arange(n, device=dev), C1_SEED)
    ptrs = o_d + slab.data_ptr()
    order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        hash_device(ptrs, l_d, out, order=order, stream=stream)
    dt, _ = _time_events(lambda: hash_device(ptrs, l_d, out, order=order, stream=stream), 20, stream)
    nbytes = int(lens.sum())
    host = slab.cpu().numpy()
    hp = offs.astype(np.uint64) + np.uint64(host.ctypes.data)
    want = hash_ref.fold64_c_batch(hp, lens.astype(np.uint64), threads=host_cores())
    verified = bool(np.array_equal(out.cpu().numpy().view(np.uint64), want))
    # e2e from pinned host buffers
    pin = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    pin.copy_(slab)
    pp = offs.astype(np.uint64) + np.uint64(pin.data_ptr())
    hout = np.zeros(n, np.uint64)
    hash_host_arrays(pp, lens.astype(np.uint64), hout)
    e2e_s = _wall(lambda: hash_host_arrays(pp, lens.astype(np.uint64), hout), 10)
    peak, peak_src = peaks()
    chain = int(lens.max()) / 8 * 10 / 1.965e9
    return _line("C1-hash", nbytes / dt / 1e9, "GB/s", dt * 1e3, buffers=n, bytes=nbytes, verified=verified,
                 roofline=_roofline(nbytes / dt / 1e9, peak, peak_src, traffic=ncu_traffic("c1_warp_ncu_summary.json"),
                                    algorithmic_bytes_per_launch=nbytes,
                                    note=f"bound by the longest buffer's serial chain (~{chain * 1e3:.2f} ms at "
                                         f"~10 cycles/word for {int(lens.max())} B), not HBM (floor "
                                         f"{nbytes / peak / 1e6:.3f} ms)"),
                 e2e={"value": round(nbytes / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": nbytes,
                      "d2h_bytes_per_step": 8 * n, "api": "b2l_hash_host (pinned host buffers)",
                      "digests_match": bool(np.array_equal(hout, want))},
                 cpu_baseline=None if args.no_cpu else _cpu_hash_port(hp, lens.astype(np.uint64), 30.0, "C1"))


def _c3_hash(args, dev):
    import numpy as np
    import torch

    from oracle import hash_ref
    from paper_2601_12713_b200.hashing import hash_host_arrays, hash_large_many
    size, k = C3_BUF_BYTES, C3_BUFS
    slab = torch.empty(size * k, dtype=torch.uint8, device=dev)
    offs = torch.arange(k, dtype=torch.int64, device=dev) * size
    _fill(slab, offs, torch.full((k,), size, dtype=torch.int64, device=dev), torch.arange(k, device=dev), C3_SEED)
    out = torch.empty(k, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    ptrs = [slab.data_ptr() + i * size for i in range(k)]

    def step():  # the 16 arrays in one call: K2 over every array at once (b2l_hash_large_many)
        hash_large_many(ptrs, [size] * k, out.data_ptr(), stream)
    step()
    dt, per = _time_events(step, 3, stream)
    got = out.cpu().numpy().view(np.uint64)
    hsamp = slab[:4 * size].cpu().numpy()
    hp = np.arange(4, dtype=np.uint64) * np.uint64(size) + np.uint64(hsamp.ctypes.data)
    want = hash_ref.fold64_c_batch(hp, np.full(4, size, np.uint64), threads=4)
    verified = bool(np.array_equal(got[:4], want))
    cpu = None
    if not args.no_cpu:
        cpu = _cpu_hash_port(hp, np.full(4, size, np.uint64), 0.0, "C3 (4 of 16)")
    # e2e: 4 arrays from pinned host memory through b2l_hash_host (K2 per buffer)
    pin = torch.empty(4 * size, dtype=torch.uint8, pin_memory=True)
    pin.copy_(slab[:4 * size])
    pp = np.arange(4, dtype=np.uint64) * np.uint64(size) + np.uint64(pin.data_ptr())
    hout = np.zeros(4, np.uint64)
    hash_host_arrays(pp, np.full(4, size, np.uint64), hout)
    e2e_s = _wall(lambda: hash_host_arrays(pp, np.full(4, size, np.uint64), hout), 2)
    peak, peak_src = peaks()
    return _line("C3-hash", k * size / dt / 1e9, "GB/s", dt * 1e3, buffers=k, buffer_bytes=size,
                 ms_per_buffer=round(dt / k * 1e3, 3), verified=verified,
                 roofline=_roofline(k * size / dt / 1e9, peak, peak_src, traffic=ncu_traffic("k2_many_ncu_summary.json"),
                                    algorithmic_bytes_per_launch=k * size,
                                    kernel="k_hash_planes (K2, the 16 arrays in one launch)",
                                    note="ALU/latency bound: one serial FNV chain per buffer resolved as 16 "
                                         "dependent 4-bit groups, each array by its own share of the GPU's "
                                         "CTAs (DESIGN.md K2)"),
                 e2e={"value": round(4 * size / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * size,
                      "d2h_bytes_per_step": 32, "api": "b2l_hash_host, 4 arrays from pinned memory",
                      "digests_match": bool(np.array_equal(hout, want))},
                 cpu_baseline=cpu)


def _analysis_line(name, cols, dev, args, iters=10, verify=True, e2e_steps=10, cpu=True, label=None):
    step_s, cf, sv, _ = _analysis_device(cols, dev, iters)
    peak, peak_src = peaks()
    kw = {"events": cols.n, "counts": cf.counts(),
          "roofline": _roofline(cols.n * EVENT_BYTES / step_s / 1e9, peak, peak_src,
                                algorithmic_bytes_per_step=cols.n * EVENT_BYTES)}
    if verify:
        ok, why = _verify(cols, cf, sv)
        kw["verified"] = ok
        if why:
            kw["verify_mismatch"] = why
        ok_s, why_s = _verify(cols, _strict(cols, dev), None, strict=True)
        kw["verified_strict_rt"] = ok_s
    if e2e_steps:  # at least ~0.5 s of steps (see run_analysis: scheduling stalls on a shared host)
        kw["e2e"] = _analysis_e2e(cols, min(2000, max(e2e_steps, int(0.5 / max(2 * step_s, 5e-5)))))
    if cpu and not args.no_cpu:
        kw["cpu_baseline"] = _ref_analysis_cpu(cols, label or name) or _oracle_analysis_cpu(cols, label or name)
    return _line(name, cols.n / step_s / 1e6, "M events/s", step_s * 1e3, **kw)


def _strict(cols, dev):
    from paper_2601_12713_b200.analysis import DeviceColumns, analyze_columns
    return analyze_columns(DeviceColumns(cols, dev), strict=True)


def _c1_analysis(args, dev):
    from paper_2601_12713_b200.synth import c2_trace
    return _analysis_line("C1-analysis", c2_trace(10_000, seed=C1_SEED), dev, args, iters=30, e2e_steps=30)


def _c3_analysis(args, dev):
    from paper_2601_12713_b200.synth import c3_trace
    return _analysis_line("C3-analysis", c3_trace(10_000), dev, args, iters=30, e2e_steps=30)


def _c4_analysis(args, dev):
    from paper_2601_12713_b200.synth import c4_trace
    return _analysis_line("C4-analysis", c4_trace(1_000_000), dev, args, iters=10, e2e_steps=20)


def _c4_10m(args, dev):
    from paper_2601_12713_b200.synth import c4_trace
    ln = _analysis_line("C4-10M-analysis", c4_trace(10_000_000), dev, args, iters=4, verify=False, e2e_steps=3,
                        cpu=False)
    ln["verified"] = None
    ln["note"] = "timing only; parity at C4 is checked on the 1M-event C4 line and in tests/test_parity_configs_gpu.py"
    return ln


def _c5_slice(args, dev):
    from paper_2601_12713_b200.synth import c2_trace
    cols = c2_trace(args.c5_events, seed=5)
    ln = _analysis_line("C5-slice-analysis", cols, dev, args, iters=3, verify=False, e2e_steps=0, cpu=False)
    ln["verified"] = None
    ln["note"] = ("timing only (C2-style cycles at 100M events; parity of the same pipeline is checked at 1M); "
                  "the multi-GPU C5 run shards this trace by key range (bench.py --gpus N)")
    return ln


def run_analysis_sharded(args, rank, world, local):
    """N>1: one global C2 trace of world x n_events events, seq-range sharded over the ranks,
    analysed with the key-range sharded pipeline (one NCCL all-to-all + final gather)."""
    import torch
    import torch.distributed as dist

    from paper_2601_12713_b200 import sharded
    from paper_2601_12713_b200.analysis import DeviceColumns
    from paper_2601_12713_b200.synth import c2_trace

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
                                  f"key-range sharded analysis: device-resident routing, one NCCL all-to-all of "
                                  f"event rows, engine per sub-trace, findings gathered and merged on rank 0",
                      "events_total": cols.n},
           "timing": "wall clock around analyze_sharded_device, max over ranks",
           "distributed": {"value": round(cols.n / dist_s / 1e6, 3), "unit": "M events/s",
                           "ms_per_step": round(dist_s * 1e3, 3),
                           "note": "same pipeline, findings left on their key-range ranks (no gather / merge)"}}
    if rank == 0 and res is not None:
        out["counts"] = res.counts()
    return out


# ----------------------------------------------------------------------------- reference arm
def _ref_hash_worker(jobs, steps, warmup, start, stop, q):
    """One host process: generate its share of the buffers (not timed), then hash them `steps` times
    with dmlens.hashing.hash_bytes between two barriers shared with the parent."""
    sys.path.insert(0, REF_PATH)
    from dmlens.hashing import hash_bytes  # the unmodified reference
    from oracle import hash_ref  # payload bytes only (input generation, not timed)
    pays = [hash_ref.payload(n, seed, cid) for n, seed, cid in jobs]
    for _ in range(warmup):
        for p in pays:
            hash_bytes(p)
    start.wait()
    nb = 0
    for _ in range(steps):
        for p in pays:
            hash_bytes(p)
            nb += len(p)
    stop.wait()
    q.put(nb)


def _ref_hash(jobs_per_worker, steps, warmup):
    """dmlens.hashing.hash_bytes on every host core (one process each, `hash_bytes` is pure) over
    the given (len, seed, content id) buffers; the parent times from the moment every process is
    ready to the moment the last one finishes.  Returns (GB/s, bytes per step, seconds per step)."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    k = len(jobs_per_worker)
    start, stop, q = ctx.Barrier(k + 1), ctx.Barrier(k + 1), ctx.Queue()
    procs = [ctx.Process(target=_ref_hash_worker, args=(j, steps, warmup, start, stop, q)) for j in jobs_per_worker]
    for p in procs:
        p.start()
    start.wait()
    t0 = time.perf_counter()
    stop.wait()
    dt = time.perf_counter() - t0
    total = sum(q.get() for _ in procs)
    for p in procs:
        p.join()
    return total / dt / 1e9, total / max(steps, 1), dt / max(steps, 1)


def _split_jobs(jobs, cores):
    """Deal buffers to workers by LPT on their lengths (balanced per-step work)."""
    out = [[] for _ in range(cores)]
    load = [0] * cores
    for j in sorted(jobs, key=lambda j: -j[0]):
        w = min(range(cores), key=lambda i: load[i])
        out[w].append(j)
        load[w] += j[0]
    return out


def _time_reference_analysis(cols, steps):
    """analyze + estimate + attribute of the unmodified reference on `cols` as dmlens objects."""
    sys.path.insert(0, REF_PATH)
    from dmlens import analyze, attribute, estimate
    from dmlens.model import CodeLocation, EventKind, Trace, TraceEvent
    kinds = [EventKind.TRANSFER, EventKind.ALLOC, EventKind.DELETE, EventKind.KERNEL]
    loc = CodeLocation()
    L = lambda a: a.tolist()  # noqa: E731
    ev = [TraceEvent(q, kinds[k], a, b, s_, d, sa, da, nb, h, loc) for q, k, a, b, s_, d, sa, da, nb, h in zip(
        L(cols.seq), L(cols.kind), L(cols.start_ns), L(cols.end_ns), L(cols.src_device), L(cols.dst_device),
        L(cols.src_addr), L(cols.dst_addr), L(cols.bytes), L(cols.hash))]
    tr = Trace(1, cols.num_devices_total, cols.host_device, cols.wall_time_ns, ev)
    best = None
    for _ in range(steps):
        t0 = time.perf_counter()
        f = analyze(tr)
        estimate(tr, f)
        attribute(tr, f)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, cols.n


def run_reference(args, rank, world):
    if rank != 0:
        return None
    if not os.path.isdir(os.path.join(REF_PATH, "dmlens")):
        return {"impl": "reference", "unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    import numpy as np
    cores = host_cores()
    # C2 hash: a prefix of the same 400,000 buffers (same content ids, so the same bytes) -- 400 per
    # core per step (~0.5 s at the reference's ~33 MB/s/core)
    cids = content_ids(args.n_bufs, 0)
    per = 400
    jobs = [(BUF_BYTES, SEED, int(cids[i])) for i in range(min(args.n_bufs, per * cores))]
    gbs, bstep, sstep = _ref_hash(_split_jobs(jobs, cores), args.steps, args.warmup)
    sample = (f"each step: the first {len(jobs)} of the {args.n_bufs} C2 buffers ({bstep / 1e9:.2f} GB, same bytes "
              f"as the GPU arm) through dmlens.hashing.hash_bytes on {cores} processes (unmodified reference)")
    rec = {
        "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sstep * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": hash_config(args.n_bufs, world), "impl": "reference",
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if not args.no_analysis:
        from paper_2601_12713_b200.synth import c2_trace  # input generation only (not timed)
        cols = c2_trace(args.n_events, seed=SEED)
        dt, n = _time_reference_analysis(cols, steps=max(1, min(args.steps, 2)))
        v = round(n / dt / 1e6, 4)
        rec["analysis"] = {
            "metric": "M trace events/s analysed", "value": v, "unit": "M events/s", "ms_per_step": round(dt * 1e3, 1),
            "config": analysis_config(n),
            "cpu_baseline": {"value": v, "unit": "M events/s", "cores": 1, "kind": "reference",
                             "sample": f"the full {n}-event C2 trace as dmlens objects; analyze + estimate + "
                                       f"attribute, best of {max(1, min(args.steps, 2))} (single-threaded by design)"},
            "e2e": {"value": v, "unit": "M events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_configs:
        rec["configs"] = run_configs_reference(args, cores)
    return rec


def run_configs_reference(args, cores):
    import numpy as np

    from paper_2601_12713_b200.synth import c2_trace, c3_trace, c4_trace  # inputs only
    out = []

    def ref_line(name, value, unit, ms, sample, kind_cores):
        return {"name": name, "metric": CONFIGS[name]["metric"], "value": round(value, 4), "unit": unit,
                "ms_per_step": round(ms, 3), "config": {"workload": CONFIGS[name]["workload"]},
                "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": kind_cores, "kind": "reference",
                                 "sample": sample}}
    # C1 hash: all 4,000 buffers (the same bytes), every core
    lens = c1_lens()
    jobs = [(int(n), C1_SEED, i) for i, n in enumerate(lens)]
    gbs, b, s = _ref_hash(_split_jobs(jobs, cores), 2, 1)
    out.append(ref_line("C1-hash", gbs, "GB/s", s * 1e3, f"all {len(jobs)} C1 buffers ({b / 1e9:.2f} GB) through "
                        f"dmlens.hashing.hash_bytes on {cores} processes", cores))
    # C3 hash: 4 of the 16 arrays (~8 s each on one core), one per process
    jobs = [(C3_BUF_BYTES, C3_SEED, i) for i in range(4)]
    gbs, b, s = _ref_hash(_split_jobs(jobs, min(cores, 4)), 1, 0)
    out.append(ref_line("C3-hash", gbs, "GB/s", s * 1e3, f"4 of the {C3_BUFS} 256 MiB C3 arrays ({b / 1e9:.2f} GB) "
                        f"through dmlens.hashing.hash_bytes, one process each", min(cores, 4)))
    # analyses on one core (single-threaded by design)
    for name, cols in (("C1-analysis", c2_trace(10_000, seed=C1_SEED)), ("C3-analysis", c3_trace(10_000)),
                       ("C4-analysis", c4_trace(1_000_000))):
        dt, n = _time_reference_analysis(cols, steps=2 if n_small(cols) else 1)
        out.append(ref_line(name, n / dt / 1e6, "M events/s", dt * 1e3,
                            f"the full {n}-event trace as dmlens objects: analyze + estimate + attribute, "
                            f"{'best of 2' if n_small(cols) else '1 step'}", 1))
    for name in ("C4-10M-analysis", "C5-slice-analysis"):
        out.append({"name": name, "metric": CONFIGS[name]["metric"], "config": {"workload": CONFIGS[name]["workload"]},
                    "not_run": "the reference needs ~200 B/event of Python objects and minutes per step at this "
                               "size; its per-event rate is the C4 (1M) / C2 (1M) line's"})
    del np
    return out


def n_small(cols):
    return cols.n <= 100_000


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
        rec = run_ours(args, rank, world, local)
        if not args.no_analysis:
            try:
                rec["analysis"] = run_analysis_ours(args, rank, world, local)
            except Exception as exc:  # the hash line above stands on its own
                rec["analysis"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if world == 1 and not args.no_configs:
            rec["configs"] = run_configs_ours(args, torch.device("cuda", local))
    rec["clocks"] = clk.summary()
    rec["clocks"]["window"] = "sampled every 100 ms across every leg (warm-up + timed regions)"
    if rank == 0:
        print(json.dumps(rec), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
