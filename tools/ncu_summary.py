#!/usr/bin/env python3
"""Summarise an ncu --set full report (.ncu-rep) into a small JSON + text
file under profiles/ (the .ncu-rep itself stays in gpurun_out/, git-ignored).

  python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/x.json [--algo-bytes N]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__inst_executed.sum": "instructions",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    algo = None
    if "--algo-bytes" in sys.argv:
        algo = float(sys.argv[sys.argv.index("--algo-bytes") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * SCALE.get(units[i], 1)
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if "dram_read" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0)
            if "duration" in d:
                d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
            if algo:
                d["algorithmic_bytes"] = algo
                d["achieved_algorithmic_gbs"] = algo / d["duration"] / 1e9
        kernels.append(d)
    doc = {"report": rep, "kernels": kernels}
    if kernels and "dram_bytes_per_launch" in kernels[0]:
        doc["dram_bytes_per_launch"] = kernels[0]["dram_bytes_per_launch"]
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc, indent=1)[:3000])


if __name__ == "__main__":
    main()
