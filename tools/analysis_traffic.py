"""Per-step DRAM traffic of the analysis pipeline from an ncu CSV launch list collected with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum

usage: python tools/analysis_traffic.py launches.csv iters events out.json
Sums every kernel of `iters` identical analyze+savings iterations and divides by iters."""
import collections
import csv
import json
import sys


def main():
    path, iters, events, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    hdr, per = None, collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.Counter()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0]
        metric, unit = r[hdr.index("Metric Name")], r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}.get(unit, 1)
        per[name][metric] += v * scale
        if metric == "gpu__time_duration.sum":
            launches[name] += 1
    tot = collections.defaultdict(float)
    for m in per.values():
        for k, v in m.items():
            tot[k] += v / iters
    kernels = sorted(({"kernel": k, "launches": launches[k] / iters,
                       "time_us": m["gpu__time_duration.sum"] / iters * 1e6,
                       "dram_bytes": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / iters,
                       "l2_bytes": m.get("lts__t_bytes.sum", 0.0) / iters} for k, m in per.items()),
                     key=lambda x: -x["time_us"])
    dram = tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]
    res = {"source": path, "events": events, "iterations": iters,
           "launches_per_step": sum(launches.values()) / iters,
           "kernel_time_us_per_step": tot["gpu__time_duration.sum"] * 1e6,
           "dram_bytes_per_step": dram, "l2_bytes_per_step": tot.get("lts__t_bytes.sum", 0.0),
           "dram_bytes_per_event": dram / events, "algorithmic_bytes_per_event": 64,
           "dram_gbs_over_kernel_time": dram / tot["gpu__time_duration.sum"] / 1e9,
           "note": "ncu serialises kernels and replays cold (--clock-control none): per-kernel times are "
                   "cold-cache upper bounds; byte counts are what each kernel moved to/from HBM",
           "kernels": kernels[:40]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main()
