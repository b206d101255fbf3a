"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

usage: python tools/launch_summary.py launches.csv [iters] [top]
Totals are divided by `iters` (the number of identical pipeline iterations captured)."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    hdr, per = None, collections.defaultdict(lambda: [0.0, 0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0]
        us = float(r[hdr.index("Metric Value")].replace(",", "")) / 1e3
        per[name][0] += us
        per[name][1] += 1
    tot = sum(v[0] for v in per.values()) / iters
    nl = sum(v[1] for v in per.values()) / iters
    print(f"# per iteration: {nl:.0f} launches, {tot:.1f} us kernel time (serialised, cold-cache)")
    print("# total_us  launches  kernel")
    for k, v in sorted(per.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v[0] / iters:10.1f} {v[1] / iters:6.0f}  {k}")


if __name__ == "__main__":
    main()
