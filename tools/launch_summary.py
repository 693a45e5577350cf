"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel.

    python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/rNN_launch_summary.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, cmd=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:72]
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v for _, v in agg.values())
    print(f"ncu launch list: {cmd}")
    print("(cold-cache, serialised per-launch device times: compare SHARES, not absolutes)")
    print(f"{'kernel':72s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>7s}")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:72s} {n:8d} {v:11.1f} {v / n:9.1f} {v / tot:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
