"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel
launches, avg/total device time and share (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys


def main(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[r[ui]]
        name = r[ki].split("(")[0].replace("void ", "")
        if "<" in name:
            name = name.split("<")[0]
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':45s} {'launches':>8s} {'avg_us':>9s} {'total_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:45s} {len(v):8d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot:6.3f}")
    print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
