"""Aggregate an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import collections
import csv
import sys


def main(path, top=25):
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
              "ms": 1e3, "msecond": 1e3,
              "second": 1e6}.get(d["Metric Unit"], 1.0)
        a = agg[d["Kernel Name"].split("(")[0]]
        a[0] += 1
        a[1] += v
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':64s} {'launches':>8s} {'total_us':>11s} "
          f"{'avg_us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[:64]:64s} {c:8d} {t:11.1f} {t / c:9.1f} "
              f"{100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
