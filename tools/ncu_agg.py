"""Aggregate an ncu --csv --metrics launch list per kernel: launches, time, DRAM read/write."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if len(r) > 10 and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0][-40:]
        a = agg.setdefault(k, collections.defaultdict(float))
        v = d["Metric Value"].replace(",", "")
        a[d["Metric Name"]] += float(v) if v not in ("n/a", "") else 0.0
        if d["Metric Name"] == "gpu__time_duration.sum":
            a["n"] += 1
    for k, a in agg.items():
        print(f"{k:42s} n={int(a['n']):4d} t={a['gpu__time_duration.sum'] / 1e6:8.3f} ms "
              f"rd={a.get('dram__bytes_read.sum', 0) / 1e9:6.2f} GB wr={a.get('dram__bytes_write.sum', 0) / 1e9:6.2f} GB")


if __name__ == "__main__":
    main(sys.argv[1])
