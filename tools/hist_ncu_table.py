"""Per-kernel table of the last histogram_fd call in an ncu --csv launch list (tools/hist_probe.py)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
ids = sorted({int(r[0]) for r in rows})
first = max(i for i in ids if any(int(r[0]) == i and ("k_minmax" in r[4] or "k_hist_init" in r[4]) for r in rows))
agg = collections.OrderedDict()
for r in rows:
    if int(r[0]) >= first:
        agg.setdefault((int(r[0]), r[4].split("(")[0].replace("unnamed>::", "")), {})[r[12]] = float(r[14].replace(",", ""))
tot = 0.0
print("| id | kernel | us | DRAM MB | GB/s |\n|---|---|---|---|---|")
for (i, n), m in agg.items():
    us = m["gpu__time_duration.sum"] / 1e3
    mb = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / 1e6
    tot += us
    print(f"| {i} | {n} | {us:.1f} | {mb:.1f} | {mb / us * 1e3:.0f} |")
print(f"\ntotal device time {tot:.1f} us")
