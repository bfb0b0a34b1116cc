"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total ms and count per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    hdr = None
    agg = {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"][:100]
                agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:top]:
        print(f"{len(v):4d} {sum(v) / 1e6:10.3f} ms  {k}")


if __name__ == "__main__":
    main()
