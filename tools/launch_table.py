"""Markdown table of an ncu --csv launch list with gpu__time_duration.sum and dram__bytes_{read,write}.sum:
launches, total / mean time, total DRAM bytes and share per kernel.

    python tools/launch_table.py gpurun_out/f2/launches.csv [title] > profiles/ncu_r2_launches.md
"""
import collections
import csv
import re
import sys

TU = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BU = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, dr, c = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"^void ", "", r[ki]).replace("edgc::<unnamed>::", "").split("(")[0]
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            t[name] += v * TU[r[ui]]
            c[name] += 1
        elif r[mi].startswith("dram__bytes"):
            dr[name] += v * BU[r[ui]]
    tot = sum(t.values())
    print(f"# {title}\n")
    print("| kernel | launches | total us | mean us | DRAM GB (all launches) | share |")
    print("|---|---|---|---|---|---|")
    for k in sorted(t, key=lambda k: -t[k])[:24]:
        print(f"| `{k[:72]}` | {c[k]} | {t[k]:.1f} | {t[k] / c[k]:.1f} | {dr[k] / 1e9:.2f} | {100 * t[k] / tot:.1f}% |")


if __name__ == "__main__":
    main()
