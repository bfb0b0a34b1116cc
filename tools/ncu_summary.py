"""Summarise ncu output into profiles/ (run here, on the CPU box, after a gpurun).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        [--report gpurun_out/prof.ncu-rep] --tag r1 [--bench gpurun_out/bench.json]

Writes profiles/ncu_<tag>_launches.md (per-kernel device time and share of the
step, from the `--metrics gpu__time_duration.sum --clock-control none` pass),
profiles/ncu_<tag>_<kernel>.md (DRAM bytes / throughput / occupancy of the
`--set full` capture) and updates profiles/ncu_summary.json, which bench.py
reads for roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    m = re.search(r"(k_[A-Za-z0-9_]+)", name)
    return m.group(1) if m else name[:60]


def parse_launches(path):
    rows = []
    with open(path) as fh:
        text = fh.read()
    # ncu --csv --log-file prefixes ==PROF== lines; keep the CSV block
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rd = csv.DictReader(io.StringIO("\n".join(lines)))
    for row in rd:
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        val = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        rows.append((short(row["Kernel Name"]), val * scale))
    return rows


def launches_md(rows, tag):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, us in rows:
        tot[k] += us
        cnt[k] += 1
    all_us = sum(tot.values())
    out = [f"# ncu launch list ({tag})", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches:",
           "compare shares, not absolute times).", "",
           "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {100 * tot[k] / all_us:.1f}% |")
    return "\n".join(out) + "\n", {k: {"launches": cnt[k], "total_us": tot[k], "share": tot[k] / all_us}
                                  for k in tot}


METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def parse_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in raw.splitlines() if ln.startswith('"')]
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    if len(rd) < 3:
        return {}
    head, units, data = rd[0], rd[1], rd[2:]
    out = defaultdict(list)
    for row in data:
        rec = dict(zip(head, row))
        k = short(rec.get("Kernel Name", "?"))
        vals = {}
        for mname in METRICS:
            if mname in rec:
                try:
                    u = units[head.index(mname)]
                    v = float(rec[mname].replace(",", ""))
                    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                            "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
                    if mname == "gpu__time_duration.sum" and u not in ("nsecond", "usecond", "msecond", "ns", "us",
                                                                       "ms", "second"):
                        mult = 1e-9
                    vals[mname] = v * mult
                except (ValueError, IndexError):
                    pass
        out[k].append(vals)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--alg-bytes", type=float, default=None, help="algorithmic bytes per launch of the profiled kernel")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(summ_path)) if os.path.exists(summ_path) else {"kernels": {}}
    if args.launches:
        md, shares = launches_md(parse_launches(args.launches), args.tag)
        with open(os.path.join(PROF, f"ncu_{args.tag}_launches.md"), "w") as fh:
            fh.write(md)
        summary["launch_shares_" + args.tag] = shares
        print(md)
    if args.report:
        rep = parse_report(args.report)
        lines = [f"# ncu --set full ({args.tag})", "", "| kernel | launch | dram read MB | dram write MB | time us | "
                 "DRAM % peak | warps active % | regs |", "|---|---|---|---|---|---|---|---|"]
        for k, lst in rep.items():
            for i, v in enumerate(lst):
                rd = v.get("dram__bytes_read.sum", 0.0)
                wr = v.get("dram__bytes_write.sum", 0.0)
                t = v.get("gpu__time_duration.sum", 0.0)
                pct = v.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                            v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", float("nan")))
                lines.append(f"| `{k}` | {i} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {t * 1e6:.1f} | {pct:.1f} | "
                             f"{v.get('sm__warps_active.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                             f"{v.get('launch__registers_per_thread', float('nan')):.0f} |")
            rec = lst[-1]
            summary["kernels"][k] = {
                "launches_captured": len(lst),
                "dram_bytes_all_launches": sum(v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
                                               for v in lst),
                "dram_bytes_per_launch": rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0),
                "dram_read": rec.get("dram__bytes_read.sum"), "dram_write": rec.get("dram__bytes_write.sum"),
                "time_s_ncu": rec.get("gpu__time_duration.sum"), "tag": args.tag, "metrics": rec,
            }
        with open(os.path.join(PROF, f"ncu_{args.tag}_full.md"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        print("\n".join(lines))
    with open(summ_path, "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
