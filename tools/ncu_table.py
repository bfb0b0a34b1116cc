"""Markdown table of selected metrics from an ncu report (run here after a gpurun).

    python tools/ncu_table.py gpurun_out/x.ncu-rep > profiles/x.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("ms", "gpu__time_duration.sum", 1e-6),
    ("DRAM read GB", "dram__bytes_read.sum", 1e-9),
    ("DRAM write GB", "dram__bytes_write.sum", 1e-9),
    ("tensor pipe active %", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {}
    for i, h in enumerate(hdr):   # some metrics carry a section prefix ("TPC.TriageCompute.<name>")
        idx.setdefault(h, i)
        idx.setdefault(h.split(".", 2)[-1] if h.count(".") >= 3 and h.split(".")[0].isupper() else h, i)
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---|" + "---|" * len(METRICS))
    for r in data:
        name = r[idx["Kernel Name"]]
        name = name.split("(")[0].split("::")[-1] if "k_tc" not in name else name.split("unnamed>::")[-1].split(">")[0]
        vals = []
        for _, key, scale in METRICS:
            v = r[idx[key]] if key in idx else ""
            try:
                x = float(v.replace(",", "")) * scale
                unit = units[idx[key]]
                if key == "gpu__time_duration.sum" and unit == "ms":
                    x = float(v.replace(",", ""))
                elif key == "gpu__time_duration.sum" and unit == "us":
                    x = float(v.replace(",", "")) / 1e3
                if key.startswith("dram__bytes") and unit in ("Gbyte", "GB"):
                    x = float(v.replace(",", ""))
                elif key.startswith("dram__bytes") and unit in ("Mbyte", "MB"):
                    x = float(v.replace(",", "")) / 1e3
                vals.append(f"{x:.3g}" if x < 100 else f"{x:.0f}")
            except ValueError:
                vals.append(v or "-")
        print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
