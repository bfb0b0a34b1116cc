"""Top CUDA source lines of one kernel in an ncu report, by executed warp instructions and stall samples.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = next(x for x in r if "Instructions Executed" in x)
    start = r.index(h) + 1
    f = lambda v: float(v.replace(",", "")) if v not in ("-", "") else 0.0
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    src, seen = [], set()
    for x in r[start:]:
        if len(x) != len(h) or x[0] == "" or x[0] == "Line No":
            continue
        if x[0] in seen:   # one launch only
            break
        seen.add(x[0])
        src.append(x)
    tot, tots = sum(f(x[ie]) for x in src), sum(f(x[ws]) for x in src)
    print(f"{kern}: {tot:.3g} warp instructions, {tots:.0f} stall samples")
    for x in sorted(src, key=lambda x: -f(x[ws]))[:n]:
        print(f"{x[0]:>5} {int(f(x[ie])):>12} {int(f(x[ws])):>7}  {x[1][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
