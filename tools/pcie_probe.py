"""PCIe copy bandwidth on the box: pinned host <-> HBM, one direction at a time and both at
once (full duplex), for the e2e leg's 9.2 GB per step and direction.

    python tools/pcie_probe.py [--gb 4]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    a = ap.parse_args()
    n = int(a.gb * 1e9 / 4)
    dev = torch.device("cuda", 0)
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float32, device=dev)
    d_out = torch.ones(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}

    def timed(fn, reps=3):
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 4.0 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        return best

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    res["h2d_GBps"] = round(timed(h2d), 1)
    res["d2h_GBps"] = round(timed(d2h), 1)
    res["duplex_GBps_per_direction"] = round(timed(both), 1)
    res["gb"] = a.gb
    print(json.dumps(res))


if __name__ == "__main__":
    main()
