"""Throughput of EDGT replay + device analyze-trace on a GPT2-2.5B-layer-shaped trace.

One frame = one GPT-2 2.5B layer (QKV 1920x5760, proj 1920x1920, fc1 1920x7680,
fc2 7680x1920; 44.2M fp32 = 177 MB).  Reports
  replay GB/s   : file -> pinned chunks -> HBM (replay_trace alone, page cache warm)
  analyze GB/s  : analyze_trace (histogram estimator, alpha=1 so every frame is
                  FD-histogrammed per layer, correlations on 4 iterations)
  cpu GB/s      : the reference's per-frame work in NumPy (np.histogram(bins="fd")
                  per layer of one frame: cli.py:631-635), 1 thread, as a baseline
Usage: python tools/trace_bench.py [--iters 8] [--dir /tmp]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10333_b200.trace import analyze_trace, replay_trace, write_trace  # noqa: E402

SHAPES = [(1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    frame0 = [rng.standard_normal(s, dtype=np.float32) for s in SHAPES]
    path = os.path.join(a.dir, "bench.edgt")
    write_trace(path, ([(f * np.float32(0.97 ** t)) for f in frame0] for t in range(a.iters)))
    frame_bytes = sum(m * n for m, n in SHAPES) * 4
    total = frame_bytes * a.iters
    for _ in range(2):  # warm page cache + allocator
        for _ in replay_trace(path):
            pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in replay_trace(path):
        pass
    torch.cuda.synchronize()
    t_replay = time.perf_counter() - t0
    for _ in range(2):  # the first call pays plan-workspace allocation
        t0 = time.perf_counter()
        res = analyze_trace(path, estimator="histogram", alpha=1.0, window=a.iters, correlation_iterations=4)
        torch.cuda.synchronize()
        t_an = time.perf_counter() - t0
    from paper_2511_10333_b200.entropy import histogram_fd
    dev = [torch.from_numpy(f).cuda() for f in frame0]
    hist_ms = []
    for d in dev:
        histogram_fd(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        histogram_fd(d)
        hist_ms.append(1e3 * (time.perf_counter() - t0))
    t0 = time.perf_counter()
    for f in frame0:
        np.histogram(f.astype(np.float64).ravel(), bins="fd")
    t_cpu = time.perf_counter() - t0
    print(json.dumps({"workload": "EDGT trace of GPT2-2.5B layer frames", "frame_bytes": frame_bytes,
                      "iterations": a.iters, "replay_gbs": total / t_replay / 1e9,
                      "analyze_gbs": total / t_an / 1e9, "analyze_ms_per_frame": 1e3 * t_an / a.iters,
                      "device_hist_ms_per_layer": hist_ms, "cpu_hist_gbs": frame_bytes / t_cpu / 1e9, "cpu_cores": 1,
                      "hist_rows": len(res.histograms), "corr_rows": len(res.correlations)}))
    os.remove(path)


if __name__ == "__main__":
    main()
