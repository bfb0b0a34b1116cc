"""Config 1 through the reference's own per-matrix surface: compress / decompress of one
1024 x 4096 fp32 matrix at r = 4 (compressor.py:94-133), wall clock per call on the host
(incl. the raise-before-mutate finiteness check and its sync), and the device time of the
same compress in the grouped engine (CUDA events).

    python tools/api_probe.py [--m 1024] [--n 4096] [--rank 4] [--calls 50]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--rank", type=int, default=4)
    ap.add_argument("--calls", type=int, default=50)
    args = ap.parse_args()
    import statistics

    import torch

    import paper_2511_10333_b200 as e
    from paper_2511_10333_b200.calibrate import measure_compressor_gpu
    dev = torch.device("cuda", 0)
    g = torch.randn(args.m, args.n, device=dev) * 1e-2
    st = e.CompressorState(args.m, args.n, args.rank, rng_seed=0)
    for _ in range(3):
        e.decompress(e.compress(g, st))
    torch.cuda.synchronize()
    tc, td = [], []
    for _ in range(args.calls):
        t0 = time.perf_counter()
        f = e.compress(g, st)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        out = e.decompress(f)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        tc.append(t1 - t0)
        td.append(t2 - t1)
    sweep = measure_compressor_gpu(args.m, args.n, [args.rank], repeats=args.calls, device=dev)
    _ = out
    print(json.dumps({"shape": [args.m, args.n], "rank": args.rank,
                      "api_compress_us_median": statistics.median(tc) * 1e6,
                      "api_decompress_us_median": statistics.median(td) * 1e6,
                      "engine_device_compress_us": sweep[0][1] * 1e6,
                      "engine_device_decompress_us": sweep[0][2] * 1e6}))


if __name__ == "__main__":
    main()
