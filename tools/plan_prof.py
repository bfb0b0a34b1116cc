"""Build the sampled-index plans of one GPT2-2.5B sampled iteration (for ncu / timing).

    python tools/plan_prof.py [--reps R] [--full-idx]
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--full-idx", action="store_true")
    ap.add_argument("--ahead", action="store_true", help="side-stream packing (the tracker's prefetch)")
    args = ap.parse_args()
    import torch
    from paper_2511_10333_b200.engine import gpt2_shapes
    from paper_2511_10333_b200.entropy import sample_count, sample_plans
    from paper_2511_10333_b200.seeds import subsample_seed
    shapes = gpt2_shapes("2.5B", None)
    specs = [(m * n, sample_count(m * n, 0.25), subsample_seed(0, 10, k)) for k, (m, n) in enumerate(shapes)]
    ts, hs = [], []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        h0 = time.perf_counter()
        _, _, st = sample_plans(specs, bitmaps=True, indices=args.full_idx, check=False, ahead=args.ahead)
        hs.append((time.perf_counter() - h0) * 1e3)   # host enqueue time of the call
        b.record()
        torch.cuda.synchronize()
        assert int(st.max()) == 0
        ts.append(a.elapsed_time(b))
    print(json.dumps({"plan_ms": ts, "host_ms": hs, "steps": sum(c for _, c, _ in specs), "ahead": args.ahead,
                      "full_idx": args.full_idx}))


if __name__ == "__main__":
    main()
