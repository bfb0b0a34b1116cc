"""Time the sampled iteration's Gaussian pass (edgc_entropy_gaussian over the membership bitmaps)
on the GPT2-2.5B bucket set, plans built once beforehand.

    [EDGC_LIB_PATH=alt_libs/x.so] python tools/gauss_probe.py [--iters 10]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2511_10333_b200.engine import BucketEngine, gpt2_shapes
    from paper_2511_10333_b200.entropy import SamplerConfig, _gaussian_launch, _layer_specs, sample_plans
    shapes = gpt2_shapes("2.5B", None)
    eng = BucketEngine(shapes, rank=4, seed=0)
    eng.grad_arena.normal_(0.0, 1e-2)
    flats = [g.reshape(-1) for g in eng.grads]
    cfg = SamplerConfig(alpha=0.1, beta=0.25, rng_seed=0)
    specs = _layer_specs(flats, 10, cfg)
    dev = flats[0].device
    plans, bms, status = sample_plans(specs, dev, bitmaps=True, check=False, indices=False)
    items = [(f, p, c, bm) for f, p, bm, (_, c, _) in zip(flats, plans, bms, specs)]
    ts = []
    for it in range(args.iters + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h, hstat = _gaussian_launch(items, 0, dev)
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b))
    total = sum(f.numel() for f in flats)
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"lib": os.environ.get("EDGC_LIB_PATH", "in-tree"), "gauss_ms_median": round(ms, 4),
                      "TBps": round(4 * total / ms / 1e9, 3), "h0": float(h[0])}))


if __name__ == "__main__":
    main()
