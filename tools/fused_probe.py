"""Pass 1 with and without the fused sampled-iteration statistics on a few GPT2-2.5B layers
(alpha = 0.5: every other step is sampled), for ncu:

    ncu -k regex:k_pass1t ... python tools/fused_probe.py --layers 4
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    import torch

    from paper_2511_10333_b200.engine import BucketEngine, gpt2_shapes
    from paper_2511_10333_b200.entropy import EntropyTracker, SamplerConfig
    shapes = gpt2_shapes("2.5B", args.layers)
    eng = BucketEngine(shapes, rank=4, seed=0)
    eng.grad_arena.normal_(0.0, 1e-2)
    tr = EntropyTracker(SamplerConfig(alpha=0.5, beta=0.25), window=100)
    for t in range(args.steps):
        fused = tr.fused_request(t, eng, eng.grads)
        eng.compress()
        tr.observe(t, eng.grads, fused=fused)
        eng.reconstruct()
        eng.advance()
    torch.cuda.synchronize()
    eng.check_status()


if __name__ == "__main__":
    main()
