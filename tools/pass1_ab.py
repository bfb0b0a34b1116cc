"""Time the compress phases of the GPT2-2.5B bucket set for one library build.

    EDGC_LIB_PATH=alt_libs/x.so python tools/pass1_ab.py [--layers L] [--iters N]

Prints one JSON line: mean device ms per phase (CUDA events, after warm-up).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rank", type=int, default=4)
    args = ap.parse_args()
    import torch
    from paper_2511_10333_b200 import _lib
    from paper_2511_10333_b200.engine import BucketEngine, gpt2_shapes
    shapes = gpt2_shapes("2.5B", args.layers)
    eng = BucketEngine(shapes, rank=args.rank, seed=0)
    eng.grad_arena.normal_(0.0, 1e-2)
    st = torch.cuda.current_stream()
    phases = [("pass1", _lib.PHASE_PASS1), ("factor", _lib.PHASE_FACTOR),
              ("pass2_finalize", _lib.PHASE_PASS2 | _lib.PHASE_FINALIZE)]
    tot = {k: 0.0 for k, _ in phases}
    tot["reconstruct"] = 0.0
    for it in range(args.iters + 3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(st)
        for i, (_, ph) in enumerate(phases):
            eng.compress(ph)
            ev[i + 1].record(st)
        eng.exchange()
        eng.reconstruct()
        ev[4].record(st)
        eng.advance()
        torch.cuda.synchronize()
        if it >= 3:
            for i, (k, _) in enumerate(phases):
                tot[k] += ev[i].elapsed_time(ev[i + 1]) / args.iters
            tot["reconstruct"] += ev[3].elapsed_time(ev[4]) / args.iters
    eng.check_status()
    total = sum(m * n for m, n in shapes)
    print(json.dumps({"lib": os.environ.get("EDGC_LIB_PATH", "in-tree"), "elems": total,
                      "ms": {k: round(v, 3) for k, v in tot.items()},
                      "pass1_TBps": round(12 * total / tot["pass1"] / 1e9, 3)}))


if __name__ == "__main__":
    main()
