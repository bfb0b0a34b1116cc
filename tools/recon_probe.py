"""Time the averaged reconstruction (1/W) sum_w P_w Q_w^T of the GPT2-2.5B set on ONE GPU
for W = 1, 2, 4, 8 ranks' worth of (random) gathered factors -- the multi-GPU step's
reconstruction without the collective, so it can be profiled in a single process.

    python tools/recon_probe.py [--rank 4] [--iters 10]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=4)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    import torch
    from paper_2511_10333_b200 import _lib
    from paper_2511_10333_b200.engine import _Plan, gpt2_shapes
    dev = torch.device("cuda", 0)
    shapes = gpt2_shapes("2.5B", None)
    r = args.rank
    total = sum(m * n for m, n in shapes)
    out_arena = torch.empty(total, dtype=torch.float32, device=dev)
    outs, o = [], 0
    for m, n in shapes:
        outs.append(out_arena[o:o + m * n].view(m, n))
        o += m * n
    res = {}
    for W in [int(x) for x in args.worlds.split(",")]:
        size = sum(r * (m + n) for m, n in shapes)   # packed [P_k | Q_k] per rank
        fac = torch.randn(W * size, dtype=torch.float32, device=dev) * 1e-2
        descs, off = [], 0
        for (m, n), out in zip(shapes, outs):
            descs.append(_lib.ReconDesc(_lib.ptr(fac[off:]), _lib.ptr(fac[off + m * r:]), _lib.ptr(out), m, n, n,
                                        size, size, r, W, 1.0 / W, 0))
            off += r * (m + n)
        plan = _Plan("recon", descs, dev)
        st = torch.cuda.current_stream(dev)
        for _ in range(3):
            plan.run(st.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.iters):
            plan.run(st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        res[W] = {"ms": round(ms, 3), "write_TBps": round(4 * total / ms / 1e9, 3),
                  "TFLOPs": round(2 * W * r * total / ms / 1e9, 1)}
        del plan, fac
    print(json.dumps({"rank": r, "recon": res}))


if __name__ == "__main__":
    main()
