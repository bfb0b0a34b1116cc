"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Cases: the r <= 4 Z path (k_pass1t cluster kernel, with and without the fused sampled-iteration
statistics), the narrow and CUDA-core GEMM paths (r = 8, 16), the tcgen05 wide path (r = 32)
with the averaged reconstruction at W = 1, the sample plans (warp walk, set-mode and full-index
resolves, Floyd head table) and the FD histogram.  Exit 0 iff every result is finite.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import oracle
    from paper_2511_10333_b200.engine import BucketEngine
    from paper_2511_10333_b200.entropy import (EntropyTracker, SamplerConfig, histogram_fd, sample_count,
                                               sample_plans)
    dev = torch.device("cuda", 0)
    ok = True
    shapes = [(256, 1536), (512, 512), (96, 200)]
    for rank in (4, 8, 16, 32):
        eng = BucketEngine(shapes, rank=rank, seed=1)
        tr = EntropyTracker(SamplerConfig(alpha=0.5, beta=0.25), window=4) if rank == 4 else None
        for t in range(3):
            gs = [torch.from_numpy(oracle.synth_matrix(2, t, k, 0, m, n, 1e-2)).to(dev) for k, (m, n) in
                  enumerate(shapes)]
            for d, g in zip(eng.grads, gs):
                d.copy_(g)
            fused = tr.fused_request(t, eng, eng.grads) if tr is not None else None
            outs = eng.step()
            if tr is not None:
                tr.observe(t, eng.grads, fused=fused)
        torch.cuda.synchronize()
        eng.check_status()
        ok &= all(bool(torch.isfinite(o).all()) for o in outs)
        if tr is not None:
            tr.flush()
        print("engine rank", rank, "ok", flush=True)
    specs = [(n, sample_count(n, b), s) for n, b, s in [(200_000, 0.25, 3), (70_000, 0.5, 4), (100_000, 0.05, 5)]]
    for idx in (True, False):
        plans, bms, st = sample_plans(specs, dev, bitmaps=True, indices=idx)
        torch.cuda.synchronize()
        ok &= int(st.max()) == 0
        print("plans indices", idx, "ok", flush=True)
    c, e, h = histogram_fd(torch.randn(300_001, device=dev))
    ok &= bool(torch.isfinite(torch.tensor(h)))
    print("histogram ok", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
