"""Multi-GPU parity check of the DP exchange (run under torchrun, one process per GPU).

Every rank runs BucketEngine with NCCL; each step rank 0 compares the averaged
reconstruction with the reference's sequential W-worker DP step
(grad_source.py:389-408, restated in oracle.dp_step) computed from the same
per-worker gradients and seeds.  Chained over a few steps at a rank well below
min(m, n).  Prints one JSON line on rank 0; exit code 0 iff within tolerance.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2511_10333_b200.engine import BucketEngine  # noqa: E402

SHAPES = [(192, 576), (192, 192), (192, 768), (768, 192), (50, 70)]


def main():
    world = int(os.environ["WORLD_SIZE"])
    me = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", me))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, steps = 4, 4
    eng = BucketEngine(SHAPES, rank=rank, seed=0, world_size=world, rank_id=me)
    seeds = oracle.state_seeds(0, world, len(SHAPES))
    ost = [[oracle.OracleState(m, n, min(rank, m, n), seeds[(w, k)]) for k, (m, n) in enumerate(SHAPES)]
           for w in range(world)] if me == 0 else None
    worst = 0.0
    for t in range(steps):
        mine = [oracle.synth_matrix(3, t, k, me, m, n, 1e-2) for k, (m, n) in enumerate(SHAPES)]
        outs = eng.step([torch.from_numpy(g).to(dev) for g in mine], check=True)
        if me == 0:
            allg = [[oracle.synth_matrix(3, t, k, w, m, n, 1e-2).astype(np.float64) for k, (m, n) in enumerate(SHAPES)]
                    for w in range(world)]
            ref = oracle.dp_step(allg, ost)
            for o, r in zip(outs, ref):
                worst = max(worst, float(np.linalg.norm(o.cpu().numpy() - r) / np.linalg.norm(r)))
    # every rank must hold the same average
    probe = eng.out_arena[:4096].clone()
    gathered = [torch.empty_like(probe) for _ in range(world)]
    dist.all_gather(gathered, probe)
    same = all(torch.equal(gathered[0], g) for g in gathered)
    ok = True
    if me == 0:
        ok = worst <= 5e-5 and same
        print(json.dumps({"world": world, "worst_rel_err": worst, "ranks_identical": same, "ok": ok}), flush=True)
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
