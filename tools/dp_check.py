"""Multi-GPU parity check of the DP exchange (run under torchrun, one process per GPU).

Every rank runs the device path with NCCL; rank 0 compares against the
reference's sequential W-worker DP step (grad_source.py:389-408, restated in
oracle.dp_step) computed from the same per-worker gradients and basis seeds
(grad_source.py:440-447).  Cases:

* ``engine_*``: BucketEngine chained over a few steps at r well below
  min(m, n): r = 4 (CUDA-core reconstruction; the factors gathered by the
  device-initiated NVLink pull, and the same through NCCL), r = 8, r = 32
  (W r >= 64: the rank-blocked tcgen05 reconstruction), r = 128 (tcgen05
  compress + recon), and one full GPT2-2.5B layer per rank at r = 4;
* ``driver``: EdgcDataParallel through warm-up (uncompressed NCCL average) into
  the active phase, with the window decisions broadcast from rank 0 only on
  window-close iterations.  The rank history must equal the LIVE reference's
  (tests/golden/dp.json: worker-0 entropies -> controller), and every step's
  average must match the oracle's DP step from the ranks' own states
  (re-synced each step: the driver's r_max ~ 0.85 min(m, n) amplifies fp32
  rounding in the error-feedback iteration, see tests/test_gpu_debug_rank.py).

Prints one JSON line per case on rank 0 (also appended to --out) and exits 0
iff every case is within tolerance.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2511_10333_b200.engine import GPT2_2P5B_LAYER, BucketEngine  # noqa: E402

SMALL = [(192, 576), (192, 192), (192, 768), (768, 192), (50, 70)]
MID = [(256, 768), (256, 256), (256, 1024), (1024, 256)]
WIDE = [(1024, 3072), (1024, 1024), (1024, 4096), (4096, 1024)]

CASES = {
    "engine_r4": dict(shapes=SMALL, rank=4, steps=4, tol=5e-5),
    "engine_r4_nccl": dict(shapes=SMALL, rank=4, steps=4, tol=5e-5, exchange="nccl"),
    "engine_r8_p2p": dict(shapes=MID, rank=8, steps=4, tol=5e-5, exchange="p2p"),
    "engine_r4_graph": dict(shapes=MID, rank=4, steps=5, tol=5e-5, graph=True),
    "engine_r32": dict(shapes=MID, rank=32, steps=4, tol=5e-5),
    "engine_r128": dict(shapes=WIDE, rank=128, steps=3, tol=5e-5),
    "engine_gpt2_layer_r4": dict(shapes=list(GPT2_2P5B_LAYER), rank=4, steps=2, tol=5e-5),
}
DRIVER_TOL = 1e-4


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def gather_np(t, world):
    """All ranks' copies of a device tensor, as float64 NumPy arrays on every rank (rank order)."""
    t = t.contiguous()
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.double().cpu().numpy() for o in out]


def engine_case(name, spec, world, me, dev):
    shapes, rank, steps = spec["shapes"], spec["rank"], spec["steps"]
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    eng = BucketEngine(shapes, rank=rank, seed=0, world_size=world, rank_id=me,
                       exchange=spec.get("exchange", "auto"))
    seeds = oracle.state_seeds(0, world, len(shapes))
    ost = [[oracle.OracleState(m, n, min(rank, m, n), seeds[(w, k)]) for k, (m, n) in enumerate(shapes)]
           for w in range(world)] if me == 0 else None
    worst = 0.0
    for t in range(steps):
        mine = [oracle.synth_matrix(3, t, k, me, m, n, 1e-2) for k, (m, n) in enumerate(shapes)]
        if spec.get("graph") and t >= 1:
            # the steady-state step as CUDA graphs (compress, NVLink exchange, reconstruction)
            if t == 1:
                eng.capture_graphs()
            for dst, g in zip(eng.grads, mine):
                dst.copy_(torch.from_numpy(g))
            outs = eng.graph_step(check=True)
        else:
            outs = eng.step([torch.from_numpy(g).to(dev) for g in mine], check=True)
        if me == 0:
            allg = [[oracle.synth_matrix(3, t, k, w, m, n, 1e-2).astype(np.float64) for k, (m, n) in
                     enumerate(shapes)] for w in range(world)]
            ref = oracle.dp_step(allg, ost)
            for o, r in zip(outs, ref):
                worst = max(worst, rel(o.double().cpu().numpy(), r))
    copies = gather_np(eng.out_arena[:1 << 16].clone(), world)  # every rank must hold the same average
    same = all(np.array_equal(c, copies[0]) for c in copies)
    mode = "p2p" if eng._p2p else "nccl"
    rec = {"case": name, "world": world, "rank": rank, "shapes": [list(s) for s in shapes], "steps": steps,
           "exchange": mode, "worst_rel_err": worst, "tol": spec["tol"], "ranks_identical": same,
           "recon_rank": world * rank, "wall_s": round(time.perf_counter() - t0, 2)}
    rec["ok"] = bool(worst <= spec["tol"] and same) if me == 0 else None
    return rec


def driver_case(world, me, dev):
    from paper_2511_10333_b200.controller import PHASE_ACTIVE
    from paper_2511_10333_b200.dp import EdgcDataParallel
    from paper_2511_10333_b200.entropy import SamplerConfig
    from tests.golden.specs import DP_SCENARIO, dp_scenario_grads
    from tests.helpers import load_json
    sc = DP_SCENARIO
    shapes = [tuple(s) for s in sc["shapes"]]
    gold = load_json("dp.json")["driver"]
    t0 = time.perf_counter()
    dp = EdgcDataParallel(shapes, total_iterations=sc["iters"], seed=0, world_size=world, rank_id=me,
                          sampler=SamplerConfig(sc["alpha"], sc["beta"], 0), window=sc["window"])
    eng = dp.engine
    seeds = oracle.state_seeds(0, world, len(shapes))
    ost = None
    worst, where, warm_worst, active_steps = 0.0, None, 0.0, 0
    for t in range(sc["iters"]):
        active = dp.ctl.phase == PHASE_ACTIVE
        if active:
            # every rank's state, re-synced into the oracle's per-worker states
            res = [gather_np(eng.residual(k), world) for k in range(len(shapes))]
            qw = [gather_np(eng.q_warm[k][:, :eng.ranks[k]], world) for k in range(len(shapes))]
            if me == 0:
                if ost is None:
                    ost = [[oracle.OracleState(m, n, eng.ranks[k], seeds[(w, k)]) for k, (m, n) in
                            enumerate(shapes)] for w in range(world)]
                for w in range(world):
                    for k, st in enumerate(ost[w]):
                        st.residual, st.q_warm, st.rank = res[k][w], qw[k][w].copy(), eng.ranks[k]
        outs = dp.step(t, [torch.from_numpy(g).to(dev) for g in dp_scenario_grads(t, me)])
        if me == 0:
            allg = [[g.astype(np.float64) for g in dp_scenario_grads(t, w)] for w in range(world)]
            if active:
                ref = oracle.dp_step(allg, ost)
                active_steps += 1
            else:
                ref = [sum(allg[w][k] for w in range(world)) / world for k in range(len(shapes))]
            for k, (o, r) in enumerate(zip(outs, ref)):
                e = rel(o.double().cpu().numpy(), r)
                if active and e > worst:
                    worst, where = e, (t, k, list(eng.ranks))
                if not active:
                    warm_worst = max(warm_worst, e)
    dp.flush()
    dp.check_status()
    hist = [None if d.ranks is None else d.ranks[0] for d in dp.rank_history] if me == 0 else None
    rank_t = torch.tensor(eng.ranks, dtype=torch.int64, device=dev)
    g = [torch.empty_like(rank_t) for _ in range(world)]
    dist.all_gather(g, rank_t)
    ranks_all = [x.tolist() for x in g]
    rec = {"case": "driver", "world": world, "shapes": [list(s) for s in shapes], "iters": sc["iters"],
           "window": sc["window"], "active_steps": active_steps, "rank_history": hist,
           "reference_history": gold["history"], "worst_rel_err_active": worst, "where": where,
           "worst_rel_err_warmup": warm_worst, "tol": DRIVER_TOL, "final_ranks_all_ranks": ranks_all,
           "wall_s": round(time.perf_counter() - t0, 2)}
    if me == 0:
        rec["ok"] = bool(hist == gold["history"] and worst <= DRIVER_TOL and warm_worst <= 1e-6
                         and all(r == ranks_all[0] for r in ranks_all) and active_steps > 0)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(list(CASES) + ["driver"]))
    ap.add_argument("--out", default=None, help="append the JSON lines here (rank 0)")
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    me = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", me))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ok = True
    for name in args.cases.split(","):
        rec = driver_case(world, me, dev) if name == "driver" else engine_case(name, CASES[name], world, me, dev)
        if me == 0:
            ok &= bool(rec["ok"])
            line = json.dumps(rec)
            print(line, flush=True)
            if args.out:
                with open(args.out, "a") as fh:
                    fh.write(line + "\n")
        dist.barrier(device_ids=[local])
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    if me == 0:
        print(json.dumps({"world": world, "ok": bool(flag.item())}), flush=True)
    return 0 if flag.item() else 1


if __name__ == "__main__":
    sys.exit(main())
