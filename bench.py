"""EDGC data-parallel hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): EDGC grad GB/s — gradient bytes (4 B per fp32
element, all ranks) pushed through entropy + compress + exchange + decompress
per second, plus the fraction of the HBM roofline.  Workload (BASELINE.json
configs[1]): the GPT2-2.5B-shaped bucket set (52 layers x {QKV 1920x5760,
proj 1920x1920, fc1 1920x7680, fc2 7680x1920} = 208 matrices, 2.30e9 fp32
elements = 9.2 GB per GPU) at rank 4, GSR beta = 0.25, ISR alpha = 0.1
(entropy on every 10th iteration, as the reference's default SamplerConfig).

A step = (sampled iterations only) device entropy of the worker-0 raw
gradients [sampled indices -> fused gather + Gaussian plug-in], then the
bucket engine: grouped compress with error feedback, NCCL all-gather of the
packed factors (N > 1), averaged reconstruction.  Inputs are resident in HBM
and 9.2 GB per GPU >> the 126 MB L2, so no flush is needed between steps.
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  `e2e` repeats the step through the same public API
with the gradients copied in from pinned host memory and the averaged
gradients copied back every step.

`--impl reference` times the reference's CPU path (the oracle port: NumPy
float64 compress/decompress + Generator.choice + std, exactly the calls
train_toy makes) on the host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TF32_FALLBACK = 1100.0   # TFLOP/s dense, B200_PROFILING.md (used only if the measurement fails)
METRIC = "EDGC grad GB/s (entropy+compress+AR+decompress) @1/2/4/8 B200; % HBM roofline"
UNIT = "GB/s"
SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
REASON_NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=["2.5B", "12.1B"], default="2.5B")
    ap.add_argument("--layers", type=int, default=None, help="layers of the model shape set (default: all)")
    ap.add_argument("--rank", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=0.1)
    ap.add_argument("--beta", type=float, default=0.25)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--entropy", choices=["prefetch", "inline", "off"], default="prefetch",
                    help="diagnostics: entropy plans built ahead on a side stream (default), inline, or no tracker")
    ap.add_argument("--no-hi-prio", dest="hi_prio", action="store_false",
                    help="run the step on the default stream instead of a high-priority one (the entropy "
                         "tracker's plan kernels run on a low-priority side stream and yield SMs to the step)")
    ap.add_argument("--alias-output", action="store_true",
                    help="averaged gradients overwrite the raw ones (default for the 12.1B set, to fit in HBM)")
    ap.add_argument("--fuse-entropy", dest="fuse_entropy", action="store_true",
                    help="gather the sampled-iteration statistics inside pass 1 instead of a separate Gaussian "
                         "pass over the bitmaps (measured: the separate pass is cheaper -- 9.2 GB at ~HBM speed "
                         "vs +47%% instructions in pass 1)")
    ap.add_argument("--exchange", choices=["auto", "p2p", "nccl"], default="auto",
                    help="N > 1: read the peers' factors in place over NVLink (p2p, the default where the "
                         "reconstruction allows it) or all-gather them with NCCL first")
    ap.add_argument("--cpu-steps", type=int, default=6, help="EF steps in the bounded CPU sample")
    return ap.parse_args()


def load_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measure_tf32_peak(dev, n: int = 8192, reps: int = 10):
    """Dense TF32 tensor-core throughput measured here: cuBLAS fp32 GEMM with TF32 math, n^3.

    MEASURED_PEAKS.json carries HBM and bf16 figures only; the wide path's roofline is TF32.
    """
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(3):
            a @ b
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            a @ b
        e1.record()
        torch.cuda.synchronize(dev)
        tf = 2.0 * n ** 3 * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
        return tf, f"measured here: cuBLAS TF32 GEMM {n}^3, mean of {reps} back-to-back launches"
    except Exception as exc:   # pragma: no cover
        return TF32_FALLBACK, f"fallback (B200_PROFILING.md; measurement failed: {exc})"
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def load_traffic(kernel: str):
    """DRAM bytes of one step's launches of `kernel` (the roofline's unit) from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
        k = rec["kernels"][kernel]
        # one capture of all the phase's launches (pass 1 runs one launch per cluster width)
        return k.get("dram_bytes_all_launches", k["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
        self.proc = None
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(gpu_index)], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "nvidia-smi unavailable"}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons, n = [], None, set(), 0
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                n += 1
                for name, val in zip(REASON_NAMES, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": n}


# ----------------------------------------------------------------- CPU side

def cpu_reference_sample(shapes, rank, alpha, beta, seed, steps):
    """Time the reference's CPU path (oracle port) on one layer; returns (GB/s, detail)."""
    import numpy as np

    import oracle
    cores = len(os.sched_getaffinity(0))
    layer = shapes[:4]
    elems = sum(m * n for m, n in layer)
    grads = [oracle.synth_matrix(seed, 0, k, 0, m, n, 1e-2).astype(np.float64) for k, (m, n) in enumerate(layer)]
    seeds = oracle.state_seeds(seed, 1, len(layer))
    states = [[oracle.OracleState(m, n, min(rank, m, n), seeds[(0, k)]) for k, (m, n) in enumerate(layer)]]
    oracle.dp_step([grads], states)  # warm call (BLAS thread pool, page faults)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.dp_step([grads], states)
    t_step = (time.perf_counter() - t0) / steps
    # worker-0 entropy of one sampled iteration: NumPy Generator.choice + gather + std (entropy.py:67-90)
    t0 = time.perf_counter()
    for k, g in enumerate(grads):
        n_el = g.size
        cnt = oracle.sample_count(n_el, beta)
        sub = g.ravel() if cnt == n_el else g.ravel()[
            np.random.default_rng(oracle.subsample_seed(seed, 0, k)).choice(n_el, size=cnt, replace=False,
                                                                          shuffle=False)]
        oracle.gaussian_entropy(sub)
    t_ent = time.perf_counter() - t0
    per_step = t_step + alpha * t_ent
    gbs = 4.0 * elems / per_step / 1e9
    sample = (f"1 GPT-2 layer ({len(layer)} matrices, {elems / 1e6:.1f}M fp32 elements) of the bucket set: "
              f"{steps} error-feedback steps of compress+decompress (NumPy f64/OpenBLAS) at r={rank}, plus one "
              f"sampled-iteration entropy pass (Generator.choice + std, beta={beta}) weighted by alpha={alpha}; "
              f"{t_step * 1e3:.0f} ms/step + {t_ent * 1e3:.0f} ms/entropy pass")
    return gbs, {"cores": cores, "sample": sample, "t_step_s": t_step, "t_entropy_s": t_ent}


def run_reference(args):
    """The reference's CPU path (oracle port) for W + K steps, each a bounded sample of the workload:
    one GPT-2 layer (4 matrices) through train_toy's per-step calls -- compress -> decompress with
    error feedback (compressor.py:94-133) and, on every round(1/alpha)-th step, the worker-0 entropy
    of the layer (Generator.choice + std, entropy.py:67-90) -- timed per step on the host."""
    rank_env = int(os.environ.get("RANK", "0"))
    if rank_env != 0:
        return 0
    import numpy as np

    import oracle
    from paper_2511_10333_b200.engine import gpt2_shapes
    shapes = gpt2_shapes(args.model, args.layers)
    layer = shapes[:4]
    elems = sum(m * n for m, n in layer)
    cores = len(os.sched_getaffinity(0))
    grads = [oracle.synth_matrix(args.seed, 0, k, 0, m, n, 1e-2).astype(np.float64) for k, (m, n) in enumerate(layer)]
    seeds = oracle.state_seeds(args.seed, 1, len(layer))
    states = [[oracle.OracleState(m, n, min(args.rank, m, n), seeds[(0, k)]) for k, (m, n) in enumerate(layer)]]
    period = max(1, round(1.0 / args.alpha))

    def one_step(t):
        oracle.dp_step([grads], states)
        if t % period == 0:
            for k, g in enumerate(grads):
                cnt = oracle.sample_count(g.size, args.beta)
                sub = g.ravel() if cnt == g.size else g.ravel()[np.random.default_rng(
                    oracle.subsample_seed(args.seed, t, k)).choice(g.size, size=cnt, replace=False, shuffle=False)]
                oracle.gaussian_entropy(sub)

    for t in range(args.warmup):
        one_step(t)
    t0 = time.perf_counter()
    for t in range(args.warmup, args.warmup + args.steps):
        one_step(t)
    dt = time.perf_counter() - t0
    value = 4.0 * elems * args.steps / dt / 1e9
    sample = (f"each step: 1 GPT-2 layer ({len(layer)} matrices, {elems / 1e6:.1f}M fp64 elements) of the "
              f"{len(shapes)}-matrix set through compress+decompress with error feedback at r={args.rank} "
              f"(NumPy f64 / OpenBLAS), plus the layer's entropy (Generator.choice + std, beta={args.beta}) on "
              f"every {period}th step; {args.steps} timed steps after {args.warmup} warm-up steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, shapes),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference CPU path = oracle port (NumPy float64, OpenBLAS on all host cores; choice/MGS "
                "single-threaded as in NumPy); a step is the one-layer sample, so ms_per_step is measured, "
                "not extrapolated",
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, shapes):
    total = sum(m * n for m, n in shapes)
    return {"workload": f"GPT2-{args.model} bucket set: {len(shapes)} matrices, {total / 1e9:.3f}e9 fp32 "
                        f"elements ({4 * total / 1e9:.2f} GB) per GPU",
            "rank": args.rank, "alpha": args.alpha, "beta": args.beta, "estimator": "gaussian_plugin",
            "l2": "inputs 9.2 GB/GPU >> 126 MB L2 (no flush needed)" if args.model == "2.5B" and args.layers is None
            else "inputs larger than L2", "parallelism": f"dp{args.gpus}",
            "exchange": getattr(args, "exchange_eff", getattr(args, "exchange", "auto")) if args.gpus > 1
            else "none (1 rank)",
            "entropy_stats": "gathered in pass 1" if getattr(args, "fuse_entropy", True) else "separate Gaussian pass",
            "entropy_plans": {"prefetch": "side stream, built during the preceding iterations",
                              "inline": "built inside the sampled iteration", "off": "tracker disabled"}[args.entropy],
            "streams": "step on a high-priority stream, entropy plans on a low-priority side stream"
            if getattr(args, "hi_prio", True) else "step on the default stream"}


# ------------------------------------------------------------------ GPU side

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_10333_b200 import _lib
    from paper_2511_10333_b200.engine import BucketEngine, gpt2_shapes
    from paper_2511_10333_b200.entropy import EntropyTracker, SamplerConfig, sample_count

    world = int(os.environ.get("WORLD_SIZE", "1"))
    me = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    shapes = gpt2_shapes(args.model, args.layers)
    total = sum(m * n for m, n in shapes)
    alias = args.alias_output or args.model == "12.1B"
    eng = BucketEngine(shapes, rank=args.rank, seed=args.seed, world_size=world, rank_id=me, alias_output=alias,
                       exchange=args.exchange)
    if world > 1:
        args.exchange_eff = ("p2p: device-initiated pull of every rank's factors over NVLink (CUDA IPC, "
                             "device flags), no collective call" if eng._p2p else "nccl all_gather_into_tensor")
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + me)
    chunk = 1 << 28
    for a in range(0, total, chunk):
        b = min(total, a + chunk)
        eng.grad_arena[a:b].normal_(0.0, 1e-2, generator=gen)
    cfg = SamplerConfig(alpha=args.alpha, beta=args.beta, rng_seed=args.seed)
    tracker = None
    if me == 0 and args.entropy != "off":
        tracker = EntropyTracker(cfg, window=max(100, args.steps + args.warmup + 10),
                                 prefetch=args.entropy == "prefetch")
    if args.hi_prio:
        torch.cuda.set_stream(torch.cuda.Stream(dev, priority=-1))
    period = max(1, round(1.0 / args.alpha))
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def one_step(t, ev=None):
        marks = []
        # sampled iteration: pass 1 also gathers the Gaussian statistics of the sampled elements
        fused = tracker.fused_request(t, eng, eng.grads) if tracker is not None and args.fuse_entropy else None
        if ev is not None:
            marks = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
            marks[0].record(stream)
        eng.compress(_lib.PHASE_PASS1)
        if ev is not None:
            marks[1].record(stream)
        eng.compress(_lib.PHASE_FACTOR)
        if ev is not None:
            marks[2].record(stream)
        eng.compress(_lib.PHASE_PASS2 | _lib.PHASE_FINALIZE)
        if ev is not None:
            marks[3].record(stream)
        if tracker is not None:
            # train_toy order (grad_source.py:416): the tracker sees worker 0's raw gradients after
            # the step's compression -- before the reconstruction, which may overwrite them
            tracker.observe(t, eng.grads, fused=fused)   # non-sampled iterations only schedule the next plan
        if ev is not None:
            marks[4].record(stream)
            if t % period == 0:
                ev["ent"].append((marks[3], marks[4]))
        eng.exchange()
        if ev is not None:
            marks[5].record(stream)
        eng.reconstruct()
        if ev is not None:
            marks[6].record(stream)
            ev["marks"].append(marks)
        eng.advance()

    for t in range(args.warmup):
        one_step(t)
    eng.check_status()
    barrier()
    clocks = ClockSampler(local) if me == 0 else None
    launches0 = L.edgc_launch_count()
    ev = {"ent": [], "marks": []}
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    start.record(stream)
    for t in range(args.warmup, args.warmup + args.steps):
        one_step(t, ev)
    if tracker is not None and tracker._pf_stream is not None:
        # the plans prefetched for the next sampled iteration belong to the timed steps: each
        # period of round(1/alpha) steps carries one plan build, so the window must contain the
        # build launched inside it (the one before the window finished during warm-up)
        stream.wait_stream(tracker._pf_stream)
    stop.record(stream)
    barrier()
    launches = L.edgc_launch_count() - launches0
    clk = clocks.stop() if clocks is not None else None
    eng.check_status()
    elapsed = start.elapsed_time(stop) / 1e3
    t_max = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_all = float(t_max.item())
    value = world * 4.0 * total * args.steps / t_all / 1e9
    # per-phase device times (ms, mean over timed steps)
    names = ["pass1", "factor", "pass2_finalize", "entropy", "exchange", "reconstruct"]
    ph = {n: 0.0 for n in names}
    for mk in ev["marks"]:
        for i, n in enumerate(names):
            ph[n] += mk[i].elapsed_time(mk[i + 1]) / len(ev["marks"])
    # sampled vs other steps (timed step t = warmup + i): pass 1 and whole-step device time
    starts_all = [mk[0] for mk in ev["marks"]] + [stop]
    samp = {"pass1": [], "step": []}
    rest = {"pass1": [], "step": []}
    for i, mk in enumerate(ev["marks"]):
        dst = samp if (args.warmup + i) % period == 0 else rest
        dst["pass1"].append(mk[0].elapsed_time(mk[1]))
        dst["step"].append(starts_all[i].elapsed_time(starts_all[i + 1]))
    ph["sampled_steps_ms"] = {k: statistics.mean(v) for k, v in samp.items() if v}
    ph["other_steps_ms"] = {k: statistics.mean(v) for k, v in rest.items() if v}
    ent_ms = [a.elapsed_time(b) for a, b in ev["ent"]]
    ph["entropy_per_sampled_step"] = statistics.mean(ent_ms) if ent_ms else 0.0
    ph["entropy_sampled_steps"] = len(ent_ms)
    starts = [mk[0] for mk in ev["marks"]] + [stop]
    step_ms = sorted(a.elapsed_time(b) for a, b in zip(starts[:-1], starts[1:]))
    ph["step_ms"] = {"min": step_ms[0], "median": statistics.median(step_ms), "max": step_ms[-1]}
    peak, peak_src = load_peak()
    # dominant kernel: pass 1 (error feedback + P = W Q): reads g and w, writes w: 12 B per element
    alg_bytes = {"pass1": 12.0 * total, "pass2_finalize": 4.0 * total, "reconstruct": 4.0 * total}
    dom = max(alg_bytes, key=lambda k: ph[k])
    dom_ms = ph[dom]
    achieved = alg_bytes[dom] / (dom_ms / 1e3) / 1e9
    # the committed ncu capture is of the r <= 4 kernels (k_pass1t / k_pass2 / k_recon4)
    traffic = (load_traffic({"pass1": "k_pass1t", "pass2_finalize": "k_pass2", "reconstruct": "k_recon4"}[dom])
               if args.rank <= 4 else None)
    tensor = None
    # ranks up to 32 run on CUDA cores (HBM roofline above); the tcgen05 path above 32, or above
    # 16 with EDGC_SKEF32=0
    tc_min = 16 if os.environ.get("EDGC_SKEF32", "1") == "0" else 32
    if args.rank > tc_min:
        # wide path on tcgen05 (3xTF32: three MMAs per product): the bound is the tensor pipe.
        # tensor FLOP per phase: pass 1 = EF update (2 N r_res) + P_raw (2 N r); pass 2 = Q (2 N r);
        # reconstruct = 2 N (W r); x3 for the hi/lo split
        tfl = {"pass1": 3 * 4.0 * total * args.rank, "pass2_finalize": 3 * 2.0 * total * args.rank,
               "reconstruct": 3 * 2.0 * total * args.rank * world}
        tdom = max(tfl, key=lambda k: ph[k])
        tf32_peak, tf32_src = measure_tf32_peak(dev)
        tensor = {"bound": "tensor", "kernel": tdom, "achieved": tfl[tdom] / (ph[tdom] / 1e3) / 1e12,
                  "peak": tf32_peak, "unit": "TFLOP/s", "frac": tfl[tdom] / (ph[tdom] / 1e3) / 1e12 / tf32_peak,
                  "traffic": None, "flop_per_launch": tfl[tdom], "peak_source": tf32_src,
                  "flop_accounting": "tensor-core FLOP incl. the 3xTF32 split (3 MMAs per fp32 product)"}
    n_sampled = len(ent_ms)
    ent_bytes = 4.0 * sum(sample_count(m * n, args.beta) for m, n in shapes) * n_sampled / max(1, args.steps)
    step_frac = (16.0 * total + ent_bytes) / (t_all / args.steps) / 1e9 / peak
    line = None
    if me == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_all / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, shapes),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes[dom], "peak_source": peak_src,
                         "step_hbm_frac": step_frac,
                         "step_alg_bytes": "16 B/elem (read g, read e, write e', write out) + 4 B/sample on "
                                           "sampled iterations (SURVEY.md 8(d))"},
            "phases_ms": ph,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if tensor is not None:
            tensor["hbm"] = line["roofline"]
            line["roofline"] = tensor
    # ---------------------------------------------------------------- e2e
    # Every step copies its gradients in from pinned host memory and its averaged gradients
    # back out.  PCIe is full duplex, so the copies are pipelined across steps on two copy
    # streams: step t+1's H2D and step t's D2H overlap step t's compute (device staging
    # buffers decouple them from the engine's arenas at the cost of two device copies).
    if not args.no_e2e:
        ke = max(1, args.e2e_steps)
        host_g = torch.empty(total, dtype=torch.float32, pin_memory=True)
        host_out = torch.empty(total, dtype=torch.float32, pin_memory=True)
        host_g.copy_(eng.grad_arena)
        dev_in = torch.empty(total, dtype=torch.float32, device=dev)
        dev_out = torch.empty(total, dtype=torch.float32, device=dev)
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = args.warmup + args.steps
        s0.record(stream)
        h2d_s.wait_event(s0)
        with torch.cuda.stream(h2d_s):
            dev_in.copy_(host_g, non_blocking=True)
        in_ready = ev()
        in_ready.record(h2d_s)
        out_free = None
        for t in range(t0, t0 + ke):
            stream.wait_event(in_ready)
            eng.grad_arena.copy_(dev_in)                  # this step's inputs, now on the device
            in_free = ev()
            in_free.record(stream)
            if t + 1 < t0 + ke:                           # next step's H2D overlaps this step
                h2d_s.wait_event(in_free)
                with torch.cuda.stream(h2d_s):
                    dev_in.copy_(host_g, non_blocking=True)
                in_ready = ev()
                in_ready.record(h2d_s)
            fused = tracker.fused_request(t, eng, eng.grads) if tracker is not None and args.fuse_entropy else None
            eng.compress()
            if tracker is not None:
                tracker.observe(t, eng.grads, fused=fused)
            eng.exchange()
            eng.reconstruct()
            eng.advance()
            if out_free is not None:
                stream.wait_event(out_free)
            dev_out.copy_(eng.out_arena)
            out_ready = ev()
            out_ready.record(stream)
            d2h_s.wait_event(out_ready)                   # this step's D2H overlaps the next step
            with torch.cuda.stream(d2h_s):
                host_out.copy_(dev_out, non_blocking=True)
            out_free = ev()
            out_free.record(d2h_s)
        stream.wait_event(out_free)
        s1.record(stream)
        barrier()
        te = torch.tensor([s0.elapsed_time(s1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        if line is not None:
            line["e2e"] = {"value": world * 4.0 * total * ke / float(te.item()) / 1e9, "unit": UNIT,
                           "h2d_bytes_per_step": 4 * total, "d2h_bytes_per_step": 4 * total, "steps": ke,
                           "path": "BucketEngine.step with every step's gradients H2D from pinned host memory and "
                                   "its averaged gradients D2H, the copies pipelined across steps on two copy "
                                   "streams (PCIe full duplex)"}
        del host_g, host_out, dev_in, dev_out
    # ------------------------------------------------------- CPU baseline
    if line is not None and world == 1 and not args.no_cpu_baseline:
        v, det = cpu_reference_sample(shapes, args.rank, args.alpha, args.beta, args.seed, args.cpu_steps)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": det["cores"], "kind": "port",
                                "sample": det["sample"]}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    _ = np
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
