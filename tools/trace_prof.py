"""Where analyze_trace's per-frame time goes (replay / tracker / full histograms / correlations)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10333_b200 import trace as tr
from paper_2511_10333_b200.entropy import EntropyTracker, SamplerConfig, entropy_histogram, histogram_fd

SHAPES = [(1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920)]
rng = np.random.default_rng(0)
f0 = [rng.standard_normal(s, dtype=np.float32) for s in SHAPES]
path = "/tmp/p.edgt"
tr.write_trace(path, ([f * np.float32(0.97 ** t) for f in f0] for t in range(8)))
def clock(name, fn, reps=2):
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(f"{name}: {1e3*(time.perf_counter()-t0)/8:.1f} ms/frame", flush=True)
for readers in (4, 1):
    tr._READERS = readers
    clock(f"replay readers={readers}", lambda: [None for _ in tr.replay_trace(path)])
tr._READERS = 4
def tracker_only():
    t = EntropyTracker(SamplerConfig(alpha=1.0, beta=0.25), 8, estimator=entropy_histogram)
    for i, m in enumerate(tr.replay_trace(path)):
        t.observe(i, m)
clock("replay+tracker(hist)", tracker_only)
def hists():
    for m in tr.replay_trace(path):
        for x in m:
            c, e, _ = histogram_fd(x.data); c.cpu().tolist(); e.cpu().tolist()
clock("replay+full hist", hists)
def corr():
    for m in tr.replay_trace(path):
        tr.layer_correlations(m)
clock("replay+corr(all frames)", corr)
clock("analyze", lambda: tr.analyze_trace(path, alpha=1.0, window=8, correlation_iterations=4))
