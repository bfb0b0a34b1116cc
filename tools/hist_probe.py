"""One FD histogram of a full 1920x7680 fp32 layer (ncu target for the histogram kernels)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10333_b200.entropy import histogram_fd
x = torch.from_numpy(np.random.default_rng(0).standard_normal((1920, 7680), dtype=np.float32)).cuda()
for _ in range(3):
    c, e, h = histogram_fd(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    histogram_fd(x)
print(f"histogram_fd 1920x7680: {1e3 * (time.perf_counter() - t0) / 20:.3f} ms/call (host-synchronising API), nb={c.numel()}")
