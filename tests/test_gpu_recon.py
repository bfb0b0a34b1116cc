"""GPU: the averaged reconstruction (1/W) sum_w P_w Q_w^T (grad_source.py:404-408) through
the recon plan C-ABI, for W*r from 4 to 32 (the float4 kernels), W*r = 64 with 4 ∤ r
(tiled CUDA-core kernel) and the tensor-core cases (W*r >= EDGC_TC_RECON_MIN with 4 | r:
3xTF32, fp32 accumulation in 128-K chunks; at W > 1 the K index concatenates the ranks'
r-wide blocks), against a plain torch fp64 reference of the same packed factor layout."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TC_RECON_MIN = int(os.environ.get("EDGC_TC_RECON_MIN", "33"))


@pytest.mark.parametrize("W,r", [(1, 4), (2, 4), (4, 4), (8, 4), (4, 16), (2, 3), (1, 48), (2, 32), (4, 64), (2, 36),
                                 (2, 34), (8, 8)])
def test_reconstruction_matches_fp64(W, r):
    from paper_2511_10333_b200 import _lib
    from paper_2511_10333_b200.engine import _Plan
    dev = torch.device("cuda", 0)
    shapes = [(192, 576), (640, 128), (70, 52), (1024, 1920)]
    size = sum(r * (m + n) for m, n in shapes)
    g = torch.Generator(device=dev)
    g.manual_seed(W * 100 + r)
    fac = torch.randn(W * size, dtype=torch.float32, device=dev, generator=g)
    outs = [torch.empty(m, n, dtype=torch.float32, device=dev) for m, n in shapes]
    descs, off = [], 0
    for (m, n), o in zip(shapes, outs):
        descs.append(_lib.ReconDesc(_lib.ptr(fac[off:]), _lib.ptr(fac[off + m * r:]), _lib.ptr(o), m, n, n,
                                    size, size, r, W, 1.0 / W, 0))
        off += r * (m + n)
    plan = _Plan("recon", descs, dev)
    plan.run(torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize()
    off = 0
    for (m, n), o in zip(shapes, outs):
        ref = torch.zeros(m, n, dtype=torch.float64, device=dev)
        for w in range(W):
            base = w * size + off
            P = fac[base:base + m * r].view(m, r).double()
            Q = fac[base + m * r:base + r * (m + n)].view(n, r).double()
            ref += P @ Q.T
        ref /= W
        err = float((o.double() - ref).norm() / ref.norm())
        # fp32 FMA kernels: 1e-6; tensor cores (3xTF32, ~1e-6 from the split and the
        # chunked fp32 accumulation): 4e-6
        tc = W * r >= TC_RECON_MIN and r % 4 == 0
        assert err <= (4e-6 if tc else 1e-6), (W, r, m, n, err)
        off += r * (m + n)


@pytest.mark.parametrize("W,r", [(4, 4), (8, 4), (2, 8), (3, 4)])
def test_narrow_rank_blocks_on_tensor_cores(W, r):
    """W r = 12..32 forced onto the tensor cores (EDGC_TC_RECON_MIN=8): K shorter than one
    32-wide block and rank blocks of 4 or 8 columns per 32-wide K block."""
    env = dict(os.environ, EDGC_TC_RECON_MIN="8")
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); "
            f"from tests.test_gpu_recon import test_reconstruction_matches_fp64 as t; t({W}, {r})")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
