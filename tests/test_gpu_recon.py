"""GPU: the averaged reconstruction (1/W) sum_w P_w Q_w^T (grad_source.py:404-408) through
the recon plan C-ABI, for W*r from 4 to 32 (the float4 kernels), W*r = 64 with r % 32 != 0
(tiled CUDA-core kernel) and the tensor-core cases (W*r > 32 with W = 1 or r % 32 == 0:
3xTF32, fp32 accumulation in 128-K chunks), against a plain torch fp64 reference of the
same packed factor layout."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,r", [(1, 4), (2, 4), (4, 4), (8, 4), (4, 16), (2, 3), (1, 48), (2, 32), (4, 64), (2, 36)])
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
        tc = W * r > 32 and r % 4 == 0 and (W == 1 or r % 32 == 0)
        assert err <= (4e-6 if tc else 1e-6), (W, r, m, n, err)
        off += r * (m + n)
