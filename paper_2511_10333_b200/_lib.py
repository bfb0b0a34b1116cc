"""ctypes binding of libedgc_b200.so (include/edgc_b200.h).

The CUDA library is the only compute path: if it cannot be loaded, or no CUDA
device is present, every device operation raises ``RuntimeError`` — there is
no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import DegenerateInputError

HERE = os.path.dirname(os.path.abspath(__file__))
# EDGC_LIB_PATH selects an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("EDGC_LIB_PATH", os.path.join(HERE, "libedgc_b200.so"))

EDGC_OK = 0
EDGC_EINVAL = 1
EDGC_ENONFINITE = 2
EDGC_EDEGENERATE = 3
EDGC_ECUDA = 4
EDGC_ETOOMANYBINS = 6
EDGC_ECAPACITY = 7
EDGC_EDRAWS = 8

PHASE_PASS1, PHASE_FACTOR, PHASE_PASS2, PHASE_FINALIZE, PHASE_ALL = 1, 2, 4, 8, 15
PLAN_BITMAP_ONLY = 1
PLAN_LATENCY = 2

c_i32, c_i64, c_u64, c_f32, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float,
                                           ctypes.c_double, ctypes.c_void_p)


class PlanDesc(ctypes.Structure):
    _fields_ = [("state_hi", c_u64), ("state_lo", c_u64), ("inc_hi", c_u64), ("inc_lo", c_u64),
                ("n_elems", c_i64), ("count", c_i64), ("idx", c_vp), ("bitmap", c_vp),
                ("flags", c_i64)]


class GaussDesc(ctypes.Structure):
    _fields_ = [("src", c_vp), ("idx", c_vp), ("count", c_i64), ("bitmap", c_vp), ("n_elems", c_i64)]


class SampleDesc(ctypes.Structure):
    _fields_ = [("bitmap", c_vp), ("first", c_vp)]


class CompressDesc(ctypes.Structure):
    _fields_ = [("g", c_vp), ("w", c_vp), ("p_res", c_vp), ("q_res", c_vp), ("q_warm", c_vp), ("basis", c_vp),
                ("p_out", c_vp), ("q_out", c_vp), ("precond", c_vp), ("m", c_i64), ("n", c_i64), ("ld_g", c_i64),
                ("r", c_i32), ("r_res", c_i32), ("ld_q", c_i32), ("ld_s", c_i32)]


class ReconDesc(ctypes.Structure):
    _fields_ = [("p", c_vp), ("q", c_vp), ("out", c_vp), ("m", c_i64), ("n", c_i64), ("ld_out", c_i64),
                ("p_rank_stride", c_i64), ("q_rank_stride", c_i64), ("r", c_i32), ("n_ranks", c_i32),
                ("scale", c_f32), ("pad_", c_i32)]


# name -> (restype, argtypes); must match include/edgc_b200.h
SIGNATURES = {
    "edgc_abi_version": (c_i32, []),
    "edgc_last_error": (ctypes.c_char_p, []),
    "edgc_launch_count": (c_i64, []),
    "edgc_sample_plan_workspace_bytes": (c_i64, [ctypes.POINTER(PlanDesc), c_i32]),
    "edgc_sample_plan": (c_i32, [ctypes.POINTER(PlanDesc), c_i32, c_vp, c_vp, c_i64, c_vp]),
    "edgc_gather": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "edgc_entropy_gaussian_workspace_bytes": (c_i64, [ctypes.POINTER(GaussDesc), c_i32]),
    "edgc_entropy_gaussian": (c_i32, [c_i32, ctypes.POINTER(GaussDesc), c_i32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "edgc_entropy_histogram_workspace_bytes": (c_i64, [c_i64]),
    "edgc_entropy_histogram": (c_i32, [c_i32, c_vp, c_i64, c_f64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_i64, c_vp]),
    "edgc_compress_plan_create": (c_i32, [ctypes.POINTER(CompressDesc), c_i32, ctypes.POINTER(c_vp)]),
    "edgc_compress_plan_workspace_bytes": (c_i64, [c_vp]),
    "edgc_compress_plan_bind": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "edgc_compress_plan_run": (c_i32, [c_vp, c_f64, c_vp, c_i32, c_vp]),
    "edgc_compress_plan_sample_slots": (c_i64, [c_vp]),
    "edgc_compress_plan_set_sampling": (c_i32, [c_vp, ctypes.POINTER(SampleDesc), c_i32, c_vp, c_vp]),
    "edgc_entropy_gaussian_partials": (c_i32, [c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "edgc_compress_plan_destroy": (None, [c_vp]),
    "edgc_compress_workspace_bytes": (c_i64, [ctypes.POINTER(CompressDesc), c_i32]),
    "edgc_compress": (c_i32, [ctypes.POINTER(CompressDesc), c_i32, c_f64, c_vp, c_vp, c_i64, c_vp]),
    "edgc_recon_plan_create": (c_i32, [ctypes.POINTER(ReconDesc), c_i32, ctypes.POINTER(c_vp)]),
    "edgc_recon_plan_workspace_bytes": (c_i64, [c_vp]),
    "edgc_recon_plan_bind": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "edgc_recon_plan_run": (c_i32, [c_vp, c_vp]),
    "edgc_recon_plan_destroy": (None, [c_vp]),
    "edgc_p2p_pull": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "edgc_p2p_signal": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "edgc_ipc_handle": (c_i32, [c_vp, c_vp, c_vp]),
    "edgc_ipc_open": (c_i32, [c_vp, c_vp]),
    "edgc_ipc_close": (c_i32, [c_vp]),
    "edgc_reconstruct_workspace_bytes": (c_i64, [ctypes.POINTER(ReconDesc), c_i32]),
    "edgc_reconstruct": (c_i32, [ctypes.POINTER(ReconDesc), c_i32, c_vp, c_i64, c_vp]),
    "edgc_residual": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp, c_vp]),
    "edgc_check_work_finite": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp, c_vp]),
    "edgc_check_finite": (c_i32, [c_i32, c_vp, c_i64, c_vp, c_vp]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_2511_10333_b200._build` "
                    "(this package has no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.edgc_abi_version() != 1:
                raise RuntimeError("libedgc_b200.so ABI version mismatch")
            _lib = lib
    return _lib


def lib():
    """The library, after checking that a CUDA device is present."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_10333_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc == EDGC_OK:
        return
    msg = (_lib.edgc_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    text = f"{what}: {msg}" if what else msg
    if rc == EDGC_EINVAL:
        raise ValueError(text)
    raise RuntimeError(f"libedgc_b200 status {rc}: {text}")


def raise_device_status(code: int, what: str) -> None:
    """Map a device-side status word onto the reference's exception types."""
    if code == EDGC_OK:
        return
    if code == EDGC_EDEGENERATE:
        raise DegenerateInputError(what)
    if code in (EDGC_EINVAL, EDGC_ENONFINITE, EDGC_ETOOMANYBINS):
        raise ValueError(what)
    raise RuntimeError(f"{what} (device status {code})")


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class Workspace:
    """Per-device scratch buffer, grown on demand (never shrunk)."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, device=None) -> torch.Tensor:
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
        buf = self._bufs.get(dev)
        if buf is None or buf.numel() < nbytes:
            # the old buffer may still be in use by queued kernels on this stream;
            # the caching allocator keeps it alive until the stream reaches here
            buf = torch.empty(max(int(nbytes * 1.25), 1 << 20), dtype=torch.uint8, device=dev)
            self._bufs[dev] = buf
        return buf


WORKSPACE = Workspace()
