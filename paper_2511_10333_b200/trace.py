"""EDGT gradient traces streamed to the device, and the GPU ``analyze-trace`` pass.

SURVEY.md §8(f) row 3.  The on-disk format is the reference's
(pkg/src/edgc/grad_source.py:44-131): a little-endian header ``<4sHHIH``
(magic ``EDGT``, version 1, layer count, iteration count, element width 4),
``(m, n)`` u32 pairs, then one fp32 row-major frame per iteration.  Header
validation and its error messages follow ``read_trace_header``
(grad_source.py:82-117) so ``TraceFormatError`` matches the reference's tests.

What changes is the replay: ``replay_trace`` reads the frames sequentially into
a ring of pinned host chunks on a reader thread (``readinto`` releases the GIL)
and copies each chunk to HBM on a dedicated copy stream, so the file read, the
PCIe transfer and the consumer's kernels on frame t overlap.  The consumer's
stream waits on the frame's copy event; nothing synchronises the host except
the finiteness check each ``GradientMatrix`` performs in the reference too
(done once per frame here, grad_source.py:129 -> matrix_core.py:36-46).

``analyze_trace`` is ``cmd_analyze_trace`` (cli.py:600-659) as a library call:
the entropy tracker over the replayed frames, FD histograms of every layer on
sampled iterations through the device histogram kernel (bit-exact counts and
edges), and Pearson correlations of equal-size layers as one fp64 Gram matrix
per size group.
"""

from __future__ import annotations

import csv
import os
import queue
import struct
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from .entropy import (EntropyTracker, SamplerConfig, entropy_gaussian_plugin, entropy_histogram, histogram_fd,
                      should_sample_iteration, write_window_csv)
from .errors import ConfigError, DegenerateInputError, TraceFormatError
from .matrix_core import GradientMatrix, _device, any_nonfinite

__all__ = ["TRACE_MAGIC", "TRACE_VERSION", "write_trace", "read_trace_header", "replay_trace",
           "TraceAnalysis", "analyze_trace", "layer_correlations"]

TRACE_MAGIC = b"EDGT"
TRACE_VERSION = 1
_HEADER = struct.Struct("<4sHHIH")
_DIMS = struct.Struct("<II")
_ELEMENT_WIDTH = 4
_CHUNK_BYTES = 64 << 20
_SLOTS = 3
_READERS = 4


def _host_array(mat) -> np.ndarray:
    if isinstance(mat, GradientMatrix):
        mat = mat.data
    if isinstance(mat, torch.Tensor):
        return mat.detach().to("cpu").numpy()
    return np.asarray(mat)


def write_trace(path, iterations) -> int:
    """Serialise per-iteration lists of matrices as fp32 frames; returns the iteration count.

    Accepts GradientMatrix, torch tensors (device or host) and array-likes.  Every
    iteration must carry the first iteration's layer shapes (grad_source.py:51-74).
    """
    shapes = None
    count = 0
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(TRACE_MAGIC, TRACE_VERSION, 0, 0, _ELEMENT_WIDTH))  # patched below
        for mats in iterations:
            arrays = [_host_array(m) for m in mats]
            if shapes is None:
                shapes = [a.shape for a in arrays]
                if not shapes:
                    raise ValueError("iterations must contain at least one layer")
                for a in arrays:
                    if a.ndim != 2:
                        raise ValueError(f"expected 2-D matrices, got shape {a.shape}")
                for m, n in shapes:
                    fh.write(_DIMS.pack(m, n))
            if [a.shape for a in arrays] != shapes:
                raise ValueError("layer shapes changed between iterations")
            for a in arrays:
                fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes(order="C"))
            count += 1
        fh.seek(0)
        fh.write(_HEADER.pack(TRACE_MAGIC, TRACE_VERSION, len(shapes or []), count, _ELEMENT_WIDTH))
    return count


def read_trace_header(path) -> tuple[int, list[tuple[int, int]]]:
    """(iteration_count, layer shapes) with the full length check of grad_source.py:82-117."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        if len(head) < _HEADER.size:
            raise TraceFormatError(f"truncated header: need {_HEADER.size} bytes, file has {len(head)}")
        magic, version, layers, iterations, width = _HEADER.unpack(head)
        if magic != TRACE_MAGIC:
            raise TraceFormatError(f"bad magic {magic!r} at byte 0, expected {TRACE_MAGIC!r}")
        if version != TRACE_VERSION:
            raise TraceFormatError(f"unsupported version {version}, expected {TRACE_VERSION}")
        if width != _ELEMENT_WIDTH:
            raise TraceFormatError(f"unsupported element width {width}, expected {_ELEMENT_WIDTH}")
        table = fh.read(_DIMS.size * layers)
        if len(table) < _DIMS.size * layers:
            raise TraceFormatError(f"truncated layer table at byte {_HEADER.size}: need "
                                   f"{_DIMS.size * layers} bytes, got {len(table)}")
    shapes = [_DIMS.unpack_from(table, k * _DIMS.size) for k in range(layers)]
    for m, n in shapes:
        if m < 1 or n < 1:
            raise TraceFormatError(f"non-positive layer dimensions {(m, n)}")
    expected = _HEADER.size + _DIMS.size * layers + iterations * _frame_bytes(shapes)
    if size < expected:
        raise TraceFormatError(f"file length {size} != expected {expected} ({expected - size} bytes missing)")
    if size > expected:
        raise TraceFormatError(f"file length {size} != expected {expected} ({size - expected} trailing bytes)")
    return iterations, shapes


def _frame_bytes(shapes) -> int:
    return sum(m * n for m, n in shapes) * _ELEMENT_WIDTH


def _pread_full(fd: int, view, offset: int) -> None:
    got = 0
    while got < len(view):
        k = os.preadv(fd, [view[got:]], offset + got)
        if not k:
            raise TraceFormatError(f"trace ended early at byte {offset + got}")
        got += k


class _ChunkReader(threading.Thread):
    """Fills pinned host slots with consecutive file chunks; hands (slot, nbytes) over a queue."""

    def __init__(self, path, offset: int, frame: int, frames: int, slots):
        super().__init__(daemon=True)
        self.path, self.offset, self.frame, self.frames, self.slots = path, offset, frame, frames, slots
        self.free = queue.Queue()
        self.ready = queue.Queue()
        self.stop = threading.Event()
        for s in range(len(slots)):
            self.free.put(s)

    def run(self) -> None:
        try:
            fd = os.open(self.path, os.O_RDONLY)
            try:
                with ThreadPoolExecutor(_READERS) as pool:
                    pos, left, in_frame = self.offset, self.frame * self.frames, self.frame
                    while left > 0 and not self.stop.is_set():
                        sid = self.free.get()
                        if sid is None:
                            return
                        want = min(in_frame, self.slots[sid].numel())  # chunks never straddle frames
                        view = memoryview(self.slots[sid].numpy())
                        # page-cache -> pinned memcpy split over _READERS threads (pread releases the GIL)
                        step = -(-want // _READERS)
                        parts = [(o, min(step, want - o)) for o in range(0, want, step)]
                        for f in [pool.submit(_pread_full, fd, view[o:o + k], pos + o) for o, k in parts]:
                            f.result()
                        pos += want
                        left -= want
                        in_frame = in_frame - want or self.frame
                        self.ready.put((sid, want))
            finally:
                os.close(fd)
        except BaseException as exc:  # handed to the consumer
            self.ready.put((None, exc))

    def take(self):
        sid, val = self.ready.get()
        if sid is None:
            raise val
        return sid, val

    def close(self) -> None:
        self.stop.set()
        self.free.put(None)


def replay_trace(path, device=None):
    """Yield each iteration's layers as device ``GradientMatrix`` objects (grad_source.py:120-131).

    Each frame lands in its own fp32 HBM buffer (the matrices stay valid after the
    next frame is yielded, as the reference's arrays do); the caller's current
    stream is ordered after the frame's copy.  Memory: one frame on the device
    per live iteration plus ``_SLOTS`` pinned chunks of at most 64 MiB.
    """
    iterations, shapes = read_trace_header(path)
    if iterations == 0:
        return
    dev = torch.device(device) if device is not None else _device()
    frame = _frame_bytes(shapes)
    header = _HEADER.size + _DIMS.size * len(shapes)
    chunk = min(_CHUNK_BYTES, frame)
    chunk -= chunk % _ELEMENT_WIDTH
    slots = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(_SLOTS)]
    reader = _ChunkReader(path, header, frame, iterations, slots)
    reader.start()
    copy_stream = torch.cuda.Stream(device=dev)
    pending = []  # (event, slot) whose H2D copy may still read the slot
    try:
        for t in range(iterations):
            buf = torch.empty(frame, dtype=torch.uint8, device=dev)
            off = 0
            while off < frame:
                sid, nbytes = reader.take()
                with torch.cuda.stream(copy_stream):
                    buf[off:off + nbytes].copy_(slots[sid][:nbytes], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy_stream)
                pending.append((ev, sid))
                off += nbytes
                while pending and (len(pending) >= _SLOTS - 1 or pending[0][0].query()):
                    done, s = pending.pop(0)
                    done.synchronize()
                    reader.free.put(s)
            torch.cuda.current_stream(dev).wait_stream(copy_stream)
            flat = buf.view(torch.float32)
            if any_nonfinite(flat):
                raise ValueError(f"iteration {t}: gradient matrix contains non-finite entries")
            mats, pos = [], 0
            for k, (m, n) in enumerate(shapes):
                mats.append(GradientMatrix.trusted(flat[pos:pos + m * n].view(m, n), layer_id=k, iteration=t))
                pos += m * n
            yield mats
    finally:
        reader.close()
        for ev, _ in pending:
            ev.synchronize()


def layer_correlations(mats) -> list[tuple[int, int, float]]:
    """Pearson rho for every ordered pair of equal-size layers (cli.py:636-642, matrix_core.py:83-100).

    Layers of one element count are centred and stacked into a k x N fp64 matrix
    X; rho_ij = (X X^T)_ij / (N s_i s_j), clamped to [-1, 1], one GEMM per group.
    Row order (i outer, j inner over all layers, skipping size mismatches) is the
    reference's.
    """
    datas = [(m.data if isinstance(m, GradientMatrix) else m).reshape(-1) for m in mats]
    groups: dict[int, list[int]] = {}
    for i, d in enumerate(datas):
        groups.setdefault(d.numel(), []).append(i)
    rho = {}
    for size, idx in groups.items():
        x = torch.stack([datas[i].double() for i in idx])
        x = x - x.mean(dim=1, keepdim=True)
        s = torch.sqrt((x * x).mean(dim=1))
        if bool((s == 0).any()):
            raise DegenerateInputError("zero-variance input to correlation")
        g = (x @ x.T) / (size * s[:, None] * s[None, :])
        g = g.clamp(-1.0, 1.0).cpu().tolist()
        for a, i in enumerate(idx):
            for b, j in enumerate(idx):
                rho[(i, j)] = g[a][b]
    return [(i, j, rho[(i, j)]) for i in range(len(datas)) for j in range(len(datas)) if (i, j) in rho]


@dataclass
class TraceAnalysis:
    iterations: int
    shapes: list
    windows: list = field(default_factory=list)
    histograms: list = field(default_factory=list)    # (iteration, layer, bin_left, bin_right, count)
    correlations: list = field(default_factory=list)  # (iteration, layer_i, layer_j, pearson)


def _correlation_iterations(want, iterations: int) -> list[int]:
    if isinstance(want, int):
        count = min(want, iterations) if iterations else 0
        return sorted({round(i * (iterations - 1) / max(1, count - 1)) for i in range(count)}) if count else []
    return sorted({int(i) for i in want})


def _write_csv(path, header, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(header)
        for row in rows:
            w.writerow([repr(float(v)) if isinstance(v, float) else v for v in row])


def analyze_trace(path, *, estimator: str = "histogram", alpha: float = 0.1, beta: float = 0.25, seed: int = 0,
                  window: int = 100, correlation_iterations=4, output_dir=None, device=None) -> TraceAnalysis:
    """``cmd_analyze_trace`` (cli.py:579-659) on the device; defaults are ANALYZE_DEFAULTS (cli.py:579-587).

    With ``output_dir`` the three CSVs are written byte-for-byte in the reference's
    layout (entropy_windows.csv, gradient_histograms.csv, layer_correlations.csv).
    """
    iterations, shapes = read_trace_header(path)
    est = {"histogram": entropy_histogram, "gaussian": entropy_gaussian_plugin}.get(estimator)
    if est is None:
        raise ConfigError(f"unknown estimator {estimator!r}")
    sampler = SamplerConfig(alpha=float(alpha), beta=float(beta), rng_seed=seed)
    tracker = EntropyTracker(sampler, int(window), estimator=est)
    corr_iters = set(_correlation_iterations(correlation_iterations, iterations))
    out = TraceAnalysis(iterations, shapes)
    for t, mats in enumerate(replay_trace(path, device)):
        tracker.observe(t, mats)
        if should_sample_iteration(t, sampler.alpha):
            for k, mat in enumerate(mats):
                counts, edges, _ = histogram_fd(mat.data)
                c = counts.cpu().tolist()
                e = edges.cpu().tolist()
                out.histograms.extend((t, k, e[j], e[j + 1], c[j]) for j in range(len(c)))
        if t in corr_iters:
            out.correlations.extend((t, i, j, rho) for i, j, rho in layer_correlations(mats))
    tracker.flush()
    out.windows = list(tracker.windows)
    if output_dir is not None:
        os.makedirs(output_dir, exist_ok=True)
        write_window_csv(os.path.join(output_dir, "entropy_windows.csv"), out.windows)
        _write_csv(os.path.join(output_dir, "gradient_histograms.csv"),
                   ["iteration", "layer", "bin_left", "bin_right", "count"], out.histograms)
        _write_csv(os.path.join(output_dir, "layer_correlations.csv"),
                   ["iteration", "layer_i", "layer_j", "pearson"], out.correlations)
    return out
