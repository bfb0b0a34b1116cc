"""Gradient down-sampling (GDS) and entropy estimation on the device.

Mirrors pkg/src/edgc/entropy.py name for name.  What runs where:

* iteration gate, window bookkeeping, per-iteration layer mean: host Python,
  identical arithmetic to the reference (entropy.py:53-64, 110-121, 158-192);
* sampler seeds and PCG64 words: host NumPy (seeds.py);
* sampled indices (NumPy ``Generator.choice`` rule), gather, Gaussian plug-in
  and FD-histogram estimators: libedgc_b200.so kernels.  Indices and
  histogram counts are bit-exact with the reference; entropies agree to fp64
  reduction order (<1e-12 nats).
"""

from __future__ import annotations

import csv
import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DegenerateInputError
from .matrix_core import as_device_array, as_device_matrix
from .seeds import pcg64_words_many, subsample_seeds

__all__ = ["GAUSSIAN_ENTROPY_CONST", "SamplerConfig", "EntropyWindow", "should_sample_iteration",
           "sampling_period", "sample_count", "sample_indices", "sample_plans", "subsample_entries",
           "entropy_gaussian_plugin", "entropy_histogram", "histogram_fd", "close_window",
           "relative_change_rate", "EntropyTracker", "write_window_csv"]

GAUSSIAN_ENTROPY_CONST = 0.5 * math.log(2.0 * math.pi * math.e)



_WS_CAP = {}


_PF_AFTER_STEP = os.environ.get("EDGC_PF_AFTER_STEP") is not None


def _plan_ws_cap(device) -> int:
    """Workspace cap of one edgc_sample_plan call: a quarter of the HBM free at first use, at most
    16 GiB (>= 2 GiB).

    All plans of a batch walk concurrently (one CTA each), so fewer, larger
    batches are faster; bucket sets beyond the cap are planned in several calls.
    Cached per device (cudaMemGetInfo must not run inside a timed step).
    """
    key = torch.device(device).index
    if key not in _WS_CAP:
        free, _ = torch.cuda.mem_get_info(device)
        # the workspace pool keeps its high-water mark: 16 GiB holds the whole GPT2-2.5B set's
        # plans (one batch) and leaves the rest of HBM to the compressor at 12.1B scale
        _WS_CAP[key] = max(2 << 30, min(free // 4, 16 << 30))
    return _WS_CAP[key]


@dataclass(frozen=True)
class SamplerConfig:
    """Iteration-level rate alpha and element-level rate beta, both in (0, 1]."""

    alpha: float = 0.1
    beta: float = 0.25
    rng_seed: int = 0

    def __post_init__(self) -> None:
        for name in ("alpha", "beta"):
            v = getattr(self, name)
            if not 0.0 < v <= 1.0:
                raise ValueError(f"{name} must be in (0, 1], got {v}")


@dataclass
class EntropyWindow:
    window_index: int
    window_size: int
    mean_entropy: float
    samples_used: int
    per_iteration_entropies: list = field(default_factory=list)


def sampling_period(alpha: float) -> int:
    return max(1, round(1.0 / alpha))


def should_sample_iteration(iteration: int, alpha: float) -> bool:
    """True on every round(1/alpha)-th iteration (Python's banker's rounding, as the reference)."""
    if iteration < 0:
        raise ValueError(f"iteration must be non-negative, got {iteration}")
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must be in (0, 1], got {alpha}")
    return iteration % sampling_period(alpha) == 0


def sample_count(n_elems: int, beta: float) -> int:
    return min(n_elems, math.ceil(beta * n_elems))


def sample_plans(specs, device=None, *, bitmaps: bool = False, stream=None, workspace=None, check: bool = True,
                 indices: bool = True, ahead: bool = False):
    """Device index plans for many (n_elems, count, seed) at once.

    Returns a list of int32 CUDA tensors (None where count == n_elems, i.e. the
    reference's full copy).  Order of each plan = NumPy's output order.  With
    ``bitmaps=True`` returns (plans, bitmaps, status): per-plan int32 words with
    bit e set iff element e is sampled.  ``stream`` / ``workspace`` let the
    tracker build the next sampled iteration's plans on a side stream;
    ``check=False`` skips the synchronising status check (the caller checks
    ``status`` later).  ``indices=False`` (with ``bitmaps``) builds only the
    membership sets: each returned index tensor then holds one sampled
    element (the Gaussian estimator's shift; see EDGC_PLAN_BITMAP_ONLY).
    ``ahead=True``: the plans are built ahead of use on a side stream, so the
    sequential walk is packed onto few SMs; otherwise (EDGC_PLAN_LATENCY) it is
    spread over all of them, as the result is waited for.
    """
    if not indices and not bitmaps:
        raise ValueError("indices=False needs bitmaps=True")
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    st = torch.cuda.current_stream(dev) if stream is None else stream
    ws_pool = _lib.WORKSPACE if workspace is None else workspace
    out = [None] * len(specs)
    bms = [None] * len(specs)
    todo = []
    with torch.cuda.stream(st):
        for i, (n_elems, count, seed) in enumerate(specs):
            if count == n_elems:
                continue
            if n_elems >= 2**31:
                raise ValueError(f"sampling over {n_elems} >= 2^31 elements is outside the device plan's range")
            todo.append(i)
        # one index buffer and one (zeroed) bitmap buffer for all plans: two allocations and one
        # fill instead of one per plan; slices start on 256-byte boundaries
        pad = lambda x: (x + 63) // 64 * 64
        n_out = (lambda c: c) if indices else (lambda c: 1)
        o_all = torch.empty(max(1, sum(pad(n_out(specs[i][1])) for i in todo)), dtype=torch.int32, device=dev)
        b_all = (torch.zeros(max(1, sum(pad((specs[i][0] + 31) // 32) for i in todo)), dtype=torch.int32, device=dev)
                 if bitmaps else None)
        oo = bo = 0
        for i in todo:
            n_elems, count, _ = specs[i]
            out[i] = o_all[oo:oo + n_out(count)]
            oo += pad(n_out(count))
            if bitmaps:
                words = (n_elems + 31) // 32
                bms[i] = b_all[bo:bo + words]
                bo += pad(words)
        cap_bytes = _plan_ws_cap(dev)
        descs, sizes = {}, {}
        words = dict(zip(todo, pcg64_words_many([specs[i][2] for i in todo])))
        for i in todo:
            n_elems, count, seed = specs[i]
            descs[i] = _lib.PlanDesc(*words[i], n_elems, count, _lib.ptr(out[i]), _lib.ptr(bms[i]),
                                     (0 if indices else _lib.PLAN_BITMAP_ONLY) |
                                     (0 if ahead else _lib.PLAN_LATENCY))
            sizes[i] = L.edgc_sample_plan_workspace_bytes((_lib.PlanDesc * 1)(descs[i]), 1) + 4096
        status_all = torch.zeros(max(1, len(todo)), dtype=torch.int32, device=dev)
        k = 0
        while k < len(todo):
            batch, acc = [], 0
            while k < len(todo) and (not batch or acc + sizes[todo[k]] <= cap_bytes):
                batch.append(descs[todo[k]])
                acc += sizes[todo[k]]
                k += 1
            arr = (_lib.PlanDesc * len(batch))(*batch)
            need = L.edgc_sample_plan_workspace_bytes(arr, len(batch))
            if need < 0:
                _lib.check(_lib.EDGC_EINVAL, "sample plan layout")
            ws = ws_pool.get(need, dev)
            status = status_all[k - len(batch):k]
            _lib.check(L.edgc_sample_plan(arr, len(batch), _lib.ptr(status), _lib.ptr(ws), ws.numel(),
                                          st.cuda_stream), "edgc_sample_plan")
    if check and todo:
        _raise_plan_status(status_all)
    if bitmaps:
        return out, bms, status_all
    return out


def _raise_plan_status(status) -> None:
    code = int(status.max().item())
    if code == 0:
        return
    if code & _lib.EDGC_EDRAWS:
        raise RuntimeError("sample plan exhausted its pre-generated draws")
    raise RuntimeError(f"sample plan failed on the device (status {code})")


def sample_indices(n_elems: int, beta: float, seed: int, device=None) -> torch.Tensor:
    """The int64 flat indices subsample_entries draws (entropy.py:75-78), on the device."""
    if not 0.0 < beta <= 1.0:
        raise ValueError(f"beta must be in (0, 1], got {beta}")
    count = sample_count(n_elems, beta)
    plan = sample_plans([(n_elems, count, seed)], device)[0]
    if plan is None:
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        return torch.arange(n_elems, dtype=torch.int64, device=dev)
    return plan.to(torch.int64)


def subsample_entries(matrix, beta: float, seed: int) -> torch.Tensor:
    """ceil(beta*m*n) row-major entries without replacement, NumPy's order (entropy.py:67-79).

    Returns a float64 CUDA tensor (values are the fp32 device entries, exactly).
    """
    if not 0.0 < beta <= 1.0:
        raise ValueError(f"beta must be in (0, 1], got {beta}")
    flat = as_device_matrix(matrix).reshape(-1)
    count = sample_count(flat.numel(), beta)
    if count == flat.numel():
        return flat.to(torch.float64)
    idx = sample_plans([(flat.numel(), count, seed)], flat.device)[0]
    out = torch.empty(count, dtype=torch.float64, device=flat.device)
    L = _lib.lib()
    _lib.check(L.edgc_gather(0, _lib.ptr(flat), _lib.ptr(idx), count, 1, _lib.ptr(out), _lib.stream_ptr()),
               "edgc_gather")
    return out


def _samples_tensor(samples) -> torch.Tensor:
    if isinstance(samples, torch.Tensor) and samples.is_cuda and samples.dtype in (torch.float32, torch.float64):
        return samples.reshape(-1).contiguous()
    return as_device_array(np.asarray(samples, dtype=np.float64).ravel()
                           if not isinstance(samples, torch.Tensor) else samples.double().reshape(-1),
                           torch.float64)


def _dtype_code(t: torch.Tensor) -> int:
    return 0 if t.dtype == torch.float32 else 1


def _gaussian_launch(items, dtype_code: int, device):
    """Queue the batched Gaussian estimator; returns device (h, status) without synchronising.

    items: (src, idx or None, count[, bitmap]).
    """
    L = _lib.lib()
    n = len(items)
    rows = []
    for it in items:
        src, idx, cnt = it[:3]
        bm = it[3] if len(it) > 3 else None
        rows.append(_lib.GaussDesc(_lib.ptr(src), _lib.ptr(idx), cnt, _lib.ptr(bm), src.numel() if bm is not None else 0))
    descs = (_lib.GaussDesc * n)(*rows)
    need = L.edgc_entropy_gaussian_workspace_bytes(descs, n)
    ws = _lib.WORKSPACE.get(need, device)
    h = torch.empty(n, dtype=torch.float64, device=device)
    status = torch.empty(n, dtype=torch.int32, device=device)
    _lib.check(L.edgc_entropy_gaussian(dtype_code, descs, n, _lib.ptr(h), _lib.ptr(status), _lib.ptr(ws),
                                       ws.numel(), _lib.stream_ptr(device)), "edgc_entropy_gaussian")
    return h, status


def _gaussian_collect(h, status, plan_status=None) -> list:
    h_host = h.cpu().tolist()
    st_host = status.cpu().tolist()
    if plan_status is not None:
        _raise_plan_status(plan_status)
    for code in st_host:
        if code == _lib.EDGC_EINVAL:
            raise ValueError("need at least 2 samples")
        if code == _lib.EDGC_EDEGENERATE:
            raise DegenerateInputError("zero-variance sample has no differential entropy")
        _lib.raise_device_status(code, "entropy_gaussian_plugin")
    return h_host


def _gaussian_batch(items, dtype_code: int, device) -> list:
    """items: (src, idx or None, count[, bitmap]) -> per-item entropies (floats; synchronises)."""
    return _gaussian_collect(*_gaussian_launch(items, dtype_code, device))


class _DeferredMean:
    """A sampled iteration's layer mean whose device entropies are read only when needed."""

    def __init__(self, h, status, plan_status):
        self.h, self.status, self.plan_status = h, status, plan_status

    def value(self) -> float:
        # np.mean over the per-layer Python floats, as entropy.py:177 does
        return float(np.mean(_gaussian_collect(self.h, self.status, self.plan_status)))


def entropy_gaussian_plugin(samples) -> float:
    """ln(sigma_hat) + 0.5 ln(2 pi e) with the ddof=1 deviation (entropy.py:82-90)."""
    x = _samples_tensor(samples)
    if x.numel() < 2:
        raise ValueError(f"need at least 2 samples, got {x.numel()}")
    return _gaussian_batch([(x, None, x.numel())], _dtype_code(x), x.device)[0]


def histogram_fd(samples, bins="fd"):
    """Device np.histogram(x, bins) for bins == "fd" or an int: (counts int64, edges float64, H).

    Counts and edges are bit-exact with NumPy 2.3.5.
    """
    x = _samples_tensor(samples)
    n = x.numel()
    if n < 2:
        raise ValueError(f"need at least 2 samples, got {n}")
    if isinstance(bins, str):
        if bins != "fd":
            raise NotImplementedError(f"bins={bins!r}: the device histogram implements 'fd' and integer bins")
        fixed = 0
    else:
        fixed = int(bins)
        if fixed < 1:
            raise ValueError("`bins` must be positive, when an integer")
    L = _lib.lib()
    dev = x.device
    ws = _lib.WORKSPACE.get(L.edgc_entropy_histogram_workspace_bytes(n), dev)
    inv_cbrt = float(n) ** (-1.0 / 3.0) if n else 0.0  # x.size ** (-1/3): same libm pow as NumPy
    cap = max(fixed, 1 << 16)
    for _ in range(2):
        counts = torch.empty(cap, dtype=torch.int64, device=dev)
        edges = torch.empty(cap + 1, dtype=torch.float64, device=dev)
        result = torch.empty(5, dtype=torch.float64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(L.edgc_entropy_histogram(_dtype_code(x), _lib.ptr(x), n, inv_cbrt, fixed, cap, _lib.ptr(counts),
                                            _lib.ptr(edges), _lib.ptr(result), _lib.ptr(status), _lib.ptr(ws),
                                            ws.numel(), _lib.stream_ptr(dev)), "edgc_entropy_histogram")
        code = int(status.item())
        res = result.cpu().tolist()
        if code == _lib.EDGC_ECAPACITY:
            cap = int(res[4])
            continue
        if code == _lib.EDGC_ENONFINITE:
            # numpy/lib/_histograms_impl.py:_get_outer_edges
            raise ValueError("autodetected range of the samples is not finite")
        if code == _lib.EDGC_EDEGENERATE:
            raise DegenerateInputError("zero-range sample has no histogram entropy")
        if code == _lib.EDGC_ETOOMANYBINS:
            raise ValueError(f"Too many bins for data range. Cannot create {int(res[4])} finite-sized bins.")
        _lib.raise_device_status(code, "entropy_histogram")
        nb = int(res[4])
        return counts[:nb], edges[:nb + 1], res[0]
    raise RuntimeError("histogram bin capacity retry failed")


def entropy_histogram(samples, bins="fd") -> float:
    """-sum p ln(p / width) over the histogram (entropy.py:93-107)."""
    return histogram_fd(samples, bins)[2]


def close_window(records, window_index: int = 0, window_size: int | None = None) -> EntropyWindow:
    values = [float(v) for v in records]
    if not values:
        raise DegenerateInputError("cannot close a window with no sampled iterations")
    return EntropyWindow(window_index=window_index,
                         window_size=len(values) if window_size is None else window_size,
                         mean_entropy=float(np.mean(values)), samples_used=len(values),
                         per_iteration_entropies=values)


def relative_change_rate(series_sampled, series_full) -> np.ndarray:
    """|H_sampled - H_full| / |H_full| per window (analysis metric, host)."""
    a = np.asarray(series_sampled, dtype=np.float64)
    b = np.asarray(series_full, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"window series lengths differ: {a.shape} vs {b.shape}")
    if np.any(b == 0.0):
        raise DegenerateInputError("zero baseline entropy in relative change rate")
    return np.abs(a - b) / np.abs(b)


def _layer_specs(flats, iteration: int, config: SamplerConfig):
    seeds = subsample_seeds(config.rng_seed, iteration, len(flats))
    return [(f.numel(), sample_count(f.numel(), config.beta), seeds[k]) for k, f in enumerate(flats)]


def layer_entropies(matrices, iteration: int, config: SamplerConfig, estimator=None, prefetched=None,
                    deferred: bool = False, workspace=None):
    """Per-layer entropies of one sampled iteration, all layers batched on the device.

    Gaussian plug-in (the default): each matrix is streamed once against the
    plan's membership bitmap (coalesced) instead of gathered at random.
    ``prefetched`` = (specs, plans, bitmaps, status) built earlier on a side stream.
    """
    estimator = entropy_gaussian_plugin if estimator is None else estimator
    flats = [as_device_matrix(m).reshape(-1) for m in matrices]
    if not flats:
        return []
    specs = _layer_specs(flats, iteration, config)
    dev = flats[0].device
    if estimator is entropy_gaussian_plugin:
        for (n, c, _) in specs:
            if c < 2:
                raise ValueError(f"need at least 2 samples, got {c}")
        if prefetched is not None and prefetched[0] == specs:
            _, plans, bms, status = prefetched
        else:
            plans, bms, status = sample_plans(specs, dev, bitmaps=True, check=False, indices=False,
                                              workspace=workspace)
        items = [(f, p, c) if p is None else (f, p, c, bm) for f, p, bm, (_, c, _) in zip(flats, plans, bms, specs)]
        h, hstat = _gaussian_launch(items, 0, dev)
        if deferred:
            return _DeferredMean(h, hstat, status)
        return _gaussian_collect(h, hstat, status)
    plans = sample_plans(specs, dev)
    out = []
    L = _lib.lib()
    for f, p, (n, c, _) in zip(flats, plans, specs):
        if estimator is entropy_histogram:
            if p is None:
                sub = f
            else:
                sub = torch.empty(c, dtype=torch.float32, device=f.device)
                _lib.check(L.edgc_gather(0, _lib.ptr(f), _lib.ptr(p), c, 0, _lib.ptr(sub), _lib.stream_ptr()),
                           "edgc_gather")
            out.append(entropy_histogram(sub))
        else:
            sub = f.double() if p is None else f.double()[p.long()]
            out.append(float(estimator(sub)))
    return out


class EntropyTracker:
    """Per-iteration layer matrices -> fixed-size entropy windows (entropy.py:135-192).

    Sampled iterations run one batched device pipeline over all layers and one
    device-to-host copy of the per-layer entropies; the layer mean and window
    logic are the reference's, on the host.  Because sampled indices do not
    depend on the gradients, the plans (and membership bitmaps) of the next
    sampled iteration are built on a side stream while the intervening
    iterations run (``prefetch=True``); results are unchanged.
    """

    def __init__(self, config: SamplerConfig, window: int, estimator=entropy_gaussian_plugin,
                 prefetch: bool = True):
        if window < 1:
            raise ValueError(f"window must be positive, got {window}")
        period = sampling_period(config.alpha)
        if window < period:
            raise ValueError(f"window {window} shorter than the sampling period {period}: "
                             "windows could close empty")
        self.config = config
        self.window = window
        self.estimator = estimator
        self.windows: list[EntropyWindow] = []
        self._pending: list[float] = []
        self._current = 0
        self.prefetch = prefetch and estimator is entropy_gaussian_plugin
        self._pf = {}              # iteration -> (specs, plans, bitmaps, status, event)
        self._pf_stream = None
        self._pf_ws = _lib.Workspace()
        # the plan workspace is shared by the side-stream prefetches and the (rare) inline builds on
        # the step stream: each side waits only for the other's last use, not for the whole stream
        # (at alpha = 1 the next plan then overlaps this step instead of queueing behind it)
        self._ws_pf_done = None      # event after the last prefetch
        self._ws_inline_done = None  # event after the last inline build

    def _launch_prefetch(self, iteration: int, matrices) -> None:
        flats = [as_device_matrix(m).reshape(-1) for m in matrices]
        if not flats:
            return
        dev = flats[0].device
        if self._pf_stream is None:
            # alpha = 1: the plans are needed by the very next iteration, so they run at the step's
            # (high) priority and overlap it; otherwise low priority, yielding SMs to the step
            prio = -1 if sampling_period(self.config.alpha) == 1 else 0
            self._pf_stream = torch.cuda.Stream(dev, priority=prio)
        specs = _layer_specs(flats, iteration, self.config)
        if any(c < 2 for _, c, _ in specs):
            return
        if self._ws_inline_done is not None:
            self._pf_stream.wait_event(self._ws_inline_done)
        if _PF_AFTER_STEP:   # A/B: start the build only after the work queued on the step stream
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(dev))
            self._pf_stream.wait_event(ready)
        # packed onto few SMs when several iterations of slack remain; spread when the plan is
        # needed by the very next iteration (alpha = 1)
        ahead = sampling_period(self.config.alpha) > 1
        plans, bms, status = sample_plans(specs, dev, bitmaps=True, stream=self._pf_stream, ahead=ahead,
                                          workspace=self._pf_ws, check=False, indices=False)
        ev = torch.cuda.Event()
        ev.record(self._pf_stream)
        self._ws_pf_done = ev
        self._pf[iteration] = (specs, plans, bms, status, ev)

    def _inline_ws(self, dev):
        """The shared plan workspace for a build on the current stream (after the last prefetch)."""
        if self._ws_pf_done is not None:
            torch.cuda.current_stream(dev).wait_event(self._ws_pf_done)
        return self._pf_ws

    def _inline_done(self, dev):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        self._ws_inline_done = ev

    def _take_prefetch(self, iteration: int):
        rec = self._pf.pop(iteration, None)
        if rec is None:
            return None
        specs, plans, bms, status, ev = rec
        cur = torch.cuda.current_stream(status.device)
        cur.wait_event(ev)
        for t in list(plans) + list(bms) + [status]:
            if t is not None:
                t.record_stream(cur)
        return specs, plans, bms, status

    def fused_request(self, iteration: int, engine, matrices):
        """On a sampled iteration (Gaussian estimator), arm `engine`'s next pass 1 to gather the
        sample statistics while it streams the raw gradients -- `matrices` must be the engine's
        gradient tensors.  Returns a handle for ``observe(iteration, matrices, fused=handle)``,
        or None when the step cannot fuse (then observe computes the entropies itself)."""
        if not should_sample_iteration(iteration, self.config.alpha) or self.estimator is not entropy_gaussian_plugin:
            return None
        slots = engine.sample_slots()
        mats = list(matrices)
        if slots <= 0 or not mats:
            return None
        flats = [as_device_matrix(m).reshape(-1) for m in mats]
        specs = _layer_specs(flats, iteration, self.config)
        if any(c < 2 or c == n for n, c, _ in specs):
            return None                      # beta = 1 copies have no membership bitmap
        dev = flats[0].device
        pre = self._take_prefetch(iteration)
        if pre is not None and pre[0] == specs:
            _, plans, bms, status = pre
        else:
            plans, bms, status = sample_plans(specs, dev, bitmaps=True, check=False, indices=False,
                                              workspace=self._inline_ws(dev))
            self._inline_done(dev)
        # slots beyond a matrix's own CTA count stay zero
        partials = torch.zeros((len(specs), slots, 2), dtype=torch.float64, device=dev)
        engine.set_sampling(bms, plans, partials)
        key = tuple(c for _, c, _ in specs)
        if getattr(self, "_counts_key", None) != key:
            self._counts = torch.tensor(key, dtype=torch.int64, device=dev)
            self._counts_key = key
        return (iteration, partials, slots, self._counts, status, (plans, bms))

    def observe(self, iteration: int, matrices, fused=None) -> EntropyWindow | None:
        closed = None
        win = iteration // self.window
        if win < self._current:
            raise ValueError(f"iteration {iteration} precedes window {self._current}")
        if win > self._current:
            closed = self._close()
            self._current = win
        mats = list(matrices)
        if should_sample_iteration(iteration, self.config.alpha) and fused is not None and fused[0] == iteration:
            # pass 1 gathered the shifted sums; finish them into per-layer entropies (read lazily)
            _, partials, slots, counts, status, _keep = fused
            n = partials.shape[0]
            h = torch.empty(n, dtype=torch.float64, device=partials.device)
            hstat = torch.empty(n, dtype=torch.int32, device=partials.device)
            _lib.check(_lib.lib().edgc_entropy_gaussian_partials(_lib.ptr(partials), slots, _lib.ptr(counts), n,
                                                                 _lib.ptr(h), _lib.ptr(hstat),
                                                                 _lib.stream_ptr(partials.device)),
                       "edgc_entropy_gaussian_partials")
            self._pending.append(_DeferredMean(h, hstat, status))
        elif should_sample_iteration(iteration, self.config.alpha):
            pre = self._take_prefetch(iteration)
            if self.estimator is entropy_gaussian_plugin and mats:
                # read back lazily: the host needs the value only when the window closes
                dev = as_device_matrix(mats[0]).device
                inline = pre is None or [n for n, _, _ in pre[0]] != [as_device_matrix(m).numel() for m in mats]
                self._pending.append(layer_entropies(mats, iteration, self.config, self.estimator,
                                                     prefetched=pre, deferred=True,
                                                     workspace=self._inline_ws(dev)))
                if inline:
                    self._inline_done(dev)
            else:
                per_layer = layer_entropies(mats, iteration, self.config, self.estimator, prefetched=pre)
                if per_layer:
                    self._pending.append(float(np.mean(per_layer)))
        period = sampling_period(self.config.alpha)
        if self.prefetch and mats and (period == 1 or not should_sample_iteration(iteration, self.config.alpha)):
            # build the next sampled iteration's plans on the side stream; launched from a
            # non-sampled iteration so the sampled one stays a single short device pass -- or,
            # when every iteration is sampled (alpha = 1), from this one, overlapping the next step
            nxt = (iteration // period + 1) * period
            if nxt not in self._pf:
                self._launch_prefetch(nxt, mats)
        return closed

    def flush(self) -> EntropyWindow | None:
        if not self._pending:
            return None
        out = self._close()
        self._current += 1
        return out

    def _close(self) -> EntropyWindow:
        self._pending = [v.value() if isinstance(v, _DeferredMean) else v for v in self._pending]
        rec = close_window(self._pending, window_index=self._current, window_size=self.window)
        self.windows.append(rec)
        self._pending = []
        return rec


def write_window_csv(path, windows) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh, lineterminator="\n")
        out.writerow(["window_index", "mean_entropy", "samples_used"])
        for w in windows:
            out.writerow([w.window_index, repr(w.mean_entropy), w.samples_used])


_ = ctypes  # ctypes structures are built in _lib
