"""EDGC data-parallel step driver: train_toy's EDGC wiring on real ranks.

Composes the hot path exactly as the reference's toy DP loop does
(grad_source.py:311-343 setup, 385-419 step, 450-479 window update), with one
process per GPU instead of simulated workers:

* setup: Eq. 2 rank bounds from a cost-free byte model (eta = 4 sum(m+n)/B),
  the g-table of the largest matrix (transposed so m <= n), r_max clamped
  below table.m, every CompressorState at r_max;
* each step: while the controller is in warm-up the gradients are averaged
  uncompressed (NCCL all-reduce); once active, the bucket engine compresses,
  all-gathers the factors and reconstructs the worker-order average;
* rank 0 feeds its raw (pre-compression) gradients to the entropy tracker;
  at a window close it runs the controller and broadcasts the decision; all
  ranks then apply set_rank.
The warm-up SVD probe of the reference (grad_source.py:454-465) is write-only
(controller.py:231) and is skipped; eps_ini falls back to the model value.
"""

from __future__ import annotations

import torch

from .controller import (PHASE_ACTIVE, PHASE_WARMUP, CommModel, RankBounds, RankControllerState, RankDecision,
                         adjust_rank_window, compute_rank_bounds, warmup_step)
from .engine import BucketEngine, broadcast_decision
from .entropy import EntropyTracker, SamplerConfig
from .rank_model import g_table

__all__ = ["EdgcDataParallel", "edgc_setup"]


def edgc_setup(shapes, *, table_trials: int = 64, seed: int = 0, bandwidth: float = 1e9, element_size: int = 4):
    """train_toy's EDGC setup (grad_source.py:311-327): byte model, Eq. 2 bounds, g-table, r_max < table.m.

    Returns (CommModel, RankBounds, GTable).  Host-only; pinned to the reference by tests/golden/dp.json.
    """
    shapes = [(int(m), int(n)) for m, n in shapes]
    per_rank = sum(m + n for m, n in shapes)
    raw = sum(m * n for m, n in shapes)
    model = CommModel(eta=element_size * per_rank / bandwidth, bandwidth=bandwidth, element_size=element_size)
    bounds = compute_rank_bounds(model, element_size * raw, shapes)
    big = max(shapes, key=lambda s: s[0] * s[1])
    table = g_table(min(big), max(big), table_trials, seed)
    if bounds.r_max >= table.m:
        r_max = table.m - 1
        bounds = RankBounds(r_min=min(bounds.r_min, r_max), r_max=r_max)
    return model, bounds, table


class EdgcDataParallel:
    def __init__(self, shapes, *, total_iterations: int, seed: int = 0, world_size: int = 1, rank_id: int = 0,
                 group=None, sampler: SamplerConfig = SamplerConfig(), window: int = 100, step_limit: int = 8,
                 warmup_floor: float = 0.10, table_trials: int = 64, bandwidth: float = 1e9, element_size: int = 4,
                 exchange: str = "auto"):
        self.shapes = [(int(m), int(n)) for m, n in shapes]
        self.world, self.me, self.group = world_size, rank_id, group
        self.model, bounds, self.table = edgc_setup(self.shapes, table_trials=table_trials, seed=seed,
                                                    bandwidth=bandwidth, element_size=element_size)
        self.bounds = bounds
        self.ctl = RankControllerState(bounds=bounds, window=window, step_limit=step_limit,
                                       warmup_floor=warmup_floor, total_iterations=total_iterations)
        self.tracker = EntropyTracker(sampler, window) if rank_id == 0 else None
        self.engine = BucketEngine(self.shapes, rank=bounds.r_max, seed=seed, world_size=world_size,
                                   rank_id=rank_id, group=group, rank_cap=bounds.r_max, exchange=exchange)
        self.rank_history: list[RankDecision] = []
        self.bytes_per_step: list[float] = []
        self._raw_avg = None

    @property
    def grads(self):
        """Per-matrix gradient buffers the backward pass writes into (views of one arena)."""
        return self.engine.grads

    def _average_raw(self):
        eng = self.engine
        if self._raw_avg is None:
            self._raw_avg = eng.out_arena
        self._raw_avg.copy_(eng.grad_arena)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self._raw_avg, group=self.group)
            self._raw_avg.mul_(1.0 / self.world)
        return eng.outs

    def step(self, t: int, grads=None):
        """One DP iteration t; returns the averaged gradients (views, valid until the next step)."""
        eng = self.engine
        if grads is not None:
            for dst, src in zip(eng.grads, grads):
                if dst.data_ptr() != src.data_ptr():
                    dst.copy_(src, non_blocking=True)
        fused = None
        if self.ctl.phase == PHASE_ACTIVE:
            if self.tracker is not None:
                # sampled iteration: pass 1 also gathers the sample's Gaussian statistics
                fused = self.tracker.fused_request(t, eng, eng.grads)
            outs = eng.step()
            self.bytes_per_step.append(float(self.world * eng.wire_bytes()))
        else:
            outs = self._average_raw()
            self.bytes_per_step.append(float(self.world * 4 * eng.total_elems))
        decision = None
        closed = None
        if self.tracker is not None:
            closed = self.tracker.observe(t, eng.grads, fused=fused)
            if closed is not None:
                decision = self._window_update(closed)
        if self.world > 1 and self.closes_window(t):
            # a window can close only when t // window advances (entropy.py:161-166), which every
            # rank knows: only those iterations pay for the broadcast (-1 = none / still warm-up)
            decision = broadcast_decision(decision, eng.device, self.group)
        if decision is not None:
            eng.set_rank(decision)
            if self.ctl.phase != PHASE_ACTIVE:
                self.ctl.phase = PHASE_ACTIVE  # non-zero ranks mirror rank 0's phase switch
        return outs

    def closes_window(self, t: int) -> bool:
        """True iff observing iteration t can close a window: t // window advanced past the previous one."""
        return t > 0 and t // self.ctl.window > (t - 1) // self.ctl.window

    def flush(self):
        """Close the trailing partial window (entropy.py:180-186); every rank applies the decision."""
        decision = None
        if self.tracker is not None:
            closed = self.tracker.flush()
            decision = None if closed is None else self._window_update(closed)
        if self.world > 1:
            decision = broadcast_decision(decision, self.engine.device, self.group)
        if decision is not None:
            self.engine.set_rank(decision)
            if self.ctl.phase != PHASE_ACTIVE:
                self.ctl.phase = PHASE_ACTIVE
        return decision

    def _window_update(self, win):
        ctl = self.ctl
        t_pred = None
        if ctl.phase == PHASE_WARMUP:
            warmup_step(ctl, win.mean_entropy, (win.window_index + 1) * ctl.window, self.table)
            rank = ctl.r_prev if ctl.phase == PHASE_ACTIVE else None
        else:
            rank, t_pred = adjust_rank_window(ctl, win.mean_entropy, self.table, self.model)
        self.rank_history.append(RankDecision(window_index=win.window_index, mean_entropy=win.mean_entropy,
                                              ranks=None if rank is None else [rank], t_pred=t_pred))
        return rank

    def check_status(self):
        self.engine.check_status()

    def synchronize(self):
        torch.cuda.synchronize(self.engine.device)
