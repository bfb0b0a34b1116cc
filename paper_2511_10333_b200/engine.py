"""Data-parallel bucket engine: the B200 form of train_toy's EDGC step.

One process per GPU.  Each rank owns its gradient matrices and one
CompressorState per matrix, seeded exactly as the reference seeds worker w's
states (grad_source.py:440-447).  A step is (grad_source.py:389-419):

  1. compress every matrix of this rank (one grouped launch per phase:
     pass 1, factor, pass 2, finalize) into a packed factor buffer
     [P_0 | Q_0 | P_1 | Q_1 | ...];
  2. exchange: one all-gather of the packed buffers over NCCL (W > 1);
  3. reconstruct the DP average out_k = (1/W) sum_w P_{k,w} Q_{k,w}^T in
     worker order (grad_source.py:404-408) — one grouped launch.

Rank decisions come from the worker-0 entropy tracker (rank 0) and are
broadcast; every rank then applies set_rank (grad_source.py:416-418, 469-471).

Memory (per rank, fp32): gradients, the error-feedback base w and the output
are m*n each; factors are 2 x sum (m + n) r_cap, basis and warm start
sum n r_cap each.  Kernel plans (descriptor + tile tables) are uploaded once
per rank configuration and reused, so a steady-state step is launches only.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .compressor import DEVICE_COLUMN_TOL, basis_columns
from .errors import DivergenceError
from .seeds import state_seeds

__all__ = ["BucketEngine", "GPT2_2P5B_LAYER", "GPT2_12P1B_LAYER", "gpt2_shapes"]

# per-layer weight gradients (QKV, proj, fc1, fc2)
GPT2_2P5B_LAYER = ((1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920))
GPT2_12P1B_LAYER = ((3584, 10752), (3584, 3584), (3584, 14336), (14336, 3584))


def gpt2_shapes(which: str = "2.5B", layers: int | None = None):
    layer, default = {"2.5B": (GPT2_2P5B_LAYER, 52), "12.1B": (GPT2_12P1B_LAYER, 76)}[which]
    return [s for _ in range(default if layers is None else layers) for s in layer]


def packed_offsets(shapes, ranks):
    """Offsets of (P_k, Q_k) in one rank's packed factor buffer and its total size (elements).

    Layout: [P_0 (m_0 x r_0) | Q_0 (n_0 x r_0) | P_1 | Q_1 | ...], row-major, ld = r_k.
    """
    offs, cur = [], 0
    for (m, n), r in zip(shapes, ranks):
        offs.append((cur, cur + m * r))
        cur += (m + n) * r
    return offs, cur


def gather_packed(send, gathered, world: int, group=None) -> None:
    """All-gather every rank's packed factors into gathered[w * size:(w + 1) * size] (rank order).

    NCCL: one all_gather_into_tensor.  Other backends (gloo in the CPU tests):
    all_gather into views of the same buffer, so the layout is identical.
    """
    import torch.distributed as dist
    size = send.numel()
    out = gathered[:world * size]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.view(world, size), send, group=group)
    else:
        views = list(out.view(world, size).unbind(0))
        dist.all_gather(views, send, group=group)


def broadcast_decision(rank, device, group=None, src: int = 0):
    """Rank `src`'s window decision (an int or None) on every rank (grad_source.py:469-471 on all workers)."""
    import torch.distributed as dist
    t = torch.tensor([-1 if rank is None else int(rank)], dtype=torch.int64, device=device)
    dist.broadcast(t, src=src, group=group)
    v = int(t.item())
    return None if v < 0 else v


class _Plan:
    """Owns one bound C plan (compress or reconstruct) and its workspace."""

    def __init__(self, kind: str, descs, device):
        L = _lib.lib()
        self.kind = kind
        self.L = L
        h = ctypes.c_void_p()
        n = len(descs)
        if kind == "compress":
            arr = (_lib.CompressDesc * n)(*descs)
            _lib.check(L.edgc_compress_plan_create(arr, n, ctypes.byref(h)), "compress plan")
            nbytes = L.edgc_compress_plan_workspace_bytes(h)
            self.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            _lib.check(L.edgc_compress_plan_bind(h, _lib.ptr(self.ws), self.ws.numel(), _lib.stream_ptr(device)),
                       "compress plan bind")
        else:
            arr = (_lib.ReconDesc * n)(*descs)
            _lib.check(L.edgc_recon_plan_create(arr, n, ctypes.byref(h)), "recon plan")
            nbytes = L.edgc_recon_plan_workspace_bytes(h)
            self.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            _lib.check(L.edgc_recon_plan_bind(h, _lib.ptr(self.ws), self.ws.numel(), _lib.stream_ptr(device)),
                       "recon plan bind")
        self.h = h
        self.descs = arr

    def sample_slots(self) -> int:
        """Fused-sampling partial slots per matrix (0: the plan cannot fuse the Gaussian statistics)."""
        return int(self.L.edgc_compress_plan_sample_slots(self.h)) if self.kind == "compress" else 0

    def set_sampling(self, descs, partials, stream):
        arr = (_lib.SampleDesc * len(descs))(*descs)
        _lib.check(self.L.edgc_compress_plan_set_sampling(self.h, arr, len(descs), _lib.ptr(partials), stream),
                   "compress plan sampling")

    def run(self, stream, *, col_tol=None, status=None, phases=_lib.PHASE_ALL):
        if self.kind == "compress":
            _lib.check(self.L.edgc_compress_plan_run(self.h, col_tol, _lib.ptr(status), phases, stream),
                       "compress run")
        else:
            _lib.check(self.L.edgc_recon_plan_run(self.h, stream), "recon run")

    def __del__(self):
        try:
            if self.h:
                (self.L.edgc_compress_plan_destroy if self.kind == "compress" else self.L.edgc_recon_plan_destroy)(
                    self.h)
        except Exception:
            pass


class BucketEngine:
    """One DP rank's bucket set: compress + exchange + averaged reconstruction."""

    def __init__(self, shapes, rank: int, seed: int = 0, *, world_size: int = 1, rank_id: int = 0, group=None,
                 rank_cap: int | None = None, col_tol: float = DEVICE_COLUMN_TOL, device=None,
                 alias_output: bool = False, exchange: str = "auto"):
        """exchange (W > 1): "p2p" gathers every rank's packed factors with a device-initiated pull over
        NVLink (CUDA IPC mappings, a device flag per rank and step, no collective call); "nccl" with
        all_gather_into_tensor; "auto" = p2p on an NCCL process group (one node)."""
        self.L = _lib.lib()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.shapes = [(int(m), int(n)) for m, n in shapes]
        if not self.shapes:
            raise ValueError("need at least one matrix")
        self.world, self.me, self.group = int(world_size), int(rank_id), group
        if exchange not in ("auto", "p2p", "nccl"):
            raise ValueError(f"exchange must be 'auto', 'p2p' or 'nccl', got {exchange!r}")
        self._p2p = False
        if self.world > 1 and exchange != "nccl":
            import torch.distributed as dist
            self._p2p = exchange == "p2p" or dist.get_backend(group) == "nccl"
        self._flags = None          # p2p: int64[W] completion flags, written by the peers
        self.col_tol = float(col_tol)
        self.cap = max(int(rank), int(rank_cap or rank))
        seeds = state_seeds(seed, self.world, len(self.shapes))
        self.basis_seeds = [seeds[(self.me, k)] for k in range(len(self.shapes))]
        dev = self.device
        numel = [m * n for m, n in self.shapes]
        self._mat_off = np.concatenate([[0], np.cumsum(numel)]).astype(np.int64)
        total = int(self._mat_off[-1])
        self.total_elems = total
        self.grad_arena = torch.zeros(total, dtype=torch.float32, device=dev)
        self.w_arena = torch.zeros(total, dtype=torch.float32, device=dev)
        # alias_output: the averaged reconstruction overwrites the gradients (one 4 B/elem arena less,
        # e.g. GPT2-12.1B: 46.9 GB); the raw gradients are then valid only until reconstruct()
        self.alias_output = bool(alias_output)
        self.out_arena = self.grad_arena if self.alias_output else torch.zeros(total, dtype=torch.float32, device=dev)
        self.grads = [self.grad_arena[a:b].view(m, n) for (a, b), (m, n) in zip(self._spans(), self.shapes)]
        self.outs = [self.out_arena[a:b].view(m, n) for (a, b), (m, n) in zip(self._spans(), self.shapes)]
        self.ws_views = [self.w_arena[a:b].view(m, n) for (a, b), (m, n) in zip(self._spans(), self.shapes)]
        self._alloc_rank_buffers(self.cap)
        self.ranks = [min(int(rank), min(m, n)) for m, n in self.shapes]
        self._res = None            # (parity, ranks, offsets) of the residual factor pair
        self._parity = 0
        self._plans = {}
        self.status = torch.zeros(len(self.shapes), dtype=torch.int32, device=dev)
        self.steps = 0

    # ------------------------------------------------------------ buffers
    def _spans(self):
        return [(int(self._mat_off[k]), int(self._mat_off[k + 1])) for k in range(len(self.shapes))]

    def _alloc_rank_buffers(self, cap: int, old=None):
        dev = self.device
        bsz = sum(n * cap for _, n in self.shapes)
        basis = torch.empty(bsz, dtype=torch.float32, device=dev)
        qwarm = torch.empty(bsz, dtype=torch.float32, device=dev)
        offs, cur = [], 0
        for k, (m, n) in enumerate(self.shapes):
            offs.append(cur)
            old_cap = 0 if old is None else old["cap"]
            view_b = basis[cur:cur + n * cap].view(n, cap)
            view_q = qwarm[cur:cur + n * cap].view(n, cap)
            if old is not None:
                view_b[:, :old_cap] = old["basis"][k]
                view_q[:, :old_cap] = old["q_warm"][k]
            if cap > old_cap:
                fresh = torch.from_numpy(basis_columns(self.basis_seeds[k], n, old_cap, cap)).to(dev)
                view_b[:, old_cap:] = fresh
                view_q[:, old_cap:] = fresh
            cur += n * cap
        self._basis_arena, self._qwarm_arena = basis, qwarm
        pre = torch.zeros(len(self.shapes), cap, cap, dtype=torch.float64, device=dev)
        pre[:] = torch.eye(cap, dtype=torch.float64, device=dev)
        if old is not None:
            pre[:, :old["cap"], :old["cap"]] = old["precond"]
        self.precond = pre
        self.basis = [basis[o:o + n * cap].view(n, cap) for o, (_, n) in zip(offs, self.shapes)]
        self.q_warm = [qwarm[o:o + n * cap].view(n, cap) for o, (_, n) in zip(offs, self.shapes)]
        fsz = sum((m + n) * cap for m, n in self.shapes)
        new_fac = [torch.zeros(fsz, dtype=torch.float32, device=dev) for _ in range(2)]
        if old is not None:
            for i in range(2):
                new_fac[i][:old["factors"][i].numel()] = old["factors"][i]
        self.factors = new_fac
        self.cap = cap
        self._gathered = None
        self._fsz = fsz
        if self.world > 1 and not self._p2p:
            self._gathered = torch.empty(self.world * fsz, dtype=torch.float32, device=dev)
        if self._p2p:
            self._share_factors()

    def _share_factors(self):
        """Map every rank's two factor buffers and flag array into this process on this rank's device
        (CUDA IPC handles of the allocations holding them, exchanged once per buffer allocation
        through the process group) and build the device pointer tables."""
        import torch.distributed as dist
        dev = self.device
        if self._flags is None:
            self._flags = torch.zeros(self.world, dtype=torch.int64, device=dev)
            self._epoch_dev = torch.zeros(1, dtype=torch.int64, device=dev)   # steps published (device)
        mine = []
        for t in (self.factors[0], self.factors[1], self._flags):
            handle = ctypes.create_string_buffer(64)
            off = ctypes.c_int64()
            _lib.check(self.L.edgc_ipc_handle(ctypes.c_void_p(t.data_ptr()), handle, ctypes.byref(off)),
                       "edgc_ipc_handle")
            mine.append((handle.raw, int(off.value)))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=self.group)
        self._close_peers()
        opened = {}
        table = []
        ok = True
        try:
            for w, recs in enumerate(everyone):
                if w == self.me:
                    table.append([t.data_ptr() for t in (self.factors[0], self.factors[1], self._flags)])
                    continue
                row = []
                for handle, off in recs:
                    if handle not in opened:   # one mapping per allocation (buffers may share one)
                        p = ctypes.c_void_p()
                        _lib.check(self.L.edgc_ipc_open(ctypes.c_char_p(handle), ctypes.byref(p)), "edgc_ipc_open")
                        opened[handle] = p.value
                    row.append(opened[handle] + off)
                table.append(row)
        except RuntimeError:
            ok = False
        self._ipc_mapped = list(opened.values())
        # all ranks agree: if any rank could not map its peers, every rank uses the NCCL all-gather
        agree = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(agree, op=dist.ReduceOp.MIN, group=self.group)
        if not int(agree.item()):
            self._close_peers()
            self._p2p = False
            self._ensure_gathered()
            return
        self._peer_bases = [torch.tensor([row[par] for row in table], dtype=torch.int64, device=dev)
                            for par in (0, 1)]
        self._peer_flags = torch.tensor([row[2] for row in table], dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)
        # every rank must hold its mappings before any rank starts publishing into them
        dist.barrier(group=self.group)

    def _close_peers(self):
        for p in getattr(self, "_ipc_mapped", []):
            try:
                self.L.edgc_ipc_close(ctypes.c_void_p(p))
            except Exception:
                pass
        self._ipc_mapped = []

    def _ensure_gathered(self):
        if self._gathered is None:
            self._gathered = torch.empty(self.world * self._fsz, dtype=torch.float32, device=self.device)

    def _packed_offsets(self, ranks):
        return packed_offsets(self.shapes, ranks)

    # -------------------------------------------------------------- plans
    def _compress_plan(self):
        ranks = tuple(self.ranks)
        res = self._res
        key = ("c", self._parity, ranks, None if res is None else (res[0], res[1]),
               tuple(g.data_ptr() for g in self.grads))
        plan = self._plans.get(key)
        if plan is not None:
            return plan
        offs, _ = self._packed_offsets(ranks)
        out_buf = self.factors[self._parity]
        descs = []
        for k, ((m, n), r) in enumerate(zip(self.shapes, ranks)):
            p_res = q_res = None
            r_res = 0
            if res is not None:
                rbuf = self.factors[res[0]]
                (po, qo), r_res = res[2][k], res[1][k]
                p_res = rbuf[po:]
                q_res = rbuf[qo:]
            po, qo = offs[k]
            g = self.grads[k]
            descs.append(_lib.CompressDesc(_lib.ptr(g), _lib.ptr(self.ws_views[k]), _lib.ptr(p_res), _lib.ptr(q_res),
                                           _lib.ptr(self.q_warm[k]), _lib.ptr(self.basis[k]),
                                           _lib.ptr(out_buf[po:]), _lib.ptr(out_buf[qo:]),
                                           _lib.ptr(self.precond[k]), m, n, g.stride(0), r, r_res, self.cap,
                                           self.cap))
        self._evict("c", ranks, key)
        plan = _Plan("compress", descs, self.device)
        self._plans[key] = plan
        return plan

    def _evict(self, kind: str, ranks, keep) -> None:
        """Release every cached plan of `kind` that the current ranks can no longer use.

        A steady-state compress plan has ranks == residual ranks == the current
        ranks (one per factor-buffer parity); the residual-free first-step plan
        and the one-step transition plan after a rank change are used once.  Each
        plan owns fp64 scratch sized by its ranks, so keeping stale ones would
        grow HBM use with every controller decision.
        """
        for k in list(self._plans):
            if k[0] != kind or k == keep:
                continue
            if k[2] != ranks or (kind == "c" and (k[3] is None or k[3][1] != ranks)):
                del self._plans[k]

    def _recon_plan(self):
        ranks = tuple(self.ranks)
        key = ("r", self._parity, ranks, tuple(o.data_ptr() for o in self.outs))
        plan = self._plans.get(key)
        if plan is not None:
            return plan
        offs, size = self._packed_offsets(ranks)
        if self.world > 1:
            self._ensure_gathered()
        src = self.factors[self._parity] if self.world == 1 else self._gathered
        descs = []
        for k, ((m, n), r) in enumerate(zip(self.shapes, ranks)):
            po, qo = offs[k]
            o = self.outs[k]
            descs.append(_lib.ReconDesc(_lib.ptr(src[po:]), _lib.ptr(src[qo:]), _lib.ptr(o), m, n, o.stride(0),
                                        size, size, r, self.world, 1.0 / self.world, 0))
        self._evict("r", ranks, key)
        plan = _Plan("recon", descs, self.device)
        self._plans[key] = plan
        return plan

    # --------------------------------------------------------------- step
    def compress(self, phases: int = _lib.PHASE_ALL):
        """Phase 1: compress every matrix of this rank into the packed factor buffer.

        `phases` selects sub-steps (pass 1, factor, pass 2, finalize) so a caller
        can bracket each with CUDA events; issuing them in order == PHASE_ALL.
        """
        stream = _lib.stream_ptr(self.device)
        self._compress_plan().run(stream, col_tol=self.col_tol, status=self.status, phases=phases)

    def sample_slots(self) -> int:
        """Partial slots per matrix when the next pass 1 can also gather the sampled-iteration
        Gaussian statistics (every matrix on the Z path), else 0."""
        return self._compress_plan().sample_slots()

    def set_sampling(self, bitmaps, firsts, partials):
        """Arm the next pass 1 to accumulate, per matrix k, the fp64 shifted sums of the raw
        gradient over bitmaps[k] (shift = element firsts[k][0]) into partials[k] (float64,
        [n, slots, 2]); see edgc_compress_plan_set_sampling."""
        descs = [_lib.SampleDesc(_lib.ptr(b), _lib.ptr(f)) for b, f in zip(bitmaps, firsts)]
        self._compress_plan().set_sampling(descs, partials, _lib.stream_ptr(self.device))

    def exchange(self):
        """Phase 2, W > 1: every rank's packed factors into the gathered buffer, in rank order.
        p2p: publish a device flag into every rank's flag array, then pull each rank's buffer over
        NVLink once its flag for this step is up (no host synchronisation, no collective call);
        nccl: one all_gather_into_tensor.  No-op at W = 1."""
        if self.world == 1:
            return
        self._ensure_gathered()
        _, size = self._packed_offsets(self.ranks)
        if self._p2p:
            stream = _lib.stream_ptr(self.device)
            _lib.check(self.L.edgc_p2p_signal(_lib.ptr(self._peer_flags), self.me, self.world,
                                              _lib.ptr(self._epoch_dev), stream), "edgc_p2p_signal")
            # every rank's packed buffer has the same layout: rank w's first `size` floats go to
            # gathered[w size ..) (the gathered layout's rank stride is the packed size)
            _lib.check(self.L.edgc_p2p_pull(_lib.ptr(self._peer_bases[self._parity]), _lib.ptr(self._gathered), size,
                                            self.world, _lib.ptr(self._flags), _lib.ptr(self._epoch_dev), stream),
                       "edgc_p2p_pull")
            return
        gather_packed(self.factors[self._parity][:size], self._gathered, self.world, self.group)

    def reconstruct(self):
        """Phase 3: out_k = (1/W) sum_w P_kw Q_kw^T in worker order."""
        self._recon_plan().run(_lib.stream_ptr(self.device))

    def step(self, grads=None, check: bool = False):
        """One DP step; returns the per-matrix averaged reconstructions (views of out_arena)."""
        if grads is not None:
            for dst, src in zip(self.grads, grads):
                if dst.data_ptr() != src.data_ptr():
                    dst.copy_(src, non_blocking=True)
        self.compress()
        self.exchange()
        self.reconstruct()
        self.advance()
        if check:
            self.check_status()
        return self.outs

    def capture_graphs(self):
        """Record the steady-state step (compress, exchange, reconstruct) as two CUDA graphs, one per
        factor-buffer parity; `graph_step` then replays the current parity's graph.

        Needs one eager step first (the residual-free first step uses its own plan).  The graphs hold
        the current plans' device pointers, so `set_rank` drops them.
        """
        if self._res is None:
            raise ValueError("run one eager step before capturing the step graphs")
        saved = (self._parity, self._res, self.steps)
        graphs = {}
        cap = torch.cuda.Stream(self.device)
        cap.wait_stream(torch.cuda.current_stream(self.device))
        for _ in range(2):
            par = self._parity
            # plans are built (allocations, uploads) before capture; capture only records launches
            self._compress_plan()
            self._recon_plan()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                self.compress()
                self.exchange()
                self.reconstruct()
            graphs[par] = g
            self.advance()   # host bookkeeping only: which buffer holds the residual pair
        torch.cuda.current_stream(self.device).wait_stream(cap)
        self._parity, self._res, self.steps = saved
        self._graphs = graphs

    def graph_step(self, check: bool = False):
        """One DP step by graph replay (capture_graphs); same results as `step`."""
        g = getattr(self, "_graphs", None)
        if not g:
            raise ValueError("capture_graphs() first")
        g[self._parity].replay()
        self.advance()
        if check:
            self.check_status()
        return self.outs

    def advance(self):
        """Close a step issued phase by phase: the factors just written become the residual pair."""
        offs, _ = self._packed_offsets(self.ranks)
        self._res = (self._parity, tuple(self.ranks), offs)
        self._parity ^= 1
        self.steps += 1

    def check_status(self):
        """Raise DivergenceError if any matrix saw a non-finite work entry (synchronises)."""
        bad = torch.nonzero(self.status).flatten().tolist()
        if bad:
            raise DivergenceError(f"non-finite gradient or residual in matrices {bad[:8]}")

    # ---------------------------------------------------------- state API
    def set_rank(self, r: int):
        """Apply a controller decision to every matrix: r_k = min(r, min(m, n)) (grad_source.py:469-471)."""
        if r < 1:
            raise ValueError(f"rank must be >= 1, got {r}")
        self._graphs = None   # captured plans no longer match
        if r > self.cap:
            old = {"cap": self.cap, "basis": [b.clone() for b in self.basis],
                   "q_warm": [q.clone() for q in self.q_warm], "factors": self.factors,
                   "precond": self.precond.clone()}
            self._alloc_rank_buffers(r, old)
            self._plans.clear()
        new = [min(int(r), min(m, n)) for m, n in self.shapes]
        for k, (ro, rn) in enumerate(zip(self.ranks, new)):
            if rn > ro:
                self.q_warm[k][:, ro:rn].copy_(self.basis[k][:, ro:rn])
                self.precond[k][:, ro:rn] = 0.0
                self.precond[k][ro:rn, ro:rn] = torch.eye(rn - ro, dtype=torch.float64, device=self.device)
        self.ranks = new

    def factors_of(self, k: int):
        """(P, Q) of matrix k from the last step (views)."""
        if self._res is None:
            raise ValueError("no step has run yet")
        parity, ranks, offs = self._res
        buf = self.factors[parity]
        (m, n), r, (po, qo) = self.shapes[k], ranks[k], offs[k]
        return buf[po:po + m * r].view(m, r), buf[qo:qo + n * r].view(n, r)

    def residual(self, k: int) -> torch.Tensor:
        """Materialised error-feedback residual of matrix k (compressor.py:112)."""
        m, n = self.shapes[k]
        w = self.ws_views[k]
        if self._res is None:
            return w.clone()
        p, q = self.factors_of(k)
        out = torch.empty_like(w)
        _lib.check(self.L.edgc_residual(_lib.ptr(w), _lib.ptr(p), _lib.ptr(q), p.shape[1], m, n, _lib.ptr(out),
                                        _lib.stream_ptr(self.device)), "edgc_residual")
        return out

    def wire_bytes(self) -> int:
        """Logical bytes this worker sends per step: 4 r (m + n) per matrix (grad_source.py:398-403)."""
        return sum(4 * r * (m + n) for (m, n), r in zip(self.shapes, self.ranks))
