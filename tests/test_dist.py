"""CPU, world_size 2 over gloo: the multi-rank host logic of the DP exchange.

Each process plays one DP worker: it compresses its own gradients with its
own seeded states (oracle compress — the device kernels are covered by the
GPU tests), packs the factors in the engine's layout, all-gathers them with
the engine's gather_packed, reconstructs the worker-order average from the
gathered buffer, and checks it against the reference's sequential DP step
(grad_source.py:389-408, restated in oracle.dp_step).  The rank-decision
broadcast is checked the same way.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SHAPES = [(24, 40), (40, 24), (16, 16)]
RANK = 3
WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import oracle
        from paper_2511_10333_b200.engine import broadcast_decision, gather_packed, packed_offsets
        seeds = oracle.state_seeds(5, WORLD, len(SHAPES))
        ranks = [min(RANK, m, n) for m, n in SHAPES]
        offs, size = packed_offsets(SHAPES, ranks)
        states = [oracle.OracleState(m, n, r, seeds[(rank, k)]) for k, ((m, n), r) in enumerate(zip(SHAPES, ranks))]
        worst = 0.0
        for t in range(3):
            grads = [oracle.synth_matrix(5, t, k, rank, m, n, 1e-2).astype(np.float64)
                     for k, (m, n) in enumerate(SHAPES)]
            send = torch.zeros(size, dtype=torch.float64)
            for k, g in enumerate(grads):
                p, q, _ = oracle.compress(g, states[k])
                po, qo = offs[k]
                send[po:po + p.size] = torch.from_numpy(p.ravel())
                send[qo:qo + q.size] = torch.from_numpy(q.ravel())
            gathered = torch.empty(WORLD * size, dtype=torch.float64)
            gather_packed(send, gathered, WORLD)
            # worker-order average from the gathered buffer (what the reconstruct kernel computes)
            for k, ((m, n), r) in enumerate(zip(SHAPES, ranks)):
                po, qo = offs[k]
                acc = np.zeros((m, n))
                for w in range(WORLD):
                    base = w * size
                    P = gathered[base + po:base + po + m * r].numpy().reshape(m, r)
                    Q = gathered[base + qo:base + qo + n * r].numpy().reshape(n, r)
                    acc += P @ Q.T
                avg = acc / WORLD
                # the reference's sequential DP step over both workers, from scratch states
                if t == 0:
                    ref_states = [[oracle.OracleState(mm, nn, rr, seeds[(w, kk)])
                                   for kk, ((mm, nn), rr) in enumerate(zip(SHAPES, ranks))] for w in range(WORLD)]
                    all_grads = [[oracle.synth_matrix(5, 0, kk, w, mm, nn, 1e-2).astype(np.float64)
                                  for kk, (mm, nn) in enumerate(SHAPES)] for w in range(WORLD)]
                    ref = oracle.dp_step(all_grads, ref_states)[k]
                    worst = max(worst, float(np.max(np.abs(avg - ref))))
        decided = broadcast_decision(17 if rank == 0 else None, torch.device("cpu"))
        none = broadcast_decision(None if rank == 0 else 5, torch.device("cpu"))
        result_q.put((rank, worst, decided, none))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_matches_sequential_reference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = sorted(q.get(timeout=5) for _ in range(WORLD))
    for rank, worst, decided, none in results:
        assert worst <= 1e-12, (rank, worst)
        assert decided == 17
        assert none is None


def test_packed_offsets_layout():
    from paper_2511_10333_b200.engine import packed_offsets
    offs, size = packed_offsets([(2, 3), (4, 5)], [2, 1])
    assert offs == [(0, 4), (10, 14)] and size == 19
