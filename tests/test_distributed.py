"""Multi-GPU host logic on CPU: chain sharding and the best-of-ranks exchange, run as a real
world_size-2 process group over gloo (127.0.0.1). The GPU side of the same path is covered by
the slice-independence test in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_14966_b200.distributed import LocalBest, chain_slice, exchange_best, pick_winner


def test_chain_slice_partitions_the_chain_space():
    for total in (1, 7, 16384, 16385):
        for world in (1, 2, 3, 8):
            spans = [chain_slice(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        chain_slice(10, 2, 2)


def test_pick_winner_order():
    rec = np.array([[1.0, 5.0, 3, 0], [2.0, 9.0, 7, 1], [2.0, 8.0, 9, 2], [2.0, 8.0, 4, 3]])
    assert pick_winner(rec) == 3  # highest g, then lowest t, then lowest chain id
    rec = np.array([[-np.inf, 0.0, -1, 0], [1e-7, 1.0, 0, 1]])
    assert pick_winner(rec) == 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for case in cases:
            g, t, chain, seq, sizes = case[rank]
            local = LocalBest(g, t, chain, np.asarray(seq, dtype=np.int32), np.asarray(sizes, dtype=np.int32))
            win, wseq, wsizes = exchange_best(local, len(seq))
            results.append((win, wseq.tolist(), wsizes.tolist()))
        out_q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_exchange_best_world_size_2_gloo():
    n = 6
    cases = [
        # rank 1 has the higher G
        [(1e-6, 100.0, 5, [0, 1, 2, 3, 4, 5], [2, 2, 2]), (2e-6, 90.0, 9, [5, 4, 3, 2, 1, 0], [1, 1, 4])],
        # equal G: lower t wins
        [(3e-6, 80.0, 1, [1, 0, 2, 3, 4, 5], [3, 3]), (3e-6, 81.0, 0, [0, 1, 2, 3, 4, 5], [6])],
        # equal G and t: lower chain id wins
        [(3e-6, 80.0, 11, [2, 1, 0, 3, 4, 5], [1, 2, 3]), (3e-6, 80.0, 10, [3, 4, 5, 0, 1, 2], [2, 4])],
        # a rank that ran no chain never wins
        [(0.0, 0.0, -1, [0] * n, [n]), (0.0, 50.0, 2, [5, 0, 4, 1, 3, 2], [2, 2, 1, 1])],
    ]
    want = [(1, cases[0][1][3], cases[0][1][4]), (0, cases[1][0][3], cases[1][0][4]),
            (1, cases[2][1][3], cases[2][1][4]), (1, cases[3][1][3], cases[3][1][4])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):  # every rank agrees on the winner and its schedule
        for (win, seq, sizes), (wwin, wseq, wsizes) in zip(got[rank], want):
            assert win == wwin and seq == list(wseq) and sizes == list(wsizes)
