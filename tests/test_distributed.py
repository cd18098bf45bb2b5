"""Multi-GPU host logic on CPU: chain sharding, the slot protocol of the device-side exchange
(csrc/exchange.cuh, restated in numpy by distributed.pack_slot / pick_slot) and the unique-id
distribution, run as a real world_size-2 process group over gloo (127.0.0.1). The GPU side of the
same path (NCCL communicator, device exchange) is covered in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_14966_b200.distributed import chain_slice, pack_slot, pick_slot, pick_winner, slot_bytes


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
    rec = np.array([[5.0, 0.0, -1, 0], [1e-7, 1.0, 0, 1]])
    assert pick_winner(rec) == 1  # a rank that ran no chain never wins
    assert pick_winner(np.array([[0.0, 0.0, -1], [0.0, 0.0, -1]])) == -1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, out_q):
    import torch
    import torch.distributed as dist

    from paper_2504_14966_b200.distributed import share_unique_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = share_unique_id(lambda: bytes(range(128)))
        results = []
        for case in cases:
            g, t, chain, ent, bits = case[rank]
            slot = pack_slot(g, t, chain, np.asarray(ent, dtype=np.uint16), np.asarray(bits, dtype=np.uint32),
                             proposals=100 + rank)
            mine = torch.frombuffer(bytearray(slot), dtype=torch.uint8)
            allb = torch.empty(world * len(slot), dtype=torch.uint8)
            dist.all_gather_into_tensor(allb, mine)
            w, head, went, wbits, props = pick_slot(allb.numpy().tobytes(), world)
            results.append((w, None if head is None else head[2], None if went is None else went[:len(ent)].tolist(),
                            None if wbits is None else wbits[:len(bits)].tolist(), props))
        out_q.put((rank, uid, results))
    finally:
        dist.destroy_process_group()


def test_slot_size_matches_engine_layout():
    # ExHead (128 B) + 1024*U 16-bit entries + 32*U 32-bit words, rounded to 128 B
    assert slot_bytes(1) == 128 + 2048 + 128
    assert slot_bytes(4) == 128 + 8192 + 512


def test_exchange_world_size_2_gloo():
    cases = [
        # rank 1 has the higher G
        [(1e-6, 100.0, 5, [0, 1, 2, 3], [8]), (2e-6, 90.0, 9, [3, 2, 1, 0], [9])],
        # equal G: lower t wins
        [(3e-6, 80.0, 1, [1, 0, 2, 3], [10]), (3e-6, 81.0, 0, [0, 1, 2, 3], [8])],
        # equal G and t: lower chain id wins
        [(3e-6, 80.0, 11, [2, 1, 0, 3], [12]), (3e-6, 80.0, 10, [3, 0, 1, 2], [10])],
        # a rank that ran no chain never wins
        [(0.0, 0.0, -1, [0, 0, 0, 0], [0]), (0.0, 50.0, 2, [2, 0, 3, 1], [15])],
        # nobody ran a chain
        [(0.0, 0.0, -1, [0, 0, 0, 0], [0]), (0.0, 0.0, -1, [0, 0, 0, 0], [0])],
    ]
    want = [(1, 9, [3, 2, 1, 0], [9]), (0, 1, [1, 0, 2, 3], [10]), (1, 10, [3, 0, 1, 2], [10]),
            (1, 2, [2, 0, 3, 1], [15]), (-1, None, None, None)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {r: (uid, res) for r, uid, res in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):  # every rank holds rank 0's id and agrees on the winner and its schedule
        uid, res = got[rank]
        assert uid == bytes(range(128))
        for k, ((w, chain, ent, bits, props), want_k) in enumerate(zip(res, want)):
            assert (w, chain, ent, bits) == want_k
            ran = [r for r in (0, 1) if cases[k][r][2] >= 0]
            assert props == sum(100 + r for r in ran)
