"""Multi-GPU annealing, one process per GPU: chains shard across ranks, one device-side exchange
picks the best.

The exchange itself lives in the engine (csrc/exchange.cuh): every rank's context carries an
NCCL communicator (slo_ctx_comm_init), and the chain launch enqueues, behind the rank's own
best-of-chains, an all-gather of one slot per rank (header + winner state) and an on-device
pick -- nothing crosses the host between the chain kernel and the job-wide winner. This module
is the torch.distributed plumbing around it: the NCCL unique id travels over the process group
once, and `anneal_distributed` is `anneal()` with the rank's context.

Chain ids are global and each chain's moves depend only on (seed, chain id), so the N-rank job
runs exactly the chains one device would run over the same ids (tests/test_gpu_parity.py).

`pack_slot` / `pick_slot` restate the slot format and the pick order of k_pack / k_pick in numpy:
the checker of the multi-rank tests (tests/test_distributed.py), never on the product path.
"""
from __future__ import annotations

import os
import struct
from dataclasses import replace
from typing import List, Optional, Sequence, Tuple

import numpy as np


def chain_slice(total_chains: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced slice [begin, end) of the global chain ids for `rank` (the split the
    engine applies to a rank context with chain_end < 0, and slo_group_anneal_chains per member)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total_chains, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def pick_winner(records: np.ndarray) -> int:
    """Index of the best row of [g, t, chain] records (g desc, t asc, chain asc; chain < 0 = a rank
    that ran no chain, never picked unless every row is empty) -- k_pick's order."""
    best = -1
    for r in range(len(records)):
        g, t, c = records[r, 0], records[r, 1], records[r, 2]
        if c < 0:
            continue
        if best < 0:
            best = r
            continue
        bg, bt, bc = records[best, 0], records[best, 1], records[best, 2]
        if g > bg or (g == bg and (t < bt or (t == bt and c < bc))):
            best = r
    return best


# ---- slot format of csrc/exchange.cuh (ExHead + entries + batch-end bits), for the checkers
_HEAD = struct.Struct("<ddq5Q4i6Q")  # g, t, chain, proposals, accepted, scan1, scan2, exact, n_met, runs, lev, pad


def slot_bytes(units_per_lane: int) -> int:
    ew, bw = 1024 * units_per_lane, 32 * units_per_lane
    return (128 + ew * 2 + bw * 4 + 127) & ~127


def pack_slot(g: float, t: float, chain: int, entries: np.ndarray, bits: np.ndarray, units_per_lane: int = 1,
              proposals: int = 0, n_met: int = 0) -> bytes:
    buf = bytearray(slot_bytes(units_per_lane))
    _HEAD.pack_into(buf, 0, g, t, chain, proposals, 0, 0, 0, 0, n_met, 1 if chain >= 0 else 0, 1, 0, 0, 0, 0, 0, 0, 0)
    e = np.zeros(1024 * units_per_lane, dtype=np.uint16)
    e[:len(entries)] = entries
    b = np.zeros(32 * units_per_lane, dtype=np.uint32)
    b[:len(bits)] = bits
    buf[128:128 + e.nbytes] = e.tobytes()
    buf[128 + e.nbytes:128 + e.nbytes + b.nbytes] = b.tobytes()
    return bytes(buf)


def pick_slot(gathered: bytes, nslots: int, units_per_lane: int = 1):
    """(winner slot index, header tuple, entries, bits, summed proposals) of gathered slots."""
    sb = slot_bytes(units_per_lane)
    heads = [_HEAD.unpack_from(gathered, s * sb) for s in range(nslots)]
    w = pick_winner(np.array([[h[0], h[1], h[2]] for h in heads], dtype=np.float64))
    props = sum(h[3] for h in heads if h[2] >= 0)
    if w < 0:
        return -1, None, None, None, props
    off = w * sb + 128
    ew = 1024 * units_per_lane
    ent = np.frombuffer(gathered, dtype=np.uint16, count=ew, offset=off)
    bits = np.frombuffer(gathered, dtype=np.uint32, count=32 * units_per_lane, offset=off + 2 * ew)
    return w, heads[w], ent, bits, props


# ---- torch.distributed plumbing
def share_unique_id(make_id, group=None) -> bytes:
    """Rank 0 of `group` makes the id (make_id()), every rank returns it (one object broadcast)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    obj: List[Optional[bytes]] = [make_id() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def local_device(device: int = -1) -> int:
    """The rank's GPU: the requested one, else torch's current device, else LOCAL_RANK."""
    if device is not None and device >= 0:
        return device
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:
        pass
    return int(os.environ.get("LOCAL_RANK", "0"))


class RankComm:
    """This rank's engine context with an NCCL communicator over the ranks of `group`
    (collective: every rank constructs it). `handle` goes into AnnealConfig.comm_ctx."""

    def __init__(self, device: int = -1, group=None):
        import torch.distributed as dist

        from .engine import Engine, comm_unique_id

        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.device = local_device(device)
        uid = share_unique_id(comm_unique_id, group)
        self.engine = Engine(self.device)
        self.engine.comm_init(self.world, self.rank, uid)

    @property
    def handle(self) -> int:
        return self.engine.handle

    def close(self):
        self.engine.close()


def anneal_distributed(workload, request_ids: Sequence[int], coeffs, config, max_batch: int, group=None,
                       comm: Optional[RankComm] = None):
    """anneal() with config.chains chains sharded over the ranks of `group`; every rank returns the
    same AnnealResult (the job-wide best chain, floored by the start candidates). Pass a RankComm to
    reuse its communicator across calls (creating one is a collective of tens of ms)."""
    from .slosched import anneal

    own = comm is None
    if own:
        comm = RankComm(config.device, group)
    try:
        cfg = replace(config, comm_ctx=comm.handle, device=comm.device, devices=(), chain_begin=0, chain_end=-1)
        return anneal(workload, request_ids, coeffs, cfg, max_batch)
    finally:
        if own:
            comm.close()
