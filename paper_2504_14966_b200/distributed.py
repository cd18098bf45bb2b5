"""Multi-GPU annealing: chains shard across ranks, one tiny exchange picks the best.

One process per GPU (torch.distributed, NCCL on GPUs; gloo works for the host logic).
Chain ids are global and every chain's trajectory depends only on (seed, chain id), so the
N-GPU result equals the 1-GPU result over the same chains (tests/test_gpu_parity.py checks
slice independence). The exchange is the one data-path collective of the path:

* all_gather of a 4-double record (engine G, engine t, chain id, rank) per rank,
* every rank picks the same winner: higher G, then lower t, then lower chain id
  (the key of the on-device best-of-chains argmax, engine.cu k_argmax),
* broadcast of the winner's priority sequence and batch sizes (2 x n int32) from its rank.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import List, Sequence, Tuple

import numpy as np


def chain_slice(total_chains: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced slice [begin, end) of the global chain ids for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total_chains, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def pick_winner(records: np.ndarray) -> int:
    """Index of the best row of [g, t, chain, rank] records (g desc, t asc, chain asc)."""
    best = 0
    for r in range(1, len(records)):
        g, t, c = records[r, 0], records[r, 1], records[r, 2]
        bg, bt, bc = records[best, 0], records[best, 1], records[best, 2]
        if g > bg or (g == bg and (t < bt or (t == bt and c < bc))):
            best = r
    return best


@dataclass
class LocalBest:
    g: float                 # engine objective of this rank's best chain
    t: float                 # its summed latency
    chain: int               # its global chain id (-1: no chain ran here)
    sequence: np.ndarray     # priority sequence (request ids), length n
    sizes: np.ndarray        # batch sizes
    exact_g: float = 0.0     # the rank's final (exactly evaluated, floored) objective
    exact_n: int = 0         # and its SLO count


def exchange_best(local: LocalBest, n: int, group=None, device=None, return_record: bool = False):
    """All-gather the per-rank records, agree on the winner rank, broadcast its schedule.

    Returns (winner_rank, sequence, sizes) on every rank, plus the winner's (exact_g, exact_n)
    when return_record is set."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    g = local.g if local.chain >= 0 else -np.inf
    rec = torch.tensor([g, local.t, float(local.chain), float(rank), local.exact_g, float(local.exact_n)],
                       dtype=torch.float64, device=dev)
    allrec = torch.empty(world * 6, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allrec, rec, group=group)
    records = allrec.view(world, 6).cpu().numpy()
    wi = pick_winner(records)
    win = int(records[wi, 3])
    buf = torch.zeros(2 * n + 1, dtype=torch.int32, device=dev)
    if rank == win:
        k = len(local.sizes)
        buf[:n] = torch.as_tensor(np.asarray(local.sequence, dtype=np.int32), device=dev)
        buf[n:n + k] = torch.as_tensor(np.asarray(local.sizes, dtype=np.int32), device=dev)
        buf[2 * n] = k
    dist.broadcast(buf, src=dist.get_global_rank(group, win) if group is not None else win, group=group)
    out = buf.cpu().numpy()
    k = int(out[2 * n])
    if return_record:
        return win, out[:n].copy(), out[n:n + k].copy(), (float(records[wi, 4]), int(records[wi, 5]))
    return win, out[:n].copy(), out[n:n + k].copy()


def anneal_distributed(workload, request_ids: Sequence[int], coeffs, config, max_batch: int, group=None,
                       device_index: int = None):
    """anneal() with config.chains chains sharded over the ranks of `group`; every rank returns
    the same AnnealResult (the best over all chains, floored by the start candidates)."""
    import torch
    import torch.distributed as dist

    from .slosched import AnnealStats, Schedule, _unflatten, anneal_flat, evaluate

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    begin, end = chain_slice(config.chains, rank, world)
    cfg = replace(config, chain_begin=begin, chain_end=end,
                  device=config.device if device_index is None else device_index)
    seq, sizes, n_met, t, g, st = anneal_flat(workload, request_ids, coeffs, cfg, max_batch)
    n = len(request_ids)
    dev = f"cuda:{cfg.device}" if torch.cuda.is_available() and cfg.device >= 0 else None
    if st.shortcut:  # identical on every rank (same start candidates)
        return _result(evaluate(_unflatten(seq, sizes), coeffs, workload), st)
    local = LocalBest(st.engine_g, st.engine_t, st.best_chain, seq, sizes)
    _, wseq, wsizes = exchange_best(local, n, group=group, device=dev)
    # summed counters over all ranks
    cnt = torch.tensor([float(st.proposals), float(st.accepted), float(st.chains_run)], dtype=torch.float64,
                       device=dev or "cpu")
    dist.all_reduce(cnt, group=group)
    stats = replace(st, proposals=int(cnt[0]), accepted=int(cnt[1]), chains_run=int(cnt[2]))
    return _result(evaluate(_unflatten(wseq, wsizes), coeffs, workload), stats)


def _result(best, stats):
    from .slosched import AnnealResult
    return AnnealResult(best, stats)
