"""K5, the chain kernel for short queues (n <= 32, csrc/chains_small.cuh): the same chains as K3
in another shape, so (1) each chain follows the sequential model of the chain specification
(tests/k3_model.py) move for move, and (2) K5 and K3 (SLOSCHED_SMALL_KERNEL=0) return the same
winner, scores and counts -- many chains, scale ladders, parked chains, negative exec times."""
import os

import numpy as np
import pytest

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E
from test_gpu_parity import _start_schedule, _three_class

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = E.Engine(0)
    yield e
    e.close()


def _batches(bp, bs):
    out, q = [], 0
    for s in bs:
        out.append([int(x) for x in bp[q:q + s]])
        q += s
    return out


@pytest.mark.parametrize("n,mb,three,kind,chains", [(2, 4, False, "mixed", 2), (3, 4, True, "full", 1),
                                                     (6, 4, False, "mixed", 3), (13, 8, True, "mixed", 2),
                                                     (20, 16, True, "mixed", 1), (31, 2, False, "full", 2),
                                                     (32, 4, True, "mixed", 2), (9, 1, True, "full", 1)])
def test_short_queue_kernel_matches_model(eng, n, mb, three, kind, chains):
    import k3_model as K
    w = _three_class(n, 170 + n) if three else S.generate_mixed(n, 170 + n)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    perm, sizes = _start_schedule(n, mb, kind, n)
    start, q = [], 0
    for s in sizes:
        start.append(perm[q:q + s])
        q += s
    f0 = prob.score(start)[2]
    seed, t0, t_thres, tau, it = 777 + n, 500.0, 20.0, 0.7, 45
    scale = t0 / f0 if f0 > 0 else t0
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=chains, t0=t0, t_thres=t_thres, tau=tau, iter=it, seed=seed,
                                  objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, seed, t0, t_thres, tau, it, scale) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    assert (r.n_met, r.t, r.g) == runs[win]["best"]
    assert _batches(bp, bs) == runs[win]["best_batches"]


def _both(eng, perm, sizes, **kw):
    out = []
    for flag in ("1", "0"):  # K5, then K3
        os.environ["SLOSCHED_SMALL_KERNEL"] = flag
        try:
            bp, bs, r = eng.anneal_chains(perm, sizes, **kw)
        finally:
            os.environ.pop("SLOSCHED_SMALL_KERNEL", None)
        out.append((_batches(bp, bs), r.chain, r.proposals, r.accepted, r.n_met, r.t, r.g, r.chains_run,
                    r.levels_run))
    return out


@pytest.mark.parametrize("n,mb,chains,max_blocks", [(4, 4, 512, 0), (9, 8, 1024, 0), (17, 4, 2048, 0),
                                                    (32, 4, 4096, 0), (12, 4, 700, 2), (5, 1, 256, 0),
                                                    (27, 16, 300, 1)])
def test_short_queue_kernel_matches_k3(eng, n, mb, chains, max_blocks):
    """Many chains over the online driver's scale ladder; max_blocks 1-2 parks chains between levels."""
    w = _three_class(n, 40 + n)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    perm, sizes = _start_schedule(n, mb, "mixed", 3 + n)
    k5, k3 = _both(eng, perm, sizes, chains=chains, t0=500.0, t_thres=20.0, tau=0.7, iter=30, seed=99 + n,
                   objective_scale=1.0, scale_ladder=(1.0, 10.0, 100.0, 1e3, 1e4, 1e5), max_blocks=max_blocks)
    assert k5 == k3


@pytest.mark.parametrize("n,mb,delta_p", [(24, 4, -400.0), (11, 8, -2500.0), (7, 4, -2500.0)])
def test_short_queue_kernel_negative_exec(eng, n, mb, delta_p):
    base = S.table_coefficients()
    c = S.LatencyCoefficients(base.alpha_p, base.beta_p, base.gamma_p, delta_p, base.alpha_d, base.beta_d,
                              base.gamma_d, base.delta_d)
    w = _three_class(n, 90 + n)
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    assert (ex < 0).any()
    eng.set_problem(ex, dl)
    perm, sizes = _start_schedule(n, mb, "mixed", 5)
    k5, k3 = _both(eng, perm, sizes, chains=640, t0=100.0, t_thres=20.0, tau=0.7, iter=30, seed=31 + n,
                   objective_scale=1e4)
    assert k5 == k3


def test_short_queue_near_deadlines_take_the_exact_path(eng):
    """Batches of one (mb = 1): a position's elapsed time is a sum of execs of the requests before
    it. Latest starts set to such sums (the reference's left-to-right fp64 order) put the chains'
    SLO tests on the tick grid's uncertified margin: K5 decides them with the reference's fp64 sum
    and still equals K3."""
    n, mb = 16, 1
    w = S.generate_mixed(n, 5)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    rs = np.random.default_rng(2)
    order = rs.permutation(n)
    sums = np.cumsum(ex[0][order])  # sequential fp64 sums
    dl = dl.copy()
    dl[0] = sums[rs.integers(0, n - 1, size=n)]
    eng.set_problem(ex, dl)
    perm, sizes = [int(x) for x in order], [1] * n
    k5, k3 = _both(eng, perm, sizes, chains=512, t0=200.0, t_thres=20.0, tau=0.7, iter=30, seed=5,
                   objective_scale=1e4)
    assert k5 == k3
    _, _, r = eng.anneal_chains(perm, sizes, chains=512, t0=200.0, t_thres=20.0, tau=0.7, iter=30, seed=5,
                                objective_scale=1e4)
    assert r.exact_walks > 0


def test_short_queues_through_the_public_api():
    """anneal() at online-window sizes: valid schedules, never below the starts, no worse than K3."""
    c = S.table_coefficients()
    for n in (2, 3, 5, 8, 16, 32):
        w = S.generate_mixed(n, n)
        cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=30, chains=max(256, 64 * n), seed=n,
                             scale_ladder=(1.0, 10.0, 100.0, 1e3, 1e4, 1e5))
        r = S.anneal(w, w.ids(), c, cfg, 4)
        assert r.best.schedule.is_partition_of(w.ids(), 4)
        assert r.best.g >= max(r.stats.g_sorted_start, r.stats.g_input_start)
        os.environ["SLOSCHED_SMALL_KERNEL"] = "0"
        try:
            r3 = S.anneal(w, w.ids(), c, cfg, 4)
        finally:
            os.environ.pop("SLOSCHED_SMALL_KERNEL", None)
        assert r.best.schedule.batches == r3.best.schedule.batches and r.best.g == r3.best.g


def test_short_queue_budget_stops_early():
    c = S.table_coefficients()
    w = _three_class(7, 6)  # (the sorted start misses SLOs: no shortcut)
    cfg = S.AnnealConfig(t0=500.0, tau=0.99, iter=2000, chains=256, budget_ms=0.2, seed=1)
    r = S.anneal(w, w.ids(), c, cfg, 4)
    assert 0 < r.stats.proposals < 256 * 2000 * r.stats.levels_run + 1
    assert r.stats.kernel_ms < 0.2 + 0.1
    assert r.best.schedule.is_partition_of(w.ids(), 4)
    assert r.best.g >= max(r.stats.g_sorted_start, r.stats.g_input_start)


def test_short_queue_over_device_groups():
    """K5 behind the multi-device paths: a device list (two contexts on GPU 0, peer exchange) and a
    rank context with an NCCL communicator return the one-context schedule."""
    c = S.table_coefficients()
    w = _three_class(14, 8)
    base = dict(seed=4, chains=777, t0=300.0, iter=30, scale_ladder=(1.0, 1e2, 1e4))
    one = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, device=0), 4)
    two = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, devices=(0, 0)), 4)
    assert two.best.schedule.batches == one.best.schedule.batches and two.best.g == one.best.g
    assert two.stats.best_chain == one.stats.best_chain and two.stats.proposals == one.stats.proposals
    e = E.Engine(0)
    e.comm_init(1, 0, E.comm_unique_id())
    got = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, comm_ctx=e.handle, device=0, chain_begin=0, chain_end=-1), 4)
    assert got.best.schedule.batches == one.best.schedule.batches and got.stats.exchange_ms > 0.0
    e.close()
