"""GPU parity: the CUDA path (through the C ABI) against the oracle and the golden vectors.

1. K1 slo_evaluate_batch vs the oracle's CostModel::score -- n_met, t, g bit-exact.
2. K2 replay (xoshiro) vs the reference walk -- identical final schedule, n, t, g,
   proposals and accepted counts (golden vectors + live oracle port, many seeds).
3. K3/K4 chains (Philox) -- valid partitions, never below either start, deterministic,
   independent of how chains are sliced; the engine's incremental objective is bit-exact
   against a full evaluation of its winner on the tick grid (and within the grid's rounding
   of the exact objective); attainment >= the reference's single chain.
"""
import math

import numpy as np
import pytest

from conftest import golden, unhex
from oracle import TABLE_COEFFS, FlatWorkload

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E

pytestmark = pytest.mark.gpu


def _flat(w: S.Workload) -> FlatWorkload:
    a = w.arrays
    return FlatWorkload(id=a["id"], cls=a["cls"], in_len=a["in_len"], true_out=a["true_out"], pred_out=a["pred_out"],
                        arrival=a["arrival"], class_id=a["class_id"], kind=a["kind"], e2e=a["e2e"], ttft=a["ttft"],
                        tpot=a["tpot"])


def _three_class(n, seed):
    """Config-1 style queue: code (E2E 30 s) / chat (TTFT 10 s + TPOT 50 ms) / offline (E2E 1e9)."""
    base = S.generate_mixed(n, seed)
    code, chat = S.default_slo_classes()
    offline = S.TaskClass(2, "offline", S.SloSpec.e2e(1e9))
    reqs = [S.Request(r.id, 2 if r.id % 3 == 2 else r.task_class_id, r.input_len, r.true_output_len,
                      r.predicted_output_len) for r in base.requests]
    return S.Workload(reqs, [code, chat, offline])


def _random_partitions(rs, n, mb, count):
    perms = np.stack([rs.permutation(n) for _ in range(count)]).astype(np.uint16)
    sizes = []
    for _ in range(count):
        s, left = [], n
        while left:
            k = int(rs.integers(1, min(mb, left) + 1))
            s.append(k)
            left -= k
        sizes.append(s)
    return perms, sizes


@pytest.fixture(scope="module")
def eng():
    e = E.Engine(0)
    yield e
    e.close()


# ---------------------------------------------------------------- K1
@pytest.mark.parametrize("n,mb,count", [(1, 1, 4), (8, 2, 500), (64, 4, 2000), (256, 4, 100000), (256, 8, 20000),
                                        (1024, 4, 2000), (300, 16, 500), (4096, 4, 64)])
def test_evaluate_batch_bit_exact(eng, port, n, mb, count):
    w = _three_class(n, 1000 + n)
    c = S.table_coefficients()
    ex, dl = E.build_tables(w, w.ids(), c, mb)
    eng.set_problem(ex, dl)
    rs = np.random.default_rng(n * mb)
    perms, sizes = _random_partitions(rs, n, mb, count)
    n_met, t, g = eng.evaluate_batch(perms, E.end_bits(sizes, n))
    o_n, o_t, o_g = port.score_batch(_flat(w), TABLE_COEFFS, sorted(w.ids()), mb, perms.astype(np.int32), sizes)
    np.testing.assert_array_equal(n_met, o_n)
    np.testing.assert_array_equal(t, o_t)  # bit-exact, not approx
    np.testing.assert_array_equal(g, o_g)


def test_evaluate_batch_matches_public_evaluate(eng):
    w = S.generate_mixed(100, 5)
    c = S.table_coefficients()
    ex, dl = E.build_tables(w, w.ids(), c, 4)
    eng.set_problem(ex, dl)
    rs = np.random.default_rng(9)
    perms, sizes = _random_partitions(rs, 100, 4, 50)
    n_met, t, g = eng.evaluate_batch(perms, E.end_bits(sizes, 100))
    ids = sorted(w.ids())
    for q in range(50):
        flat = [ids[i] for i in perms[q]]
        batches, pos = [], 0
        for s in sizes[q]:
            batches.append(flat[pos:pos + s])
            pos += s
        ev = S.evaluate(S.Schedule(batches), c, w)
        assert (ev.n, ev.t_ms, ev.g) == (n_met[q], t[q], g[q])


def test_evaluate_batch_rejects_bad_input(eng):
    w = S.generate_mixed(10, 1)
    ex, dl = E.build_tables(w, w.ids(), S.table_coefficients(), 2)
    eng.set_problem(ex, dl)
    perm = np.arange(10, dtype=np.uint16)[None]
    with pytest.raises(S.DataError):  # batch of 3 > mb
        eng.evaluate_batch(perm, E.end_bits([[3, 3, 2, 2]], 10))
    with pytest.raises(S.DataError):  # last position not a batch end
        eng.evaluate_batch(perm, np.zeros((1, 1), dtype=np.uint32))
    bad = perm.copy()
    bad[0, 4] = 10
    with pytest.raises(S.DataError):  # dense index out of range
        eng.evaluate_batch(bad, E.end_bits([[2] * 5], 10))
    # validation runs on the device, per candidate: one bad row among good ones still fails the call
    rows = np.repeat(perm, 64, axis=0)
    rows[37, 2] = 11
    with pytest.raises(S.DataError):
        eng.evaluate_batch(rows, E.end_bits([[2] * 5] * 64, 10))
    nm, t, g = eng.evaluate_batch(np.repeat(perm, 64, axis=0), E.end_bits([[2] * 5] * 64, 10))
    assert (nm == nm[0]).all() and (t == t[0]).all()


# ---------------------------------------------------------------- K2 replay
def _replay_cfg(seed, **kw):
    return S.AnnealConfig(seed=seed, mode=S.SearchMode.REPLAY, **kw)


def test_replay_matches_golden_anneal():
    c = S.table_coefficients()
    for case in golden("anneal"):
        w = S.generate_mixed(case["n"], case["wseed"])
        res = S.anneal(w, w.ids(), c, _replay_cfg(case["seed"], **case["cfg"]), case["mb"])
        assert res.best.schedule.batches == case["batches"], case
        assert res.best.n == case["n_met"]
        assert res.best.g == unhex(case["g"]) and res.best.t_ms == unhex(case["t"])
        assert res.stats.shortcut == case["shortcut"]
        if not case["shortcut"]:
            assert res.stats.proposals == case["proposals"] and res.stats.accepted == case["accepted"]
        assert res.stats.objective_scale_used == unhex(case["scale"])


@pytest.mark.parametrize("n", [8, 64, 256])
@pytest.mark.parametrize("mb", [1, 2, 4])
def test_replay_matches_oracle_many_seeds(port, n, mb):
    c = S.table_coefficients()
    w = _three_class(n, 77 + n)
    fw = _flat(w)
    seeds = range(20) if n < 256 else range(4)
    cfg = {} if n < 256 else {"t0": 100.0, "iter": 30}
    for seed in seeds:
        res = S.anneal(w, w.ids(), c, _replay_cfg(seed, **cfg), mb)
        o = port.anneal(fw, TABLE_COEFFS, w.ids(), mb, seed=seed, **cfg)
        assert res.best.schedule.batches == o["batches"], (n, mb, seed)
        assert (res.best.n, res.best.t_ms, res.best.g) == (o["n"], o["t"], o["g"])
        assert (res.stats.proposals, res.stats.accepted) == (o["proposals"], o["accepted"])


@pytest.mark.parametrize("n,mb", [(200, 8), (150, 16), (1024, 4), (61, 16)])
def test_replay_long_batches_and_full_size(port, n, mb):
    """K2's staged operands across long batches (a swap restages two 16-position batches, a squeeze
    or delay up to 32 positions) and at the headline size: the reference walk, bit for bit."""
    c = S.table_coefficients()
    w = _three_class(n, 5 + n)
    fw = _flat(w)
    cfg = {"t0": 100.0, "iter": 40} if n >= 1024 else {}
    for seed in (0, 1, 2):
        res = S.anneal(w, w.ids(), c, _replay_cfg(seed, **cfg), mb)
        o = port.anneal(fw, TABLE_COEFFS, w.ids(), mb, seed=seed, **cfg)
        assert res.best.schedule.batches == o["batches"], (n, mb, seed)
        assert (res.best.n, res.best.t_ms, res.best.g) == (o["n"], o["t"], o["g"])
        assert (res.stats.proposals, res.stats.accepted) == (o["proposals"], o["accepted"])


def test_replay_many_chains_in_one_launch(eng, port):
    """K2 with C chains: chain c reproduces the reference walk with seed + c."""
    n, mb = 48, 4
    w = S.generate_mixed(n, 3)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    s, i = S.initial_candidates(w, ids, c, mb)
    gs, gi = S.evaluate(s, c, w).g, S.evaluate(i, c, w).g
    st = s if gs >= gi else i
    start = [ids.index(x) for x in st.flatten()]
    sizes = [len(b) for b in st.batches]
    g0 = max(gs, gi)
    bp, bs, res = eng.anneal_chains(start, sizes, t0=80.0, iter=20, seed=11, objective_scale=80.0 / g0, replay=True,
                                    chains=16)
    levels, t = 0, 80.0
    while t >= 20.0:
        levels, t = levels + 1, t * 0.95
    assert res.chains_run == 16 and res.proposals == 16 * levels * 20
    fw = _flat(w)
    best = max(range(16), key=lambda k: (port.anneal(fw, TABLE_COEFFS, ids, mb, seed=11 + k, t0=80.0, iter=20,
                                                     objective_scale=80.0 / g0)["g"], -k))
    assert res.chain == best


def test_reference_binding_drop_in(ref):
    """integration/reference_anneal_gpu.cpp compiled into the unmodified reference: the
    reference's own anneal() types routed through the C ABI give the reference's result
    (replay) and a dominant result (chains)."""
    from oracle import refshim
    if not refshim.available():
        pytest.skip("oracle/_ref/libslosched_refshim.so not built")
    for n, mb, seed in [(16, 2, 0), (64, 4, 3), (200, 8, 7)]:
        fw = ref.generate_mixed(n, 50 + n, 1)
        ids = list(fw.id)
        want = ref.anneal(fw, TABLE_COEFFS, ids, mb, seed=seed, t0=200.0, iter=50)
        got = refshim.anneal_gpu(fw, TABLE_COEFFS, ids, mb, seed=seed, mode=1, t0=200.0, iter=50)
        assert got["batches"] == want["batches"] and got["g"] == want["g"] and got["n"] == want["n"]
        assert (got["proposals"], got["accepted"]) == (want["proposals"], want["accepted"])
        many = refshim.anneal_gpu(fw, TABLE_COEFFS, ids, mb, seed=seed, mode=0, chains=512, t0=200.0, iter=50)
        assert many["g"] >= max(want["g_sorted_start"], want["g_input_start"])


def test_schedule_all_replay_matches_golden():
    c = S.table_coefficients()
    for case in golden("schedule_all"):
        w = S.generate_mixed(case["n"], case["wseed"])
        insts = [S.InstanceState(i, 2**35, 2**35, 0.9, 262144.0, case["mb"]) for i in range(case["k"])]
        res = S.schedule_all(w, insts, c, _replay_cfg(case["seed"]))
        assert res.epochs == case["epochs"]
        for got, want in zip(res.per_instance, case["per_instance"]):
            assert got.schedule.batches == want["batches"]
            assert got.n == want["n_met"] and got.g == unhex(want["g"])


def test_schedule_all_concurrent_instances_equal_sequential():
    """Chains mode: the k per-instance anneals run concurrently (own thread, context, stream and
    1/k of the SMs); chain results do not depend on the grid, so the schedules are identical to
    one-after-another runs, and every instance result dominates its starts."""
    c = S.table_coefficients()
    w = _three_class(160, 12)
    insts = [S.InstanceState(i, 2**35, 2**35, 0.9, 262144.0, 4) for i in range(4)]
    base = dict(seed=5, chains=1024, t0=100.0, iter=30, scale_ladder=(1.0, 100.0, 1e4))
    conc = S.schedule_all(w, insts, c, S.AnnealConfig(**base))
    seq = S.schedule_all(w, insts, c, S.AnnealConfig(**base, sequential_instances=True))
    assert conc.epochs == seq.epochs
    for a, b in zip(conc.per_instance, seq.per_instance):
        assert a.schedule.batches == b.schedule.batches and a.g == b.g
    ids = sorted(i for ev in conc.per_instance for i in ev.schedule.flatten())
    assert ids == sorted(w.ids())


def test_cpp_example_runs_against_the_cpp_api(port):
    """examples/anneal_example.cpp: a C++ caller of include/slosched_b200.hpp (no Python)."""
    import os
    import re
    import subprocess

    from conftest import ROOT
    exe = os.path.join(ROOT, "examples", "_build", "anneal_example")
    if not os.path.exists(exe):
        pytest.skip("example not built")
    out = subprocess.run([exe, "256"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rep = re.search(r"replay: n_met=(\d+) g=(\S+) proposals=(\d+) accepted=(\d+)", out.stdout)
    w = S.generate_mixed(256, 0)
    o = port.anneal(_flat(w), TABLE_COEFFS, w.ids(), 4, seed=0)
    assert int(rep.group(1)) == o["n"] and float(rep.group(2)) == float(f"{o['g']:.9e}")
    assert (int(rep.group(3)), int(rep.group(4))) == (o["proposals"], o["accepted"])
    assert "schedule_all: instances=4" in out.stdout


def test_distributed_path_over_nccl_single_rank():
    """The multi-process path on real NCCL (one rank here: the box has one GPU per call): the rank
    context's communicator (slo_ctx_comm_init, id shared over torch.distributed), the device-side
    exchange enqueued behind the chains, and anneal_distributed == anneal over the same chains."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2504_14966_b200.distributed import RankComm, anneal_distributed

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        c = S.table_coefficients()
        w = _three_class(96, 31)
        cfg = S.AnnealConfig(seed=2, chains=512, t0=80.0, iter=20, scale_ladder=(1.0, 1e3), device=0)
        want = S.anneal(w, w.ids(), c, cfg, 4)
        comm = RankComm(0)
        assert comm.engine.comm_info() == (1, 0)
        for _ in range(2):  # the communicator is reused across calls
            got = anneal_distributed(w, w.ids(), c, cfg, 4, comm=comm)
            assert got.best.schedule.batches == want.best.schedule.batches and got.best.g == want.best.g
            assert got.stats.proposals == want.stats.proposals and got.stats.best_chain == want.stats.best_chain
            assert got.stats.devices == 1 and got.stats.exchange_ms > 0.0
        comm.engine.comm_check()
        comm.close()
        got = anneal_distributed(w, w.ids(), c, cfg, 4)  # a communicator of its own
        assert got.best.schedule.batches == want.best.schedule.batches
    finally:
        dist.destroy_process_group()


def test_rank_with_empty_slice_takes_part_in_the_exchange():
    """A rank given no chain (fewer chains than ranks) still contributes an empty slot; with no
    chain anywhere the fetch reports it instead of returning garbage."""
    w = _three_class(64, 5)
    c = S.table_coefficients()
    e = E.Engine(0)
    e.comm_init(1, 0, E.comm_unique_id())
    ex, dl = E.build_tables(w, w.ids(), c, 4)
    e.set_problem(ex, dl)
    s_sched, _ = S.initial_candidates(w, w.ids(), c, 4)
    pos = {rid: k for k, rid in enumerate(sorted(w.ids()))}
    sp, ss = [pos[x] for x in s_sched.flatten()], [len(b) for b in s_sched.batches]
    e.prepare(sp, ss, t0=50.0, iter=5, chains=4, chain_begin=0, chain_end=0, objective_scale=1e6)
    e.launch()
    with pytest.raises(Exception, match="no chain"):
        e.fetch()
    e.prepare(sp, ss, t0=50.0, iter=5, chains=4, chain_begin=0, chain_end=4, objective_scale=1e6)
    e.launch()
    _, _, res = e.fetch()
    assert res.nranks == 1 and res.chains_run == 4 and 0 <= res.chain < 4
    # a rank that failed before its launch joins the exchange with an empty slot
    from paper_2504_14966_b200._lib import lib
    assert lib().slo_ctx_exchange_empty(e._ctx, 64) == 0
    with pytest.raises(Exception, match="prepared|no chain"):
        e.fetch()
    e.close()


def test_device_group_equals_one_context():
    """anneal() over a device list (here two contexts on GPU 0: the peer-copy exchange) returns the
    schedule one context returns over the same chain ids; Group{0} runs the NCCL transport."""
    c = S.table_coefficients()
    w = _three_class(300, 8)
    base = dict(seed=4, chains=2049, t0=120.0, iter=25, scale_ladder=(1.0, 1e4))
    one = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, device=0), 4)
    two = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, devices=(0, 0)), 4)
    assert two.best.schedule.batches == one.best.schedule.batches and two.best.g == one.best.g
    assert two.stats.best_chain == one.stats.best_chain and two.stats.proposals == one.stats.proposals
    assert two.stats.devices == 2
    g = E.Group([0])
    assert g.transport == "nccl"
    g.close()
    g = E.Group([0, 0])
    assert g.transport == "peer"
    g.close()


def test_cpp_multi_gpu_example():
    """examples/multi_gpu_example.cpp: the C++ entry point over device groups ({0}: NCCL with one
    device, {0,0} / {0,0,0}: two / three contexts on one GPU) and schedule_all placement."""
    import os
    import subprocess

    from conftest import ROOT
    exe = os.path.join(ROOT, "examples", "_build", "multi_gpu_example")
    if not os.path.exists(exe):
        pytest.skip("example not built")
    out = subprocess.run([exe, "400"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") >= 5 and "FAIL" not in out.stdout


# ---------------------------------------------------------------- exhaustive oracle
def test_exhaustive_matches_golden():
    c = S.table_coefficients()
    for case in golden("exhaustive"):
        w = S.generate_mixed(case["n"], case["seed"], predict=False)
        r = S.exhaustive(w, w.ids(), c, case["mb"])
        assert r.best.schedule.batches == case["batches"]
        assert r.best.n == case["n_met"] and r.best.g == unhex(case["g"])
        assert r.schedules_evaluated == case["evaluated"]


def test_exhaustive_counts_ties_and_cap():
    c = S.table_coefficients()
    assert S.exhaustive(S.generate_mixed(1, 0, predict=False), [0], c, 1).schedules_evaluated == 1
    w3 = S.generate_mixed(3, 1, predict=False)
    assert S.exhaustive(w3, w3.ids(), c, 1).schedules_evaluated == 6
    assert S.exhaustive(w3, w3.ids(), c, 3).schedules_evaluated == 24
    loose = S.TaskClass(0, "loose", S.SloSpec.e2e(1e9))  # indistinguishable requests: lexicographic tie-break
    w = S.Workload([S.Request(i, 0, 100, 10, 10) for i in range(3)], [loose])
    assert S.exhaustive(w, [0, 1, 2], c, 1).best.schedule.flatten() == [0, 1, 2]
    w12 = S.generate_mixed(12, 2)
    with pytest.raises(S.CapacityError, match="exceed"):
        S.exhaustive(w12, w12.ids(), c, 1, 10)
    empty = S.Workload([], list(S.default_slo_classes()))
    r = S.exhaustive(empty, [], c, 2)
    assert r.best.schedule.batches == [] and r.schedules_evaluated == 1


@pytest.mark.parametrize("n,mb", [(5, 2), (7, 3), (8, 2), (9, 1), (11, 1)])
def test_exhaustive_matches_reference_live(ref, n, mb):
    c = S.table_coefficients()
    for seed in (3, 4):
        fw = ref.generate_mixed(n, 500 + seed, 1)
        want = ref.exhaustive(fw, TABLE_COEFFS, list(fw.id), mb, n_cap=12)
        w = S.generate_mixed(n, 500 + seed)
        got = S.exhaustive(w, w.ids(), c, mb, n_cap=12)
        assert got.best.schedule.batches == want["batches"]
        assert (got.best.n, got.best.g, got.schedules_evaluated) == (want["n"], want["g"], want["evaluated"])


def test_sa_reaches_exhaustive_parity():
    """Acceptance criterion 1 (P:tests/acceptance/acceptance.cpp:83-113): n in {4,6,8,10}, mb 1,
    20 seeds: G >= 0.99 x exhaustive on >= 90 % of runs, attainment equal at n in {4,6} -- here with
    GPU chains, and exhaustive is never beaten."""
    c = S.table_coefficients()
    ok = total = 0
    for n in (4, 6, 8, 10):
        for s in range(20):
            w = S.generate_mixed(n, 1000 * n + s)
            sa = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=s, chains=256), 1)
            ex = S.exhaustive(w, w.ids(), c, 1)
            assert sa.best.g <= ex.best.g * (1 + 1e-12)
            total += 1
            ok += sa.best.g >= 0.99 * ex.best.g if ex.best.g > 0 else sa.best.g >= ex.best.g
            if n in (4, 6):
                assert sa.best.n == ex.best.n
    assert ok >= 0.9 * total


# ---------------------------------------------------------------- K3/K4 chains
@pytest.mark.parametrize("n,mb,chains", [(2, 2, 8), (9, 3, 64), (64, 4, 512), (256, 4, 1024), (1024, 4, 256),
                                         (200, 16, 128), (4096, 4, 32)])
def test_chains_valid_and_dominant(n, mb, chains):
    c = S.table_coefficients()
    w = _three_class(n, 5 + n)
    cfg = S.AnnealConfig(seed=3, chains=chains, t0=100.0, iter=20 if n < 4096 else 5)
    res = S.anneal(w, w.ids(), c, cfg, mb)
    assert res.best.schedule.is_partition_of(w.ids(), mb)
    if not res.stats.shortcut:
        assert res.best.g >= res.stats.g_sorted_start and res.best.g >= res.stats.g_input_start
        assert res.best.g >= res.stats.g_deadline_start > 0.0  # the third start is a floor too
        assert res.stats.chains_run == chains
        assert res.stats.proposals == chains * res.stats.levels_run * cfg.iter
        # the engine's objective (exec rounded to a 2^-k ms grid, max exec < 2^27 ticks) is within
        # the grid's rounding of the exact evaluation of its winner
        if res.best.g > max(res.stats.g_sorted_start, res.stats.g_input_start, res.stats.g_deadline_start):
            assert abs(res.stats.engine_g - res.best.g) <= 2.0 ** -26 * res.best.g


@pytest.mark.parametrize("n,mb", [(256, 4), (1024, 4), (1024, 8), (3000, 4)])
def test_chain_winner_objective_matches_exact_evaluation(n, mb):
    """Whichever start wins the final floor, the engine's own winner -- fetched through the engine
    C ABI -- has the n_met of the reference's evaluate() exactly and t within 2^-26."""
    c = S.table_coefficients()
    w = _three_class(n, 77 + n)
    ids = sorted(w.ids())
    s_sched, i_sched = S.initial_candidates(w, ids, c, mb)
    ev = max([S.evaluate(x, c, w) for x in (s_sched, i_sched, S.deadline_first_candidate(w, ids, c, mb))],
             key=lambda e: e.g)
    pos = {r: k for k, r in enumerate(ids)}
    eng = E.Engine(0)
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    bp, bs, res = eng.anneal_chains([pos[x] for x in ev.schedule.flatten()], [len(b) for b in ev.schedule.batches],
                                    t0=200.0, iter=40, seed=9, objective_scale=1e6 * 200.0 / ev.g, chains=2048,
                                    scale_ladder=(1.0, 100.0))
    eng.close()
    sched = S.Schedule([[ids[k] for k in bp[p0:p0 + z]] for p0, z in zip(np.cumsum([0] + list(bs[:-1])), bs)])
    exact = S.evaluate(sched, c, w)
    assert res.n_met == exact.n
    assert abs(res.t - exact.t_ms) <= 2.0 ** -26 * exact.t_ms


def tick_objective(ex, dl, tick, perm, sizes):
    """Full evaluation with the chain kernel's arithmetic: the total latency in Python integers on
    the grid (exec rounded half-even to ticks); n_met the reference's (fp64 elapsed, summed left to
    right, <= the fp64 latest start; +inf deadlines always met)."""
    xt = np.rint(ex / tick).astype(np.int64)
    elapsed = total = met = pos = 0
    elapsed_f = 0.0
    for sz in sizes:
        mk, mk_f = 0, 0.0
        for _ in range(sz):
            i = int(perm[pos]); pos += 1
            x = int(xt[sz - 1, i]); d = float(dl[sz - 1, i])
            total += elapsed + x
            met += elapsed_f <= d
            mk = max(mk, x)
            e = float(ex[sz - 1, i])
            mk_f = e if mk_f < e else mk_f
        elapsed += mk
        elapsed_f = elapsed_f + mk_f
    t = float(total) * tick
    return met, t, (met * (1.0 / t) if t > 0 else 0.0)


@pytest.mark.parametrize("n,mb,chains,three", [(64, 4, 256, True), (256, 4, 1024, False), (1024, 4, 2048, False),
                                               (1024, 8, 512, True), (200, 16, 256, True), (4096, 4, 64, False)])
def test_chains_objective_is_tick_exact(eng, n, mb, chains, three):
    """The winner's (n_met, t, g) reported by the kernel -- accumulated move by move from the
    few batches each move rebuilds -- equals a from-scratch evaluation of the winning schedule on
    the same grid, bit for bit."""
    w = _three_class(n, 40 + n) if three else S.generate_mixed(n, 40 + n)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    tick = eng.tick_ms
    assert tick > 0 and np.rint(ex / tick).max() < 2 ** 27 and np.log2(tick) == int(np.log2(tick))
    s, _ = S.initial_candidates(w, ids, c, mb)
    start = [ids.index(x) for x in s.flatten()]
    sizes = [len(b) for b in s.batches]
    bp, bs, r = eng.anneal_chains(start, sizes, chains=chains, t0=200.0, iter=30, seed=11, objective_scale=1e7,
                                  scale_ladder=(1e-3, 1.0, 1e3))
    assert sorted(bp.tolist()) == list(range(n)) and bs.sum() == n and bs.max() <= mb
    nm, t, g = tick_objective(ex, dl, tick, bp, bs)
    assert (r.n_met, r.t, r.g) == (nm, t, g)
    assert r.proposals == chains * r.levels_run * 30


def test_chains_deterministic_and_slice_independent():
    c = S.table_coefficients()
    w = _three_class(128, 21)
    base = dict(seed=9, chains=300, t0=60.0, iter=25, scale_ladder=(1.0, 100.0, 1e4))
    a = S.anneal(w, w.ids(), c, S.AnnealConfig(**base), 4)
    b = S.anneal(w, w.ids(), c, S.AnnealConfig(**base), 4)
    assert a.best.schedule.batches == b.best.schedule.batches
    a.stats.kernel_ms = b.stats.kernel_ms = 0.0  # device timing is the only non-deterministic field
    assert a.stats == b.stats
    # the same 300 chains split over two "devices": the better half-winner is the full winner
    h1 = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, chain_begin=0, chain_end=150), 4)
    h2 = S.anneal(w, w.ids(), c, S.AnnealConfig(**base, chain_begin=150, chain_end=300), 4)
    win = max((h1, h2), key=lambda r: (r.stats.engine_g, -r.best.t_ms, -r.stats.best_chain))
    assert win.stats.best_chain == a.stats.best_chain
    assert win.best.schedule.batches == a.best.schedule.batches


def test_chains_state_parking_is_transparent(eng):
    """More chains than resident warps (state parked in HBM between levels) gives each chain
    exactly the trajectory it has when it stays resident."""
    n, mb = 256, 4
    w = _three_class(n, 8)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    s, _ = S.initial_candidates(w, ids, c, mb)
    start = [ids.index(x) for x in s.flatten()]
    sizes = [len(b) for b in s.batches]
    kw = dict(t0=50.0, iter=10, seed=5, objective_scale=1e6)
    many = eng.sm_count * 32 * 2 + 7   # forces several chains per warp
    _, _, r_all = eng.anneal_chains(start, sizes, chains=many, **kw)
    lo = r_all.chain
    _, _, r_one = eng.anneal_chains(start, sizes, chains=many, chain_begin=lo, chain_end=lo + 1, **kw)
    assert r_one.chain == lo and r_one.g == r_all.g and r_one.t == r_all.t


def test_chains_attainment_at_least_reference(port):
    c = S.table_coefficients()
    wins = 0
    for seed in range(4):
        w = S.generate_mixed(256, seed)
        ref_res = port.anneal(_flat(w), TABLE_COEFFS, w.ids(), 4, seed=seed)
        gpu = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=seed, chains=2048,
                                                     scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4)), 4)
        assert gpu.best.n >= ref_res["n"] or gpu.best.g >= ref_res["g"]
        wins += gpu.best.g > ref_res["g"]
    assert wins >= 3
    # the bench configuration (configs[2]): 10 ms budget vs the reference's default single chain
    w = S.generate_mixed(1024, 0)
    ref_res = port.anneal(_flat(w), TABLE_COEFFS, w.ids(), 4, seed=0)
    gpu = S.anneal(w, w.ids(), c, S.AnnealConfig(t0=500.0, tau=0.7, iter=60, chains=16384, budget_ms=9.5,
                                                 scale_ladder=(1e4, 1e5, 1e6, 1e7, 1e8)), 4)
    assert gpu.stats.kernel_ms < 10.0
    assert gpu.best.n > ref_res["n"] and gpu.best.g > ref_res["g"]


def test_chains_edge_cases():
    c = S.table_coefficients()
    code, chat = S.default_slo_classes()
    tight = S.TaskClass(0, "tight", S.SloSpec.e2e(1e-6))
    one = S.Workload([S.Request(0, 0, 100, 10, 10)], [tight])
    r = S.anneal(one, [0], c, S.AnnealConfig(chains=4, t0=30.0, iter=5), 1)
    assert r.best.schedule.batches == [[0]] and r.stats.proposals == 4 * 5 * r.stats.levels_run
    loose = S.Workload([S.Request(i, 0, 100 * (i + 1), 10, 10) for i in range(3)], [S.TaskClass(0, "l", S.SloSpec.e2e(1e12))])
    r = S.anneal(loose, [0, 1, 2], c, S.AnnealConfig(), 1)
    assert r.stats.shortcut and r.stats.proposals == 0 and r.best.schedule.flatten() == [0, 1, 2]
    empty = S.Workload([], [code, chat])
    r = S.anneal(empty, [], c, S.AnnealConfig(), 2)
    assert r.stats.shortcut and r.best.schedule.batches == [] and r.best.g == 0.0
    w = S.generate_mixed(5000, 0)
    with pytest.raises(S.CapacityError):
        S.anneal(w, w.ids(), c, S.AnnealConfig(), 4)


def test_budget_stops_early():
    c = S.table_coefficients()
    w = S.generate_mixed(1024, 0)
    r = S.anneal(w, w.ids(), c, S.AnnealConfig(chains=16384, budget_ms=2.0), 4)
    assert 0 < r.stats.proposals < 16384 * 63 * 100
    assert r.stats.kernel_ms < 2.0 + 0.1  # the budget is checked every 8 proposals
    assert r.best.schedule.is_partition_of(w.ids(), 4)
    assert r.best.g >= max(r.stats.g_sorted_start, r.stats.g_input_start)


def _start_schedule(n, mb, kind, seed):
    rs = np.random.default_rng(seed)
    perm = [int(x) for x in rs.permutation(n)]
    if kind == "full":
        sizes = [mb] * (n // mb) + ([n % mb] if n % mb else [])
    else:  # mixed sizes: squeezes and delays apply often
        sizes, left, k = [], n, 0
        while left:
            s = min(1 + (k % mb), left)
            sizes.append(s)
            left -= s
            k += 1
    return perm, sizes


@pytest.mark.parametrize("n,mb,three,kind,chains", [(64, 4, True, "full", 1), (64, 4, False, "mixed", 1),
                                                     (200, 8, True, "mixed", 1), (150, 4, False, "full", 3),
                                                     (40, 16, True, "mixed", 2), (37, 2, False, "mixed", 1),
                                                     (1500, 4, True, "mixed", 1), (3000, 4, False, "full", 1)])
def test_chain_trajectory_matches_model(eng, n, mb, three, kind, chains):
    """K3 chains follow exactly the trajectory of a plain-Python model of their specification
    (tests/k3_model.py: the reference's proposal discipline on Philox words, the tick-grid
    objective evaluated from scratch, fp32 Metropolis): same winner schedule, (n_met, t, g),
    proposals and accepted counts. This pins the kernel's incremental scoring (rebuilt-batch
    deltas, anchor shifts, SLO walks), its move flags and its lazy swap writes."""
    import k3_model as K
    w = _three_class(n, 70 + n) if three else S.generate_mixed(n, 70 + n)
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
    seed, t0, t_thres, tau, it = 12345 + n, 100.0, 20.0, 0.8, 40
    scale = t0 / f0 if f0 > 0 else t0
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=chains, t0=t0, t_thres=t_thres, tau=tau, iter=it, seed=seed,
                                  objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, seed, t0, t_thres, tau, it, scale) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    assert r.chain == win
    assert r.proposals == sum(x["proposals"] for x in runs)
    assert r.accepted == sum(x["accepted"] for x in runs)
    assert (r.n_met, r.t, r.g) == runs[win]["best"]
    got, q = [], 0
    for s in bs:
        got.append([int(x) for x in bp[q:q + s]])
        q += s
    assert got == runs[win]["best_batches"]


@pytest.mark.parametrize("n,start_kind", [(1024, "deadline_first"), (1024, "mixed"), (2048, "deadline_first"),
                                          (3000, "deadline_first")])
def test_chain_trajectory_through_the_speculative_stage(eng, n, start_kind):
    """The bench shape (N=1024, mb=4, generate_mixed): only a short prefix of the 32-position
    units is live (elapsed <= the largest finite deadline), so most proposals are swaps in the
    dead region and K3 scores up to four of them at once, consuming the leading rejected ones.
    The chains must still follow the sequential model exactly (1, 2 and 4 units per lane)."""
    import k3_model as K
    mb = 4
    w = S.generate_mixed(n, 11)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    if start_kind == "deadline_first":
        pos = {r: k for k, r in enumerate(ids)}
        start = [[pos[r] for r in b] for b in S.deadline_first_candidate(w, ids, c, mb).batches]
    else:
        perm, sizes = _start_schedule(n, mb, "mixed", 7)
        start, q = [], 0
        for sz in sizes:
            start.append(perm[q:q + sz])
            q += sz
    # the dead region exists: live units (E <= largest finite deadline, in ticks) are a short prefix
    finite = dl[np.isfinite(dl) & (dl >= 0)]
    dg = math.floor(finite.max() / eng.tick_ms)
    elapsed, unit_e, q = 0, [], 0
    for bt in start:
        for _ in bt:
            if q % 32 == 0:
                unit_e.append(elapsed)
            q += 1
        elapsed += max(int(prob.xt[len(bt) - 1, i]) for i in bt)
    assert sum(e <= dg for e in unit_e) <= 8
    f0 = prob.score(start)[2]
    seed, t0, t_thres, tau, it, chains = 4242, 500.0, 20.0, 0.7, 40, 2
    perm = [i for b in start for i in b]
    bp, bs, r = eng.anneal_chains(perm, [len(b) for b in start], chains=chains, t0=t0, t_thres=t_thres, tau=tau,
                                  iter=it, seed=seed, objective_scale=t0 / f0 * 1e5)
    runs = [K.run_chain(prob, start, cid, seed, t0, t_thres, tau, it, t0 / f0 * 1e5) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    got, q = [], 0
    for sz in bs:
        got.append([int(x) for x in bp[q:q + sz]])
        q += sz
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"]


def test_parked_chains_match_model(eng):
    """More chains than resident warps (one block: each warp runs two or three chains, parking
    each in HBM between temperature levels): every chain still follows the sequential model,
    through the speculative stage and across park/resume."""
    import k3_model as K
    n, mb, chains = 256, 4, 60
    w = S.generate_mixed(n, 21)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    pos = {r: k for k, r in enumerate(ids)}
    start = [[pos[r] for r in b] for b in S.deadline_first_candidate(w, ids, c, mb).batches]
    f0 = prob.score(start)[2]
    seed, t0, t_thres, tau, it = 777, 500.0, 20.0, 0.7, 20
    scale = t0 / f0 * 1e4
    bp, bs, r = eng.anneal_chains([i for b in start for i in b], [len(b) for b in start], chains=chains, t0=t0,
                                  t_thres=t_thres, tau=tau, iter=it, seed=seed, objective_scale=scale, max_blocks=1)
    runs = [K.run_chain(prob, start, cid, seed, t0, t_thres, tau, it, scale) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    got, q = [], 0
    for sz in bs:
        got.append([int(x) for x in bp[q:q + sz]])
        q += sz
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"]


@pytest.mark.parametrize("scale", [1e-3, 1e4])
def test_chain_trajectory_matches_model_at_other_time_scales(eng, scale):
    """The tick grid follows the problem's scale (largest exec < 2^27 ticks): the same queue with
    every exec time and deadline multiplied by `scale` still matches the model exactly."""
    import k3_model as K
    n, mb = 96, 4
    w = _three_class(n, 5)
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
    ex, dl = ex * scale, dl * scale
    eng.set_problem(ex, dl)
    tick = eng.tick_ms
    assert np.rint(ex / tick).max() < 2 ** 27 and np.rint(ex / tick).max() >= 2 ** 26
    prob = K.TickProblem(ex, dl, tick)
    perm, sizes = _start_schedule(n, mb, "mixed", 3)
    start, q = [], 0
    for s in sizes:
        start.append(perm[q:q + s])
        q += s
    f0 = prob.score(start)[2]
    seed, t0, t_thres, tau, it = 99, 100.0, 20.0, 0.8, 40
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=1, t0=t0, t_thres=t_thres, tau=tau, iter=it, seed=seed,
                                  objective_scale=t0 / f0)
    model = K.run_chain(prob, start, 0, seed, t0, t_thres, tau, it, t0 / f0)
    assert (r.n_met, r.t, r.g) == model["best"] and r.accepted == model["accepted"]


@pytest.mark.parametrize("n,mb,delta_p", [(64, 4, -400.0), (300, 8, -120.0), (1024, 4, -60.0)])
def test_chains_with_negative_exec_times(eng, port, n, mb, delta_p):
    """Fitted coefficients with a negative intercept (delta_p < 0) are valid reference inputs
    (P:src/core.cpp:55-62) and give negative exec times for short requests. The chain kernel offsets
    its tick grid (makespans start at 0 as in the reference, :267-273) and still follows the model
    move for move, with the reference's n_met; the replay mode (K2) stays bit-identical to the
    reference walk; the public anneal() returns a valid schedule no worse than its starts."""
    import k3_model as K
    base = S.table_coefficients()
    c = S.LatencyCoefficients(base.alpha_p, base.beta_p, base.gamma_p, delta_p, base.alpha_d, base.beta_d,
                              base.gamma_d, base.delta_d)
    w = _three_class(n, 90 + n)
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, c, mb)
    assert (ex < 0).any(), "the coefficients must produce negative exec times"
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    perm, sizes = _start_schedule(n, mb, "mixed", 5)
    start, q = [], 0
    for s_ in sizes:
        start.append(perm[q:q + s_])
        q += s_
    f0 = prob.score(start)[2]
    seed, t0, tau, it = 31 + n, 100.0, 0.7, 30
    scale = t0 / f0 if f0 > 0 else t0
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=2, t0=t0, t_thres=20.0, tau=tau, iter=it, seed=seed,
                                  objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, seed, t0, 20.0, tau, it, scale) for cid in range(2)]
    win = min(range(2), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    got, q = [], 0
    for s_ in bs:
        got.append([int(x) for x in bp[q:q + s_]])
        q += s_
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"]
    # the K3 evaluator agrees with the reference score on random schedules
    rs = np.random.default_rng(n)
    perms, szs = _random_partitions(rs, n, mb, 500)
    coeffs = np.asarray(c.as_array(), dtype=np.float64)
    nm, t, g, _ = eng.evaluate_batch_tick(perms, E.end_bits(szs, n))
    o_n, o_t, o_g = port.score_batch(_flat(w), coeffs, ids, mb, perms.astype(np.int32), szs)
    np.testing.assert_array_equal(nm, o_n)
    np.testing.assert_allclose(t, o_t, rtol=1e-6, atol=1e-6 * np.abs(o_t).max())
    # replay: the reference walk, bit for bit
    r2 = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=3, t0=60.0, iter=15, mode=S.SearchMode.REPLAY), mb)
    o = port.anneal(_flat(w), coeffs, w.ids(), mb, seed=3, t0=60.0, iter=15)
    assert r2.best.schedule.batches == o["batches"] and r2.best.g == o["g"] and r2.best.n == o["n"]
    # chains through the public entry point
    r3 = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=1, chains=512, t0=100.0, iter=20), mb)
    assert r3.best.schedule.is_partition_of(w.ids(), mb)
    assert r3.best.g >= max(r3.stats.g_sorted_start, r3.stats.g_input_start)


@pytest.mark.parametrize("n,mb", [(40, 4), (200, 8), (700, 2)])
def test_chains_negative_exec_raw_tables(eng, n, mb):
    """Raw tables where a third of the exec times are negative (whole batches of them: the
    makespan floors at 0): the chains still follow the model move for move, and the K3 evaluator's
    n_met equals K1's exact count."""
    import k3_model as K
    rs = np.random.default_rng(n)
    ex = rs.uniform(-60.0, 120.0, size=(mb, n))
    elapsed_scale = 120.0 * n / mb
    dl = rs.uniform(-10.0, 0.6 * elapsed_scale, size=(mb, n))
    dl[rs.random((mb, n)) < 0.1] = np.inf
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    perm, sizes = _start_schedule(n, mb, "mixed", 9)
    start, q = [], 0
    for s_ in sizes:
        start.append(perm[q:q + s_])
        q += s_
    f0 = prob.score(start)[2]
    seed, t0, tau, it = 77 + n, 100.0, 0.7, 30
    scale = t0 / f0 if f0 > 0 else t0
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=2, t0=t0, t_thres=20.0, tau=tau, iter=it, seed=seed,
                                  objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, seed, t0, 20.0, tau, it, scale) for cid in range(2)]
    win = min(range(2), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    got, q = [], 0
    for s_ in bs:
        got.append([int(x) for x in bp[q:q + s_]])
        q += s_
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"]
    perms, szs = _random_partitions(rs, n, mb, 300)
    bits = E.end_bits(szs, n)
    nm, _, _, _ = eng.evaluate_batch_tick(perms, bits)
    k1, _, _ = eng.evaluate_batch(perms, bits)
    np.testing.assert_array_equal(nm, k1)


def test_chain_trajectory_random_shapes(eng):
    """Randomised shapes (N 2..300, mb 1..16, random start batchings, scales, ladders, 1-2 chains):
    K3 and the Python model agree exactly on every case."""
    import random
    import k3_model as K
    rs = random.Random(2024)
    for case in range(24):
        n = rs.choice([2, 3, 5, 9, 17, 33, 64, 100, 150, 257, 300])
        mb = rs.choice([1, 2, 3, 4, 5, 8, 16])
        w = _three_class(n, case) if rs.random() < 0.5 else S.generate_mixed(n, case)
        ids = sorted(w.ids())
        ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
        eng.set_problem(ex, dl)
        prob = K.TickProblem(ex, dl, eng.tick_ms)
        perm = list(range(n))
        rs.shuffle(perm)
        sizes, left = [], n
        while left:
            s = rs.randint(1, min(mb, left))
            sizes.append(s)
            left -= s
        start, q = [], 0
        for s in sizes:
            start.append(perm[q:q + s])
            q += s
        f0 = prob.score(start)[2]
        t0, tau, it = rs.choice([30.0, 100.0, 500.0]), rs.choice([0.5, 0.8]), rs.choice([7, 20, 33])
        scale = (t0 / f0 if f0 > 0 else t0) * rs.choice([1.0, 1e3, 1e-2])
        seed, chains = rs.randrange(1 << 40), rs.choice([1, 2])
        bp, bs, r = eng.anneal_chains(perm, sizes, chains=chains, t0=t0, t_thres=20.0, tau=tau, iter=it, seed=seed,
                                      objective_scale=scale)
        runs = [K.run_chain(prob, start, cid, seed, t0, 20.0, tau, it, scale) for cid in range(chains)]
        win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
        got, q = [], 0
        for s in bs:
            got.append([int(x) for x in bp[q:q + s]])
            q += s
        assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                       sum(x["accepted"] for x in runs)), case
        assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"], case


@pytest.mark.gpu
@pytest.mark.parametrize("n,mb,seed", [(64, 4, 1), (300, 4, 2), (1100, 4, 3), (2100, 2, 4)])
def test_chain_trajectory_loose_deadlines(eng, n, mb, seed):
    """Deadlines far beyond the exec scale (> 2^31 ticks: the cached slacks clamp to int32) mixed
    with tight, +inf and never-met ones, at temperatures that accept often: the incremental
    live-cache refresh (shifted units, clamped slacks re-read from the deadline table) keeps the
    chains on the model's trajectories (one, two and four units per lane)."""
    import k3_model as K
    rs = np.random.default_rng(seed)
    base = rs.uniform(2.0, 60.0, n)
    ex = np.stack([base * (1.0 + 0.15 * b) for b in range(mb)])  # [mb][n], growing with batch size
    mx = float(ex.max())
    kind = rs.choice(4, n, p=[0.35, 0.4, 0.15, 0.1])
    dl = np.empty_like(ex)
    for i in range(n):
        if kind[i] == 0:    # tight: met only near the head of the schedule
            dl[:, i] = rs.uniform(0.0, 4.0 * mx)
        elif kind[i] == 1:  # loose but finite: slack beyond 2^31 ticks near the head
            dl[:, i] = rs.uniform(40.0, 90.0) * mx
        elif kind[i] == 2:
            dl[:, i] = np.inf
        else:
            dl[:, i] = -np.inf
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    assert (dl[np.isfinite(dl)].max() / eng.tick_ms) > 2.0 ** 31  # the clamp is reachable
    perm = list(rs.permutation(n))
    sizes = [mb] * (n // mb) + ([n % mb] if n % mb else [])
    start, q = [], 0
    for s in sizes:
        start.append([int(x) for x in perm[q:q + s]])
        q += s
    f0 = prob.score(start)[2]
    t0, tau, it, chains = 2000.0, 0.6, 24, 2
    scale = t0 / f0 if f0 > 0 else t0
    sd = int(rs.integers(1 << 40))
    bp, bs, r = eng.anneal_chains([int(x) for x in perm], sizes, chains=chains, t0=t0, t_thres=20.0, tau=tau,
                                  iter=it, seed=sd, objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, sd, t0, 20.0, tau, it, scale) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    got, q = [], 0
    for s in bs:
        got.append([int(x) for x in bp[q:q + s]])
        q += s
    assert sum(x["accepted"] for x in runs) > 0.2 * sum(x["proposals"] for x in runs)  # accepts often
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and got == runs[win]["best_batches"]
