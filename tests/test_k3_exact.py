"""The chain kernel's (K3) SLO count is the reference's, bit for bit.

K3 keeps the total latency on an integer tick grid (2^-k ms), but its n_met must equal
CostModel::score's (P:src/priority_mapper.cpp:259-279): fp64 batch-start elapsed times summed left
to right, compared with each request's SLO. The kernel decides a test on the grid only where the
grid's rounding bound certifies it and re-sums the rest in fp64 (chains.cuh unit_walk/exact_met).

These tests check it three ways:
* slo_evaluate_batch_tick (K3's evaluator) against the oracle's score on random schedules at
  configs[1] (N=256, mb=4, 1e5 schedules) and at N=1024 / 4096;
* adversarial queues: one SLO class per request, each SLO set on its own deadline in a chosen
  schedule (exactly on it, one ulp either side, a few ticks either side, within the margin) --
  the tick grid alone gets some of these wrong, the kernel must not;
* chains run on those queues: the trajectories follow the model (tests/k3_model.py, whose n_met
  is the reference's), and the winners' n_met equals K1's exact re-score.
"""
import math

import numpy as np
import pytest

from oracle import TABLE_COEFFS, FlatWorkload

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E

pytestmark = pytest.mark.gpu

T_REL = 1e-6  # north_star: latencies within 1e-6 relative


def _flat(w: S.Workload) -> FlatWorkload:
    a = w.arrays
    return FlatWorkload(id=a["id"], cls=a["cls"], in_len=a["in_len"], true_out=a["true_out"], pred_out=a["pred_out"],
                        arrival=a["arrival"], class_id=a["class_id"], kind=a["kind"], e2e=a["e2e"], ttft=a["ttft"],
                        tpot=a["tpot"])


def _three_class(n, seed):
    base = S.generate_mixed(n, seed)
    code, chat = S.default_slo_classes()
    offline = S.TaskClass(2, "offline", S.SloSpec.e2e(1e9))
    reqs = [S.Request(r.id, 2 if r.id % 3 == 2 else r.task_class_id, r.input_len, r.true_output_len,
                      r.predicted_output_len) for r in base.requests]
    return S.Workload(reqs, [code, chat, offline])


def _random_sizes(rs, n, mb):
    s, left = [], n
    while left:
        k = int(rs.integers(1, min(mb, left) + 1))
        s.append(k)
        left -= k
    return s


def _random_partitions(rs, n, mb, count, full_frac=0.5):
    perms = np.stack([rs.permutation(n) for _ in range(count)]).astype(np.uint16)
    sizes = []
    for r in range(count):
        if r < full_frac * count:
            sizes.append([mb] * (n // mb) + ([n % mb] if n % mb else []))
        else:
            sizes.append(_random_sizes(rs, n, mb))
    return perms, sizes


def _ref_elapsed(ex, perm, sizes):
    """The reference's batch-start elapsed time of every position (fp64, left to right)."""
    el, out, q = 0.0, np.zeros(len(perm)), 0
    for sz in sizes:
        mk = 0.0
        for _ in range(sz):
            out[q] = el
            e = float(ex[sz - 1, perm[q]])
            mk = e if mk < e else mk
            q += 1
        el = el + mk
    return out


def _tick_only_met(ex, dl, tick, perm, sizes):
    """Per-position SLO flags decided on the grid alone (K3 before its tests were certified)."""
    xt = np.rint(ex / tick).astype(np.int64)
    el = q = 0
    met = []
    for sz in sizes:
        mk = 0
        for _ in range(sz):
            i = int(perm[q]); q += 1
            d = float(dl[sz - 1, i])
            met.append(d == math.inf or (d >= 0 and el <= math.floor(d / tick)))
            mk = max(mk, int(xt[sz - 1, i]))
        el += mk
    return met


def adversarial(n, mb, seed, eng):
    """A queue whose SLOs sit on their deadlines in one schedule (perm, sizes): one class per
    request, E2E or TTFT+TPOT, the SLO = the request's e2e (or TTFT) in that schedule, computed with
    the reference arithmetic, then nudged by 0, +-1 ulp, +-j ticks, a uniform draw within the
    certification margin, or far away. Returns (workload, ids, perm, sizes, tick)."""
    rs = np.random.default_rng(seed)
    base = S.generate_mixed(n, seed)
    c = S.table_coefficients()
    ids = sorted(base.ids())
    ex, dl = E.build_tables(base, ids, c, mb)
    eng.set_problem(ex, dl)
    tick, marg = eng.tick_ms, n // 2 + 2
    perm = [int(x) for x in rs.permutation(n)]
    sizes = [mb] * (n // mb) + ([n % mb] if n % mb else []) if rs.random() < 0.5 else _random_sizes(rs, n, mb)
    start = _ref_elapsed(ex, perm, sizes)
    by_id = {r.id: r for r in base.requests}
    classes, reqs, q = [], [], 0
    for sz in sizes:
        for _ in range(sz):
            i = perm[q]
            r = by_id[ids[i]]
            k = int(rs.integers(0, 9))
            if k == 0:
                pert = 0.0
            elif k in (1, 2):
                pert = None  # one ulp, below (1) or above (2)
            elif k in (3, 4):
                pert = (1 if k == 3 else -1) * int(rs.integers(1, 4)) * tick
            elif k in (5, 6):
                pert = float(rs.uniform(-(marg + 3), marg + 3)) * tick
            elif k == 7:
                pert = float(rs.uniform(-0.5, 0.5)) * tick
            else:
                pert = float(rs.choice([-1.0, 1.0])) * float(rs.uniform(1.0, 500.0))
            ttft = rs.random() < 0.3
            cost = S.predict_prefill(c, sz, r.input_len) if ttft else float(ex[sz - 1, i])
            slo = start[q] + cost
            if pert is None:
                slo = math.nextafter(slo, -math.inf if k == 1 else math.inf)
            else:
                slo = slo + pert
            slo = max(slo, 1e-3)
            cid = len(classes)
            if ttft:
                tp = S.predict_tpot(c, sz, r.input_len, r.predicted_output_len)
                classes.append(S.TaskClass(cid, f"t{cid}", S.SloSpec.ttft_tpot(slo, tp if rs.random() < 0.5 else 1e9)))
            else:
                classes.append(S.TaskClass(cid, f"e{cid}", S.SloSpec.e2e(slo)))
            reqs.append(S.Request(r.id, cid, r.input_len, r.true_output_len, r.predicted_output_len))
            q += 1
    w = S.Workload(reqs, classes)
    return w, ids, perm, sizes, tick


def _neighbours(rs, perm, sizes, count):
    """perm itself, then perturbations: swaps inside one batch (same elapsed times), swaps of two
    random positions, and a few fresh batchings of the same order."""
    n = len(perm)
    out_p, out_s = [list(perm)], [list(sizes)]
    ends = np.cumsum(sizes)
    for k in range(count - 1):
        p, s = list(perm), list(sizes)
        kind = k % 3
        if kind == 0 and max(sizes) > 1:
            b = int(rs.integers(0, len(sizes)))
            while sizes[b] < 2:
                b = int(rs.integers(0, len(sizes)))
            lo = int(ends[b] - sizes[b])
            a, c = rs.choice(sizes[b], 2, replace=False)
            p[lo + a], p[lo + c] = p[lo + c], p[lo + a]
        elif kind == 1 and n >= 2:
            for _ in range(int(rs.integers(1, 4))):
                a, c = rs.choice(n, 2, replace=False)
                p[a], p[c] = p[c], p[a]
        else:
            s = _random_sizes(rs, n, max(sizes))
        out_p.append(p)
        out_s.append(s)
    return np.array(out_p, dtype=np.uint16), out_s


@pytest.fixture(scope="module")
def eng():
    e = E.Engine(0)
    yield e
    e.close()


def _check(eng, port, w, ids, mb, perms, sizes):
    bits = E.end_bits(sizes, len(ids))
    n_met, t, g, exact = eng.evaluate_batch_tick(perms, bits)
    o_n, o_t, o_g = port.score_batch(_flat(w), TABLE_COEFFS, ids, mb, perms.astype(np.int32), sizes)
    np.testing.assert_array_equal(n_met, o_n)
    np.testing.assert_allclose(t, o_t, rtol=T_REL, atol=0)
    np.testing.assert_allclose(g, o_g, rtol=T_REL, atol=0)
    # K1 (the bit-exact checker-grade evaluator) agrees too
    k_n, k_t, k_g = eng.evaluate_batch(perms, bits)
    np.testing.assert_array_equal(k_n, o_n)
    np.testing.assert_array_equal(k_t, o_t)
    return exact


@pytest.mark.parametrize("n,mb,count,three", [(256, 4, 100000, False), (256, 4, 20000, True), (1024, 4, 20000, False),
                                              (1024, 8, 5000, True), (4096, 4, 2000, False), (300, 16, 5000, True),
                                              (37, 1, 2000, True)])
def test_tick_evaluator_matches_reference(eng, port, n, mb, count, three):
    """configs[1] (N=256, mb=4, 1e5 random schedules) and larger queues: the K3 evaluator's n_met
    equals CostModel::score's exactly, t and g within 1e-6 relative."""
    w = _three_class(n, 300 + n) if three else S.generate_mixed(n, 300 + n)
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
    eng.set_problem(ex, dl)
    rs = np.random.default_rng(n * 31 + mb)
    perms, sizes = _random_partitions(rs, n, mb, count)
    _check(eng, port, w, ids, mb, perms, sizes)


@pytest.mark.parametrize("n,mb,seed", [(16, 4, 1), (64, 1, 2), (64, 4, 3), (256, 4, 4), (256, 8, 5), (1024, 4, 6),
                                       (1024, 16, 7), (2048, 4, 8), (4096, 4, 9), (4096, 8, 10)])
def test_tick_evaluator_near_deadlines(eng, port, n, mb, seed):
    """Adversarial queues (every SLO on or within a few ticks of its deadline in one schedule): the
    grid alone misjudges some of them; the K3 evaluator's n_met is still exactly the reference's,
    and the fp64 re-sum is exercised."""
    w, ids, perm, sizes, tick = adversarial(n, mb, seed, eng)
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
    eng.set_problem(ex, dl)
    rs = np.random.default_rng(seed)
    perms, szs = _neighbours(rs, perm, sizes, 60)
    exact = _check(eng, port, w, ids, mb, perms, szs)
    assert exact > 0
    if n >= 64:  # the grid alone misjudges some request of the adversarial schedule itself
        ev = S.evaluate(S.Schedule([[ids[i] for i in b] for b in _batches(perm, sizes)]), S.table_coefficients(), w)
        assert _tick_only_met(ex, dl, eng.tick_ms, perm, sizes) != [m.slo_met for m in ev.per_request]


def _batches(perm, sizes):
    out, q = [], 0
    for s in sizes:
        out.append([int(x) for x in perm[q:q + s]])
        q += s
    return out


@pytest.mark.parametrize("n,mb,seed,chains", [(48, 4, 11, 2), (128, 4, 12, 2), (200, 8, 13, 1), (512, 4, 14, 1),
                                              (1024, 4, 15, 1)])
def test_chain_trajectory_near_deadlines(eng, n, mb, seed, chains):
    """Chains started on the adversarial schedule, at a low temperature so they stay near it,
    follow the model -- whose n_met is the reference's -- move for move, and needed the fp64
    re-sum on the way."""
    import k3_model as K
    w, ids, perm, sizes, tick = adversarial(n, mb, seed, eng)
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
    eng.set_problem(ex, dl)
    prob = K.TickProblem(ex, dl, eng.tick_ms)
    start = _batches(perm, sizes)
    f0 = prob.score(start)[2]
    seed_, t0, t_thres, tau, it = 900 + seed, 100.0, 20.0, 0.6, 40
    scale = t0 / f0 * 1e3
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=chains, t0=t0, t_thres=t_thres, tau=tau, iter=it, seed=seed_,
                                  objective_scale=scale)
    runs = [K.run_chain(prob, start, cid, seed_, t0, t_thres, tau, it, scale) for cid in range(chains)]
    win = min(range(chains), key=lambda k: (-runs[k]["best"][2], runs[k]["best"][1], k))
    assert (r.chain, r.proposals, r.accepted) == (win, sum(x["proposals"] for x in runs),
                                                   sum(x["accepted"] for x in runs))
    assert (r.n_met, r.t, r.g) == runs[win]["best"] and _batches(bp, bs) == runs[win]["best_batches"]
    assert r.exact_walks > 0


@pytest.mark.parametrize("n,mb,chains,adv", [(256, 4, 4096, True), (1024, 4, 16384, True), (1024, 4, 16384, False),
                                             (4096, 4, 2048, True), (300, 16, 2048, True)])
def test_chain_winner_n_met_is_reference(eng, port, n, mb, chains, adv):
    """Many chains (the bench's kernel path, speculative stage included): the winner's n_met is the
    reference's exact count of the winning schedule and its t within 1e-6 relative."""
    if adv:
        w, ids, perm, sizes, _ = adversarial(n, mb, 40 + n, eng)
    else:
        w = S.generate_mixed(n, 40 + n)
        ids = sorted(w.ids())
        s, _ = S.initial_candidates(w, ids, S.table_coefficients(), mb)
        perm = [ids.index(x) for x in s.flatten()]
        sizes = [len(b) for b in s.batches]
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), mb)
    eng.set_problem(ex, dl)
    bp, bs, r = eng.anneal_chains(perm, sizes, chains=chains, t0=200.0, tau=0.7, iter=40, seed=n + 1,
                                  objective_scale=1e6, scale_ladder=(1e-2, 1.0, 1e2))
    o_n, o_t, o_g = port.score_batch(_flat(w), TABLE_COEFFS, ids, mb, bp[None, :].astype(np.int32), [list(bs)])
    assert r.n_met == o_n[0]
    assert abs(r.t - o_t[0]) <= T_REL * o_t[0]
