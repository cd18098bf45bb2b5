"""The evaluation harness (csrc/harness.cpp) against the unmodified reference (oracle/_ref):

* run() / run_fcfs() -- every per-request record and the report bit-identical to the reference's
  simulator (P:src/simulator.cpp:17-123), with and without execution noise, 1-4 instances;
* realize_batches() -- run() is its special case; window bounds stop the clock as documented;
* Estimator -- Welford models and the predictions drawn from them bit-identical
  (P:src/output_estimator.cpp:10-78);
* (GPU) compare / sweep / perturb with the exact-replay mapper equal the reference's drivers, the
  chains-mode drivers equal their one-after-another runs, and evaluate_batch equals evaluate().
"""
import numpy as np
import pytest

from conftest import requires_ref
from oracle import TABLE_COEFFS, FlatWorkload
from oracle import ref

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import harness as H


def _flat(w):
    a = w.arrays
    return FlatWorkload(**{k: a[k] for k in ("id", "cls", "in_len", "true_out", "pred_out", "arrival", "class_id",
                                             "kind", "e2e", "ttft", "tpot")})


def _fleet(k, mb=4):
    return [S.InstanceState(10 + 3 * i, 2**35, 2**35, 0.9, 262144.0, mb) for i in range(k)]


def _ref_fleet(insts):
    return [dict(id=i.id, total_mem=i.total_mem, remaining_mem=i.remaining_mem, mu=i.mem_utility,
                 sigma=i.bytes_per_token, max_batch=i.max_batch_size) for i in insts]


def _random_plans(rs, ids, k, mb):
    ids = list(rs.permutation(ids))
    cut = sorted(rs.choice(np.arange(1, len(ids)), size=k - 1, replace=False)) if k > 1 else []
    parts = np.split(np.asarray(ids), cut)
    plans = []
    for p in parts:
        batches, pos = [], 0
        while pos < len(p):
            b = int(rs.integers(1, mb + 1))
            batches.append([int(x) for x in p[pos:pos + b]])
            pos += b
        plans.append(S.Schedule(batches))
    return plans


def _same_records(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.request_id == w["request_id"]
        for f in ("wait_ms", "exec_ms", "e2e_ms", "ttft_ms", "tpot_ms"):
            assert getattr(g, f) == w[f], (f, getattr(g, f), w[f])
        assert g.slo_met == w["slo_met"] and g.extrapolated == w["extrapolated"]


def _same_report(got, want):
    assert got.n_met == want["n_met"]
    for f in ("slo_attainment", "avg_latency_ms", "g", "total_latency_ms", "scheduling_overhead_ms"):
        assert getattr(got, f) == want[f], f


@requires_ref
@pytest.mark.parametrize("k", [1, 2, 4])
@pytest.mark.parametrize("noise", [0.0, 0.15])
def test_run_matches_reference_simulator(k, noise):
    rs = np.random.default_rng(k * 7 + int(noise * 100))
    c = S.table_coefficients()
    for seed in range(3):
        w = S.generate_mixed(150, seed)
        insts = _fleet(k)
        plans = _random_plans(rs, w.ids(), k, 4)
        got = H.run(plans, w, insts, c, H.SimConfig(noise_pct=noise, dispatch_gap_ms=0.1, seed=seed + 5), 1.25)
        recs, rep = ref.run(_flat(w), TABLE_COEFFS, _ref_fleet(insts), [p.batches for p in plans], noise=noise, gap=0.1,
                            seed=seed + 5, overhead=1.25)
        _same_records(got.per_request, recs)
        _same_report(got, rep)


@requires_ref
@pytest.mark.parametrize("k", [1, 3])
@pytest.mark.parametrize("noise", [0.0, 0.2])
def test_run_fcfs_matches_reference(k, noise):
    c = S.table_coefficients()
    for seed in range(3):
        w = S.generate_mixed(97, seed)
        # arrivals: ties and an unsorted order exercise the (arrival, id) order
        arr = (np.arange(len(w.requests)) * 37 % 11) * 50.0
        reqs = [S.Request(r.id, r.task_class_id, r.input_len, r.true_output_len, r.predicted_output_len, float(arr[j]))
                for j, r in enumerate(w.requests)]
        w = S.Workload(reqs, list(S.default_synth_classes()))
        insts = [S.InstanceState(i, 2**35, 2**35, 0.9, 262144.0, 2 + i) for i in range(k)]
        got = H.run_fcfs(w, insts, c, H.SimConfig(noise_pct=noise, seed=seed))
        plans, recs, rep = ref.run_fcfs(_flat(w), TABLE_COEFFS, _ref_fleet(insts), noise=noise, seed=seed)
        assert [p.batches for p in got.schedules] == plans
        _same_records(got.report.per_request, recs)
        _same_report(got.report, rep)


def test_realize_batches_windows_and_run_special_case():
    c = S.table_coefficients()
    w = S.generate_mixed(40, 2)
    plan = S.Schedule([w.ids()[i:i + 4] for i in range(0, 40, 4)])
    rep = H.run([plan], w, _fleet(1), c, H.SimConfig(dispatch_gap_ms=0.1))
    recs, clock, started = H.realize_batches(plan.batches, w, c, 0.0, 0.0, 0.1)
    assert started == 10 and [r.e2e_ms for r in recs] == [r.e2e_ms for r in rep.per_request]
    # a window bound: batches start while the clock is below it (the bound is checked before the gap)
    ends = []
    t = 0.0
    for b in plan.batches:
        start = t + (0.1 if ends else 0.0)
        t = start + max(r.exec_ms for r in recs if r.request_id in b)
        ends.append(t)
    _, clock3, started3 = H.realize_batches(plan.batches, w, c, 0.0, 0.0, 0.1, until=ends[2])
    assert started3 == 3 and clock3 == ends[2]
    _, _, started0 = H.realize_batches(plan.batches, w, c, 5.0, 0.1, 0.1, until=5.0)
    assert started0 == 0
    # waits measured from arrival
    reqs = [S.Request(r.id, r.task_class_id, r.input_len, r.true_output_len, r.predicted_output_len, 3.0)
            for r in w.requests]
    w3 = S.Workload(reqs, list(S.default_synth_classes()))
    r3, _, _ = H.realize_batches(plan.batches[:1], w3, c, 10.0, 0.5, 0.1, from_arrival=True)
    assert all(r.wait_ms == 10.5 - 3.0 for r in r3)


@requires_ref
def test_estimator_matches_reference():
    code, chat = S.default_synth_classes()
    rng_cls = S.TaskClass(2, "range", S.SloSpec.e2e(1e4), ("range", 10, 20))
    bare = S.TaskClass(3, "bare", S.SloSpec.e2e(1e4))
    classes = [code, chat, rng_cls, bare]
    rs = np.random.default_rng(3)
    for n_obs in (0, 1, 2, 7, 200):
        obs = [(int(rs.choice([0, 1, 2])), int(rs.integers(1, 2000))) for _ in range(n_obs)]
        pred_cls = [int(x) for x in rs.choice([0, 1, 2, 3], size=64)]
        got, models = H.estimator_run(classes, obs, pred_cls, seed=n_obs + 11)
        want, wmodels = ref.estimator([c.id for c in classes], [c.output_prior for c in classes], obs, pred_cls,
                                      seed=n_obs + 11)
        assert got == want
        assert [(m.count, m.mean, m.m2) for m in models] == wmodels
    with pytest.raises(S.DataError):
        H.estimator_run(classes, [(0, 0)], [], 1)
    with pytest.raises(S.DataError):
        H.estimator_run(classes, [], [9], 1)


def test_median():
    assert H.median([]) == 0.0 and H.median([3.0, 1.0, 2.0]) == 2.0 and H.median([4.0, 1.0]) == 2.5


# ---------------------------------------------------------------- GPU drivers
def _replay_cfg(**kw):
    return S.AnnealConfig(mode=S.SearchMode.REPLAY, t0=80.0, iter=15, **kw)


@pytest.mark.gpu
@requires_ref
def test_compare_replay_mode_matches_reference_compare():
    """With the exact-replay mapper, compare() is the reference's compare() row for row."""
    c = S.table_coefficients()
    w = S.generate_mixed(18, 4)  # 6 requests per instance: the exhaustive oracle stays small
    insts = _fleet(3, mb=4)
    t = H.compare(w, insts, c, ["sa", "fcfs", "exhaustive"], [1, 2], _replay_cfg(), H.SimConfig(noise_pct=0.1),
                  exhaustive_cap=10)
    rows, med = ref.compare(_flat(w), TABLE_COEFFS, _ref_fleet(insts), [0, 2, 1], [1, 2], noise=0.1, n_cap=10,
                            t0=80.0, iter=15)
    assert len(t.rows) == 6
    for got, want in zip(t.rows, rows):
        assert got.policy == {0: "sa", 1: "exhaustive", 2: "fcfs"}[int(want[0])] and got.seed == int(want[1])
        assert (got.attainment, got.avg_latency_ms, got.g_req_per_ms) == (want[2], want[3], want[4])
    for got, want in zip(t.medians, med):
        assert (got.attainment, got.avg_latency_ms, got.g_req_per_ms) == (want[2], want[3], want[4])


@pytest.mark.gpu
@requires_ref
def test_sweep_and_perturb_replay_mode_match_reference_loops():
    c = S.table_coefficients()
    insts = _fleet(2)
    seeds = [3, 4]
    rows = H.sweep(48, seeds, insts, c, _replay_cfg(), [60.0, 120.0], [10, 20])
    assert len(rows) == 8
    for t0, it, seed, g in rows:  # the reference's sweep cell: schedule_all, G = sum n / sum t
        fw = ref.generate_mixed(48, seed)
        per, _ = ref.schedule_all(fw, TABLE_COEFFS, _ref_fleet(insts), seed=seed, t0=t0, iter=it)
        met, tot = 0, 0.0
        for ev in per:
            met += ev["n"]
            tot += ev["t"]
        assert g == (met / tot if tot > 0 else 0.0)
    prow = H.perturb(48, seeds, insts, c, _replay_cfg(), H.SimConfig(), ["beta_p", "delta_d"], [0.5, 2.0])
    assert len(prow) == 8
    for p, f, seed, g, base, deg in prow:
        fw = ref.generate_mixed(48, seed)
        pert = list(TABLE_COEFFS)
        pert[["alpha_p", "beta_p", "gamma_p", "delta_p", "alpha_d", "beta_d", "gamma_d", "delta_d"].index(p)] *= f
        want = []
        for coeffs in (TABLE_COEFFS, pert):
            per, _ = ref.schedule_all(fw, coeffs, _ref_fleet(insts), seed=seed, t0=80.0, iter=15)
            _, rep = ref.run(fw, TABLE_COEFFS, _ref_fleet(insts), [ev["batches"] for ev in per], seed=seed)
            want.append(rep["g"])
        assert (base, g) == (want[0], want[1])
        assert deg == ((want[0] - want[1]) / want[0] * 100.0 if want[0] > 0 else 0.0)


@pytest.mark.gpu
def test_sweep_chains_mode_equals_sequential_cells():
    """Cells run concurrently on SM shares; chain results do not depend on the grid."""
    c = S.table_coefficients()
    insts = _fleet(2)
    cfg = S.AnnealConfig(chains=512, scale_ladder=(1.0, 1e3), seed=0)
    rows = H.sweep(200, [7], insts, c, cfg, [100.0, 300.0], [15])
    for t0, it, seed, g in rows:
        w = S.generate_mixed(200, seed)
        r = S.schedule_all(w, insts, c, S.AnnealConfig(chains=512, scale_ladder=(1.0, 1e3), seed=seed, t0=t0, iter=it))
        met = sum(ev.n for ev in r.per_instance)
        tot = 0.0
        for ev in r.per_instance:
            tot += ev.t_ms
        assert g == met / tot


@pytest.mark.gpu
def test_evaluate_batch_equals_evaluate():
    c = S.table_coefficients()
    w = S.generate_mixed(300, 9)
    rs = np.random.default_rng(1)
    plans = []
    for _ in range(40):
        plans.append(_random_plans(rs, w.ids(), 1, 6)[0])
    nm, t, g = H.evaluate_batch(plans, c, w, 6)
    for k, p in enumerate(plans):
        ev = S.evaluate(p, c, w)
        assert (int(nm[k]), float(t[k]), float(g[k])) == (ev.n, ev.t_ms, ev.g)
    with pytest.raises(S.DataError):
        H.evaluate_batch([plans[0], S.Schedule([w.ids()[:5]])], c, w, 6)


@pytest.mark.gpu
def test_cpp_harness_example():
    """examples/harness_example.cpp: the harness through the C++ API (Estimator, run_fcfs, compare
    with GPU chains, evaluate_batch, run)."""
    import os
    import subprocess

    from conftest import ROOT
    exe = os.path.join(ROOT, "examples", "_build", "harness_example")
    if not os.path.exists(exe):
        pytest.skip("example not built")
    out = subprocess.run([exe, "150"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 5 and "FAIL" not in out.stdout
