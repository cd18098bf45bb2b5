"""CPU-only checks of the product library: it loads, exports every symbol its headers
declare, and its host-side logic (the reference's O(N) setup/teardown around the GPU
loop) matches the oracle and the golden vectors. No compute call needs a GPU here."""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, unhex
from oracle import TABLE_COEFFS

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import _lib
from paper_2504_14966_b200 import engine as E


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**((?:slo|slosched)_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared("slosched_gpu.h") | _declared("slosched_api.h")
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED) == declared


def test_version_and_no_silent_fallback():
    assert b"sm_100a" in _lib.lib().slo_version()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        w = S.generate_mixed(16, 0)
        with pytest.raises(S.EngineError):
            S.anneal(w, w.ids(), S.table_coefficients(), S.AnnealConfig(chains=4), 2)


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32_10
    assert list(E.philox4x32_10([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    f = 0xFFFFFFFF
    assert list(E.philox4x32_10([f, f, f, f], [f, f])) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert list(E.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_latency_model_matches_golden():
    c = S.table_coefficients()
    for case in golden("latency"):
        b, li, lo = case["b"], case["li"], case["lo"]
        assert S.predict_prefill(c, b, li) == unhex(case["prefill"])
        assert S.predict_decode_total(c, b, li, lo) == unhex(case["decode_total"])
        assert S.predict_exec(c, b, li, lo) == unhex(case["exec"])
        assert S.predict_tpot(c, b, li, lo) == unhex(case["tpot"])
    with pytest.raises(ValueError):
        S.predict_tpot(c, 1, 100, 0)


def test_generate_mixed_matches_golden():
    for case in golden("generate_mixed"):
        w = S.generate_mixed(case["n"], case["seed"], predict=case["mode"] == 1)
        a = w.arrays
        for k in ("id", "cls", "in_len", "true_out", "pred_out"):
            assert list(a[k]) == case[k], k


def test_evaluate_matches_golden():
    c = S.table_coefficients()
    for case in golden("evaluate"):
        w = S.generate_mixed(case["n"], case["seed"])
        ev = S.evaluate(S.Schedule(case["batches"]), c, w)
        assert ev.n == case["n_met"] and ev.t_ms == unhex(case["t"]) and ev.g == unhex(case["g"])
        assert [m.wait_ms for m in ev.per_request] == [unhex(x) for x in case["wait"]]
        assert [int(m.slo_met) for m in ev.per_request] == case["met"]


def test_initial_candidates_and_neighbor_match_golden():
    c = S.table_coefficients()
    for case in golden("initial_candidates"):
        w = S.generate_mixed(case["n"], case["seed"])
        s, i = S.initial_candidates(w, w.ids(), c, case["mb"])
        assert s.batches == case["sorted"] and i.batches == case["input"]
    for case in golden("neighbor_walk"):
        out = S.neighbor_walk(S.Schedule(case["start"]), case["seed"], case["steps"], case["mb"])
        assert out.batches == case["out"]


def test_initial_candidates_break_ties_by_id():
    """The candidates order by (key, id) (P:src/priority_mapper.cpp:297-308): with every key tied,
    both are the ids in ascending order whatever order the caller passes them in (negative ids
    included), and evaluate() agrees with a direct restatement of the objective on them."""
    c = S.table_coefficients()
    code, chat = S.default_slo_classes()
    rs = np.random.RandomState(5)
    ids = [int(x) for x in rs.choice(np.arange(-5000, 5000), 300, replace=False)]
    reqs = [S.Request(i, code.id if k % 2 else chat.id, 120, 60, 60, 7.0) for k, i in enumerate(ids)]
    w = S.Workload(reqs, [code, chat])
    for mb in (1, 3, 4):
        s, inp = S.initial_candidates(w, ids, c, mb)
        assert s.flatten() == sorted(ids) and inp.flatten() == sorted(ids)
        ev = S.evaluate(s, c, w)
        elapsed, tot, met = 0.0, 0.0, 0
        for b in s.batches:
            e = S.predict_exec(c, len(b), 120, 60)
            for _ in b:
                tot += elapsed + e
            elapsed += e
        assert ev.t_ms == tot and len(ev.per_request) == 300


def test_errors_follow_reference_contract():
    code, chat = S.default_slo_classes()
    with pytest.raises(S.DataError):  # duplicate id
        S.Workload([S.Request(0, 0, 10, 10, 10), S.Request(0, 0, 10, 10, 10)], [code])
    with pytest.raises(S.DataError):  # unknown class
        S.Workload([S.Request(0, 7, 10, 10, 10)], [code])
    with pytest.raises(S.DataError):  # bad SLO
        S.Workload([], [S.TaskClass(0, "x", S.SloSpec.e2e(-1.0))])
    w = S.Workload([S.Request(0, 0, 10, 10, None)], [code])
    with pytest.raises(S.DataError):  # missing prediction
        S.evaluate(S.Schedule([[0]]), S.table_coefficients(), w)
    with pytest.raises(S.DataError):  # bad AnnealConfig is rejected before any GPU work
        S.anneal(S.generate_mixed(4, 0), [0, 1, 2, 3], S.table_coefficients(), S.AnnealConfig(t0=10.0), 2)


def test_latest_start_is_the_exact_deadline():
    rs = np.random.default_rng(3)
    for _ in range(20000):
        s = float(rs.choice([30000.0, 10000.0, 1e9, rs.uniform(1, 1e5)]))
        c = float(rs.uniform(0, 5e4))
        d = S.latest_start(s, c)
        assert d + c <= s or math.isinf(d)
        up = math.nextafter(d, math.inf)
        assert not (up + c <= s)
        for x in (d, up, math.nextafter(d, -math.inf), d + rs.uniform(-1e-9, 1e-9) * abs(d)):
            if x >= 0:
                assert (x <= d) == (x + c <= s)


def test_latest_start_near_zero_slack():
    """SLO == cost (zero slack) or within a few ulps of it: the answer lies many ulps of d away
    from s - c (up to ~half an ulp of c above 0); found by bisection, not an ulp-by-ulp walk."""
    rs = np.random.default_rng(4)
    cases = [(c, c) for c in (1e-3, 0.1, 1.0, 100.0, 2.5e4, 1e9)]
    for _ in range(2000):
        c = float(rs.uniform(1e-3, 5e4))
        s = c
        for _ in range(int(rs.integers(0, 4))):
            s = math.nextafter(s, math.inf if rs.random() < 0.5 else -math.inf)
        cases.append((s, c))
    cases += [(5.0, 5.0 + 1e-12), (1e-300, 1e-300), (1e300, 1e300), (1.0, 0.0), (0.5, 1.5)]
    for s, c in cases:
        d = S.latest_start(s, c)
        assert d + c <= s or d == -math.inf
        assert not (math.nextafter(d, math.inf) + c <= s)


def test_tables_fold_the_slo_test_exactly(port):
    """deadline[b][i] reproduces CostModel::met (P:src/priority_mapper.cpp:237-241) for every
    elapsed value the oracle's score visits."""
    w = S.generate_mixed(40, 11)
    c = S.table_coefficients()
    ex, dl = E.build_tables(w, w.ids(), c, 4)
    ids = sorted(w.ids())
    for i, rid in enumerate(ids):
        r = w.find_request(rid)
        for b in range(1, 5):
            assert ex[b - 1, i] == S.predict_exec(c, b, r.input_len, r.predicted_output_len)
    rs = np.random.default_rng(0)
    for i, rid in enumerate(ids):
        r = w.find_request(rid)
        cls = w.classes[r.task_class_id]
        for b in range(1, 5):
            for el in rs.uniform(0, 40000, 50):
                if cls.slo.kind == S.SloKind.E2E:
                    met = el + ex[b - 1, i] <= cls.slo.e2e_ms
                else:
                    met = (el + S.predict_prefill(c, b, r.input_len) <= cls.slo.ttft_ms and
                           S.predict_tpot(c, b, r.input_len, r.predicted_output_len) <= cls.slo.tpot_ms)
                assert met == (el <= dl[b - 1, i])


def test_end_bits_layout():
    bits = E.end_bits([[2, 1, 3], [1] * 40], 40)
    assert bits.shape == (2, 2)
    assert bits[0, 0] == (1 << 1) | (1 << 2) | (1 << 5)
    assert bits[1, 0] == 0xFFFFFFFF and bits[1, 1] == 0xFF


def test_deadline_first_candidate():
    """The chains' third start: a partition into batches <= mb whose leading batches were timed
    with the exact tables (every request in them meets its SLO); on the bench workload it beats
    the reference's sorted start (74 vs 65 SLOs)."""
    c = S.table_coefficients()
    for n, seed, mb in [(1, 0, 4), (7, 1, 2), (64, 2, 4), (256, 0, 4), (1024, 0, 4), (300, 3, 16)]:
        w = S.generate_mixed(n, seed)
        s = S.deadline_first_candidate(w, w.ids(), c, mb)
        assert s.is_partition_of(w.ids(), mb)
        ev = S.evaluate(s, c, w)
        lead = ev.per_request[0]
        assert ev.n == 0 or lead.slo_met  # the first kept request starts at 0 and was admitted
    w = S.generate_mixed(1024, 0)
    s_sorted, _ = S.initial_candidates(w, w.ids(), c, 4)
    ev_dl = S.evaluate(S.deadline_first_candidate(w, w.ids(), c, 4), c, w)
    ev_sorted = S.evaluate(s_sorted, c, w)
    assert ev_dl.n >= 74 and ev_dl.n > ev_sorted.n and ev_dl.g > ev_sorted.g


def test_deadline_first_candidate_is_stable():
    """The deadline-first start seeds every chain, so its output is part of the K3 trajectories:
    pinned (sha256 of the batches) across host-side rewrites of the admission loop."""
    import hashlib
    c = S.table_coefficients()
    h = hashlib.sha256()
    for n in (5, 37, 256, 1024):
        for seed in (0, 1):
            w = S.generate_mixed(n, seed)
            for mb in (1, 4, 8):
                h.update(repr(S.deadline_first_candidate(w, w.ids(), c, mb).batches).encode())
    assert h.hexdigest() == "5f97608dae55a47f831bd1a9fac3033712984cf2fec6b586558384cbc3949d57"


def test_k3_model_philox_and_tick_objective():
    """The K3 model used by the GPU trajectory tests (tests/k3_model.py): its Philox matches the
    Random123 known answers; its SLO count is exactly CostModel::score's and its total latency
    within the grid's rounding of it, on random schedules."""
    import k3_model as K
    f = 0xFFFFFFFF
    assert K.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert K.philox4x32_10([f, f, f, f], [f, f]) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert K.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]
    import numpy as np
    from oracle import TABLE_COEFFS
    from oracle import port
    w = S.generate_mixed(48, 3)
    a = w.arrays
    from oracle import FlatWorkload
    fw = FlatWorkload(**{k: a[k] for k in ("id", "cls", "in_len", "true_out", "pred_out", "arrival", "class_id",
                                           "kind", "e2e", "ttft", "tpot")})
    ids = sorted(w.ids())
    ex, dl = E.build_tables(w, ids, S.table_coefficients(), 4)
    tick = 2.0 ** -int(np.floor(np.log2((2 ** 27 - 1) / ex.max())))
    prob = K.TickProblem(ex, dl, tick)
    rs = np.random.default_rng(5)
    for _ in range(20):
        perm = rs.permutation(48)
        sizes, left = [], 48
        while left:
            k = int(rs.integers(1, min(4, left) + 1))
            sizes.append(k)
            left -= k
        batches, q = [], 0
        for s in sizes:
            batches.append([int(x) for x in perm[q:q + s]])
            q += s
        nm, t, g = prob.score(batches)
        o_n, o_t, o_g = port.score_batch(fw, TABLE_COEFFS, ids, 4, perm[None, :].astype(np.int32), [sizes])
        assert abs(t - o_t[0]) <= 48 * 48 * tick and nm == o_n[0]


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the driver's reference arm) runs the unmodified reference on the
    host cores and prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--n", "256"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "evals/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the same config object as the GPU arm's line (bench_config), so the driver can pair the arms
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    assert line["config"] == bench.bench_config(argparse.Namespace(n=256, mb=4, budget_ms=10.0, chains=16384), 1)


def test_bench_reference_arm_never_loads_the_product():
    """The reference arm runs the reference's own generator and anneal(): libslosched_b200.so stays
    unmapped in that process."""
    import subprocess
    import sys
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', '--n', '64'];"
            "import bench; bench.main(); maps = open('/proc/self/maps').read();"
            "print('MAPPED', 'libslosched_b200' in maps, 'libslosched_ref' in maps)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "MAPPED False True"
