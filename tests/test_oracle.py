"""Pin the C restatement (oracle/slo_oracle.c) before trusting it.

1. Against the committed golden vectors produced by the unmodified reference
   (tests/golden/make_golden.py) -- always runs.
2. Against oracle/_ref live on fresh random cases -- when the reference library
   is built (it travels to the GPU box with the snapshot).
Everything here is CPU-only.
"""
import numpy as np
import pytest

from conftest import golden, unhex
from oracle import TABLE_COEFFS, FlatWorkload


def _gen(port, n, seed, mode=1):
    return port.generate_mixed(n, seed, mode)


def test_rng_streams_match_golden(port):
    g = golden("rng")
    for seed, vals in g["u64"].items():
        r = port.Rng(int(seed))
        assert [r.next_u64() for _ in vals] == [int(v) for v in vals]
    for seed, vals in g["uniform"].items():
        r = port.Rng(int(seed))
        assert [r.uniform() for _ in vals] == [unhex(v) for v in vals]
    for seed, vals in g["normal"].items():
        r = port.Rng(int(seed))
        assert [r.normal() for _ in vals] == [unhex(v) for v in vals]
    for case in g["index"]:
        r = port.Rng(case["seed"])
        assert [r.uniform_index(int(b)) for b in case["bounds"]] == [int(v) for v in case["out"]]
    for seed, stream, want in g["derive"]:
        assert port.derive(seed, stream) == int(want)


def test_latency_known_answers(port):
    # P:tests/test_latency_model.cpp:63-116 known answers
    c = TABLE_COEFFS
    assert port.predict(c, 1, 100, 2)[3] == pytest.approx(92.83924, rel=1e-12)
    assert port.predict(c, 1, 100, 2)[0] == pytest.approx(60.37, rel=1e-12)
    assert port.predict(c, 4, 500, 1)[0] == pytest.approx(271.47, rel=1e-12)
    assert port.predict(c, 1, 100, 2)[2] == pytest.approx(32.46924, rel=1e-12)
    assert port.predict(c, 1, 100, 2)[4] == pytest.approx(16.23462, rel=1e-12)
    for case in golden("latency"):
        v = port.predict(c, case["b"], case["li"], case["lo"])
        assert v[0] == unhex(case["prefill"])
        assert v[2] == unhex(case["decode_total"])
        assert v[3] == unhex(case["exec"])
        assert v[4] == unhex(case["tpot"])


def test_generate_mixed_matches_golden(port):
    for case in golden("generate_mixed"):
        w = port.generate_mixed(case["n"], case["seed"], case["mode"])
        for k in ("id", "cls", "in_len", "true_out", "pred_out"):
            assert list(getattr(w, k)) == case[k], k


def test_evaluate_matches_golden(port):
    for case in golden("evaluate"):
        w = _gen(port, case["n"], case["seed"])
        nm, t, g, per = port.evaluate(w, TABLE_COEFFS, case["batches"])
        assert nm == case["n_met"]
        assert t == unhex(case["t"]) and g == unhex(case["g"])
        assert [float(x) for x in per["wait"]] == [unhex(x) for x in case["wait"]]
        assert [float(x) for x in per["e2e"]] == [unhex(x) for x in case["e2e"]]
        assert list(per["met"]) == case["met"]


def test_evaluate_known_answers(port):
    # P:tests/test_objective.cpp:109-148: identity coefficients, exec = input_len
    ident = (0, 0, 1.0, 0, 0, 0, 0, 0)
    w = FlatWorkload(id=[0, 1, 2], cls=[0, 0, 1], in_len=[300, 500, 800], true_out=[1, 1, 1],
                     pred_out=[1, 1, 1], arrival=[0, 0, 0], class_id=[0, 1], kind=[0, 0],
                     e2e=[1e9, 1500.0], ttft=[0, 0], tpot=[0, 0])
    nm, t, g, per = port.evaluate(w, ident, [[0], [1], [2]])
    assert nm == 2 and t == 2700.0 and g * 1000 == pytest.approx(0.74, rel=0.005)
    assert list(per["wait"]) == [0.0, 300.0, 800.0]
    nm, t, g, _ = port.evaluate(w, ident, [])
    assert (nm, t, g) == (0, 0.0, 0.0)


def test_initial_candidates_match_golden(port):
    for case in golden("initial_candidates"):
        w = _gen(port, case["n"], case["seed"])
        s, i = port.initial_candidates(w, TABLE_COEFFS, list(w.id), case["mb"])
        assert s == case["sorted"] and i == case["input"]


def test_anneal_matches_golden(port):
    for case in golden("anneal"):
        w = _gen(port, case["n"], case["wseed"])
        res = port.anneal(w, TABLE_COEFFS, list(w.id), case["mb"], seed=case["seed"], **case["cfg"])
        assert res["batches"] == case["batches"], case["n"]
        assert res["n"] == case["n_met"] and res["g"] == unhex(case["g"]) and res["t"] == unhex(case["t"])
        assert res["proposals"] == case["proposals"] and res["accepted"] == case["accepted"]
        assert res["shortcut"] == case["shortcut"]
        assert res["objective_scale_used"] == unhex(case["scale"])


def test_anneal_edge_cases(port):
    w = _gen(port, 4, 1)
    res = port.anneal(w, TABLE_COEFFS, [], 2)  # empty set: vacuous shortcut
    assert res["shortcut"] and res["batches"] == [] and res["g"] == 0.0
    with pytest.raises(ValueError):
        port.anneal(w, TABLE_COEFFS, list(w.id), 2, t0=10.0, t_thres=20.0)
    with pytest.raises(ValueError):
        port.anneal(w, TABLE_COEFFS, [999], 2)


@pytest.mark.parametrize("n,mb", [(8, 2), (64, 4), (200, 8)])
def test_port_matches_reference_live(ref, port, n, mb):
    rs = np.random.default_rng(n * 31 + mb)
    for trial in range(3):
        seed = int(rs.integers(0, 2**62))
        w = ref.generate_mixed(n, seed % 1000, 1)
        a = ref.anneal(w, TABLE_COEFFS, list(w.id), mb, seed=seed, t0=100.0, iter=30)
        b = port.anneal(w, TABLE_COEFFS, list(w.id), mb, seed=seed, t0=100.0, iter=30)
        assert a == b
        batches = a["batches"]
        ra, rb = ref.evaluate(w, TABLE_COEFFS, batches), port.evaluate(w, TABLE_COEFFS, batches)
        assert ra[:3] == rb[:3]
