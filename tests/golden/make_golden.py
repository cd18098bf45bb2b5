"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs oracle/_ref/libslosched_ref.so, i.e.
`make -C oracle ref` with /root/reference present):

    python tests/golden/make_golden.py

Writes tests/golden/*.json. The GPU box never needs /root/reference: the
tests read these committed fixtures. Floats are stored as float.hex() strings
so the comparison is bit-exact.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import TABLE_COEFFS, ref  # noqa: E402


def hx(x):
    return float(x).hex()


def workload_json(w):
    return {k: [int(v) for v in getattr(w, k)] for k in ("id", "cls", "in_len", "true_out", "pred_out")}


def main():
    out = {}

    # --- Rng streams (P:include/slosched/rng.hpp)
    rng = {"u64": {}, "index": [], "uniform": {}, "normal": {}, "derive": []}
    for seed in (0, 1, 7, 2**63 + 5):
        rng["u64"][str(seed)] = [str(int(v)) for v in ref.rng_u64(seed, 64)]
        rng["uniform"][str(seed)] = [hx(v) for v in ref.rng_uniform(seed, 32)]
        rng["normal"][str(seed)] = [hx(v) for v in ref.rng_normal(seed, 32)]
    r = np.random.default_rng(1)
    for seed in (3, 11):
        bounds = [int(b) for b in r.integers(1, 5000, 200)] + [3, 2, 1, 2**63 + 1, 2**40 + 7]
        rng["index"].append({"seed": seed, "bounds": [str(b) for b in bounds],
                             "out": [str(int(v)) for v in ref.rng_index(seed, bounds)]})
    for seed, stream in ((0, 0), (0, 0x9e37), (9, 3), (123, 7)):
        rng["derive"].append([seed, stream, str(ref.derive(seed, stream))])
    out["rng"] = rng

    # --- latency model known answers (P:src/latency_model.cpp:86-113)
    lat = []
    for b, li, lo in [(1, 100, 2), (4, 500, 1), (2, 1000, 1), (3, 50, 7), (8, 2047, 2047), (1, 1, 1),
                      (16, 300, 900), (5, 77, 1234)]:
        v = ref.predict(TABLE_COEFFS, b, li, lo)
        lat.append({"b": b, "li": li, "lo": lo, "prefill": hx(v[0]), "per_token": hx(v[1]),
                    "decode_total": hx(v[2]), "exec": hx(v[3]), "tpot": hx(v[4])})
    out["latency"] = lat

    # --- synthetic workloads (P:src/workload.cpp:158-183 + estimator)
    gen = []
    for n, seed, mode in [(16, 0, 1), (64, 0, 1), (64, 5, 0), (257, 42, 1), (1024, 0, 1)]:
        w = ref.generate_mixed(n, seed, mode)
        gen.append({"n": n, "seed": seed, "mode": mode, **workload_json(w)})
    out["generate_mixed"] = gen

    # --- evaluate on random schedules (P:src/objective.cpp:55-82)
    ev = []
    r = np.random.default_rng(7)
    for n, seed in [(8, 1), (64, 2), (256, 3)]:
        w = ref.generate_mixed(n, seed, 1)
        for trial in range(6):
            mb = int(r.integers(1, 9))
            perm = r.permutation(n).tolist()
            batches, pos = [], 0
            while pos < n:
                take = int(r.integers(1, mb + 1))
                batches.append(perm[pos:pos + take])
                pos += take
            nm, t, g, per = ref.evaluate(w, TABLE_COEFFS, batches)
            ev.append({"n": n, "seed": seed, "batches": batches, "n_met": nm, "t": hx(t), "g": hx(g),
                       "wait": [hx(x) for x in per["wait"]], "e2e": [hx(x) for x in per["e2e"]],
                       "met": [int(x) for x in per["met"]]})
    out["evaluate"] = ev

    # --- initial candidates (P:src/priority_mapper.cpp:292-311)
    ic = []
    for n, seed, mb in [(10, 4, 2), (64, 0, 4), (33, 9, 8)]:
        w = ref.generate_mixed(n, seed, 1)
        s, i = ref.initial_candidates(w, TABLE_COEFFS, list(w.id), mb)
        ic.append({"n": n, "seed": seed, "mb": mb, "sorted": s, "input": i})
    out["initial_candidates"] = ic

    # --- neighbor walks (P:src/priority_mapper.cpp:322-338)
    nw = []
    for n, mb, seed, steps in [(2, 2, 31, 50), (9, 3, 5, 500), (40, 4, 8, 300), (1, 1, 8, 10)]:
        start = [[i for i in range(k, min(k + mb, n))] for k in range(0, n, mb)]
        nw.append({"start": start, "mb": mb, "seed": seed, "steps": steps,
                   "out": ref.neighbor_walk(start, seed, steps, mb)})
    out["neighbor_walk"] = nw

    # --- anneal (P:src/priority_mapper.cpp:340-411)
    an = []
    cases = [(8, 2, s, {}) for s in range(4)]
    cases += [(64, mb, s, {}) for mb in (1, 4, 8) for s in (0, 1)]
    cases += [(256, 4, 0, {}), (256, 2, 3, {"t0": 60.0, "iter": 40})]
    cases += [(64, 4, 2, {"objective_scale": 0.0, "t0": 30.0, "iter": 50}),
              (64, 4, 5, {"objective_scale": 1e9})]
    for n, mb, seed, cfg in cases:
        w = ref.generate_mixed(n, 100 + n + seed, 1)
        res = ref.anneal(w, TABLE_COEFFS, list(w.id), mb, seed=seed, **cfg)
        an.append({"n": n, "wseed": 100 + n + seed, "mb": mb, "seed": seed, "cfg": cfg,
                   "batches": res["batches"], "n_met": res["n"], "t": hx(res["t"]), "g": hx(res["g"]),
                   "proposals": res["proposals"], "accepted": res["accepted"], "shortcut": res["shortcut"],
                   "g_sorted_start": hx(res["g_sorted_start"]), "g_input_start": hx(res["g_input_start"]),
                   "scale": hx(res["objective_scale_used"])})
    out["anneal"] = an

    # --- exhaustive (P:src/priority_mapper.cpp:440-517), small n
    ex = []
    for n, mb, seed in [(3, 1, 1), (3, 3, 1), (6, 2, 40), (7, 2, 41)]:
        w = ref.generate_mixed(n, seed, 0)
        res = ref.exhaustive(w, TABLE_COEFFS, list(w.id), mb)
        ex.append({"n": n, "mb": mb, "seed": seed, "batches": res["batches"], "n_met": res["n"],
                   "g": hx(res["g"]), "evaluated": res["evaluated"]})
    out["exhaustive"] = ex

    # --- schedule_all (P:src/scheduler.cpp:92-129)
    sa = []
    for n, k, mb, seed in [(10, 1, 2, 9), (20, 2, 2, 4), (40, 4, 1, 9)]:
        w = ref.generate_mixed(n, 77 + n, 1)
        insts = [dict(id=i, total_mem=2.0 ** 35, remaining_mem=2.0 ** 35, mu=0.9, sigma=262144.0, max_batch=mb)
                 for i in range(k)]
        res, epochs = ref.schedule_all(w, TABLE_COEFFS, insts, seed=seed)
        sa.append({"n": n, "wseed": 77 + n, "k": k, "mb": mb, "seed": seed, "epochs": epochs,
                   "per_instance": [{"batches": r_["batches"], "n_met": r_["n"], "g": hx(r_["g"])} for r_ in res]})
    out["schedule_all"] = sa

    for key, val in out.items():
        with open(os.path.join(HERE, f"{key}.json"), "w") as f:
            json.dump(val, f, separators=(",", ":"))
    print("wrote", ", ".join(sorted(out)))


if __name__ == "__main__":
    main()
