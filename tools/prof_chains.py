"""Fixed-work chain launch for ncu and A/B timing (no device budget, so every replay of the
kernel does identical work).

    python tools/prof_chains.py [n] [chains] [reps] [3class]
        legacy shape: reference start, t0=500 tau=0.5 iter=32, scale ladder 1..1e5
    python tools/prof_chains.py --bench [--n 1024] [--chains 16384] [--levels 8] [--reps 1]
        bench.py's configuration (best of the three starts, t0=500 tau=0.7 iter=300, scale ladder
        1e4..1e8) for a fixed number of temperature levels (8 ~ the levels the 9 ms device
        budget allows at N=1024), so the ncu instruction count per proposal describes the bench run
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14966_b200 as S  # noqa: E402
from paper_2504_14966_b200 import engine as E  # noqa: E402

BENCH_LADDER = (1e4, 1e5, 1e6, 1e7, 1e8)  # bench.py SCALE_LADDER


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pos", nargs="*")
    ap.add_argument("--bench", action="store_true")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--mb", type=int, default=4)
    ap.add_argument("--chains", type=int, default=16384)
    ap.add_argument("--levels", type=int, default=8)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    n, chains, reps, three = a.n, a.chains, a.reps, False
    if a.pos:
        n = int(a.pos[0])
        chains = int(a.pos[1]) if len(a.pos) > 1 else 16384
        reps = int(a.pos[2]) if len(a.pos) > 2 else 3
        three = len(a.pos) > 3 and a.pos[3] == "3class"
    w = S.generate_mixed(n, 0)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    if three:  # configs[0] mix: code / chat / offline (E2E 1e9 ms)
        code, chat = S.default_slo_classes()
        reqs = [S.Request(r.id, 2 if r.id % 3 == 2 else r.task_class_id, r.input_len, r.true_output_len,
                          r.predicted_output_len) for r in w.requests]
        w = S.Workload(reqs, [code, chat, S.TaskClass(2, "offline", S.SloSpec.e2e(1e9))])
    s, i = S.initial_candidates(w, ids, c, a.mb)
    ev_s, ev_i = S.evaluate(s, c, w), S.evaluate(i, c, w)
    pos = {r: k for k, r in enumerate(ids)}
    eng = E.Engine(0)
    ex, dl = E.build_tables(w, ids, c, a.mb)
    eng.set_problem(ex, dl)
    if a.bench:
        start, f0 = (s, ev_s.g) if ev_s.g >= ev_i.g else (i, ev_i.g)
        d = S.deadline_first_candidate(w, ids, c, a.mb)
        ev_d = S.evaluate(d, c, w)
        if ev_d.g > f0:
            start, f0 = d, ev_d.g
        t0, tau, it = 500.0, 0.7, 300
        t_thres = t0 * tau ** (a.levels - 0.5)
        kw = dict(t0=t0, tau=tau, iter=it, t_thres=t_thres, seed=0, objective_scale=t0 / f0, chains=chains,
                  scale_ladder=BENCH_LADDER)
    else:
        start = s
        kw = dict(t0=500.0, tau=0.5, iter=32, seed=0, objective_scale=500.0 / ev_s.g, chains=chains,
                  scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5))
    eng.prepare([pos[x] for x in start.flatten()], [len(b) for b in start.batches], **kw)
    for r in range(reps):
        eng.launch()
        bp, bs, res = eng.fetch()
        print(f"rep {r}: {res.proposals} proposals in {res.kernel_ms:.3f} ms = "
              f"{res.proposals / res.kernel_ms * 1e3:.3e}/s, g={res.g:.4e} n={res.n_met} levels={res.levels_run} "
              f"exact_tests={getattr(res, 'exact_walks', -1)}")


if __name__ == "__main__":
    main()
