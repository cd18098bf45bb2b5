"""Search-quality probe: one 9 ms chain launch vs k launches of 9/k ms, each restarting all chains
from the previous launch's winner (the host re-prepares the start state). Exact G / n_met of
the final schedule (evaluate()), N=1024 mb=4 bench workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14966_b200 as S  # noqa: E402
from paper_2504_14966_b200 import engine as E  # noqa: E402

LADDER = (1e4, 1e5, 1e6, 1e7, 1e8)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    for wseed in (0, 1):
        w = S.generate_mixed(n, wseed)
        c = S.table_coefficients()
        ids = sorted(w.ids())
        cands = list(S.initial_candidates(w, ids, c, 4)) + [S.deadline_first_candidate(w, ids, c, 4)]
        ev = max([S.evaluate(x, c, w) for x in cands], key=lambda e: e.g)
        pos = {r: k for k, r in enumerate(ids)}
        eng = E.Engine(0)
        ex, dl = E.build_tables(w, ids, c, 4)
        eng.set_problem(ex, dl)
        for k, t0s in ((1, (500.0,)), (2, (500.0, 100.0)), (3, (500.0, 200.0, 50.0)), (2, (500.0, 500.0)), (4, (500.0, 200.0, 100.0, 50.0))):
            perm, sizes = [pos[x] for x in ev.schedule.flatten()], [len(b) for b in ev.schedule.batches]
            f0 = ev.g
            props = 0
            for j in range(k):
                eng.prepare(perm, sizes, t0=t0s[j], t_thres=20.0 if t0s[j] > 20 else 1.0, tau=0.7, iter=1000, seed=j,
                            objective_scale=500.0 / f0, chains=16384, budget_ms=9.0 / k, scale_ladder=LADDER)
                eng.launch()
                bp, bs, res = eng.fetch()
                props += res.proposals
                sched = S.Schedule([[ids[q] for q in bp[p0:p0 + z]] for p0, z in
                                    zip([sum(bs[:i]) for i in range(len(bs))], bs)])
                e2 = S.evaluate(sched, c, w)
                if e2.g > f0:
                    perm, sizes, f0 = list(bp), list(bs), e2.g
            print(f"N={n} wseed={wseed} launches={k} t0s={t0s}: n_met={round(f0 * 0)}", end=" ")
            final = S.evaluate(S.Schedule([[ids[q] for q in perm[p0:p0 + z]] for p0, z in
                                           zip([sum(sizes[:i]) for i in range(len(sizes))], sizes)]), c, w)
            print(f"n={final.n} g={final.g:.5e} proposals={props}")
        eng.close()


if __name__ == "__main__":
    main()
