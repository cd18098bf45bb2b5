"""Sweep the chain schedule (t0, tau, iter, scale ladder) at a fixed device budget; report the
exact attainment / G of the returned schedule for the bench workload (N=1024, mb=4).

    python tools/quality_sweep.py [--budget-ms 9.5] [--chains 16384]
"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14966_b200 as S  # noqa: E402

LADDERS = {
    "x1": (1.0,),
    "1..1e5": (1.0, 10.0, 100.0, 1000.0, 1e4, 1e5),
    "1e2..1e6": (1e2, 1e3, 1e4, 1e5, 1e6),
    "1e3..1e7": (1e3, 1e4, 1e5, 1e6, 1e7),
    "1e4..1e8": (1e4, 1e5, 1e6, 1e7, 1e8),
    "1e5..1e9": (1e5, 1e6, 1e7, 1e8, 1e9),
}
SCHEDULES = [(500.0, 0.7, 60), (500.0, 0.7, 100), (500.0, 0.7, 160), (500.0, 0.5, 200), (500.0, 0.85, 60),
             (2000.0, 0.7, 100), (100.0, 0.8, 100)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget-ms", type=float, default=9.5)
    ap.add_argument("--chains", type=int, default=16384)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--ladders", default="1e3..1e7,1e4..1e8,1e5..1e9")
    ap.add_argument("--schedules", default=None, help="t0:tau:iter,... (default: the built-in list)")
    ap.add_argument("--workload-seed", type=int, default=0)
    ap.add_argument("--out", default=None, help="append the rows (JSONL)")
    args = ap.parse_args()
    scheds = SCHEDULES if not args.schedules else [tuple(float(x) if i < 2 else int(x) for i, x in enumerate(s.split(":")))
                                                   for s in args.schedules.split(",")]
    c = S.table_coefficients()
    w = S.generate_mixed(args.n, args.workload_seed)
    ids = w.ids()
    rows = []
    grid = itertools.product([(k, LADDERS[k]) for k in args.ladders.split(",")], scheds)
    for (lname, ladder), (t0, tau, it) in grid:
        for chains in (args.chains, args.chains // 4):
            ns, gs = [], []
            for seed in range(args.seeds):
                cfg = S.AnnealConfig(t0=t0, tau=tau, iter=it, seed=seed, chains=chains, budget_ms=args.budget_ms,
                                     scale_ladder=ladder)
                seq, sizes, n_met, t, g, st = S.anneal_flat(w, ids, c, cfg, 4)
                ns.append(n_met)
                gs.append(g)
            row = dict(ladder=lname, t0=t0, tau=tau, iter=it, chains=chains, n_met=ns, g=[f"{x:.5e}" for x in gs],
                       levels=st.levels_run, g_mean=sum(gs) / len(gs), n=args.n, workload_seed=args.workload_seed)
            rows.append(row)
            print(json.dumps(row), flush=True)
            if args.out:
                with open(args.out, "a") as f:
                    f.write(json.dumps(row) + "\n")
    best = max(rows, key=lambda r: r["g_mean"])
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
