"""Fixed-work K2 (exact replay) launch for timing / ncu: `chains` independent reference walks
(chain c = Rng(seed + c)) of the default AnnealConfig at N requests.

    python tools/prof_replay.py [--n 1024] [--chains 1] [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14966_b200 as S  # noqa: E402
from paper_2504_14966_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--mb", type=int, default=4)
    ap.add_argument("--chains", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    w = S.generate_mixed(a.n, 0)
    c = S.table_coefficients()
    ids = sorted(w.ids())
    s, i = S.initial_candidates(w, ids, c, a.mb)
    ev_s, ev_i = S.evaluate(s, c, w), S.evaluate(i, c, w)
    start, f0 = (s, ev_s.g) if ev_s.g >= ev_i.g else (i, ev_i.g)
    pos = {r: k for k, r in enumerate(ids)}
    eng = E.Engine(0)
    ex, dl = E.build_tables(w, ids, c, a.mb)
    eng.set_problem(ex, dl)
    kw = dict(t0=500.0, t_thres=20.0, iter=100, tau=0.95, seed=0, objective_scale=500.0 / f0, replay=True,
              chains=a.chains)
    eng.prepare([pos[x] for x in start.flatten()], [len(b) for b in start.batches], **kw)
    for r in range(a.reps):
        t = time.perf_counter()
        eng.launch()
        bp, bs, res = eng.fetch()
        wall = time.perf_counter() - t
        print(f"rep {r}: {res.proposals} proposals in {res.kernel_ms:.3f} ms = "
              f"{res.kernel_ms * 1e3 / max(1, res.proposals / a.chains):.2f} us/proposal/chain, "
              f"{res.proposals / res.kernel_ms * 1e3:.3e}/s total, g={res.g:.6e} n={res.n_met}, wall {wall*1e3:.1f} ms")


if __name__ == "__main__":
    main()
