"""Small invocation of every kernel, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14966_b200 as S  # noqa: E402
from paper_2504_14966_b200 import engine as E  # noqa: E402

c = S.table_coefficients()
for n, mb, chains in [(5, 2, 8), (70, 4, 64), (300, 8, 100), (200, 16, 50), (1500, 4, 40), (3000, 4, 20)]:
    w = S.generate_mixed(n, n)
    r = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=1, chains=chains, t0=60.0, iter=40,
                                               scale_ladder=(1.0, 100.0)), mb)
    assert r.best.schedule.is_partition_of(w.ids(), mb)
    r = S.anneal(w, w.ids(), c, S.AnnealConfig(seed=2, t0=40.0, iter=20, mode=S.SearchMode.REPLAY), mb)
    eng = E.Engine(0)
    ex, dl = E.build_tables(w, w.ids(), c, mb)
    eng.set_problem(ex, dl)
    rs = np.random.default_rng(n)
    perms = np.stack([rs.permutation(n) for _ in range(16)]).astype(np.uint16)
    eng.evaluate_batch(perms, E.end_bits([[1] * n] * 16, n))
    eng.close()
w = S.generate_mixed(7, 3)
S.exhaustive(w, w.ids(), c, 2)
# more chains than resident warps: exercises parking
w = S.generate_mixed(64, 9)
S.anneal(w, w.ids(), c, S.AnnealConfig(seed=3, chains=148 * 24 + 50, t0=30.0, iter=8), 4)
# short queues (K5): every segmented-max depth, negative execs, parked chains, the fp64 path
for n, mb in [(6, 1), (12, 2), (9, 4), (20, 8), (31, 16)]:
    w = S.generate_mixed(n, 40 + n)
    S.anneal(w, w.ids(), c, S.AnnealConfig(seed=4, chains=96, t0=500.0, iter=30, scale_ladder=(1.0, 1e4)), mb)
base = S.table_coefficients()
cneg = S.LatencyCoefficients(base.alpha_p, base.beta_p, base.gamma_p, -2500.0, base.alpha_d, base.beta_d,
                             base.gamma_d, base.delta_d)
w = S.generate_mixed(11, 101)
S.anneal(w, w.ids(), cneg, S.AnnealConfig(seed=5, chains=64, t0=100.0, iter=30, max_blocks=1), 8)
eng = E.Engine(0)
n = 16
w = S.generate_mixed(n, 5)
ex, dl = E.build_tables(w, w.ids(), c, 1)
dl = dl.copy()
dl[0] = np.cumsum(ex[0])[np.arange(n) % (n - 1)]
eng.set_problem(ex, dl)
eng.anneal_chains(list(range(n)), [1] * n, chains=100, t0=200.0, t_thres=20.0, tau=0.7, iter=30, seed=5,
                  objective_scale=1e4, max_blocks=1)
eng.close()
print("sanitize run complete")
