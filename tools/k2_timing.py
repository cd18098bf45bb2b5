"""Where K2's time per proposal goes (one exact reference chain, N=1024, default AnnealConfig):
cycles in the sequential score vs propose + apply + restage, from a -DSLO_K2_TIMING build.

    bash tools/build_variant.sh k2t -DSLO_K2_TIMING
    SLOSCHED_LIB=paper_2504_14966_b200/_variants/k2t.so python tools/k2_timing.py
"""
import sys, os
sys.path.insert(0, '.')
import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E
w = S.generate_mixed(1024, 0); c = S.table_coefficients(); ids = sorted(w.ids()); mb = 4
s, i = S.initial_candidates(w, ids, c, mb)
ev_s, ev_i = S.evaluate(s, c, w), S.evaluate(i, c, w)
start, f0 = (s, ev_s.g) if ev_s.g >= ev_i.g else (i, ev_i.g)
pos = {r: k for k, r in enumerate(ids)}
eng = E.Engine(0); ex, dl = E.build_tables(w, ids, c, mb); eng.set_problem(ex, dl)
kw = dict(t0=500.0, t_thres=20.0, iter=100, tau=0.95, seed=0, objective_scale=500.0 / f0, replay=True, chains=1)
bp, bs, r = eng.anneal_chains([pos[x] for x in start.flatten()], [len(b) for b in start.batches], **kw)
P = r.proposals
print("kernel_ms", r.kernel_ms, "us/prop", r.kernel_ms * 1e3 / P, "score cycles/prop", r.positions_pass1 / P, "pre cycles/prop", r.positions_pass2 / P, "total cycles/prop", r.kernel_ms * 1.965e6 / P)
