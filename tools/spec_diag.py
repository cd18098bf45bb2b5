"""Why proposals leave K3's speculative stage: build the library with -DSLO_DIAG (the scan
statistics then carry category counts) and run this against it, e.g.
    SLO_EXTRA_NVCC=-DSLO_DIAG python -m paper_2504_14966_b200.build --force && cp ... libDIAG.so
    SLOSCHED_LIB=.../libDIAG.so python tools/spec_diag.py
(64 chains, so the 16-bit fields cannot overflow)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E
c = S.table_coefficients()
MB = int(os.environ.get("MB", "4"))
for n in (1024, 4096):
    w = S.generate_mixed(n, 0); ids = sorted(w.ids())
    s, i = S.initial_candidates(w, ids, c, MB); d = S.deadline_first_candidate(w, ids, c, MB)
    ev = max([S.evaluate(x, c, w) for x in (s, i, d)], key=lambda e: e.g)
    pos = {r: k for k, r in enumerate(ids)}
    eng = E.Engine(0); ex, dl = E.build_tables(w, ids, c, MB); eng.set_problem(ex, dl)
    for lev in (3, 7):
        t0, tau = 500.0, 0.7
        eng.prepare([pos[x] for x in ev.schedule.flatten()], [len(b) for b in ev.schedule.batches], t0=t0, tau=tau, iter=100,
                    t_thres=t0 * tau ** (lev - 0.5), seed=0, objective_scale=t0 / ev.g, chains=64, scale_ladder=(1e4, 1e5, 1e6, 1e7, 1e8))
        eng.launch(); bp, bs, r = eng.fetch()
        p1, p2 = r.positions_pass1, r.positions_pass2
        print(n, lev, "proposals", r.proposals, "accepted", r.accepted, "general: squeeze/delay", p2 & 0xffff, "live-region swap", p2 >> 16,
              "dead-region general (accepted/shift)", p1)
