"""One online-window-shaped anneal (short queue, online settings: t0=500 tau=0.7 iter=30, six
scales, 64 chains per request, at least 256; no device budget) for ncu: where the per-proposal
latency of short queues goes.

    python tools/prof_small.py [n] [reps]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14966_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = S.generate_mixed(n, 1)
c = S.table_coefficients()
cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=30, chains=min(4096, max(256, 64 * n)), budget_ms=0.0,
                     scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5))
for _ in range(reps):
    st = S.anneal_flat(w, w.ids(), c, cfg, 4)[5]
    print(f"n={n} chains={cfg.chains} kernel_ms={st.kernel_ms:.3f} proposals={st.proposals} "
          f"accepted={st.accepted} levels={st.levels_run}", flush=True)
