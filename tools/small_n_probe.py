"""Planning cost of the short queues an online window holds: one anneal() per n with
the online driver's settings (ladder t0=500, tau=0.7, iter=30, six scales, 64 chains per request,
at least 256), wall time per call, kernel time, proposals and levels."""
import sys
import time

sys.path.insert(0, '.')
import paper_2504_14966_b200 as S  # noqa: E402

c = S.table_coefficients()
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,6,8,12,16,24,48").split(",")]:
    w = S.generate_mixed(n, 1)
    cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=30, chains=min(4096, max(256, 64 * n)), budget_ms=9.3,
                         scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5))
    S.anneal_flat(w, w.ids(), c, cfg, 4)
    t = time.perf_counter()
    for _ in range(20):
        st = S.anneal_flat(w, w.ids(), c, cfg, 4)[5]
    print(n, "chains", cfg.chains, "wall %.3f ms" % ((time.perf_counter() - t) * 50), "kernel %.3f ms" % st.kernel_ms,
          "props", st.proposals, "levels", st.levels_run, flush=True)
