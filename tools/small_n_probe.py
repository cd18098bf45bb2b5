import time, sys
sys.path.insert(0, '.')
import paper_2504_14966_b200 as S
c = S.table_coefficients()
for n in (8, 16, 24, 48):
    w = S.generate_mixed(n, 1)
    for mb in (0, 18):
        cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=30, chains=4096, budget_ms=9.3, scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5), max_blocks=mb)
        S.anneal_flat(w, w.ids(), c, cfg, 4)
        t = time.perf_counter()
        for _ in range(10):
            st = S.anneal_flat(w, w.ids(), c, cfg, 4)[5]
        print(n, mb, "wall %.3f ms" % ((time.perf_counter() - t) * 100), "kernel %.3f ms" % st.kernel_ms, "props", st.proposals, "levels", st.levels_run)
