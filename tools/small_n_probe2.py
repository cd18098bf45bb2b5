"""Short-queue chain throughput vs chain count, iterations per level and SM share (n = 6, 16, 48):
kernel time, proposals, proposals/s and acceptance per configuration."""
import sys, time
sys.path.insert(0, '.')
import paper_2504_14966_b200 as S
c = S.table_coefficients()
for n in (6, 16, 48):
    w = S.generate_mixed(n, 1)
    for ch, it, mbk in ((384, 30, 0), (384, 300, 0), (4096, 30, 0), (384, 30, 128)):
        cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=it, chains=ch, budget_ms=9.3, scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5), max_blocks=mbk)
        S.anneal_flat(w, w.ids(), c, cfg, 4)
        ks = []
        for _ in range(10):
            st = S.anneal_flat(w, w.ids(), c, cfg, 4)[5]
            ks.append(st.kernel_ms)
        k = sorted(ks)[5]
        print(n, ch, it, mbk, "kernel %.3f ms" % k, "props", st.proposals, "rate %.3e" % (st.proposals / k * 1e3), "acc %.2f" % (st.accepted / max(1, st.proposals)), flush=True)
