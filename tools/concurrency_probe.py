"""Wall time of k concurrent short-queue anneal() calls (the online driver's per-window planning):
sequential vs one host thread per instance, SM share per instance as the driver sets it."""
import sys
import threading
import time

sys.path.insert(0, '.')
import paper_2504_14966_b200 as S  # noqa: E402

c = S.table_coefficients()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ws = [S.generate_mixed(n, 10 + j) for j in range(k)]


def cfg(j):
    return S.AnnealConfig(t0=500.0, tau=0.7, iter=30, chains=max(256, 64 * n), budget_ms=9.0, seed=j,
                          scale_ladder=(1.0, 10.0, 100.0, 1e3, 1e4, 1e5), max_blocks=148 // k)


def one(j, out):
    t = time.perf_counter()
    r = S.anneal(ws[j], ws[j].ids(), c, cfg(j), 4)
    out[j] = ((time.perf_counter() - t) * 1e3, r.stats.kernel_ms, r.stats.shortcut)


for rep in range(3):
    out = [None] * k
    t = time.perf_counter()
    for j in range(k):
        one(j, out)
    seq = (time.perf_counter() - t) * 1e3
    out2 = [None] * k
    th = [threading.Thread(target=one, args=(j, out2)) for j in range(k)]
    t = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    par = (time.perf_counter() - t) * 1e3
    print(f"k={k} n={n} sequential {seq:.2f} ms (per call {[round(o[0], 2) for o in out]}, kernel "
          f"{[round(o[1], 2) for o in out]}) | threads {par:.2f} ms (per call {[round(o[0], 2) for o in out2]})",
          flush=True)
