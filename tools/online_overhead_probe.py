"""Per-window planning wall of the native online driver vs the instance count (same per-instance
load), with K5 and with K3 for the short queues (SLOSCHED_SMALL_KERNEL=0)."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2504_14966_b200 import online as O  # noqa: E402

mu = O.service_rate_per_s()
for flag in ("1", "0"):
    os.environ["SLOSCHED_SMALL_KERNEL"] = flag
    for k in (1, 2, 4, 8):
        s = O.make_stream(400 * k, rate_per_s=0.9 * k * mu, seed=3)
        r = O.run_online(s, "sa", n_instances=k, window_ms=5000.0, budget_ms=10.0, chains=4096)
        ov = np.asarray(r.overhead_ms[5:])
        print(f"K5={flag} k={k} windows={r.windows} overhead mean {ov.mean():.3f} p50 {np.median(ov):.3f} "
              f"p99 {np.percentile(ov, 99):.3f} ms, attainment {r.n_met / r.n:.4f}", flush=True)
