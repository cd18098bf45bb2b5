"""Per-decision comparison behind configs[4]: the same instance-queue snapshots (queue, planning
time) planned by the GPU chains and by the unmodified reference's CPU anneal(), scored by the
objective both optimise (G = SLOs met / summed latency over the queue, remaining-slack SLOs;
evaluate(), P:src/objective.cpp:55-82).

    python tools/online_decisions.py [--n 20000] [--every 25] [--out profiles/r2/online_decisions.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2504_14966_b200 as S  # noqa: E402
from paper_2504_14966_b200 import online as O  # noqa: E402
from tools.online_bench import reference_planner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--every", type=int, default=25)
    ap.add_argument("--chains", type=int, default=4096)
    ap.add_argument("--budget-ms", type=float, default=10.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    mu = O.service_rate_per_s()
    stream = O.make_stream(a.n, 0.9 * a.instances * mu, seed=0)
    snaps = []
    O.run_online(stream, "fcfs", n_instances=a.instances, snapshots=snaps, snapshot_every=a.every)
    c = S.table_coefficients()
    ref_plan = reference_planner()
    share = max(1, 148 // a.instances)
    rows = []
    for ids, start in snaps:
        w = O.window_workload(stream, ids, start)
        cfg = S.AnnealConfig(t0=500.0, tau=0.7, iter=30, seed=len(rows), chains=a.chains, budget_ms=a.budget_ms - 1.0,
                             scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5), max_blocks=share, deadline_start=False)
        gpu = S.anneal(w, [int(i) for i in ids], c, cfg, 4).best
        ref = S.evaluate(S.Schedule(ref_plan(stream, ids, start)), c, w)
        rows.append((len(ids), gpu.g, ref.g, gpu.n, ref.n))
    r = np.asarray(rows, dtype=np.float64)
    out = {"snapshots": len(rows), "queue_len_mean": float(r[:, 0].mean()),
           "gpu_g_ge_ref": float(np.mean(r[:, 1] >= r[:, 2])), "gpu_g_gt_ref": float(np.mean(r[:, 1] > r[:, 2])),
           "gpu_n_ge_ref": float(np.mean(r[:, 3] >= r[:, 4])),
           "g_ratio_mean_where_ref_positive": float(np.mean(r[r[:, 2] > 0, 1] / r[r[:, 2] > 0, 2])),
           "n_met_gpu": int(r[:, 3].sum()), "n_met_ref": int(r[:, 4].sum())}
    lose = r[:, 1] < r[:, 2]
    if lose.any():
        gap = (r[lose, 2] - r[lose, 1]) / r[lose, 2]
        out["gpu_below_ref_rel_gap"] = {"count": int(lose.sum()), "max": float(gap.max()), "median": float(np.median(gap)),
                                        "queue_len_mean": float(r[lose, 0].mean())}
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
