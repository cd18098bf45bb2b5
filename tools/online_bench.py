"""BASELINE configs[4]: online rolling-window rescheduling over a Poisson stream.

    python tools/online_bench.py [--n 100000] [--instances 8] [--load 0.9] [--window-ms 5000]
                                 [--budget-ms 10] [--chains 4096] [--out profiles/r1/online.json]

Prints one JSON object: the stream (rate = load x instances x per-instance service rate), and
per policy (GPU SA, FCFS) realized attainment, average latency, G and the per-window scheduling
overhead (wall ms for planning all instances of a window concurrently).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_14966_b200 import online as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--load", type=float, default=0.9)
    ap.add_argument("--window-ms", type=float, default=5000.0)
    ap.add_argument("--budget-ms", type=float, default=10.0)
    ap.add_argument("--chains", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policies", default="sa,fcfs")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    mu = O.service_rate_per_s()
    rate = args.load * args.instances * mu
    stream = O.make_stream(args.n, rate, seed=args.seed)
    out = {"config": "configs[4]: online rolling-window rescheduling, Poisson arrivals",
           "requests": args.n, "instances": args.instances, "load": args.load,
           "service_rate_per_instance_req_s": mu, "arrival_rate_req_s": rate, "window_ms": args.window_ms,
           "budget_ms_per_window": args.budget_ms, "chains_per_instance": args.chains, "results": {}}
    for pol in args.policies.split(","):
        t = time.perf_counter()
        r = O.run_online(stream, pol, n_instances=args.instances, window_ms=args.window_ms,
                         budget_ms=args.budget_ms, chains=args.chains, seed=args.seed)
        s = r.summary()
        s["wall_s"] = time.perf_counter() - t
        out["results"][pol] = s
        print(json.dumps({pol: s}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
