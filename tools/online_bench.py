"""BASELINE configs[4]: online rolling-window rescheduling over a Poisson stream.

    python tools/online_bench.py [--n 100000] [--instances 8] [--load 0.9] [--window-ms 5000]
                                 [--budget-ms 10] [--chains 4096] [--out profiles/r1/online.json]

Prints one JSON object: the stream (rate = load x instances x per-instance service rate), and
per policy realized attainment, average latency, G and the per-window scheduling overhead (wall ms
for planning all instances of a window concurrently). Policies:
  sa    the GPU chains, instances placed round-robin on --devices (default: every visible GPU)
  sa-dlstart  the same, with the deadline-first candidate among the chains' starts
  sa-full     every plan gets all --chains chains (the default sa arm scales them with the queue:
              64 per request, at least 256, so a short queue's plan ends well inside the budget)
  sa-py the sa arm through the Python dispatch loop (online._run_online_py) instead of the library's
        slosched_run_online: same plans, host overhead of the Python loop
  fcfs  arrival order, greedy batches (the reference's FCFS baseline)
  ref   the UNMODIFIED reference's CPU anneal() (oracle/_ref, default AnnealConfig) per window and
        instance, with the same remaining-slack SLOs the GPU arm plans with -- the reference
        scheduler run online on the host cores (one thread per instance)
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_14966_b200 import online as O  # noqa: E402


def reference_planner(max_batch=4, seed=0):
    """Per window: the reference's own anneal() on the instance queue (test infrastructure)."""
    import numpy as np

    from oracle import TABLE_COEFFS, FlatWorkload
    from oracle import ref

    def plan(stream, ids, start_ms):
        n = len(ids)
        waited = start_ms - stream.arrival_ms[ids]
        code = stream.cls[ids] == 0
        e2e = np.where(code, np.maximum(30000.0 - waited, O._IMPOSSIBLE_MS), 0.0)
        ttft = np.where(code, 0.0, np.maximum(10000.0 - waited, O._IMPOSSIBLE_MS))
        fw = FlatWorkload(id=np.asarray(ids), cls=np.arange(n), in_len=stream.input_len[ids],
                          true_out=stream.true_out[ids], pred_out=stream.pred_out[ids],
                          arrival=stream.arrival_ms[ids], class_id=np.arange(n), kind=np.where(code, 0, 1),
                          e2e=e2e, ttft=ttft, tpot=np.where(code, 0.0, 50.0))
        return ref.anneal(fw, TABLE_COEFFS, [int(i) for i in ids], max_batch, seed=seed)["batches"]
    return plan


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
    ap.add_argument("--devices", default=None, help="comma list of GPUs for the instances (default: all visible)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    mu = O.service_rate_per_s()
    rate = args.load * args.instances * mu
    stream = O.make_stream(args.n, rate, seed=args.seed)
    out = {"config": "configs[4]: online rolling-window rescheduling, Poisson arrivals",
           "requests": args.n, "instances": args.instances, "load": args.load,
           "service_rate_per_instance_req_s": mu, "arrival_rate_req_s": rate, "window_ms": args.window_ms,
           "budget_ms_per_window": args.budget_ms, "chains_per_instance": args.chains, "results": {}}
    if args.devices:
        devices = [int(d) for d in args.devices.split(",")]
    else:
        try:
            import torch
            devices = list(range(max(1, torch.cuda.device_count())))
        except Exception:
            devices = [0]
    out["devices"] = devices
    for pol in args.policies.split(","):
        t = time.perf_counter()
        if pol == "ref":
            kw = dict(policy="custom", planner=reference_planner(seed=args.seed))
        elif pol == "sa-dlstart":  # the chains also start from the deadline-first candidate
            kw = dict(policy="sa", anneal_kw=dict(deadline_start=True))
        elif pol == "sa-full":  # every window's plan gets all --chains chains (fills the budget)
            kw = dict(policy="sa", chains_per_request=1 << 30)
        else:
            kw = dict(policy=pol)
        fn = O.run_online
        if pol == "sa-py":
            kw, fn = dict(policy="sa"), O._run_online_py
        r = fn(stream, n_instances=args.instances, window_ms=args.window_ms, budget_ms=args.budget_ms,
                         chains=args.chains, seed=args.seed, devices=devices, **kw)
        s = r.summary()
        s["policy"] = pol
        s["wall_s"] = time.perf_counter() - t
        out["results"][pol] = s
        print(json.dumps({pol: s}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
