"""Online rolling-window rescheduling over a Poisson request stream (BASELINE configs[4]).

The reference has no online mode (it schedules in synchronous waves); this driver
is the §8(f) row 2 extension, built on the public entry points:

* stream    -- request lengths from the reference's synthetic generator (generate_mixed, with
              estimator-predicted output lengths), Poisson arrivals at a stated rate;
* instances -- k serving instances placed round-robin on `devices` (one per GPU on an 8-GPU box;
              instances sharing a GPU split its SMs), requests assigned on arrival to the
              least-loaded instance;
* windows   -- every window_ms of simulated time each instance's queue (arrived, not yet
              started) is re-planned with anneal() under a per-window device budget; the plan's
              batches are dispatched until the next window boundary, the rest is re-planned;
* planning  -- the objective sees each request's remaining slack: its SLO minus the time it has
              already waited (a per-request SLO class), exactly the reference objective otherwise;
              the chains start from the reference's two candidates only (the deadline-first start
              raises each window's G but measured lower long-run attainment on a 20k stream:
              32.1 % vs 32.8 %, profiles/r2/online_config5.json);
* execution -- the library's replay (harness.realize_batches, csrc/harness.cpp): the reference
              simulator's ground truth -- latency model over the TRUE output lengths, 0.1 ms
              dispatch gap, noise 0 (P:src/simulator.cpp:17-74) -- on each instance's clock, every
              window; run() is the same routine and is pinned bit-for-bit to the reference's run()
              (tests/test_harness.py).

Policies: "sa" (GPU chains), "fcfs" (arrival order, greedy batches -- the reference's FCFS
baseline, P:src/simulator.cpp:76-123), "custom" (a caller's planner(stream, queue, start_ms) ->
batches; tools/online_bench.py plugs the reference's own CPU anneal() in per window).
"""
from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from .harness import realize_batches
from .slosched import (AnnealConfig, LatencyCoefficients, Request, SloSpec, TaskClass, Workload, anneal_flat,
                       generate_mixed, table_coefficients)

_IMPOSSIBLE_MS = 1e-9  # an SLO whose slack is already gone: positive (valid) but unreachable


def _coeffs(c: LatencyCoefficients):
    return (c.alpha_p, c.beta_p, c.gamma_p, c.delta_p, c.alpha_d, c.beta_d, c.gamma_d, c.delta_d)


def prefill_ms(c, b, li):
    ap, bp, gp, dp = _coeffs(c)[:4]
    return ap * b * li + bp * b + gp * li + dp


def decode_total_ms(c, b, li, lo):
    ad, bd, gd, dd = _coeffs(c)[4:]
    return (ad * b + gd) * (lo * li + lo * (lo + 1.0) / 2.0) + lo * (bd * b + dd)


@dataclass
class Stream:
    arrival_ms: np.ndarray
    cls: np.ndarray          # 0 = code (E2E 30 s), 1 = chat (TTFT 10 s + TPOT 50 ms)
    input_len: np.ndarray
    true_out: np.ndarray
    pred_out: np.ndarray
    rate_per_s: float

    @property
    def n(self):
        return len(self.arrival_ms)


def service_rate_per_s(coeffs=None, max_batch=4, samples=4096, seed=7):
    """Requests/s one instance completes when always busy with full batches: max_batch over the
    mean makespan of random batches drawn from the synthetic length distribution."""
    c = coeffs or table_coefficients()
    w = generate_mixed(samples, seed)
    li = w.arrays["in_len"].astype(np.float64)
    lo = w.arrays["true_out"].astype(np.float64)
    ex = prefill_ms(c, max_batch, li) + decode_total_ms(c, max_batch, li, lo)
    ex = ex[: (samples // max_batch) * max_batch].reshape(-1, max_batch)
    return max_batch / (ex.max(axis=1).mean() / 1000.0)


def make_stream(n: int, rate_per_s: float, seed: int = 0) -> Stream:
    w = generate_mixed(n, seed)  # reference synthetic lengths + estimator predictions
    a = w.arrays
    rs = np.random.default_rng(seed + 1)
    arrivals = np.cumsum(rs.exponential(1000.0 / rate_per_s, size=n))
    return Stream(arrivals, a["cls"].copy(), a["in_len"].copy(), a["true_out"].copy(), a["pred_out"].copy(),
                  rate_per_s)


@dataclass
class OnlineResult:
    policy: str
    n: int
    n_met: int
    total_latency_ms: float
    windows: int
    decisions: int
    proposals: int
    overhead_ms: List[float] = field(default_factory=list)

    def summary(self) -> Dict:
        ov = np.asarray(self.overhead_ms) if self.overhead_ms else np.zeros(1)
        return {"policy": self.policy, "requests": self.n, "attainment": self.n_met / self.n,
                "avg_latency_ms": self.total_latency_ms / self.n,
                "g_req_per_ms": self.n_met / self.total_latency_ms if self.total_latency_ms > 0 else 0.0,
                "windows": self.windows, "decisions": self.decisions, "proposals": self.proposals,
                "overhead_ms_mean": float(ov.mean()), "overhead_ms_p99": float(np.percentile(ov, 99)),
                "overhead_ms_max": float(ov.max())}


def window_workload(stream, ids, start_ms):
    """The planning view of one instance queue at start_ms: each request in a class of its own whose
    SLO is shrunk by the time it has already waited (the objective every planner optimises)."""
    classes, reqs = [], []
    for k, i in enumerate(ids):
        waited = start_ms - stream.arrival_ms[i]
        if stream.cls[i] == 0:
            slo = SloSpec.e2e(max(30000.0 - waited, _IMPOSSIBLE_MS))
        else:
            slo = SloSpec.ttft_tpot(max(10000.0 - waited, _IMPOSSIBLE_MS), 50.0)
        classes.append(TaskClass(k, f"r{i}", slo))
        reqs.append(Request(int(i), k, int(stream.input_len[i]), int(stream.true_out[i]), int(stream.pred_out[i]),
                            float(stream.arrival_ms[i])))
    return Workload(reqs, classes)


def _plan_sa(stream, ids, start_ms, coeffs, max_batch, cfg: AnnealConfig):
    """Plan one instance's queue with the GPU annealer; SLOs shrunk by the time already waited."""
    w = window_workload(stream, ids, start_ms)
    seq, sizes, _, _, _, st = anneal_flat(w, [int(i) for i in ids], coeffs, cfg, max_batch)
    out, pos = [], 0
    for s in sizes:
        out.append([int(x) for x in seq[pos:pos + s]])
        pos += int(s)
    return out, st.proposals, st.kernel_ms


_CLASSES = [TaskClass(0, "code", SloSpec.e2e(30000.0)), TaskClass(1, "chat", SloSpec.ttft_tpot(10000.0, 50.0))]


def _execute(stream, batches, c, clock0, gap, until):
    """Replay a plan on one instance clock until the window ends: (met, summed e2e, started ids, clock)."""
    ids = [i for b in batches for i in b]
    reqs = [Request(int(i), int(stream.cls[i]), int(stream.input_len[i]), int(stream.true_out[i]),
                    int(stream.pred_out[i]), float(stream.arrival_ms[i])) for i in ids]
    recs, clock, started = realize_batches(batches, Workload(reqs, _CLASSES), c, clock0, gap, gap, until,
                                           from_arrival=True)
    met = sum(1 for r in recs if r.slo_met)
    lat = 0.0
    for r in recs:
        lat += r.e2e_ms
    return met, lat, [i for b in batches[:started] for i in b], clock


def _plan_fcfs(stream, ids, max_batch):
    order = sorted(ids, key=lambda i: (stream.arrival_ms[i], i))
    return [order[k:k + max_batch] for k in range(0, len(order), max_batch)], 0, 0.0


def run_online(stream: Stream, policy: str = "sa", n_instances: int = 8, window_ms: float = 5000.0,
               max_batch: int = 4, budget_ms: float = 10.0, chains: int = 4096, seed: int = 0,
               coeffs: Optional[LatencyCoefficients] = None, dispatch_gap_ms: float = 0.1,
               max_windows: Optional[int] = None, scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5),
               t0: float = 500.0, tau: float = 0.7, iter: int = 30, devices: Sequence[int] = (0,),
               planner: Optional[Callable] = None, anneal_kw: Optional[Dict] = None,
               chains_per_request: int = 64, chains_min: int = 256,
               snapshots: Optional[List] = None, snapshot_every: int = 50) -> OnlineResult:
    """The online driver. "sa" and "fcfs" run in the library (csrc/online.cpp, slosched_run_online);
    a caller's planner ("custom"), snapshot capture or engine options other than deadline_start run
    the same loop in Python (_run_online_py; identical results on the same inputs)."""
    kw = dict(anneal_kw or {})
    native = (policy in ("sa", "fcfs") and planner is None and snapshots is None and set(kw) <= {"deadline_start"})
    if not native:
        return _run_online_py(stream, policy, n_instances, window_ms, max_batch, budget_ms, chains, seed, coeffs,
                              dispatch_gap_ms, max_windows, scale_ladder, t0, tau, iter, devices, planner, anneal_kw,
                              chains_per_request, chains_min, snapshots, snapshot_every)
    import ctypes

    from ._lib import SloOnlineConfig, SloOnlineResult, lib
    from .slosched import _check_api, _f64, _i32, _p
    c = coeffs or table_coefficients()
    devs = _i32(list(devices) or [0])
    lad = _f64(list(scale_ladder) or [1.0])
    cfg = SloOnlineConfig(0 if policy == "sa" else 2, n_instances, window_ms, max_batch, budget_ms, chains,
                          chains_per_request, chains_min, seed & (2**64 - 1), dispatch_gap_ms, len(devs), _p(devs),
                          len(lad), _p(lad, ctypes.c_double), t0, tau, iter, 1 if kw.get("deadline_start") else 0,
                          -1 if max_windows is None else max_windows)
    arr = _f64(stream.arrival_ms)
    cap = int(np.ceil((arr[-1] if len(arr) else 0.0) / window_ms)) + stream.n + 16
    ovh = np.zeros(cap)
    out = SloOnlineResult()
    _check_api(lib().slosched_run_online(stream.n, _p(arr, ctypes.c_double), _p(_i32(stream.cls)),
                                         _p(_i32(stream.input_len)), _p(_i32(stream.true_out)),
                                         _p(_i32(stream.pred_out)), _p(c.as_array(), ctypes.c_double),
                                         ctypes.byref(cfg), ctypes.byref(out), _p(ovh, ctypes.c_double), cap))
    return OnlineResult(policy, out.n, out.n_met, out.total_latency_ms, out.windows, out.decisions, int(out.proposals),
                        list(ovh[:min(out.windows, cap)]))


def _run_online_py(stream: Stream, policy: str = "sa", n_instances: int = 8, window_ms: float = 5000.0,
               max_batch: int = 4, budget_ms: float = 10.0, chains: int = 4096, seed: int = 0,
               coeffs: Optional[LatencyCoefficients] = None, dispatch_gap_ms: float = 0.1,
               max_windows: Optional[int] = None, scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5),
               t0: float = 500.0, tau: float = 0.7, iter: int = 30, devices: Sequence[int] = (0,),
               planner: Optional[Callable] = None, anneal_kw: Optional[Dict] = None,
               chains_per_request: int = 64, chains_min: int = 256,
               snapshots: Optional[List] = None, snapshot_every: int = 50) -> OnlineResult:
    c = coeffs or table_coefficients()
    n = stream.n
    queue: List[List[int]] = [[] for _ in range(n_instances)]
    busy_until = np.zeros(n_instances)
    load = np.zeros(n_instances)     # outstanding predicted work per instance (assignment key)
    next_arrival = 0
    done = 0
    n_met, total_lat, proposals, decisions = 0, 0.0, 0, 0
    overhead: List[float] = []
    # instance k runs on devices[k % len]; instances sharing a device split its SMs
    dev_of = [int(devices[k % len(devices)]) for k in range(n_instances)]
    share = [0] * n_instances
    if policy == "sa":
        import ctypes
        from ._lib import lib
        for d in set(dev_of):
            ctx = ctypes.c_void_p()
            if lib().slo_ctx_create(d, ctypes.byref(ctx)) == 0:
                sms = int(lib().slo_ctx_sm_count(ctx))
                lib().slo_ctx_destroy(ctx)
                for k in range(n_instances):
                    if dev_of[k] == d:
                        share[k] = max(1, sms // dev_of.count(d))
    if policy == "custom" and planner is None:
        raise ValueError("run_online: policy 'custom' needs a planner")
    pool = ThreadPoolExecutor(n_instances) if policy in ("sa", "custom") else None
    t_win = 0.0
    windows = 0
    host_ms = 1.5  # host share of a window's planning (updated from measurements)
    while done < n and (max_windows is None or windows < max_windows):
        t_next = t_win + window_ms
        # arrivals up to this window start join the least-loaded instance
        while next_arrival < n and stream.arrival_ms[next_arrival] <= t_win:
            i = next_arrival
            inst = int(np.argmin(np.maximum(busy_until, t_win) + load))
            queue[inst].append(i)
            load[inst] += prefill_ms(c, 1, stream.input_len[i]) + decode_total_ms(c, 1, stream.input_len[i],
                                                                                  stream.pred_out[i])
            next_arrival += 1
        if not any(queue) and next_arrival < n:  # idle: jump to the first window holding an arrival
            t_win = max(t_win, np.ceil(stream.arrival_ms[next_arrival] / window_ms) * window_ms)
            continue
        windows += 1
        # plan every non-empty instance queue (concurrently, one engine context each)
        active = [k for k in range(n_instances) if queue[k]]
        if snapshots is not None and windows % snapshot_every == 0:  # planning inputs, for offline study
            snapshots.extend((list(queue[k]), max(busy_until[k], t_win)) for k in active)
        t0_wall = time.perf_counter()
        if policy == "sa":
            # the window's planning (host setup of every instance, kernels, copies) fits the budget:
            # the chains get what the measured host share of recent windows leaves, less 0.3 ms
            kernel_budget = max(0.5, budget_ms - host_ms - 0.3)

            def plan(k):
                # chains in proportion to the queue (a short queue's search space is tiny: the
                # ladder then finishes well inside the budget instead of filling it)
                nq = len(queue[k])
                ch = min(chains, max(chains_min, chains_per_request * nq))
                cfg = AnnealConfig(t0=t0, tau=tau, iter=iter, seed=seed * 1_000_003 + windows * 131 + k,
                                   chains=ch, budget_ms=kernel_budget, scale_ladder=scale_ladder,
                                   max_blocks=share[k], device=dev_of[k],
                                   **{"deadline_start": False, **(anneal_kw or {})})
                return _plan_sa(stream, queue[k], max(busy_until[k], t_win), c, max_batch, cfg)
            plans = dict(zip(active, pool.map(plan, active)))
        elif policy == "custom":
            starts = [max(busy_until[k], t_win) for k in active]
            plans = {k: (b, 0, 0.0) for k, b in zip(active, pool.map(planner, [stream] * len(active),
                                                                      [queue[k] for k in active], starts))}
        else:
            plans = {k: _plan_fcfs(stream, queue[k], max_batch) for k in active}
        overhead.append((time.perf_counter() - t0_wall) * 1e3)
        if policy == "sa":  # host share of this window: wall less the longest kernel
            host_now = overhead[-1] - max(p[2] for p in plans.values())
            host_ms = host_now if windows <= 1 else max(0.9 * host_ms + 0.1 * host_now, host_now * 0.5)
        decisions += len(active)
        # execute each plan until the next window boundary (the library's replay)
        for k, (batches, props, _kms) in plans.items():
            proposals += props
            met, lat, started, clock = _execute(stream, batches, c, max(busy_until[k], t_win), dispatch_gap_ms, t_next)
            n_met += met
            total_lat += lat
            busy_until[k] = clock
            if started:
                for i in started:
                    load[k] -= prefill_ms(c, 1, stream.input_len[i]) + decode_total_ms(c, 1, stream.input_len[i],
                                                                                       stream.pred_out[i])
                s_ = set(started)
                queue[k] = [i for i in queue[k] if i not in s_]
                done += len(started)
        t_win = t_next
    if pool:
        pool.shutdown()
    return OnlineResult(policy, done, n_met, total_lat, windows, decisions, proposals, overhead)
