"""Evaluation harness of the scheduler (Python face of csrc/harness.cpp through include/slosched_api.h).

Mirrors the reference's simulator / estimator / CLI-driver interface (P: = /root/reference/proj/):
  run, run_fcfs, SimConfig, MetricsReport   P:include/slosched/simulator.hpp:13-72, core.hpp:139-150
  compare, median, ComparisonRow            P:src/simulator.cpp:148-220
  sweep, perturb                            P:tools/slosched.cpp:335-448
  Estimator (LengthModel, predict)          P:include/slosched/output_estimator.hpp:10-56
plus the engine extensions realize_batches (one replay clock, used by the online driver) and
evaluate_batch (many schedules in one launch of the bit-exact evaluator).
"""
from __future__ import annotations

from ctypes import byref, c_char_p, c_double, c_int32, c_int64, c_uint64
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from ._lib import SloFleet, SloRecord, SloReport, SloRow, SloSimConfig, lib
from .slosched import (AnnealConfig, InstanceState, LatencyCoefficients, RequestMetrics, Schedule, Workload,
                       _check_api, _f64, _i32, _p, _unflatten)


@dataclass
class SimConfig:
    noise_pct: float = 0.0
    dispatch_gap_ms: float = 0.1
    seed: int = 0

    def _c(self):
        return SloSimConfig(self.noise_pct, self.dispatch_gap_ms, self.seed & (2**64 - 1))


@dataclass
class MetricsReport:
    slo_attainment: float
    avg_latency_ms: float
    g: float
    scheduling_overhead_ms: float
    per_request: List[RequestMetrics]
    n_met: int
    total_latency_ms: float


class _Fleet:
    def __init__(self, instances: Sequence[InstanceState]):
        col = lambda f, key: f([getattr(i, key) for i in instances])  # noqa: E731
        self.k = len(instances)
        self._keep = (col(_i32, "id"), col(_f64, "total_mem"), col(_f64, "remaining_mem"), col(_f64, "mem_utility"),
                      col(_f64, "bytes_per_token"), col(_i32, "max_batch_size"))
        iid, tm, rm, mu, sg, mb = self._keep
        self.c = SloFleet(self.k, _p(iid), _p(tm, c_double), _p(rm, c_double), _p(mu, c_double), _p(sg, c_double),
                          _p(mb))


def _records(buf, count) -> List[RequestMetrics]:
    return [RequestMetrics(r.request_id, r.wait_ms, r.exec_ms, r.e2e_ms, r.ttft_ms, r.tpot_ms, bool(r.slo_met),
                           bool(r.extrapolated)) for r in buf[:count]]


def _report(rep: SloReport, records) -> MetricsReport:
    return MetricsReport(rep.slo_attainment, rep.avg_latency_ms, rep.g, rep.scheduling_overhead_ms, records, rep.n_met,
                         rep.total_latency_ms)


def _flat_plans(schedules: Sequence[Schedule]):
    ids, sizes, nb = [], [], []
    for s in schedules:
        nb.append(len(s.batches))
        for b in s.batches:
            sizes.append(len(b))
            ids.extend(b)
    return _i32(ids or [0]), _i32(sizes or [0]), _i32(nb or [0])


def run(schedules: Sequence[Schedule], workload: Workload, instances: Sequence[InstanceState],
        coeffs: LatencyCoefficients, sim: SimConfig = SimConfig(), scheduling_overhead_ms: float = 0.0) -> MetricsReport:
    """Replay per-instance schedules on the synthetic backend (true lengths, noise, dispatch gap)."""
    fl = _Fleet(instances)
    ids, sizes, nb = _flat_plans(schedules)
    n = sum(s.request_count() for s in schedules)
    recs = (SloRecord * max(n, 1))()
    rep = SloReport()
    _check_api(lib().slosched_run(byref(workload._view), _p(coeffs.as_array(), c_double), byref(fl.c), _p(ids),
                                  _p(sizes), _p(nb), byref(sim._c()), scheduling_overhead_ms, recs, byref(rep)))
    return _report(rep, _records(recs, n))


@dataclass
class FcfsResult:
    report: MetricsReport
    schedules: List[Schedule]


def run_fcfs(workload: Workload, instances: Sequence[InstanceState], coeffs: LatencyCoefficients,
             sim: SimConfig = SimConfig()) -> FcfsResult:
    fl = _Fleet(instances)
    n = len(workload.requests)
    oi, osz, inb = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32), np.zeros(
        max(fl.k, 1), dtype=np.int32)
    recs = (SloRecord * max(n, 1))()
    rep = SloReport()
    _check_api(lib().slosched_run_fcfs(byref(workload._view), _p(coeffs.as_array(), c_double), byref(fl.c),
                                       byref(sim._c()), _p(oi), _p(osz), _p(inb), recs, byref(rep)))
    plans, pos, kb = [], 0, 0
    for i in range(fl.k):
        sizes = osz[kb:kb + inb[i]]
        cnt = int(sizes.sum())
        plans.append(_unflatten(oi[pos:pos + cnt], sizes))
        pos += cnt
        kb += int(inb[i])
    return FcfsResult(_report(rep, _records(recs, n)), plans)


def realize_batches(batches: Sequence[Sequence[int]], workload: Workload, coeffs: LatencyCoefficients,
                    clock0: float = 0.0, first_gap: float = 0.0, gap: float = 0.1, until: float = float("inf"),
                    noise_pct: float = 0.0, seed: int = 0, from_arrival: bool = False
                    ) -> Tuple[List[RequestMetrics], float, int]:
    """One instance clock of the replay: (records, clock, batches started)."""
    ids, sizes, _ = _flat_plans([Schedule([list(b) for b in batches])])
    n = sum(len(b) for b in batches)
    recs = (SloRecord * max(n, 1))()
    clock, started = c_double(), c_int32()
    _check_api(lib().slosched_realize_batches(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids),
                                              _p(sizes), len(batches), clock0, first_gap, gap, until, noise_pct,
                                              seed & (2**64 - 1), 1 if from_arrival else 0, recs, byref(clock),
                                              byref(started)))
    k = sum(len(b) for b in batches[:started.value])
    return _records(recs, k), clock.value, started.value


# ------------------------------------------------------------------ estimator
@dataclass
class LengthModel:
    task_class_id: int
    count: int = 0
    mean: float = 0.0
    m2: float = 0.0


def estimator_run(classes, observations: Sequence[Tuple[int, int]], predict_classes: Sequence[int], seed: int):
    """The Estimator over `classes` (TaskClass list, output_prior None / ("gaussian", mean, std) /
    ("range", low, high)): observe (class, length) pairs in order, then predict one length per entry of
    predict_classes with Rng(seed). Returns (predictions, models after the observations)."""
    kinds, pa, pb = [], [], []
    for c in classes:
        pr = c.output_prior
        if pr is None:
            kinds.append(0), pa.append(0.0), pb.append(0.0)
        elif pr[0] == "gaussian":
            kinds.append(1), pa.append(float(pr[1])), pb.append(float(pr[2]))
        else:
            kinds.append(2), pa.append(float(pr[1])), pb.append(float(pr[2]))
    cid, kd, a, b = _i32([c.id for c in classes]), _i32(kinds), _f64(pa), _f64(pb)
    oc = _i32([o[0] for o in observations] or [0])
    ol = _i32([o[1] for o in observations] or [0])
    pc = _i32(list(predict_classes) or [0])
    out = np.zeros(max(len(predict_classes), 1), dtype=np.int32)
    cnt = np.zeros(len(classes), dtype=np.int64)
    mean, m2 = np.zeros(len(classes)), np.zeros(len(classes))
    _check_api(lib().slosched_estimator(len(classes), _p(cid), _p(kd), _p(a, c_double), _p(b, c_double),
                                        len(observations), _p(oc), _p(ol), len(predict_classes), _p(pc),
                                        seed & (2**64 - 1), _p(out), _p(cnt, c_int64), _p(mean, c_double),
                                        _p(m2, c_double)))
    models = [LengthModel(c.id, int(cnt[k]), float(mean[k]), float(m2[k])) for k, c in enumerate(classes)]
    return [int(x) for x in out[:len(predict_classes)]], models


# ------------------------------------------------------------------ drivers
@dataclass
class ComparisonRow:
    policy: str
    seed: int
    n_requests: int
    max_batch: int
    attainment: float
    avg_latency_ms: float
    g_req_per_ms: float
    overhead_ms: float


@dataclass
class ComparisonTable:
    rows: List[ComparisonRow] = field(default_factory=list)
    medians: List[ComparisonRow] = field(default_factory=list)


_POLICY_NAMES = {0: "sa", 1: "exhaustive", 2: "fcfs"}


def _row(r: SloRow) -> ComparisonRow:
    return ComparisonRow(_POLICY_NAMES[r.policy], int(r.seed), r.n_requests, r.max_batch, r.attainment,
                         r.avg_latency_ms, r.g_req_per_ms, r.overhead_ms)


def compare(workload: Workload, instances: Sequence[InstanceState], coeffs: LatencyCoefficients,
            policies: Sequence[str], seeds: Sequence[int], anneal_cfg: AnnealConfig, sim: SimConfig = SimConfig(),
            exhaustive_cap: int = 10) -> ComparisonTable:
    codes = {"sa": 0, "exhaustive": 1, "fcfs": 2}
    pol = _i32([codes[p] for p in policies])
    sd = np.asarray(list(seeds), dtype=np.uint64)
    fl = _Fleet(instances)
    cfg, _keep = anneal_cfg._c()
    rows = (SloRow * max(len(pol) * len(sd), 1))()
    med = (SloRow * max(len(pol), 1))()
    _check_api(lib().slosched_compare(byref(workload._view), _p(coeffs.as_array(), c_double), byref(fl.c), len(pol),
                                      _p(pol), len(sd), _p(sd, c_uint64), byref(cfg), byref(sim._c()), exhaustive_cap,
                                      rows, med))
    return ComparisonTable([_row(r) for r in rows[:len(pol) * len(sd)]], [_row(r) for r in med[:len(pol)]])


def sweep(n_requests: int, seeds: Sequence[int], instances: Sequence[InstanceState], coeffs: LatencyCoefficients,
          base_cfg: AnnealConfig, t0_grid: Sequence[float], iter_grid: Sequence[int], predict: bool = True):
    """G of schedule_all over the (t0, iter) grid for the CLI's synthetic workload of each seed; rows
    (t0, iter, seed, g) in t0-major order."""
    sd = np.asarray(list(seeds), dtype=np.uint64)
    t0s, its = _f64(list(t0_grid)), _i32(list(iter_grid))
    fl = _Fleet(instances)
    cfg, _keep = base_cfg._c()
    g = np.zeros(len(t0s) * len(its) * len(sd))
    _check_api(lib().slosched_sweep(n_requests, 1 if predict else 0, len(sd), _p(sd, c_uint64), byref(fl.c),
                                    _p(coeffs.as_array(), c_double), byref(cfg), len(t0s), _p(t0s, c_double),
                                    len(its), _p(its), _p(g, c_double)))
    rows, k = [], 0
    for t0 in t0s:
        for it in its:
            for s in sd:
                rows.append((float(t0), int(it), int(s), float(g[k])))
                k += 1
    return rows


def perturb(n_requests: int, seeds: Sequence[int], instances: Sequence[InstanceState], truth: LatencyCoefficients,
            base_cfg: AnnealConfig, sim: SimConfig, params: Sequence[str], factors: Sequence[float],
            predict: bool = True):
    """Realized G when the mapper sees perturbed coefficients but the backend runs `truth`; rows
    (param, factor, seed, g, baseline_g, degradation_pct)."""
    sd = np.asarray(list(seeds), dtype=np.uint64)
    fs = _f64(list(factors))
    names = (c_char_p * max(len(params), 1))(*[p.encode() for p in params])
    fl = _Fleet(instances)
    cfg, _keep = base_cfg._c()
    m = len(params) * len(fs) * len(sd)
    g, base, deg = np.zeros(max(m, 1)), np.zeros(max(m, 1)), np.zeros(max(m, 1))
    _check_api(lib().slosched_perturb(n_requests, 1 if predict else 0, len(sd), _p(sd, c_uint64), byref(fl.c),
                                      _p(truth.as_array(), c_double), byref(cfg), byref(sim._c()), len(params), names,
                                      len(fs), _p(fs, c_double), _p(g, c_double), _p(base, c_double),
                                      _p(deg, c_double)))
    rows, k = [], 0
    for p in params:
        for f in fs:
            for s in sd:
                rows.append((p, float(f), int(s), float(g[k]), float(base[k]), float(deg[k])))
                k += 1
    return rows


def evaluate_batch(schedules: Sequence[Schedule], coeffs: LatencyCoefficients, workload: Workload, max_batch: int):
    """(n_met, t, g) arrays of many schedules over the same requests: one launch of the bit-exact
    evaluator (== evaluate() bit for bit)."""
    if not schedules:
        return np.zeros(0, dtype=np.int32), np.zeros(0), np.zeros(0)
    n = schedules[0].request_count()
    ids, sizes, nb = _flat_plans(schedules)
    k = len(schedules)
    nm, t, g = np.zeros(k, dtype=np.int32), np.zeros(k), np.zeros(k)
    _check_api(lib().slosched_evaluate_batch(byref(workload._view), _p(coeffs.as_array(), c_double), k, n, _p(ids),
                                             _p(sizes), _p(nb), max_batch, _p(nm), _p(t, c_double), _p(g, c_double)))
    return nm, t, g


def median(values: Sequence[float]) -> float:
    v = sorted(values)
    if not v:
        return 0.0
    m = len(v) // 2
    return v[m] if len(v) % 2 else 0.5 * (v[m - 1] + v[m])


__all__ = ["SimConfig", "MetricsReport", "FcfsResult", "run", "run_fcfs", "realize_batches", "LengthModel",
           "estimator_run", "ComparisonRow", "ComparisonTable", "compare", "sweep", "perturb", "evaluate_batch",
           "median"]
