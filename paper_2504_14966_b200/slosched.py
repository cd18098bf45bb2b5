"""Python mirror of the reference scheduler interface, backed by libslosched_b200.so.

Same names, argument meaning and error behaviour as the reference's C++ API
(P: = /root/reference/proj/):

* types: SloSpec / TaskClass / Request / LatencyCoefficients / Schedule / Workload /
  EvaluatedSchedule / RequestMetrics (P:include/slosched/core.hpp:26-170)
* predict_* / table_coefficients (P:include/slosched/latency_model.hpp:43-59)
* evaluate (P:include/slosched/objective.hpp:36-38)
* initial_candidates / shortcut_check / anneal (P:include/slosched/priority_mapper.hpp:46-69)
* schedule_all / InstanceState (P:include/slosched/scheduler.hpp:54-59)
* generate_mixed / default_synth_classes (P:include/slosched/workload.hpp:38-52)

Errors: DataError, CapacityError, ValueError (reference std::invalid_argument) and
EngineError (CUDA failures -- the annealing loop has no CPU fallback).
"""
from __future__ import annotations

import ctypes
import enum
from ctypes import byref, c_double, c_int32
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import SloAnnealConfig, SloAnnealStats, SloWorkload, lib


class DataError(RuntimeError):
    pass


class CapacityError(RuntimeError):
    pass


class EngineError(RuntimeError):
    pass


def _raise(rc: int, msg: str):
    if rc == _lib.SLO_ERR_DATA:
        raise DataError(msg)
    if rc == _lib.SLO_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == _lib.SLO_ERR_ARG:
        raise ValueError(msg)
    raise EngineError(msg)


def _check_api(rc: int):
    if rc != _lib.SLO_OK:
        _raise(rc, lib().slosched_last_error().decode())


def _check_engine(rc: int):
    if rc != _lib.SLO_OK:
        _raise(rc, lib().slo_last_error().decode())


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a, t=c_int32):
    return a.ctypes.data_as(ctypes.POINTER(t))


# ------------------------------------------------------------------ domain types
class SloKind(enum.IntEnum):
    E2E = 0
    TTFT_TPOT = 1


@dataclass(frozen=True)
class SloSpec:
    kind: SloKind = SloKind.E2E
    e2e_ms: Optional[float] = None
    ttft_ms: Optional[float] = None
    tpot_ms: Optional[float] = None

    @staticmethod
    def e2e(ms: float) -> "SloSpec":
        return SloSpec(SloKind.E2E, e2e_ms=float(ms))

    @staticmethod
    def ttft_tpot(ttft_ms: float, tpot_ms: float) -> "SloSpec":
        return SloSpec(SloKind.TTFT_TPOT, ttft_ms=float(ttft_ms), tpot_ms=float(tpot_ms))


@dataclass(frozen=True)
class TaskClass:
    id: int
    name: str
    slo: SloSpec
    output_prior: Optional[tuple] = None  # ("gaussian", mean, std) | ("range", lo, hi) | None


@dataclass
class Request:
    id: int
    task_class_id: int
    input_len: int
    true_output_len: int
    predicted_output_len: Optional[int] = None
    arrival_time_ms: float = 0.0


@dataclass(frozen=True)
class LatencyCoefficients:
    alpha_p: float = 0.0
    beta_p: float = 0.0
    gamma_p: float = 0.0
    delta_p: float = 0.0
    alpha_d: float = 0.0
    beta_d: float = 0.0
    gamma_d: float = 0.0
    delta_d: float = 0.0

    def as_array(self) -> np.ndarray:
        return _f64([self.alpha_p, self.beta_p, self.gamma_p, self.delta_p,
                     self.alpha_d, self.beta_d, self.gamma_d, self.delta_d])


def table_coefficients() -> LatencyCoefficients:
    """Built-in profile (P:src/latency_model.cpp:115-117)."""
    return LatencyCoefficients(0.1, 5.7, 0.01, 43.67, 0.0002, 0.275, 0.00088, 15.85)


@dataclass
class Schedule:
    batches: List[List[int]] = field(default_factory=list)

    def request_count(self) -> int:
        return sum(len(b) for b in self.batches)

    def flatten(self) -> List[int]:
        return [i for b in self.batches for i in b]

    def is_partition_of(self, ids: Sequence[int], max_batch: int) -> bool:
        got = self.flatten()
        if any(len(b) == 0 or (max_batch > 0 and len(b) > max_batch) for b in self.batches):
            return False
        return len(got) == len(set(got)) and sorted(got) == sorted(ids)

    def _flat(self):
        return _i32(self.flatten()), _i32([len(b) for b in self.batches])


def _unflatten(ids, sizes) -> Schedule:
    out, pos = [], 0
    for s in sizes:
        out.append([int(x) for x in ids[pos:pos + s]])
        pos += int(s)
    return Schedule(out)


@dataclass
class RequestMetrics:
    request_id: int
    wait_ms: float
    exec_ms: float
    e2e_ms: float
    ttft_ms: float
    tpot_ms: float
    slo_met: bool
    extrapolated: bool


@dataclass
class EvaluatedSchedule:
    schedule: Schedule
    per_request: List[RequestMetrics]
    n: int
    t_ms: float
    g: float


class Workload:
    """Validated workload (P:src/core.cpp:151-170), held as structure-of-arrays for the C ABI."""

    def __init__(self, requests: Sequence[Request], classes: Sequence[TaskClass]):
        self.requests = list(requests)
        self.classes = list(classes)
        self._arrays = dict(
            id=_i32([r.id for r in self.requests]),
            cls=_i32([r.task_class_id for r in self.requests]),
            in_len=_i32([r.input_len for r in self.requests]),
            true_out=_i32([r.true_output_len for r in self.requests]),
            pred_out=_i32([-1 if r.predicted_output_len is None else r.predicted_output_len for r in self.requests]),
            arrival=_f64([r.arrival_time_ms for r in self.requests]),
            class_id=_i32([c.id for c in self.classes]),
            kind=_i32([int(c.slo.kind) for c in self.classes]),
            e2e=_f64([c.slo.e2e_ms or 0.0 for c in self.classes]),
            ttft=_f64([c.slo.ttft_ms or 0.0 for c in self.classes]),
            tpot=_f64([c.slo.tpot_ms or 0.0 for c in self.classes]),
        )
        a = self._arrays
        self._view = SloWorkload(len(self.requests), _p(a["id"]), _p(a["cls"]), _p(a["in_len"]), _p(a["true_out"]),
                                 _p(a["pred_out"]), _p(a["arrival"], c_double), len(self.classes),
                                 _p(a["class_id"]), _p(a["kind"]), _p(a["e2e"], c_double), _p(a["ttft"], c_double),
                                 _p(a["tpot"], c_double))
        self._validate()

    def _validate(self):
        # the C++ validate_workload does the checking; evaluate() on an empty schedule runs it
        n_met, t, g = c_int32(), c_double(), c_double()
        z = np.zeros(1, dtype=np.int32)
        _check_api(lib().slosched_evaluate(byref(self._view), _p(table_coefficients().as_array(), c_double),
                                           _p(z), _p(z), 0, byref(n_met), byref(t), byref(g),
                                           None, None, None, None, None, None, None))

    @property
    def arrays(self):
        return self._arrays

    def ids(self) -> List[int]:
        return [r.id for r in self.requests]

    def find_request(self, rid: int) -> Optional[Request]:
        for r in self.requests:
            if r.id == rid:
                return r
        return None


def validate_workload(requests: Sequence[Request], classes: Sequence[TaskClass]) -> Workload:
    return Workload(requests, classes)


# ------------------------------------------------------------------ latency model
def _predict(c: LatencyCoefficients, b, li, lo):
    out = np.zeros(5)
    _check_api(lib().slosched_predict(_p(c.as_array(), c_double), b, li, lo, _p(out, c_double)))
    return out


def predict_prefill(c, b, input_len):
    return float(_predict(c, b, input_len, 1)[0])


def predict_per_token_decode(c, b, accumulated_len):
    return float(_predict(c, b, accumulated_len, 1)[1])


def predict_decode_total(c, b, input_len, output_len):
    return float(_predict(c, b, input_len, output_len)[2])


def predict_exec(c, b, input_len, output_len):
    return float(_predict(c, b, input_len, output_len)[3])


def predict_tpot(c, b, input_len, output_len):
    if output_len <= 0:
        raise ValueError("predict_tpot: TPOT undefined for zero output")
    return float(_predict(c, b, input_len, output_len)[4])


def latest_start(slo_ms: float, cost_ms: float) -> float:
    """Largest d with fl(d + cost) <= slo: the engine's deadline convention."""
    return float(lib().slosched_latest_start(slo_ms, cost_ms))


# ------------------------------------------------------------------ objective
def evaluate(schedule: Schedule, coeffs: LatencyCoefficients, workload: Workload) -> EvaluatedSchedule:
    ids, sizes = schedule._flat()
    n = len(ids)
    per = {k: np.zeros(max(n, 1)) for k in ("wait", "exec", "e2e", "ttft", "tpot")}
    met, ext = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    n_met, t, g = c_int32(), c_double(), c_double()
    _check_api(lib().slosched_evaluate(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), _p(sizes),
                                       len(sizes), byref(n_met), byref(t), byref(g),
                                       *(_p(per[k], c_double) for k in ("wait", "exec", "e2e", "ttft", "tpot")),
                                       _p(met), _p(ext)))
    metrics = [RequestMetrics(int(ids[i]), float(per["wait"][i]), float(per["exec"][i]), float(per["e2e"][i]),
                              float(per["ttft"][i]), float(per["tpot"][i]), bool(met[i]), bool(ext[i]))
               for i in range(n)]
    return EvaluatedSchedule(Schedule([list(b) for b in schedule.batches]), metrics, n_met.value, t.value, g.value)


# ------------------------------------------------------------------ priority mapper
class SearchMode(enum.IntEnum):
    CHAINS = 0  # thousands of independent Philox chains on the GPU, best-of-chains
    REPLAY = 1  # one chain on the reference's xoshiro stream: bit-identical to the reference


@dataclass
class AnnealConfig:
    t0: float = 500.0
    t_thres: float = 20.0
    iter: int = 100
    tau: float = 0.95
    seed: int = 0
    objective_scale: Optional[float] = None
    # engine extensions (include/slosched_b200.hpp EngineOptions)
    mode: SearchMode = SearchMode.CHAINS
    chains: int = 4096
    budget_ms: float = 0.0
    scale_ladder: Sequence[float] = ()
    device: int = -1
    chain_begin: int = 0
    chain_end: int = -1
    sequential_instances: bool = False  # schedule_all: anneal instances one after another
    max_blocks: int = 0                 # > 0: cap the chain grid (concurrent callers share the GPU)
    deadline_start: bool = True         # chains: the deadline-first candidate joins the two starts
    # multi-GPU: devices of this process sharing the chains (slo_group), or this rank's engine
    # context with an NCCL communicator (distributed.RankComm.handle) in a one-process-per-GPU job
    devices: Sequence[int] = ()
    comm_ctx: Optional[int] = None

    def _c(self):
        ladder = _f64(list(self.scale_ladder)) if len(self.scale_ladder) else None
        devs = _i32(list(self.devices)) if len(self.devices) else None
        cfg = SloAnnealConfig(self.t0, self.t_thres, self.iter, self.tau, self.seed & (2**64 - 1),
                              0 if self.objective_scale is None else 1,
                              0.0 if self.objective_scale is None else self.objective_scale, int(self.mode),
                              self.chains, self.budget_ms, 0 if ladder is None else len(ladder),
                              None if ladder is None else _p(ladder, c_double), self.device, self.chain_begin,
                              self.chain_end, 1 if self.sequential_instances else 0, self.max_blocks,
                              0 if self.deadline_start else 1, 0 if devs is None else len(devs),
                              None if devs is None else _p(devs), self.comm_ctx)
        return cfg, (ladder, devs)


@dataclass
class AnnealStats:
    proposals: int = 0
    accepted: int = 0
    shortcut: bool = False
    g_sorted_start: float = 0.0
    g_input_start: float = 0.0
    objective_scale_used: float = 1.0
    chains_run: int = 0
    levels_run: int = 0
    best_chain: int = -1
    engine_g: float = 0.0
    engine_t: float = 0.0
    kernel_ms: float = 0.0
    g_deadline_start: float = 0.0
    exchange_ms: float = 0.0  # multi-GPU: chain kernel end -> job-wide winner (device time)
    devices: int = 1          # devices whose chains the result covers

    @staticmethod
    def _from(s: SloAnnealStats) -> "AnnealStats":
        return AnnealStats(int(s.proposals), int(s.accepted), bool(s.shortcut), s.g_sorted_start, s.g_input_start,
                           s.objective_scale_used, s.chains_run, s.levels_run, s.best_chain, s.engine_g, s.engine_t,
                           s.kernel_ms, s.g_deadline_start, s.exchange_ms, s.devices)


@dataclass
class AnnealResult:
    best: EvaluatedSchedule
    stats: AnnealStats


def initial_candidates(workload: Workload, request_ids, coeffs: LatencyCoefficients, max_batch: int):
    ids = _i32(request_ids)
    n = len(ids)
    si, ss, ii, isz = (np.zeros(max(n, 1), dtype=np.int32) for _ in range(4))
    snb, inb = c_int32(), c_int32()
    _check_api(lib().slosched_initial_candidates(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), n,
                                                 max_batch, _p(si), _p(ss), byref(snb), _p(ii), _p(isz), byref(inb)))
    return _unflatten(si, ss[:snb.value]), _unflatten(ii, isz[:inb.value])


def deadline_first_candidate(workload: Workload, request_ids, coeffs: LatencyCoefficients, max_batch: int) -> Schedule:
    """The chains' third start (engine extension, include/slosched_b200.hpp): Moore-Hodgson with
    batching over the latest-start tables."""
    ids = _i32(request_ids)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb = c_int32()
    _check_api(lib().slosched_deadline_first_candidate(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids),
                                                       n, max_batch, _p(oi), _p(osz), byref(nb)))
    return _unflatten(oi, osz[:nb.value])


def shortcut_check(sorted_schedule: Schedule, coeffs, workload) -> Optional[EvaluatedSchedule]:
    ev = evaluate(sorted_schedule, coeffs, workload)
    return ev if ev.n == len(ev.per_request) else None


def neighbor_walk(schedule: Schedule, seed: int, steps: int, max_batch: int) -> Schedule:
    """`steps` chained neighbor() calls from one Rng(seed) (P:src/priority_mapper.cpp:322-338)."""
    ids, sizes = schedule._flat()
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb = c_int32()
    _check_api(lib().slosched_neighbor_walk(_p(ids), _p(sizes), len(sizes), seed, steps, max_batch, _p(oi), _p(osz),
                                            byref(nb)))
    return _unflatten(oi, osz[:nb.value])


def _evaluated_from_flat(workload, coeffs, oi, osz, nb):
    return evaluate(_unflatten(oi, osz[:nb]), coeffs, workload)


def anneal(workload: Workload, request_ids, coeffs: LatencyCoefficients, config: AnnealConfig,
           max_batch: int) -> AnnealResult:
    """SA priority mapping (P:src/priority_mapper.cpp:340-411) with the loop on the B200."""
    ids = _i32(request_ids)
    n = len(ids)
    cfg, _keep = config._c()
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g = c_int32(), c_int32(), c_double(), c_double()
    st = SloAnnealStats()
    _check_api(lib().slosched_anneal(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), n, byref(cfg),
                                     max_batch, _p(oi), _p(osz), byref(nb), byref(n_met), byref(t), byref(g),
                                     byref(st)))
    best = _evaluated_from_flat(workload, coeffs, oi, osz, nb.value)
    assert best.n == n_met.value and best.g == g.value
    return AnnealResult(best, AnnealStats._from(st))


def anneal_flat(workload: Workload, request_ids, coeffs: LatencyCoefficients, config: AnnealConfig, max_batch: int):
    """anneal() returning the raw C-ABI outputs (priority sequence, batch sizes, n, t, g, stats)
    without building per-request Python objects -- the call the benchmark times end to end."""
    ids = _i32(request_ids)
    n = len(ids)
    cfg, _keep = config._c()
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g = c_int32(), c_int32(), c_double(), c_double()
    st = SloAnnealStats()
    _check_api(lib().slosched_anneal(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), n, byref(cfg),
                                     max_batch, _p(oi), _p(osz), byref(nb), byref(n_met), byref(t), byref(g),
                                     byref(st)))
    return oi[:n], osz[:nb.value], n_met.value, t.value, g.value, AnnealStats._from(st)


@dataclass
class ExhaustiveResult:
    best: EvaluatedSchedule
    schedules_evaluated: int


def exhaustive(workload: Workload, request_ids, coeffs: LatencyCoefficients, max_batch: int,
               n_cap: int = 10) -> ExhaustiveResult:
    """Small-n oracle on the GPU (P:src/priority_mapper.cpp:440-517): every permutation x every
    batch-size composition, the reference's tie-breaking; CapacityError beyond n_cap."""
    ids = _i32(request_ids)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g, ev = c_int32(), c_int32(), c_double(), c_double(), ctypes.c_uint64()
    _check_api(lib().slosched_exhaustive(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), n,
                                         max_batch, n_cap, _p(oi), _p(osz), byref(nb), byref(n_met), byref(t),
                                         byref(g), byref(ev)))
    return ExhaustiveResult(_evaluated_from_flat(workload, coeffs, oi, osz, nb.value), int(ev.value))


# ------------------------------------------------------------------ scheduler
@dataclass
class InstanceState:
    id: int = 0
    total_mem: int = 0
    remaining_mem: int = 0
    mem_utility: float = 0.9
    bytes_per_token: float = 1.0
    max_batch_size: int = 1


@dataclass
class ScheduleAllResult:
    per_instance: List[EvaluatedSchedule]
    epochs: int
    overhead_ms: float


def schedule_all(workload: Workload, instances: Sequence[InstanceState], coeffs: LatencyCoefficients,
                 config: AnnealConfig) -> ScheduleAllResult:
    """Algorithm 2 (P:src/scheduler.cpp:92-129): assign, then anneal per instance on the GPU."""
    k = len(instances)
    col = lambda f, key: f([getattr(i, key) for i in instances])  # noqa: E731
    iid, tm, rm = col(_i32, "id"), col(_f64, "total_mem"), col(_f64, "remaining_mem")
    mu, sg, mb = col(_f64, "mem_utility"), col(_f64, "bytes_per_token"), col(_i32, "max_batch_size")
    cfg, _keep = config._c()
    n = len(workload.requests)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    inb, icnt, in_ = (np.zeros(max(k, 1), dtype=np.int32) for _ in range(3))
    it, ig = np.zeros(max(k, 1)), np.zeros(max(k, 1))
    epochs, ovh = c_int32(), c_double()
    _check_api(lib().slosched_schedule_all(byref(workload._view), _p(coeffs.as_array(), c_double), k, _p(iid),
                                           _p(tm, c_double), _p(rm, c_double), _p(mu, c_double), _p(sg, c_double),
                                           _p(mb), byref(cfg), _p(oi), _p(osz), _p(inb), _p(icnt), _p(in_),
                                           _p(it, c_double), _p(ig, c_double), byref(epochs), byref(ovh)))
    per, pos, kb = [], 0, 0
    for i in range(k):
        s = _unflatten(oi[pos:pos + icnt[i]], osz[kb:kb + inb[i]])
        per.append(evaluate(s, coeffs, workload))
        pos += int(icnt[i])
        kb += int(inb[i])
    return ScheduleAllResult(per, epochs.value, ovh.value)


# ------------------------------------------------------------------ synthetic inputs
def default_slo_classes():
    return (TaskClass(0, "code", SloSpec.e2e(30000.0)), TaskClass(1, "chat", SloSpec.ttft_tpot(10000.0, 50.0)))


def default_synth_classes():
    code, chat = default_slo_classes()
    return (TaskClass(0, "code", code.slo, ("gaussian", 900.0, 300.0)),
            TaskClass(1, "chat", chat.slo, ("gaussian", 250.0, 150.0)))


def generate_mixed(n: int, seed: int, predict: bool = True) -> Workload:
    """generate_mixed(n, seed) with default classes (P:src/workload.cpp:158-183); predict=True fills
    predicted lengths from the class priors with Rng(derive(seed, 0x9e37)) as the CLI does
    (P:tools/slosched.cpp:131-142), predict=False copies the true lengths."""
    a = {k: np.zeros(max(n, 1), dtype=np.int32) for k in ("id", "cls", "in_len", "true_out", "pred_out")}
    arr = np.zeros(max(n, 1))
    _check_api(lib().slosched_generate_mixed(n, seed, 1 if predict else 0,
                                             *(_p(a[k]) for k in ("id", "cls", "in_len", "true_out", "pred_out")),
                                             _p(arr, c_double)))
    reqs = [Request(int(a["id"][i]), int(a["cls"][i]), int(a["in_len"][i]), int(a["true_out"][i]),
                    int(a["pred_out"][i]), float(arr[i])) for i in range(n)]
    return Workload(reqs, default_synth_classes())
