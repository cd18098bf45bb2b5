"""B200-native SLO-aware simulated-annealing scheduler (arXiv 2504.14966).

The annealing loop runs as hand-written sm_100a CUDA in libslosched_b200.so
(build: ``python -m paper_2504_14966_b200.build``). Importing this package does not
touch the GPU; the first anneal()/Engine() call does, and fails loudly without one.
"""
from .slosched import (  # noqa: F401
    AnnealConfig, AnnealResult, AnnealStats, CapacityError, DataError, EngineError, EvaluatedSchedule,
    ExhaustiveResult, deadline_first_candidate, exhaustive,
    InstanceState, LatencyCoefficients, Request, RequestMetrics, Schedule, ScheduleAllResult, SearchMode, SloKind,
    SloSpec, TaskClass, Workload, anneal, anneal_flat, default_slo_classes, default_synth_classes, evaluate,
    generate_mixed, initial_candidates, latest_start, neighbor_walk, predict_decode_total, predict_exec,
    predict_per_token_decode, predict_prefill, predict_tpot, schedule_all, shortcut_check, table_coefficients,
    validate_workload)

__version__ = "0.1.0"
