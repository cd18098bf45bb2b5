"""ctypes binding of libslosched_b200.so (include/slosched_gpu.h + include/slosched_api.h).

Loading fails loudly: there is no CPU fallback for the scheduler's hot path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_double, c_float, c_int32, c_int64, c_uint32, c_uint64, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLOSCHED_LIB") or os.path.join(PKG, "libslosched_b200.so")  # override: A/B runs

# slo_status codes (include/slosched_gpu.h)
SLO_OK, SLO_ERR_DATA, SLO_ERR_CAPACITY, SLO_ERR_CUDA, SLO_ERR_COMM, SLO_ERR_STATE, SLO_ERR_ARG = range(7)
SLO_MAX_N, SLO_MAX_MB = 4096, 16
SLO_COMM_ID_BYTES = 128
SLO_RNG_PHILOX, SLO_RNG_XOSHIRO_REPLAY = 0, 1


class SloWorkload(Structure):
    _fields_ = [("n", c_int32), ("id", POINTER(c_int32)), ("cls", POINTER(c_int32)), ("in_len", POINTER(c_int32)),
                ("true_out", POINTER(c_int32)), ("pred_out", POINTER(c_int32)), ("arrival", POINTER(c_double)),
                ("n_classes", c_int32), ("class_id", POINTER(c_int32)), ("kind", POINTER(c_int32)),
                ("e2e", POINTER(c_double)), ("ttft", POINTER(c_double)), ("tpot", POINTER(c_double))]


class SloAnnealConfig(Structure):
    _fields_ = [("t0", c_double), ("t_thres", c_double), ("iter", c_int32), ("tau", c_double), ("seed", c_uint64),
                ("has_objective_scale", c_int32), ("objective_scale", c_double), ("mode", c_int32),
                ("chains", c_int32), ("budget_ms", c_double), ("n_scale_ladder", c_int32),
                ("scale_ladder", POINTER(c_double)), ("device", c_int32), ("chain_begin", c_int32),
                ("chain_end", c_int32), ("sequential_instances", c_int32), ("max_blocks", c_int32),
                ("start_policy", c_int32), ("n_devices", c_int32), ("devices", POINTER(c_int32)),
                ("comm_ctx", c_void_p)]


class SloAnnealStats(Structure):
    _fields_ = [("proposals", c_uint64), ("accepted", c_uint64), ("shortcut", c_int32),
                ("g_sorted_start", c_double), ("g_input_start", c_double), ("objective_scale_used", c_double),
                ("chains_run", c_int32), ("levels_run", c_int32), ("best_chain", c_int32),
                ("engine_g", c_double), ("engine_t", c_double), ("kernel_ms", c_double),
                ("g_deadline_start", c_double), ("exchange_ms", c_double), ("devices", c_int32)]


class SloChainParams(Structure):
    _fields_ = [("t0", c_double), ("t_thres", c_double), ("iter", c_int32), ("tau", c_double), ("seed", c_uint64),
                ("objective_scale", c_double), ("rng_mode", c_int32), ("chains", c_int32),
                ("chain_begin", c_int32), ("chain_end", c_int32), ("budget_ns", c_int64),
                ("n_scale_mult", c_int32), ("scale_mult", POINTER(c_double)), ("max_blocks", c_int32)]


class SloChainResult(Structure):
    _fields_ = [("g", c_double), ("t", c_double), ("n_met", c_int32), ("chain", c_int32),
                ("proposals", c_uint64), ("accepted", c_uint64), ("chains_run", c_int32),
                ("levels_run", c_int32), ("kernel_ms", c_float), ("positions_pass1", c_uint64),
                ("positions_pass2", c_uint64), ("exact_walks", c_uint64), ("exchange_ms", c_float),
                ("nranks", c_int32), ("local_proposals", c_uint64), ("local_positions_pass1", c_uint64),
                ("local_positions_pass2", c_uint64)]


class SloFleet(Structure):
    _fields_ = [("n", c_int32), ("id", POINTER(c_int32)), ("total_mem", POINTER(c_double)),
                ("remaining_mem", POINTER(c_double)), ("mu", POINTER(c_double)), ("sigma", POINTER(c_double)),
                ("max_batch", POINTER(c_int32))]


class SloSimConfig(Structure):
    _fields_ = [("noise_pct", c_double), ("dispatch_gap_ms", c_double), ("seed", c_uint64)]


class SloRecord(Structure):
    _fields_ = [("request_id", c_int32), ("wait_ms", c_double), ("exec_ms", c_double), ("e2e_ms", c_double),
                ("ttft_ms", c_double), ("tpot_ms", c_double), ("slo_met", c_int32), ("extrapolated", c_int32)]


class SloReport(Structure):
    _fields_ = [("slo_attainment", c_double), ("avg_latency_ms", c_double), ("g", c_double),
                ("scheduling_overhead_ms", c_double), ("n_met", c_int32), ("total_latency_ms", c_double)]


class SloRow(Structure):
    _fields_ = [("policy", c_int32), ("seed", c_uint64), ("n_requests", c_int32), ("max_batch", c_int32),
                ("attainment", c_double), ("avg_latency_ms", c_double), ("g_req_per_ms", c_double),
                ("overhead_ms", c_double)]


class SloOnlineConfig(Structure):
    _fields_ = [("policy", c_int32), ("n_instances", c_int32), ("window_ms", c_double), ("max_batch", c_int32),
                ("budget_ms", c_double), ("chains", c_int32), ("chains_per_request", c_int32),
                ("chains_min", c_int32), ("seed", c_uint64), ("dispatch_gap_ms", c_double),
                ("n_devices", c_int32), ("devices", POINTER(c_int32)), ("n_scale_ladder", c_int32),
                ("scale_ladder", POINTER(c_double)), ("t0", c_double), ("tau", c_double), ("iter", c_int32),
                ("deadline_start", c_int32), ("max_windows", c_int32)]


class SloOnlineResult(Structure):
    _fields_ = [("n", c_int32), ("n_met", c_int32), ("total_latency_ms", c_double), ("windows", c_int32),
                ("decisions", c_int32), ("proposals", c_uint64)]


_I = POINTER(c_int32)
_D = POINTER(c_double)

# (name, restype, argtypes)
_SIGNATURES = [
    ("slo_last_error", c_char_p, []),
    ("slo_version", c_char_p, []),
    ("slo_ctx_create", c_int32, [c_int32, POINTER(c_void_p)]),
    ("slo_ctx_destroy", None, [c_void_p]),
    ("slo_ctx_stream", c_void_p, [c_void_p]),
    ("slo_ctx_sync", c_int32, [c_void_p]),
    ("slo_ctx_sm_count", c_int32, [c_void_p]),
    ("slo_problem_set", c_int32, [c_void_p, c_int32, c_int32, _D, _D]),
    ("slo_problem_tick_ms", c_double, [c_void_p]),
    ("slo_evaluate_batch", c_int32, [c_void_p, c_int32, POINTER(ctypes.c_uint16), POINTER(c_uint32), _I, _D, _D]),
    ("slo_evaluate_batch_tick", c_int32, [c_void_p, c_int32, POINTER(ctypes.c_uint16), POINTER(c_uint32), _I, _D, _D,
                                          POINTER(c_uint64)]),
    ("slo_anneal_chains", c_int32, [c_void_p, POINTER(SloChainParams), _I, _I, c_int32, _I, _I, _I,
                                    POINTER(SloChainResult)]),
    ("slo_chains_prepare", c_int32, [c_void_p, POINTER(SloChainParams), _I, _I, c_int32]),
    ("slo_chains_launch", c_int32, [c_void_p]),
    ("slo_chains_fetch", c_int32, [c_void_p, _I, _I, _I, POINTER(SloChainResult)]),
    ("slo_probe_smem_bandwidth", c_int32, [c_void_p, POINTER(c_double)]),
    ("slo_comm_unique_id", c_int32, [POINTER(ctypes.c_uint8)]),
    ("slo_ctx_comm_init", c_int32, [c_void_p, c_int32, c_int32, POINTER(ctypes.c_uint8)]),
    ("slo_ctx_comm_info", c_int32, [c_void_p, _I, _I]),
    ("slo_comm_check", c_int32, [c_void_p]),
    ("slo_ctx_exchange_empty", c_int32, [c_void_p, c_int32]),
    ("slo_group_create", c_int32, [c_int32, _I, POINTER(c_void_p)]),
    ("slo_group_destroy", None, [c_void_p]),
    ("slo_group_size", c_int32, [c_void_p]),
    ("slo_group_ctx", c_void_p, [c_void_p, c_int32]),
    ("slo_group_transport", c_char_p, [c_void_p]),
    ("slo_group_problem_set", c_int32, [c_void_p, c_int32, c_int32, _D, _D]),
    ("slo_group_anneal_chains", c_int32, [c_void_p, POINTER(SloChainParams), _I, _I, c_int32, _I, _I, _I,
                                          POINTER(SloChainResult)]),
    ("slo_philox4x32_10", None, [POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint32)]),
    ("slosched_last_error", c_char_p, []),
    ("slosched_predict", c_int32, [_D, c_int32, c_int32, c_int32, _D]),
    ("slosched_latest_start", c_double, [c_double, c_double]),
    ("slosched_generate_mixed", c_int32, [c_int32, c_uint64, c_int32, _I, _I, _I, _I, _I, _D]),
    ("slosched_evaluate", c_int32, [POINTER(SloWorkload), _D, _I, _I, c_int32, _I, _D, _D, _D, _D, _D, _D, _D, _I,
                                    _I]),
    ("slosched_initial_candidates", c_int32, [POINTER(SloWorkload), _D, _I, c_int32, c_int32, _I, _I, _I, _I, _I,
                                              _I]),
    ("slosched_deadline_first_candidate", c_int32, [POINTER(SloWorkload), _D, _I, c_int32, c_int32, _I, _I, _I]),
    ("slosched_neighbor_walk", c_int32, [_I, _I, c_int32, c_uint64, c_int32, c_int32, _I, _I, _I]),
    ("slosched_anneal", c_int32, [POINTER(SloWorkload), _D, _I, c_int32, POINTER(SloAnnealConfig), c_int32, _I, _I,
                                  _I, _I, _D, _D, POINTER(SloAnnealStats)]),
    ("slosched_schedule_all", c_int32, [POINTER(SloWorkload), _D, c_int32, _I, _D, _D, _D, _D, _I,
                                        POINTER(SloAnnealConfig), _I, _I, _I, _I, _I, _D, _D, _I, _D]),
    ("slosched_build_tables", c_int32, [POINTER(SloWorkload), _D, _I, c_int32, c_int32, _D, _D]),
    ("slosched_exhaustive", c_int32, [POINTER(SloWorkload), _D, _I, c_int32, c_int32, c_int32, _I, _I, _I, _I, _D,
                                      _D, POINTER(c_uint64)]),
    ("slo_exhaustive", c_int32, [c_void_p, c_int32, _I, _I, _I, _D, _D, POINTER(c_uint64)]),
    ("slosched_run", c_int32, [POINTER(SloWorkload), _D, POINTER(SloFleet), _I, _I, _I, POINTER(SloSimConfig),
                               c_double, POINTER(SloRecord), POINTER(SloReport)]),
    ("slosched_run_fcfs", c_int32, [POINTER(SloWorkload), _D, POINTER(SloFleet), POINTER(SloSimConfig), _I, _I, _I,
                                    POINTER(SloRecord), POINTER(SloReport)]),
    ("slosched_realize_batches", c_int32, [POINTER(SloWorkload), _D, _I, _I, c_int32, c_double, c_double, c_double,
                                           c_double, c_double, c_uint64, c_int32, POINTER(SloRecord), _D, _I]),
    ("slosched_estimator", c_int32, [c_int32, _I, _I, _D, _D, c_int32, _I, _I, c_int32, _I, c_uint64, _I,
                                     POINTER(c_int64), _D, _D]),
    ("slosched_compare", c_int32, [POINTER(SloWorkload), _D, POINTER(SloFleet), c_int32, _I, c_int32,
                                   POINTER(c_uint64), POINTER(SloAnnealConfig), POINTER(SloSimConfig), c_int32,
                                   POINTER(SloRow), POINTER(SloRow)]),
    ("slosched_sweep", c_int32, [c_int32, c_int32, c_int32, POINTER(c_uint64), POINTER(SloFleet), _D,
                                 POINTER(SloAnnealConfig), c_int32, _D, c_int32, _I, _D]),
    ("slosched_perturb", c_int32, [c_int32, c_int32, c_int32, POINTER(c_uint64), POINTER(SloFleet), _D,
                                   POINTER(SloAnnealConfig), POINTER(SloSimConfig), c_int32, POINTER(c_char_p),
                                   c_int32, _D, _D, _D, _D]),
    ("slosched_run_online", c_int32, [c_int32, _D, _I, _I, _I, _I, _D, POINTER(SloOnlineConfig),
                                      POINTER(SloOnlineResult), _D, c_int32]),
    ("slosched_evaluate_batch", c_int32, [POINTER(SloWorkload), _D, c_int32, c_int32, _I, _I, _I, c_int32, _I, _D,
                                          _D]),
]

EXPORTED = [name for name, _, _ in _SIGNATURES]

_lib = None


def lib():
    """The loaded library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2504_14966_b200.build` "
                              "(the scheduler has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGNATURES:
            if os.environ.get("SLOSCHED_LIB") and not hasattr(L, name):
                continue  # an older variant library (A/B timing runs) may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
