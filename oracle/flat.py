"""Flat (structure-of-arrays) workload shared by both checkers.

Field meaning follows P:include/slosched/core.hpp:26-74: requests carry an id,
a task-class id, input length, true and predicted output length (-1 = none)
and an arrival time; classes carry an SLO kind (0 = E2E, 1 = TTFT_TPOT) and
thresholds in ms.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

# built-in profile, P:src/latency_model.cpp:115-117 (= PAPER.md:716-718)
TABLE_COEFFS = (0.1, 5.7, 0.01, 43.67, 0.0002, 0.275, 0.00088, 15.85)


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


@dataclass
class FlatWorkload:
    id: np.ndarray
    cls: np.ndarray
    in_len: np.ndarray
    true_out: np.ndarray
    pred_out: np.ndarray
    arrival: np.ndarray
    class_id: np.ndarray = field(default_factory=lambda: _i32([0, 1]))
    kind: np.ndarray = field(default_factory=lambda: _i32([0, 1]))
    e2e: np.ndarray = field(default_factory=lambda: _f64([30000.0, 0.0]))
    ttft: np.ndarray = field(default_factory=lambda: _f64([0.0, 10000.0]))
    tpot: np.ndarray = field(default_factory=lambda: _f64([0.0, 50.0]))

    def __post_init__(self):
        for k in ("id", "cls", "in_len", "true_out", "pred_out", "class_id", "kind"):
            setattr(self, k, _i32(getattr(self, k)))
        for k in ("arrival", "e2e", "ttft", "tpot"):
            setattr(self, k, _f64(getattr(self, k)))

    @property
    def n(self) -> int:
        return int(self.id.shape[0])

    @property
    def n_classes(self) -> int:
        return int(self.class_id.shape[0])


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def flatten_batches(batches):
    ids = [i for b in batches for i in b]
    sizes = [len(b) for b in batches]
    return _i32(ids), _i32(sizes)


def unflatten(ids, sizes):
    out, pos = [], 0
    for s in sizes:
        out.append([int(x) for x in ids[pos:pos + s]])
        pos += s
    return out
