"""ctypes face of oracle/_ref/libslosched_refshim.so -- TEST INFRASTRUCTURE.

The unmodified reference compiled together with integration/reference_anneal_gpu.cpp, the
binding a maintainer would add so the reference's own anneal() runs on the B200 engine.
Tests compare it with the reference's CPU anneal() in the same process image.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_ulonglong

import numpy as np

from .flat import FlatWorkload, _f64, _i32, ptr, unflatten
from .ref import _cfg, _wargs

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libslosched_refshim.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def anneal_gpu(w: FlatWorkload, coeffs, ids, max_batch, seed=0, mode=1, chains=1, **cfg):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g = c_int(), c_int(), c_double(), c_double()
    stats = np.zeros(2)
    cf = _cfg(**cfg)
    rc = lib().refshim_anneal_gpu(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), c_int(n), ptr(cf, c_double),
                                  c_ulonglong(seed), c_int(max_batch), c_int(mode), c_int(chains), ptr(oi, c_int),
                                  ptr(osz, c_int), ctypes.byref(nb), ctypes.byref(n_met), ctypes.byref(t),
                                  ctypes.byref(g), ptr(stats, c_double))
    if rc != 0:
        raise RuntimeError(f"refshim_anneal_gpu failed with code {rc}")
    return dict(batches=unflatten(oi, osz[:nb.value]), n=n_met.value, t=t.value, g=g.value,
                proposals=int(stats[0]), accepted=int(stats[1]))
