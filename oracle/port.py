"""ctypes face of slo_oracle.c, the plain-C restatement -- TEST INFRASTRUCTURE."""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, Structure, c_double, c_int, c_uint64

import numpy as np

from .flat import FlatWorkload, _f64, _i32, flatten_batches, ptr, unflatten

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libslo_oracle.so")
_lib = None


class _CWorkload(Structure):
    _fields_ = [("n", c_int), ("id", POINTER(c_int)), ("cls", POINTER(c_int)), ("in_len", POINTER(c_int)),
                ("true_out", POINTER(c_int)), ("pred_out", POINTER(c_int)), ("arrival", POINTER(c_double)),
                ("n_classes", c_int), ("class_id", POINTER(c_int)), ("kind", POINTER(c_int)),
                ("e2e", POINTER(c_double)), ("ttft", POINTER(c_double)), ("tpot", POINTER(c_double))]


class _rng(Structure):
    _fields_ = [("s", c_uint64 * 4)]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        for name in ("or_predict_prefill", "or_predict_decode_total", "or_predict_exec", "or_predict_tpot"):
            getattr(_lib, name).restype = c_double
        _lib.or_rng_next.restype = c_uint64
        _lib.or_rng_index.restype = c_uint64
        _lib.or_rng_index.argtypes = [POINTER(_rng), c_uint64]
        _lib.or_rng_uniform.restype = c_double
        _lib.or_rng_normal.restype = c_double
        _lib.or_rng_derive.restype = c_uint64
        _lib.or_rng_derive.argtypes = [c_uint64, c_uint64]
        _lib.or_rng_seed.argtypes = [POINTER(_rng), c_uint64]
    return _lib


def _cw(w: FlatWorkload):
    cw = _CWorkload(w.n, ptr(w.id, c_int), ptr(w.cls, c_int), ptr(w.in_len, c_int), ptr(w.true_out, c_int),
                    ptr(w.pred_out, c_int), ptr(w.arrival, c_double), w.n_classes, ptr(w.class_id, c_int),
                    ptr(w.kind, c_int), ptr(w.e2e, c_double), ptr(w.ttft, c_double), ptr(w.tpot, c_double))
    cw._keep = w  # keep arrays alive
    return cw


class Rng:
    """xoshiro256++ (P:include/slosched/rng.hpp:14-100) via the C port."""

    def __init__(self, seed):
        self._s = _rng()
        lib().or_rng_seed(ctypes.byref(self._s), c_uint64(seed))

    def next_u64(self):
        return int(lib().or_rng_next(ctypes.byref(self._s)))

    def uniform_index(self, n):
        return int(lib().or_rng_index(ctypes.byref(self._s), c_uint64(n)))

    def uniform(self):
        return float(lib().or_rng_uniform(ctypes.byref(self._s)))

    def normal(self):
        return float(lib().or_rng_normal(ctypes.byref(self._s)))


def derive(seed, stream):
    return int(lib().or_rng_derive(seed, stream))


def predict(coeffs, b, li, lo):
    c = _f64(coeffs)
    L = lib()
    return np.array([L.or_predict_prefill(ptr(c, c_double), b, li), 0.0,
                     L.or_predict_decode_total(ptr(c, c_double), b, li, lo),
                     L.or_predict_exec(ptr(c, c_double), b, li, lo),
                     L.or_predict_tpot(ptr(c, c_double), b, li, lo) if lo > 0 else 0.0])


def generate_mixed(n, seed, predict_mode=1) -> FlatWorkload:
    a = {k: np.zeros(n, dtype=np.int32) for k in ("id", "cls", "in_len", "true_out", "pred_out")}
    arr = np.zeros(n, dtype=np.float64)
    lib().or_generate_mixed(c_int(n), c_uint64(seed), c_int(predict_mode),
                            *(ptr(a[k], c_int) for k in ("id", "cls", "in_len", "true_out", "pred_out")),
                            ptr(arr, c_double))
    return FlatWorkload(arrival=arr, **a)


def evaluate(w: FlatWorkload, coeffs, batches):
    c = _f64(coeffs)
    ids, sizes = flatten_batches(batches)
    n = len(ids)
    n_met, t, g = c_int(), c_double(), c_double()
    per = {k: np.zeros(max(n, 1), dtype=np.float64) for k in ("wait", "exec", "e2e", "ttft", "tpot")}
    met = np.zeros(max(n, 1), dtype=np.int32)
    cw = _cw(w)
    rc = lib().or_evaluate(ctypes.byref(cw), ptr(c, c_double), ptr(ids, c_int), ptr(sizes, c_int),
                           c_int(len(sizes)), ctypes.byref(n_met), ctypes.byref(t), ctypes.byref(g),
                           *(ptr(per[k], c_double) for k in ("wait", "exec", "e2e", "ttft", "tpot")),
                           ptr(met, c_int))
    if rc != 0:
        raise ValueError("oracle evaluate: unknown request id or missing prediction")
    per = {k: v[:n] for k, v in per.items()}
    per["met"] = met[:n]
    return n_met.value, t.value, g.value, per


def score_batch(w: FlatWorkload, coeffs, ids, max_batch, perms, sizes_list):
    """CostModel::score over dense-index candidates; perms [count, n], sizes_list list of lists."""
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    perms = _i32(perms).reshape(-1, n)
    count = perms.shape[0]
    sz = np.zeros((count, max(n, 1)), dtype=np.int32)
    nb = np.zeros(count, dtype=np.int32)
    for q, s in enumerate(sizes_list):
        sz[q, :len(s)] = s
        nb[q] = len(s)
    n_met = np.zeros(count, dtype=np.int32)
    t, g = np.zeros(count), np.zeros(count)
    cw = _cw(w)
    rc = lib().or_score_batch(ctypes.byref(cw), ptr(c, c_double), ptr(ids, c_int), c_int(n), c_int(max_batch),
                              c_int(count), ptr(perms, c_int), ptr(sz, c_int), ptr(nb, c_int), ptr(n_met, c_int),
                              ptr(t, c_double), ptr(g, c_double))
    if rc != 0:
        raise ValueError("oracle score_batch: unknown request id or missing prediction")
    return n_met, t, g


def initial_candidates(w: FlatWorkload, coeffs, ids, max_batch):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    si, ss, ii, isz = (np.zeros(max(n, 1), dtype=np.int32) for _ in range(4))
    snb, inb = c_int(), c_int()
    cw = _cw(w)
    rc = lib().or_initial_candidates(ctypes.byref(cw), ptr(c, c_double), ptr(ids, c_int), c_int(n),
                                     c_int(max_batch), ptr(si, c_int), ptr(ss, c_int), ctypes.byref(snb),
                                     ptr(ii, c_int), ptr(isz, c_int), ctypes.byref(inb))
    if rc != 0:
        raise ValueError("oracle initial_candidates: unknown request id or missing prediction")
    return unflatten(si, ss[:snb.value]), unflatten(ii, isz[:inb.value])


def anneal(w: FlatWorkload, coeffs, ids, max_batch, seed=0, t0=500.0, t_thres=20.0, iter=100, tau=0.95,
           objective_scale=None):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    cf = _f64([t0, t_thres, iter, tau, 0.0 if objective_scale is None else 1.0,
               0.0 if objective_scale is None else objective_scale])
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g = c_int(), c_int(), c_double(), c_double()
    stats = np.zeros(6)
    cw = _cw(w)
    rc = lib().or_anneal(ctypes.byref(cw), ptr(c, c_double), ptr(ids, c_int), c_int(n), ptr(cf, c_double),
                         c_uint64(seed), c_int(max_batch), ptr(oi, c_int), ptr(osz, c_int), ctypes.byref(nb),
                         ctypes.byref(n_met), ctypes.byref(t), ctypes.byref(g), ptr(stats, c_double))
    if rc == -2:
        raise ValueError("oracle anneal: invalid AnnealConfig")
    if rc != 0:
        raise ValueError("oracle anneal: unknown request id or missing prediction")
    return dict(batches=unflatten(oi, osz[:nb.value]), n=n_met.value, t=t.value, g=g.value,
                proposals=int(stats[0]), accepted=int(stats[1]), shortcut=bool(stats[2]),
                g_sorted_start=stats[3], g_input_start=stats[4], objective_scale_used=stats[5])
