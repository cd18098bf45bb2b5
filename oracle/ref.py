"""ctypes face of the unmodified reference library (oracle/_ref) -- TEST INFRASTRUCTURE.

See oracle/ref_glue.cpp for the reference entry point behind each call.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_uint64

import numpy as np

from .flat import FlatWorkload, _f64, _i32, flatten_batches, ptr, unflatten

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libslosched_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle ref)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = ctypes.c_char_p
        _lib.ref_rng_derive.restype = c_uint64
        _lib.ref_rng_derive.argtypes = [c_uint64, c_uint64]
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _wargs(w: FlatWorkload):
    return (c_int(w.n), ptr(w.id, c_int), ptr(w.cls, c_int), ptr(w.in_len, c_int),
            ptr(w.true_out, c_int), ptr(w.pred_out, c_int), ptr(w.arrival, c_double),
            c_int(w.n_classes), ptr(w.class_id, c_int), ptr(w.kind, c_int), ptr(w.e2e, c_double),
            ptr(w.ttft, c_double), ptr(w.tpot, c_double))


def _cfg(t0=500.0, t_thres=20.0, iter=100, tau=0.95, objective_scale=None):
    return _f64([t0, t_thres, iter, tau, 0.0 if objective_scale is None else 1.0,
                 0.0 if objective_scale is None else objective_scale])


def rng_u64(seed, count):
    out = np.zeros(count, dtype=np.uint64)
    lib().ref_rng_u64(c_uint64(seed), c_int(count), ptr(out, c_uint64))
    return out


def rng_index(seed, bounds):
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.uint64))
    out = np.zeros(len(b), dtype=np.uint64)
    lib().ref_rng_index(c_uint64(seed), c_int(len(b)), ptr(b, c_uint64), ptr(out, c_uint64))
    return out


def rng_uniform(seed, count):
    out = np.zeros(count, dtype=np.float64)
    lib().ref_rng_uniform(c_uint64(seed), c_int(count), ptr(out, c_double))
    return out


def rng_normal(seed, count):
    out = np.zeros(count, dtype=np.float64)
    lib().ref_rng_normal(c_uint64(seed), c_int(count), ptr(out, c_double))
    return out


def derive(seed, stream):
    return int(lib().ref_rng_derive(seed, stream))


def predict(coeffs, b, li, lo):
    c = _f64(coeffs)
    out = np.zeros(5, dtype=np.float64)
    _check(lib().ref_predict(ptr(c, c_double), c_int(b), c_int(li), c_int(lo), ptr(out, c_double)))
    return out  # prefill, per_token_decode(b, li), decode_total, exec, tpot


def generate_mixed(n, seed, predict_mode=1) -> FlatWorkload:
    a = {k: np.zeros(n, dtype=np.int32) for k in ("id", "cls", "in_len", "true_out", "pred_out")}
    arr = np.zeros(n, dtype=np.float64)
    _check(lib().ref_generate_mixed(c_int(n), c_uint64(seed), c_int(predict_mode),
                                    *(ptr(a[k], c_int) for k in ("id", "cls", "in_len", "true_out", "pred_out")),
                                    ptr(arr, c_double)))
    return FlatWorkload(arrival=arr, **a)


def evaluate(w: FlatWorkload, coeffs, batches):
    c = _f64(coeffs)
    ids, sizes = flatten_batches(batches)
    n = len(ids)
    n_met, t, g = c_int(), c_double(), c_double()
    per = {k: np.zeros(n, dtype=np.float64) for k in ("wait", "exec", "e2e", "ttft", "tpot")}
    met = np.zeros(n, dtype=np.int32)
    _check(lib().ref_evaluate(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), ptr(sizes, c_int),
                              c_int(len(sizes)), ctypes.byref(n_met), ctypes.byref(t), ctypes.byref(g),
                              *(ptr(per[k], c_double) for k in ("wait", "exec", "e2e", "ttft", "tpot")),
                              ptr(met, c_int)))
    per["met"] = met
    return n_met.value, t.value, g.value, per


def initial_candidates(w: FlatWorkload, coeffs, ids, max_batch):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    si, ss, ii, isz = (np.zeros(max(n, 1), dtype=np.int32) for _ in range(4))
    snb, inb = c_int(), c_int()
    _check(lib().ref_initial_candidates(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), c_int(n),
                                        c_int(max_batch), ptr(si, c_int), ptr(ss, c_int), ctypes.byref(snb),
                                        ptr(ii, c_int), ptr(isz, c_int), ctypes.byref(inb)))
    return unflatten(si, ss[:snb.value]), unflatten(ii, isz[:inb.value])


def neighbor_walk(batches, seed, steps, max_batch):
    ids, sizes = flatten_batches(batches)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb = c_int()
    _check(lib().ref_neighbor_walk(ptr(ids, c_int), ptr(sizes, c_int), c_int(len(sizes)), c_uint64(seed),
                                   c_int(steps), c_int(max_batch), ptr(oi, c_int), ptr(osz, c_int),
                                   ctypes.byref(nb)))
    return unflatten(oi, osz[:nb.value])


def anneal(w: FlatWorkload, coeffs, ids, max_batch, seed=0, **cfg):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g = c_int(), c_int(), c_double(), c_double()
    stats = np.zeros(6, dtype=np.float64)
    cf = _cfg(**cfg)
    _check(lib().ref_anneal(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), c_int(n), ptr(cf, c_double),
                            c_uint64(seed), c_int(max_batch), ptr(oi, c_int), ptr(osz, c_int),
                            ctypes.byref(nb), ctypes.byref(n_met), ctypes.byref(t), ctypes.byref(g),
                            ptr(stats, c_double)))
    return dict(batches=unflatten(oi, osz[:nb.value]), n=n_met.value, t=t.value, g=g.value,
                proposals=int(stats[0]), accepted=int(stats[1]), shortcut=bool(stats[2]),
                g_sorted_start=stats[3], g_input_start=stats[4], objective_scale_used=stats[5])


def anneal_parallel(w: FlatWorkload, coeffs, ids, max_batch, threads, reps=1, seed0=0, **cfg):
    """`threads` independent reference anneal() chains, one std::thread each."""
    c = _f64(coeffs)
    ids = _i32(ids)
    cf = _cfg(**cfg)
    props, wall, bn, bg = c_double(), c_double(), c_int(), c_double()
    _check(lib().ref_anneal_parallel(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), c_int(len(ids)),
                                     ptr(cf, c_double), c_uint64(seed0), c_int(max_batch), c_int(threads),
                                     c_int(reps), ctypes.byref(props), ctypes.byref(wall), ctypes.byref(bn),
                                     ctypes.byref(bg)))
    return dict(proposals=props.value, wall_ms=wall.value, best_n=bn.value, best_g=bg.value)


def exhaustive(w: FlatWorkload, coeffs, ids, max_batch, n_cap=10):
    c = _f64(coeffs)
    ids = _i32(ids)
    n = len(ids)
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    nb, n_met, t, g, ev = c_int(), c_int(), c_double(), c_double(), c_double()
    _check(lib().ref_exhaustive(*_wargs(w), ptr(c, c_double), ptr(ids, c_int), c_int(n), c_int(max_batch),
                                c_int(n_cap), ptr(oi, c_int), ptr(osz, c_int), ctypes.byref(nb),
                                ctypes.byref(n_met), ctypes.byref(t), ctypes.byref(g), ctypes.byref(ev)))
    return dict(batches=unflatten(oi, osz[:nb.value]), n=n_met.value, t=t.value, g=g.value,
                evaluated=int(ev.value))


def schedule_all(w: FlatWorkload, coeffs, instances, seed=0, **cfg):
    """instances: list of dicts {id, total_mem, remaining_mem, mu, sigma, max_batch}."""
    c = _f64(coeffs)
    k = len(instances)
    col = lambda key, f: f([inst[key] for inst in instances])  # noqa: E731
    iid, tm, rm = col("id", _i32), col("total_mem", _f64), col("remaining_mem", _f64)
    mu, sg, mb = col("mu", _f64), col("sigma", _f64), col("max_batch", _i32)
    cf = _cfg(**cfg)
    oi, osz = np.zeros(max(w.n, 1), dtype=np.int32), np.zeros(max(w.n, 1), dtype=np.int32)
    inb, icnt, in_ = (np.zeros(k, dtype=np.int32) for _ in range(3))
    it, ig = np.zeros(k), np.zeros(k)
    epochs = c_int()
    _check(lib().ref_schedule_all(*_wargs(w), ptr(c, c_double), c_int(k), ptr(iid, c_int), ptr(tm, c_double),
                                  ptr(rm, c_double), ptr(mu, c_double), ptr(sg, c_double), ptr(mb, c_int),
                                  ptr(cf, c_double), c_uint64(seed), ptr(oi, c_int), ptr(osz, c_int),
                                  ptr(inb, c_int), ptr(icnt, c_int), ptr(in_, c_int), ptr(it, c_double),
                                  ptr(ig, c_double), ctypes.byref(epochs)))
    out, pos, kb = [], 0, 0
    for i in range(k):
        sizes = osz[kb:kb + inb[i]]
        out.append(dict(batches=unflatten(oi[pos:pos + icnt[i]], sizes), n=int(in_[i]), t=float(it[i]),
                        g=float(ig[i])))
        pos += int(icnt[i])
        kb += int(inb[i])
    return out, epochs.value


def _fleet(instances):
    col = lambda key, f: f([inst[key] for inst in instances])  # noqa: E731
    return (col("id", _i32), col("total_mem", _f64), col("remaining_mem", _f64), col("mu", _f64), col("sigma", _f64),
            col("max_batch", _i32))


def _fleet_args(fl):
    iid, tm, rm, mu, sg, mb = fl
    return (c_int(len(iid)), ptr(iid, c_int), ptr(tm, c_double), ptr(rm, c_double), ptr(mu, c_double),
            ptr(sg, c_double), ptr(mb, c_int))


def _unpack_records(rec, n):
    r = rec[:8 * n].reshape(n, 8)
    return [dict(request_id=int(x[0]), wait_ms=x[1], exec_ms=x[2], e2e_ms=x[3], ttft_ms=x[4], tpot_ms=x[5],
                 slo_met=bool(x[6]), extrapolated=bool(x[7])) for x in r]


def _unpack_report(rep):
    return dict(slo_attainment=rep[0], avg_latency_ms=rep[1], g=rep[2], scheduling_overhead_ms=rep[3],
                n_met=int(rep[4]), total_latency_ms=rep[5])


def run(w: FlatWorkload, coeffs, instances, plans, noise=0.0, gap=0.1, seed=0, overhead=0.0):
    """run() (P:src/simulator.cpp:49-74); plans: per instance a list of batches (request ids)."""
    fl = _fleet(instances)
    ids = _i32([i for p in plans for b in p for i in b] or [0])
    sizes = _i32([len(b) for p in plans for b in p] or [0])
    nb = _i32([len(p) for p in plans])
    n = sum(len(b) for p in plans for b in p)
    rec, rep = np.zeros(8 * max(n, 1)), np.zeros(6)
    _check(lib().ref_run(*_wargs(w), ptr(_f64(coeffs), c_double), *_fleet_args(fl), ptr(ids, c_int),
                         ptr(sizes, c_int), ptr(nb, c_int), c_double(noise), c_double(gap), c_uint64(seed),
                         c_double(overhead), ptr(rec, c_double), ptr(rep, c_double)))
    return _unpack_records(rec, n), _unpack_report(rep)


def run_fcfs(w: FlatWorkload, coeffs, instances, noise=0.0, gap=0.1, seed=0):
    fl = _fleet(instances)
    n = w.n
    oi, osz = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
    inb = np.zeros(len(instances), dtype=np.int32)
    rec, rep = np.zeros(8 * max(n, 1)), np.zeros(6)
    _check(lib().ref_run_fcfs(*_wargs(w), ptr(_f64(coeffs), c_double), *_fleet_args(fl), c_double(noise),
                              c_double(gap), c_uint64(seed), ptr(oi, c_int), ptr(osz, c_int), ptr(inb, c_int),
                              ptr(rec, c_double), ptr(rep, c_double)))
    plans, pos, kb = [], 0, 0
    for i in range(len(instances)):
        sizes = osz[kb:kb + inb[i]]
        cnt = int(sizes.sum())
        plans.append(unflatten(oi[pos:pos + cnt], sizes))
        pos += cnt
        kb += int(inb[i])
    return plans, _unpack_records(rec, n), _unpack_report(rep)


def estimator(class_ids, priors, observations, predict_classes, seed):
    """Estimator (P:src/output_estimator.cpp): priors per class None / ("gaussian", m, s) / ("range", lo, hi)."""
    kinds = [0 if p is None else (1 if p[0] == "gaussian" else 2) for p in priors]
    pa = [0.0 if p is None else float(p[1]) for p in priors]
    pb = [0.0 if p is None else float(p[2]) for p in priors]
    k = len(class_ids)
    oc, ol = _i32([o[0] for o in observations] or [0]), _i32([o[1] for o in observations] or [0])
    pc = _i32(list(predict_classes) or [0])
    out = np.zeros(max(len(predict_classes), 1), dtype=np.int32)
    cnt, mean, m2 = np.zeros(k, dtype=np.int64), np.zeros(k), np.zeros(k)
    _check(lib().ref_estimator(c_int(k), ptr(_i32(class_ids), c_int), ptr(_i32(kinds), c_int), ptr(_f64(pa), c_double),
                               ptr(_f64(pb), c_double), c_int(len(observations)), ptr(oc, c_int), ptr(ol, c_int),
                               c_int(len(predict_classes)), ptr(pc, c_int), c_uint64(seed), ptr(out, c_int),
                               ptr(cnt, ctypes.c_longlong), ptr(mean, c_double), ptr(m2, c_double)))
    return [int(x) for x in out[:len(predict_classes)]], [(int(cnt[i]), float(mean[i]), float(m2[i])) for i in range(k)]


def compare(w: FlatWorkload, coeffs, instances, policies, seeds, noise=0.0, gap=0.1, n_cap=10, **cfg):
    """compare() (P:src/simulator.cpp:148-220); policies as codes (0 sa, 1 exhaustive, 2 fcfs)."""
    fl = _fleet(instances)
    sd = np.asarray(list(seeds), dtype=np.uint64)
    rows, med = np.zeros(6 * len(policies) * len(sd)), np.zeros(6 * len(policies))
    _check(lib().ref_compare(*_wargs(w), ptr(_f64(coeffs), c_double), *_fleet_args(fl), c_int(len(policies)),
                             ptr(_i32(policies), c_int), c_int(len(sd)), ptr(sd, c_uint64), ptr(_cfg(**cfg), c_double),
                             c_double(noise), c_double(gap), c_int(n_cap), ptr(rows, c_double), ptr(med, c_double)))
    return rows.reshape(-1, 6), med.reshape(-1, 6)


__all__ = [n for n in dir() if not n.startswith("_")] + ["POINTER"]
