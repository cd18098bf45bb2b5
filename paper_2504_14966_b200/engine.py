"""Direct handle on the engine C ABI (include/slosched_gpu.h): tables, the bit-exact batch
evaluator (K1) and the split prepare / launch / fetch chain interface used for
device-resident timing."""
from __future__ import annotations

import ctypes
from ctypes import byref, c_double, c_int32, c_uint32, c_void_p

import numpy as np

from . import _lib
from ._lib import SloChainParams, SloChainResult, lib
from .slosched import LatencyCoefficients, Workload, _check_api, _check_engine, _f64, _i32, _p


def build_tables(workload: Workload, ids, coeffs: LatencyCoefficients, max_batch: int):
    """(exec, deadline) as [max_batch, n] float64 over dense indices = rank of each id."""
    ids = _i32(ids)
    n = len(ids)
    ex, dl = np.zeros(n * max_batch), np.zeros(n * max_batch)
    _check_api(lib().slosched_build_tables(byref(workload._view), _p(coeffs.as_array(), c_double), _p(ids), n,
                                           max_batch, _p(ex, c_double), _p(dl, c_double)))
    return ex.reshape(max_batch, n), dl.reshape(max_batch, n)


def end_bits(sizes_list, n):
    """Batch-end bitmask rows (uint32, ceil(n/32) words) for a list of batch-size sequences."""
    words = (n + 31) // 32
    out = np.zeros((len(sizes_list), words), dtype=np.uint32)
    for r, sizes in enumerate(sizes_list):
        ends = np.cumsum(np.asarray(sizes, dtype=np.int64)) - 1
        np.bitwise_or.at(out[r], ends >> 5, (np.uint32(1) << (ends & 31).astype(np.uint32)))
    return out


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    o = np.zeros(4, dtype=np.uint32)
    lib().slo_philox4x32_10(_p(c, c_uint32), _p(k, c_uint32), _p(o, c_uint32))
    return o


class Engine:
    """One slo_ctx (device, stream, device buffers)."""

    def __init__(self, device: int = 0):
        self._ctx = c_void_p()
        _check_engine(lib().slo_ctx_create(device, byref(self._ctx)))
        self.device = device
        self.n = 0
        self.mb = 0

    def close(self):
        if self._ctx:
            lib().slo_ctx_destroy(self._ctx)
            self._ctx = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(lib().slo_ctx_stream(self._ctx) or 0)

    @property
    def sm_count(self) -> int:
        return int(lib().slo_ctx_sm_count(self._ctx))

    def sync(self):
        _check_engine(lib().slo_ctx_sync(self._ctx))

    def set_problem(self, exec_tab: np.ndarray, deadline_tab: np.ndarray):
        mb, n = exec_tab.shape
        ex, dl = _f64(exec_tab).ravel(), _f64(deadline_tab).ravel()
        _check_engine(lib().slo_problem_set(self._ctx, n, mb, _p(ex, c_double), _p(dl, c_double)))
        self.n, self.mb = n, mb

    @property
    def tick_ms(self) -> float:
        """Grid (ms) of the chain kernel's integer objective for the current problem."""
        return float(lib().slo_problem_tick_ms(self._ctx))

    def evaluate_batch(self, perms: np.ndarray, bits: np.ndarray):
        """K1: bit-exact n_met / t / g of `count` candidates (dense-index perms [count, n])."""
        perms = np.ascontiguousarray(perms, dtype=np.uint16)
        bits = np.ascontiguousarray(bits, dtype=np.uint32)
        count = perms.shape[0]
        n_met, t, g = np.zeros(count, dtype=np.int32), np.zeros(count), np.zeros(count)
        _check_engine(lib().slo_evaluate_batch(self._ctx, count, perms.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
                                               _p(bits, c_uint32), _p(n_met), _p(t, c_double), _p(g, c_double)))
        return n_met, t, g

    def evaluate_batch_tick(self, perms: np.ndarray, bits: np.ndarray):
        """K3's own objective of `count` candidates: n_met bit-exact with CostModel::score, t and g on
        the tick grid. Returns (n_met, t, g, exact_walks)."""
        perms = np.ascontiguousarray(perms, dtype=np.uint16)
        bits = np.ascontiguousarray(bits, dtype=np.uint32)
        count = perms.shape[0]
        n_met, t, g = np.zeros(count, dtype=np.int32), np.zeros(count), np.zeros(count)
        ex = ctypes.c_uint64()
        _check_engine(lib().slo_evaluate_batch_tick(self._ctx, count,
                                                    perms.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
                                                    _p(bits, c_uint32), _p(n_met), _p(t, c_double), _p(g, c_double),
                                                    byref(ex)))
        return n_met, t, g, int(ex.value)

    def _params(self, t0=500.0, t_thres=20.0, iter=100, tau=0.95, seed=0, objective_scale=1.0, replay=False,
                chains=1, chain_begin=0, chain_end=None, budget_ms=0.0, scale_ladder=(), max_blocks=0):
        ladder = _f64(list(scale_ladder)) if len(scale_ladder) else None
        prm = SloChainParams(t0, t_thres, iter, tau, seed & (2**64 - 1), objective_scale,
                             _lib.SLO_RNG_XOSHIRO_REPLAY if replay else _lib.SLO_RNG_PHILOX, chains, chain_begin,
                             chains if chain_end is None else chain_end, int(budget_ms * 1e6),
                             0 if ladder is None else len(ladder), None if ladder is None else _p(ladder, c_double),
                             max_blocks)
        return prm, ladder

    def prepare(self, start_perm, start_sizes, **kw):
        prm, self._ladder = self._params(**kw)
        sp, ss = _i32(start_perm), _i32(start_sizes)
        _check_engine(lib().slo_chains_prepare(self._ctx, byref(prm), _p(sp), _p(ss), len(ss)))

    def launch(self):
        _check_engine(lib().slo_chains_launch(self._ctx))

    def fetch(self):
        n = self.n
        bp, bs, nb = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32), c_int32()
        res = SloChainResult()
        _check_engine(lib().slo_chains_fetch(self._ctx, _p(bp), _p(bs), byref(nb), byref(res)))
        return bp, bs[:nb.value], res

    def anneal_chains(self, start_perm, start_sizes, **kw):
        self.prepare(start_perm, start_sizes, **kw)
        self.launch()
        return self.fetch()

    # ---- multi-process exchange (include/slosched_gpu.h, multi-GPU section)
    @property
    def handle(self) -> int:
        """The slo_ctx pointer (AnnealConfig.comm_ctx of a rank context)."""
        return int(self._ctx.value or 0)

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Attach an NCCL communicator (collective over the nranks processes): launch() then also
        enqueues the device-side exchange, fetch() returns the job-wide winner on every rank."""
        buf = (ctypes.c_uint8 * _lib.SLO_COMM_ID_BYTES).from_buffer_copy(bytes(uid))
        _check_engine(lib().slo_ctx_comm_init(self._ctx, nranks, rank, buf))

    def comm_info(self):
        nr, rk = c_int32(), c_int32()
        _check_engine(lib().slo_ctx_comm_info(self._ctx, byref(nr), byref(rk)))
        return nr.value, rk.value

    def comm_check(self):
        _check_engine(lib().slo_comm_check(self._ctx))


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it; the launcher distributes it)."""
    buf = (ctypes.c_uint8 * _lib.SLO_COMM_ID_BYTES)()
    _check_engine(lib().slo_comm_unique_id(buf))
    return bytes(buf)


class Group:
    """Several devices driven by this process (slo_group): one context per device, one NCCL
    communicator over them (transport "nccl"), or peer copies onto member 0 when a device is
    listed twice (transport "peer")."""

    def __init__(self, devices):
        devs = _i32(list(devices))
        self._g = c_void_p()
        _check_engine(lib().slo_group_create(len(devs), _p(devs), byref(self._g)))
        self.devices = [int(d) for d in devs]
        self.n = 0

    def close(self):
        if self._g:
            lib().slo_group_destroy(self._g)
            self._g = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def transport(self) -> str:
        return lib().slo_group_transport(self._g).decode()

    def set_problem(self, exec_tab: np.ndarray, deadline_tab: np.ndarray):
        mb, n = exec_tab.shape
        ex, dl = _f64(exec_tab).ravel(), _f64(deadline_tab).ravel()
        _check_engine(lib().slo_group_problem_set(self._g, n, mb, _p(ex, c_double), _p(dl, c_double)))
        self.n = n

    def anneal_chains(self, start_perm, start_sizes, **kw):
        prm, _ladder = Engine._params(None, **kw)
        sp, ss = _i32(start_perm), _i32(start_sizes)
        n = self.n
        bp, bs, nb = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32), c_int32()
        res = SloChainResult()
        _check_engine(lib().slo_group_anneal_chains(self._g, byref(prm), _p(sp), _p(ss), len(ss), _p(bp), _p(bs),
                                                    byref(nb), byref(res)))
        return bp, bs[:nb.value], res
