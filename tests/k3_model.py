"""Test infrastructure: a plain-Python model of one K3 chain (paper_2504_14966_b200/csrc/chains.cuh),
written from its specification, to pin the GPU kernel's trajectory exactly.

Semantics modelled:
* proposal discipline of the reference (P:src/priority_mapper.cpp:184-198, moves :141-180) on a
  list of batches: up to 8 attempts of op = U[0,3) -- squeeze / delay / swap -- the first valid one
  wins, else a forced swap (attempt 8);
* draws from Philox4x32-10 (Random123 constants): the row of proposal `prop` of chain `cid` is
  20 words, block b = philox(ctr = (prop, cid, b, 0x5105c4ed), key = (seed lo, seed hi)); the ops of
  attempts 0-7 are the base-3 digits of U[0, 3^8) from word 0, attempt a's positions come from words
  1 + 2a and 2 + 2a (attempt 8, the forced swap: words 17, 18); U[0, m) = (word * m) >> 32; the
  acceptance uniform is word 19;
* objective: the total latency on the tick grid (exec rounded half-even to multiples of `tick`,
  every sum an integer); n_met exactly the reference's -- the batch-start elapsed time summed in
  fp64 makespan by makespan (P:src/priority_mapper.cpp:264-276) against the fp64 latest-start
  table (deadline +inf: always met); G = n_met / t;
* Metropolis: accept if G_new > G, else u < exp(-x) in float32 with x = (G - G_new) * (scale / t)
  and u = (word27 >> 8) * 2^-24; temperature t = t0, t *= tau while t >= t_thres;
* the best state is the first one reaching a new maximum G.

It is a model, not the product: it evaluates every proposal from scratch (O(n)), so it also checks
the kernel's incremental scoring (rebuilt-batch deltas, anchor shifts, SLO walks, move flags)."""
from __future__ import annotations

import math

import numpy as np

M32 = 0xFFFFFFFF
TAG_MOVE = 0x5105C4ED
ATTEMPTS = 9
ACC_WORD = 19


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = [x & M32 for x in ctr]
    k0, k1 = key[0] & M32, key[1] & M32
    for _ in range(10):
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c3 ^ k1) & M32, p0 & M32
        k0, k1 = (k0 + 0x9E3779B9) & M32, (k1 + 0xBB67AE85) & M32
    return [c0, c1, c2, c3]


def row(prop, cid, seed):
    words = []
    for b in range(5):
        words += philox4x32_10([prop, cid, b, TAG_MOVE], [seed & M32, (seed >> 32) & M32])
    return words


def mulhi(x, m):
    return (x * m) >> 32


class TickProblem:
    """exec / deadline tables [mb][n] (float64) on the tick grid."""

    def __init__(self, ex, dl, tick):
        self.mb, self.n = ex.shape
        self.tick = tick
        self.xt = np.rint(ex / tick).astype(np.int64)
        self.dl = dl
        self.ex = ex

    def met(self, elapsed_f, b, i):
        """the reference's test: fp64 batch-start elapsed <= latest start"""
        return elapsed_f <= float(self.dl[b - 1, i])

    def score(self, batches):
        elapsed = total = met = 0
        elapsed_f = 0.0  # the reference's elapsed: fp64, left to right
        for bt in batches:
            b = len(bt)
            mk, mk_f = 0, 0.0
            for i in bt:
                x = int(self.xt[b - 1, i])
                total += elapsed + x
                met += self.met(elapsed_f, b, i)
                mk = max(mk, x)
                e = float(self.ex[b - 1, i])
                mk_f = e if mk_f < e else mk_f
            elapsed += mk
            elapsed_f = elapsed_f + mk_f
        t = float(total) * self.tick
        return met, t, (met * (1.0 / t) if t > 0 else 0.0)


def _locate(batches, pos):
    """(batch index, offset) of flat position pos"""
    for k, bt in enumerate(batches):
        if pos < len(bt):
            return k, pos
        pos -= len(bt)
    raise IndexError(pos)


def propose(batches, n, mb, words):
    """Apply the first valid attempt to a copy of batches; returns the new batches (or None)."""
    ops = mulhi(words[0], 3 ** 8)
    for a in range(ATTEMPTS):
        r1, r2 = words[1 + 2 * a], words[2 + 2 * a]
        op = (ops // 3 ** a) % 3 if a < ATTEMPTS - 1 else 2
        if op == 0:  # squeeze: move pos to the end of the previous batch (:141-153)
            first = len(batches[0])
            if first >= n:
                continue
            pos = first + mulhi(r1, n - first)
            k, off = _locate(batches, pos)
            if len(batches[k - 1]) >= mb:
                continue
            nb = [list(x) for x in batches]
            x = nb[k].pop(off)
            nb[k - 1].append(x)
            if not nb[k]:
                del nb[k]
            return nb
        if op == 1:  # delay: move pos to the end of the next batch, or a new last batch (:155-170)
            pos = mulhi(r1, n)
            k, off = _locate(batches, pos)
            if k + 1 < len(batches) and len(batches[k + 1]) >= mb:
                continue
            nb = [list(x) for x in batches]
            x = nb[k].pop(off)
            if k + 1 < len(nb):
                nb[k + 1].append(x)
            else:
                nb.append([x])
            if not nb[k]:
                del nb[k]
            return nb
        if n < 2:  # swap two positions (:172-180)
            continue
        pa = mulhi(r1, n)
        pb = mulhi(r2, n - 1)
        pb += 1 if pb >= pa else 0
        flat = [i for bt in batches for i in bt]
        flat[pa], flat[pb] = flat[pb], flat[pa]
        nb, q = [], 0
        for bt in batches:
            nb.append(flat[q:q + len(bt)])
            q += len(bt)
        return nb
    return None


def run_chain(prob: TickProblem, start_batches, cid, seed, t0, t_thres, tau, iters, scale):
    """One chain; returns dict(best_batches, best=(n_met, t, g), proposals, accepted)."""
    n, mb = prob.n, prob.mb
    cur = [list(b) for b in start_batches]
    nm, t_cur, f = prob.score(cur)
    best, best_b = (nm, t_cur, f), [list(b) for b in cur]
    props = accs = 0
    temp, lev = t0, 0
    while temp >= t_thres:
        sinv = scale * (1.0 / temp)
        for it in range(iters):
            w = row(lev * iters + it, cid, seed)
            props += 1
            nb = propose(cur, n, mb, w)
            if nb is None:
                cand = cur
            else:
                cand = nb
            nm2, t2, f2 = prob.score(cand)
            accept = f2 > f
            if not accept:
                x = np.float32((f - f2) * sinv)
                u = np.float32(w[ACC_WORD] >> 8) * np.float32(2.0 ** -24)
                with np.errstate(over="ignore", under="ignore"):
                    accept = bool(u < np.exp2(np.float32(-x) * np.float32(1.4426950408889634)))
            if accept:
                accs += 1
                cur, f = cand, f2
                if f2 > best[2]:
                    best, best_b = (nm2, t2, f2), [list(b) for b in cand]
        temp *= tau
        lev += 1
    return {"best_batches": best_b, "best": best, "proposals": props, "accepted": accs}
