#!/usr/bin/env python
"""Scratch prototype (not product, not oracle): validates the schedule of the
blocked "unit" pass kernel before it is written in CUDA.

A UNIT is step j of G consecutive sweeps r0..r0+G-1 of one pass (c, t).  The
kernel executes it as: all G right reflectors (A-phase, g = 0..G-1), then all
G left reflectors (B-phase).  The oracle order interleaves A_0 B_0 A_1 B_1 ...
and runs sweep r0 to the end before sweep r0+1 starts; the unit order only
swaps pairs that commute exactly (A_g with B_g' for g' < g; B_g(j) with
A_g'(j+1) for g > g'), so the results agree up to rounding.

Checks (small n, dense numpy, fp64):
  1. unit order vs sequential (oracle) order: |d|, |e| and sigma agree to
     rounding, structural zeros exact;
  2. every unit touches only cells inside its declared L-shaped window;
  3. the inter-group rule "unit (k+1, j) after unit (k, j + dK)" (dK from the
     closed form used by the kernel) is sufficient: random interleavings
     that respect it give results BITWISE equal to the canonical group order,
     and dK is >= the brute-force minimum.
"""
from __future__ import annotations

import itertools
import sys

import numpy as np


def house(x):
    alpha = x[0]
    if len(x) == 1 or not np.any(x[1:] != 0):
        return None, 0.0, alpha
    nrm = np.sqrt(np.sum(x * x))
    beta = -nrm if alpha >= 0 else nrm
    tau = (beta - alpha) / beta
    v = x.copy()
    v[0] = 1.0
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def passes(n, b, tw):
    out = []
    c = min(b, n - 1)
    while c > 1:
        t = min(tw, c - 1)
        out.append((c, t))
        c -= t
    return out


def geo(n, c, t, r, j):
    p = r + (c - t) + j * c
    if p > n - 2:
        return None
    q = r if j == 0 else p - c
    hi = min(p + t, n - 1)
    ce = min(hi + c, n - 1)
    return q, p, hi, ce


class Tracker:
    def __init__(self):
        self.cells = set()

    def touch(self, rows, cols):
        for i in rows:
            for x in cols:
                self.cells.add((i, x))


def op_A(A, n, c, t, r, j, tr=None):
    g = geo(n, c, t, r, j)
    if g is None:
        return
    q, p, hi, ce = g
    v, tau, beta = house(A[q, p:hi + 1].copy())
    if tr is not None:
        tr.touch([q], range(p, hi + 1))
        tr.touch(range(q + 1, hi + 1), range(p, hi + 1))
    if v is not None:
        blk = A[q + 1:hi + 1, p:hi + 1]
        w = blk @ v
        blk -= tau * np.outer(w, v)
    A[q, p] = beta
    A[q, p + 1:hi + 1] = 0.0


def op_B(A, n, c, t, r, j, tr=None):
    g = geo(n, c, t, r, j)
    if g is None:
        return
    q, p, hi, ce = g
    v, tau, beta = house(A[p:hi + 1, p].copy())
    if tr is not None:
        tr.touch(range(p, hi + 1), [p])
        tr.touch(range(p, hi + 1), range(p + 1, ce + 1))
    if v is not None:
        blk = A[p:hi + 1, p + 1:ce + 1]
        w = v @ blk
        blk -= tau * np.outer(v, w)
    A[p, p] = beta
    A[p + 1:hi + 1, p] = 0.0


def seq_reduce(A, b, tw):
    A = A.copy()
    n = A.shape[0]
    for c, t in passes(n, b, tw):
        for r in range(n - 1):
            j = 0
            while geo(n, c, t, r, j) is not None:
                op_A(A, n, c, t, r, j)
                op_B(A, n, c, t, r, j)
                j += 1
    return A


def unit(A, n, c, t, G, k, j, tr=None):
    r0 = k * G
    for g in range(G):
        op_A(A, n, c, t, r0 + g, j, tr)
    for g in range(G):
        op_B(A, n, c, t, r0 + g, j, tr)


def n_units(n, c, t, G, k):
    # units of group k: steps of its first sweep (later sweeps have <= as many)
    r0 = k * G
    j = 0
    while geo(n, c, t, r0, j) is not None:
        j += 1
    return j


def window(n, c, t, G, k, j):
    """Declared L-shaped window of unit (k, j): V part rows [q0, p-1] x cols
    [p, p+t+G-1]; H part rows [p, p+t+G-1] x cols [p, p+c+t+G-1]; restricted
    to the matrix and the band offsets [-t, c+t]."""
    r0 = k * G
    p = r0 + (c - t) + j * c
    q0 = r0 if j == 0 else p - c
    cells = set()
    W = t + G
    for i in range(q0, p):
        for x in range(p, p + W):
            cells.add((i, x))
    for i in range(p, p + W):
        for x in range(p, p + c + W):
            cells.add((i, x))
    return {(i, x) for (i, x) in cells if i < n and x < n and -t <= x - i <= c + t}


def dK_closed(c, t, G):
    """Kernel rule: unit (k+1, j) may start once group k completed units
    0 .. j + dK - 1 (progress >= j + dK)."""
    # group k+1's window at unit j reaches col p+G+c+t+G-1 and row p+2G+t-1;
    # group k's unit j+d window starts at col/row p+d*c - c (V part rows
    # from p+dc-c, cols from p+dc).  Overlap while (d-1)*c <= 2G+t-1 + ...
    d = 1
    while (d - 1) * c <= 2 * G + t - 1 + c:
        d += 1
    return d


def unit_reduce(A, b, tw, Gfun, order="canonical", rng=None, check_windows=False, dK_bf=None):
    A = A.copy()
    n = A.shape[0]
    for c, t in passes(n, b, tw):
        G = Gfun(c, t)
        ns = max(0, (n - 2) - (c - t) + 1)
        ngroups = (ns + G - 1) // G
        J = [n_units(n, c, t, G, k) for k in range(ngroups)]
        if check_windows or dK_bf is not None:
            touched = {}
            B = A.copy()
            for k in range(ngroups):
                for j in range(J[k]):
                    tr = Tracker()
                    unit(B, n, c, t, G, k, j, tr)
                    tr.cells = {(i, x) for (i, x) in tr.cells if i < n and x < n}
                    touched[(k, j)] = tr.cells
                    if check_windows:
                        w = window(n, c, t, G, k, j)
                        extra = tr.cells - w
                        assert not extra, ("unit touches outside its window", c, t, G, k, j, sorted(extra)[:5])
            if dK_bf is not None:
                # brute force: unit (k+1, j) must follow every unit (k, j2) whose
                # touched cells intersect its own
                need = 0
                for k in range(ngroups - 1):
                    for j in range(J[k + 1]):
                        mine = window(n, c, t, G, k + 1, j)
                        last = -1
                        for j2 in range(J[k]):
                            if touched[(k, j2)] & mine:
                                last = j2
                        need = max(need, last - j + 1)
                dK_bf.append((c, t, G, need, dK_closed(c, t, G)))
        if order == "canonical":
            for k in range(ngroups):
                for j in range(J[k]):
                    unit(A, n, c, t, G, k, j)
        else:
            dK = dK_closed(c, t, G)
            prog = [0] * ngroups
            live = True
            while live:
                ready = []
                for k in range(ngroups):
                    j = prog[k]
                    if j >= J[k]:
                        continue
                    if k > 0 and prog[k - 1] < min(j + dK, J[k - 1]):
                        continue
                    ready.append(k)
                if not ready:
                    assert all(prog[k] >= J[k] for k in range(ngroups)), "deadlock"
                    live = False
                    continue
                k = ready[rng.integers(len(ready))]
                unit(A, n, c, t, G, k, prog[k])
                prog[k] += 1
    return A


def svals(A):
    return np.linalg.svd(A, compute_uv=False)


def main():
    rng = np.random.default_rng(1)
    cases = [(60, 8, 2, lambda c, t: max(1, min(3, c - t))),
             (90, 12, 4, lambda c, t: max(1, min(5, c - t))),
             (97, 16, 4, lambda c, t: max(1, min(8, c - t))),
             (130, 24, 8, lambda c, t: max(1, min(6, c - t))),
             (150, 32, 8, lambda c, t: max(1, min(24, c - t))),
             (77, 20, 19, lambda c, t: max(1, c - t))]
    bf = []
    for n, b, tw, Gf in cases:
        A0 = np.triu(np.tril(rng.standard_normal((n, n)), b))
        S = seq_reduce(A0, b, tw)
        U = unit_reduce(A0, b, tw, Gf, check_windows=True, dK_bf=bf)
        for name, M in (("seq", S), ("unit", U)):
            off = M - np.diag(np.diag(M)) - np.diag(np.diag(M, 1), 1)
            assert np.all(off == 0), (name, "structural zeros")
        dd = np.max(np.abs(np.abs(np.diag(S)) - np.abs(np.diag(U))))
        de = np.max(np.abs(np.abs(np.diag(S, 1)) - np.abs(np.diag(U, 1))))
        ds = np.max(np.abs(svals(S) - svals(A0)))
        du = np.max(np.abs(svals(U) - svals(A0)))
        for trial in range(3):
            R = unit_reduce(A0, b, tw, Gf, order="random", rng=np.random.default_rng(trial))
            assert np.array_equal(R, U), ("interleaving changed bits", n, b, tw, trial)
        print(f"n={n} b={b} tw={tw}: |d| diff {dd:.2e} |e| diff {de:.2e} sigma err seq {ds:.2e} unit {du:.2e}")
        assert dd < 1e-10 and de < 1e-10 and du < 1e-11
    for c, t, G, need, closed in sorted(set(bf)):
        print(f"  pass c={c} t={t} G={G}: brute-force dK {need}, closed form {closed}")
        assert closed >= need
    print("OK")


if __name__ == "__main__" and len(sys.argv) == 1:
    sys.exit(main())


# --------------------------------------------------------------------------
# CTA-level simulation of the v5 kernel's data protocol (loads, write-backs,
# half-unit progress flags) -- what the CUDA kernel does, cell for cell.
# --------------------------------------------------------------------------
def _inband(n, c, t, i, x):
    return 0 <= i < n and 0 <= x < n and -t <= x - i <= c + t


class GroupSim:
    def __init__(self, n, c, t, G, k):
        self.n, self.c, self.t, self.G, self.k = n, c, t, G, k
        self.r0 = k * G
        self.J = n_units(n, c, t, G, k)
        self.j = 0
        self.phase = 0          # 0: LV+A+WA, 1: LH+B+WB(+carry)
        self.local = {}         # (i, x) -> value (the CTA's shared memory)
        self.prog = 0

    def geo(self, j):
        c, t, G = self.c, self.t, self.G
        p = self.r0 + (c - t) + j * c
        q0 = self.r0 if j == 0 else p - c
        return p, q0, t + G

    def need(self, rule):
        """progress of the previous group this group's next phase needs;
        rule = (a0, b0): A half waits >= 2j + a0, B half >= 2j + b0"""
        j = self.j
        a0, b0 = rule
        return 2 * j + (a0 if self.phase == 0 else b0)

    def run_phase(self, Gm):
        n, c, t, G = self.n, self.c, self.t, self.G
        j = self.j
        p, q0, W = self.geo(j)
        last = j == self.J - 1
        if self.phase == 0:
            lo = q0 if j == 0 else q0 + W
            for x in range(p, p + W):
                for i in range(lo, p + W):
                    self.local[(i, x)] = Gm[i, x] if _inband(n, c, t, i, x) else 0.0
            L = np.zeros((n, n))
            for (i, x), v in self.local.items():
                if 0 <= i < n and 0 <= x < n:
                    L[i, x] = v
            for g in range(G):
                op_A(L, n, c, t, self.r0 + g, j)
            for key in list(self.local):
                i, x = key
                if 0 <= i < n and 0 <= x < n:
                    self.local[key] = L[i, x]
            for x in range(p, p + W):
                for i in range(q0, p):
                    if _inband(n, c, t, i, x):
                        Gm[i, x] = self.local[(i, x)]
            self.prog = 2 * j + 1
            self.phase = 1
        else:
            for x in range(p + W, p + W + c):
                for i in range(p, p + W):
                    self.local[(i, x)] = Gm[i, x] if _inband(n, c, t, i, x) else 0.0
            L = np.zeros((n, n))
            for (i, x), v in self.local.items():
                if 0 <= i < n and 0 <= x < n:
                    L[i, x] = v
            for g in range(G):
                op_B(L, n, c, t, self.r0 + g, j)
            for key in list(self.local):
                i, x = key
                if 0 <= i < n and 0 <= x < n:
                    self.local[key] = L[i, x]
            xend = p + W + c if last else p + c
            for x in range(p, xend):
                for i in range(p, p + W):
                    if _inband(n, c, t, i, x):
                        Gm[i, x] = self.local[(i, x)]
            self.prog = 2 * j + 2
            # carry: H-part cols [p+c, p+c+W) rows [p, p+W) become the next
            # unit's top V rows; everything else leaves shared memory
            carry = {(i, x): self.local[(i, x)] for x in range(p + c, p + c + W) for i in range(p, p + W)}
            self.local = carry
            self.j += 1
            self.phase = 0

    def done(self):
        return self.j >= self.J


def cta_sim_reduce(A, b, tw, Gfun, half_rule_fun, rng):
    A = A.copy()
    n = A.shape[0]
    for c, t in passes(n, b, tw):
        G = Gfun(c, t)
        half = half_rule_fun(c, t, G)   # (a0, b0)
        ns = max(0, (n - 2) - (c - t) + 1)
        ngroups = (ns + G - 1) // G
        gs = [GroupSim(n, c, t, G, k) for k in range(ngroups)]
        while True:
            ready = []
            for k, s in enumerate(gs):
                if s.done():
                    continue
                if k > 0 and gs[k - 1].prog < min(s.need(half), 2 * gs[k - 1].J):
                    continue
                ready.append(k)
            if not ready:
                assert all(s.done() for s in gs), "deadlock"
                break
            gs[ready[rng.integers(len(ready))]].run_phase(A)
    return A


def main_sim():
    rng = np.random.default_rng(5)
    cases = [(70, 8, 2), (95, 12, 4), (101, 16, 4), (123, 24, 8), (140, 32, 8), (77, 20, 19), (88, 17, 5)]
    for n, b, tw in cases:
        A0 = np.triu(np.tril(rng.standard_normal((n, n)), b))
        from v5_rules import minimal_rule
        for Gf, name in ((lambda c, t: max(1, min(4, (c - t) // 2)), "G<=(c-t)/2"),
                         (lambda c, t: max(1, c - t), "G=c-t"),
                         (lambda c, t: max(1, min(3, c - t)), "G<=3")):
            hf = lambda c, t, G: minimal_rule(c, t, G)
            U = unit_reduce(A0, b, tw, Gf)
            for trial in range(2):
                R = cta_sim_reduce(A0, b, tw, Gf, hf, np.random.default_rng(trial))
                assert np.array_equal(R, U), ("cta sim differs", n, b, tw, name, trial,
                                               np.max(np.abs(R - U)))
        print(f"cta sim n={n} b={b} tw={tw}: bitwise equal to canonical unit order")
    print("SIM OK")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sim":
    main_sim()
