#!/usr/bin/env python
"""Hazard checker for the unit pass kernel's (bb_pass_v5.cuh) inter-group
protocol, on the kernel's exact load / write-back rectangles.

Group k (sweeps kG .. kG+G-1) runs, per unit j (step j of its sweeps):
  LV(j)  load   rows [lo, p+W)    x cols [p, p+W)        lo = q0 (j = 0) else q0 + W
  WA(j)  write  rows [q0, p)      x cols [p, p+W)        -> progress 2j+1
  LH(j)  load   rows [p, p+W)     x cols [p+W, p+W+c)
  WB(j)  write  rows [p, p+W)     x cols [p, p+c)        (last unit: [p, p+W+c)) -> 2j+2
with p = kG + (c-t) + j*c, q0 = kG (j = 0) else p - c, W = t + G, all cells
restricted to the matrix and to band offsets [-t, c+t].  Rule (a0, b0): the
A half of unit j of group k+1 (LV, WA) starts once progress[k] >= 2j + a0,
the B half (LH, WB) once progress[k] >= 2j + b0 (both capped at 2*J_k).

A rule is SAFE when, for every pair of groups k < k' and every phase of k'
that can run while k is at the progress the chain of rules guarantees, no
later phase of k writes a cell k' loads (read too early), loads a cell k'
writes (clobbered), or writes a cell k' writes (lost update).

    python tools/v5_rules.py            # search the minimal safe rule for a grid of (c, t, G)
"""
from __future__ import annotations

import itertools
import sys

CANDIDATES = [(2, 3), (2, 4), (3, 4), (4, 5), (4, 6), (5, 6), (6, 7), (6, 8), (7, 8), (8, 9), (8, 10)]


def n_units(n, c, t, G, k):
    r0 = k * G
    first = r0 + c - t
    return 0 if first > n - 2 else (n - 2 - first) // c + 1


def phases(n, c, t, G, k):
    """list of (progress value after the phase, loads, writes) in order; each
    set is a list of rectangles (i0, i1, x0, x1) inclusive."""
    J = n_units(n, c, t, G, k)
    out = []
    W = t + G
    for j in range(J):
        p = k * G + (c - t) + j * c
        q0 = k * G if j == 0 else p - c
        lo = q0 if j == 0 else q0 + W
        out.append((2 * j + 1, [(lo, p + W - 1, p, p + W - 1)], [(q0, p - 1, p, p + W - 1)]))
        xend = p + W + c - 1 if j == J - 1 else p + c - 1
        out.append((2 * j + 2, [(p, p + W - 1, p + W, p + W + c - 1)], [(p, p + W - 1, p, xend)]))
    return out


def rect_hit(n, c, t, a, b):
    i0 = max(a[0], b[0]); i1 = min(a[1], b[1], n - 1)
    x0 = max(a[2], b[2]); x1 = min(a[3], b[3], n - 1)
    if i0 > i1 or x0 > x1:
        return False
    # some cell with -t <= x - i <= c + t
    return x1 - i0 >= -t and x0 - i1 <= c + t


def sets_hit(n, c, t, A, B):
    return any(rect_hit(n, c, t, a, b) for a in A for b in B)


def need_of(h, a0, b0):
    """progress the previous group must have for a phase whose own progress
    value is h (odd: A half of unit (h-1)/2, even: B half of unit h/2 - 1)"""
    if h % 2 == 1:
        return (h - 1) + a0
    return (h - 2) + b0


def need_of_tail(h, a0, b0, Jp, tail_b0=4):
    """need_of with the end-of-predecessor refinement: the B half of unit j
    waits for 2j + b0 while the predecessor's unit j+1 is not its last unit,
    for 2j + tail_b0 otherwise (its last unit writes back the whole H region)"""
    if h % 2 == 1:
        return (h - 1) + a0
    j = h // 2 - 1
    return 2 * j + (b0 if j + 2 < Jp else tail_b0)


def safe(n, c, t, G, a0, b0, dmax=None, kmax=4, tail_b0=None):
    ns = max(0, (n - 2) - (c - t) + 1)
    ng = (ns + G - 1) // G
    if ng < 2:
        return True
    P = [phases(n, c, t, G, k) for k in range(ng)]
    Jk = [len(P[k]) // 2 for k in range(ng)]
    if dmax is None:
        dmax = ng - 1
    for k in range(min(kmax, ng - 1)):
        for d in range(1, min(dmax, ng - 1 - k) + 1):
            kp = k + d
            nf = (lambda hh, Jp: need_of(hh, a0, b0)) if tail_b0 is None else \
                (lambda hh, Jp: need_of_tail(hh, a0, b0, Jp, tail_b0))
            for (h, L, Wr) in P[kp]:
                # guaranteed progress of groups kp-1, ..., k
                g = nf(h, Jk[kp - 1])
                for e in range(1, d):
                    g = min(g, 2 * Jk[kp - e])
                    # group kp-e has progress >= g: it executed the phase with value g
                    g = nf(g, Jk[kp - e - 1])
                g = min(g, 2 * Jk[k])
                for (h2, L2, W2) in P[k]:
                    if h2 <= g:
                        continue
                    if sets_hit(n, c, t, W2, L) or sets_hit(n, c, t, L2, Wr) or sets_hit(n, c, t, W2, Wr):
                        return False
    return True


def minimal_rule(c, t, G, n=None):
    if n is None:
        n = 8 * c + 10 * G + 7
    for a0, b0 in CANDIDATES:
        if all(safe(nn, c, t, G, a0, b0) for nn in (n, n + c // 2 + 1, n + G + 2)):
            return a0, b0
    return None


def closed_rule(c, t, G):
    """The rule bb_api.cu uses (must be >= the brute-force minimal rule)."""
    raise NotImplementedError


def main():
    rows = []
    for c in list(range(3, 33)) + [40, 48, 64, 96, 128]:
        ts = range(1, c) if c <= 32 else (8, 16, 31, 32)
        for t in ts:
            if t >= c:
                continue
            Gs = sorted({1, 2, 3, 4, 8, 16, (c - t) // 2, (c - t) // 3, c - t} & set(range(1, c - t + 1)))
            for G in Gs:
                r = minimal_rule(c, t, G)
                rows.append((c, t, G, r))
                print(c, t, G, r, flush=True)


if __name__ == "__main__":
    sys.exit(main())
