#!/usr/bin/env python
"""Executable model of the segment-ring kernel's protocol (bb_pass_v6.cuh)
for the target-bandwidth-1 pass: every group's producer / warp-groups /
writer as actors with exactly the kernel's enabling conditions, run under a
random scheduler over all groups at once.  Each half-step reads its footprint
from its CTA's ring and checks that every cell holds the version the
SEQUENTIAL order (the oracle's) would give it -- so any missing chunk, stale
copy, early reuse of a ring slot, or write-back that races a later reader is
caught.  Used by tests/test_v6_protocol.py.

Cells carry versions (the id of the last half-step that touched them), not
values: the protocol is about which copy is read when, not about arithmetic.
"""
from __future__ import annotations

import numpy as np


def sweep_len(n, c, t, r):
    first = r + c - t
    return 0 if first > n - 2 else (n - 2 - first) // c + 1


def footprint(n, c, t, r, j, half):
    p = r + (c - t) + j * c
    q = r if j == 0 else p - c
    hi = min(p + t, n - 1)
    ce = min(hi + c, n - 1)
    if half == 0:   # A: row reflector from row q over cols [p, hi], applied to rows q+1..hi
        rows, cols = range(q, hi + 1), range(p, hi + 1)
    else:           # B: column reflector from col p over rows [p, hi], applied to cols p+1..ce
        rows, cols = range(p, hi + 1), range(p, ce + 1)
    return [(i, x) for i in rows for x in cols if -t <= x - i <= c + t]


def run(n, c, G, R, seed=0, steps_limit=10 ** 7, load_need=4, a_need=4, b_need=5, write_lag=0):
    """load_need / a_need / b_need / write_lag: the kernel's rules (4, 4, 5, 0);
    other values are mutations the tests expect to be caught."""
    t = c - 1
    rng = np.random.default_rng(seed)
    ns = max(0, (n - 2) - (c - t) + 1)
    # sequential order: expected input versions of every half-step
    seq = {}
    hid = {}
    cur = {}
    h = 0
    for r in range(ns):
        for j in range(sweep_len(n, c, t, r)):
            for half in (0, 1):
                fp = footprint(n, c, t, r, j, half)
                seq[(r, j, half)] = {cell: cur.get(cell, -1) for cell in fp}
                for cell in fp:
                    cur[cell] = h
                hid[(r, j, half)] = h
                h += 1
    final = dict(cur)
    glob = {}            # global band: cell -> version (missing = initial, -1)
    ngroups = (ns + G - 1) // G
    gprog = [0] * ngroups

    class Grp:
        pass

    groups = []
    for k in range(ngroups):
        g = Grp()
        g.k, g.r0 = k, k * G
        g.glast = min(G, ns - g.r0) - 1
        g.M = (n - 1 - (g.r0 + 1)) // c + 1 if g.r0 + 1 <= n - 1 else 0
        g.J = [sweep_len(n, c, t, g.r0 + i) for i in range(g.glast + 1)]
        g.prog = [0] * (g.glast + 1)
        g.loaded = 0        # chunks loaded (in order)
        g.wb = 0            # chunks written back
        g.wj = 0            # writer's next step
        g.done = False
        g.ring = {}         # cell -> version (copies of the loaded chunks)
        g.slot = {}         # chunk index -> cells in the ring
        groups.append(g)

    def cols_of(g, m):
        x0 = g.r0 + 1 + m * c
        return range(x0, min(x0 + c, n))

    def cells_of_cols(cols):
        return [(i, x) for x in cols for i in range(x - c - t, x + t + 1) if 0 <= i < n]

    def actions(g):
        acts = []
        k = g.k
        # producer
        m = g.loaded
        if m < g.M and (m < R or g.wb >= m - R + 1):
            Jp = sweep_len(n, c, t, g.r0 - 1) if k > 0 else 0
            if k == 0 or gprog[k - 1] >= min(2 * m + load_need, 2 * Jp):
                acts.append(("load", m))
        # warp-groups
        for gi in range(g.glast + 1):
            r = g.r0 + gi
            pr = g.prog[gi]
            if pr >= 2 * g.J[gi]:
                continue
            j, half = pr // 2, pr % 2
            if gi == 0:
                need_chunk = j if half == 0 else j + 1
                ok = (need_chunk < g.loaded) or (half == 1 and g.r0 + 1 + (j + 1) * c > n - 1)
            else:
                Jprev = g.J[gi - 1]
                need = min(2 * j + (a_need if half == 0 else b_need), 2 * Jprev)
                ok = g.prog[gi - 1] >= need
            if ok:
                acts.append(("step", gi, j, half))
        # writer
        Js = g.J[g.glast]
        if g.wj < Js - 1:
            if g.prog[g.glast] >= 2 * (g.wj - write_lag) + 2:
                acts.append(("write", g.wj))
        elif not g.done and all(g.prog[gi] >= 2 * g.J[gi] for gi in range(g.glast + 1)):
            acts.append(("flush",))
        return acts

    def do(g, a):
        if a[0] == "load":
            m = a[1]
            old = m - R
            if old >= 0:
                assert old < g.wb, ("slot reused before write-back", g.k, m)
                for cell in g.slot.pop(old, []):
                    g.ring.pop(cell, None)
            cells = cells_of_cols(cols_of(g, m))
            for cell in cells:
                g.ring[cell] = glob.get(cell, -1)
            g.slot[m] = cells
            g.loaded += 1
        elif a[0] == "step":
            _, gi, j, half = a
            r = g.r0 + gi
            exp = seq[(r, j, half)]
            for cell, v in exp.items():
                assert cell in g.ring, ("cell not in the ring", g.k, r, j, half, cell)
                assert g.ring[cell] == v, ("stale copy", g.k, r, j, half, cell, g.ring[cell], v)
            me = hid[(r, j, half)]
            for cell in exp:
                g.ring[cell] = me
            g.prog[gi] += 1
        elif a[0] == "write":
            j = a[1]
            if j < g.M:
                assert j in g.slot, ("write-back of a chunk not loaded", g.k, j)
                for cell in g.slot[j]:
                    glob[cell] = g.ring[cell]
                g.wb = j + 1
            gprog[g.k] = 2 * j + 2
            g.wj += 1
        else:  # flush
            for m in range(g.wb, g.M):
                for cell in g.slot.get(m, []):
                    glob[cell] = g.ring[cell]
            g.wb = g.M
            gprog[g.k] = 2 * g.J[g.glast]
            g.done = True

    nstep = 0
    while True:
        cand = [(g, a) for g in groups if not g.done for a in actions(g)]
        if not cand:
            break
        g, a = cand[rng.integers(len(cand))]
        do(g, a)
        nstep += 1
        assert nstep < steps_limit
    assert all(g.done for g in groups), "deadlock: " + str([(g.k, g.prog, g.loaded, g.wb) for g in groups if not g.done])
    for cell, v in final.items():
        assert glob.get(cell, -1) == v, ("final global version", cell, glob.get(cell, -1), v)
    return nstep


if __name__ == "__main__":
    for (n, c, G, R) in [(70, 4, 3, 7), (90, 8, 4, 9), (131, 8, 5, 12), (100, 16, 4, 9)]:
        for s in range(3):
            print(n, c, G, R, s, run(n, c, G, R, seed=s))
