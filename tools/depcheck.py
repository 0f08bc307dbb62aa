"""Phase-level dependency checker for wavefront schedules (host-side analysis).

A step (r, j) of pass (c, t) is split into phase A (row reflector + right
application: cells rows q..hi x cols p..hi) and phase B (column reflector +
left application: rows p..hi x cols p..ce).  A schedule rule says which
progress value of sweep r-1 each phase waits for (progress counts completed
phases: 2j+1 after A(j), 2j+2 after B(j)).  The rule is VALID iff every pair
of phases with intersecting cell sets is ordered (transitively) the same way
as in sequential order -- then any execution admitted by the rule is bitwise
equal to the sequential oracle.
"""
import sys


def geometry(n, c, t, r, j):
    p = r + (c - t) + j * c
    if p > n - 2:
        return None
    q = r if j == 0 else p - c
    hi = min(p + t, n - 1)
    ce = min(hi + c, n - 1)
    return q, p, hi, ce


def cells_A(g):
    q, p, hi, ce = g
    return {(i, jj) for i in range(q, hi + 1) for jj in range(p, hi + 1)}


def cells_B(g):
    q, p, hi, ce = g
    return {(i, jj) for i in range(p, hi + 1) for jj in range(p, ce + 1)}


def check(n, c, t, need_A, need_B=None):
    """need_A(j, Jprev) / need_B(j, Jprev): progress of sweep r-1 that phase A / B
    of step j waits for (None: no extra wait).  Returns the number of violations."""
    J = []
    r = 0
    while True:
        k = 0
        while geometry(n, c, t, r, k) is not None:
            k += 1
        if k == 0:
            break
        J.append(k)
        r += 1
    nodes = []          # (r, phase) in sequential order; phase 2j = A(j), 2j+1 = B(j)
    index = {}
    for r in range(len(J)):
        for ph in range(2 * J[r]):
            index[(r, ph)] = len(nodes)
            nodes.append((r, ph))
    N = len(nodes)
    preds = [[] for _ in range(N)]
    for (r, ph), x in index.items():
        if ph > 0:
            preds[x].append(index[(r, ph - 1)])
        if r > 0:
            j = ph // 2
            f = need_A if ph % 2 == 0 else need_B
            if f is None:
                continue
            v = f(j, J[r - 1])
            v = min(v, 2 * J[r - 1])
            if v > 0:
                preds[x].append(index[(r - 1, v - 1)])
    reach = [0] * N       # bitset of ancestors
    for x in range(N):
        m = 0
        for y in preds[x]:
            m |= reach[y] | (1 << y)
        reach[x] = m
    cells = []
    for (r, ph) in nodes:
        g = geometry(n, c, t, r, ph // 2)
        cells.append(cells_A(g) if ph % 2 == 0 else cells_B(g))
    # only nearby sweeps can conflict; footprints of sweep r lie in rows >= r
    bad = 0
    for y in range(N):
        ry = nodes[y][0]
        for x in range(y):
            rx = nodes[x][0]
            if rx == ry or ry - rx > 3:
                continue
            if cells[x] & cells[y] and not (reach[y] >> x) & 1:
                bad += 1
    return bad


RULES = {
    # whole-step dependency distance s: step (r, j) waits for step j+s-1 of r-1 complete
    "s2": (lambda j, J: 2 * (j + 2), None),
    "s3": (lambda j, J: 2 * (j + 3), None),
    "s1": (lambda j, J: 2 * (j + 1), None),
    # R2: step (r, j) waits until phase A of (r-1, j+1) is done
    "R2": (lambda j, J: 2 * (j + 1) + 1, None),
    # R2b: A(r, j) waits for (r-1, j) complete; B(r, j) waits for A(r-1, j+1)
    "R2b": (lambda j, J: 2 * j + 2, lambda j, J: 2 * (j + 1) + 1),
    # R2c: step waits for (r-1, j) complete only (too weak?)
    "R2c": (lambda j, J: 2 * j + 2, None),
}

if __name__ == "__main__":
    cases = [(40, 4, 2), (40, 6, 2), (50, 8, 3), (60, 12, 5), (45, 10, 4), (40, 4, 3), (30, 6, 5), (64, 16, 4),
             (41, 9, 7), (37, 7, 3)]
    for name, (fa, fb) in RULES.items():
        res = [(n, c, t, check(n, c, t, fa, fb)) for (n, c, t) in cases]
        print(name, [(c, t, "TBW1" if c - t == 1 else "", v) for (n, c, t, v) in res])
