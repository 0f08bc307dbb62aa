"""For the multi-sweep kernel (bb_pass_v3.cuh): which cells of a group's slots are
last modified (within the group) by a WG other than the last one?  Those cells
are not written through by the last WG and must be written back when the slot
is retired.  Prints them relative to the slot origin (p0)."""
import sys
from collections import defaultdict


def geo(n, c, t, r, j):
    p = r + (c - t) + j * c
    if p > n - 2:
        return None
    q = r if j == 0 else p - c
    hi = min(p + t, n - 1)
    ce = min(hi + c, n - 1)
    return q, p, hi, ce


def cells(g):
    q, p, hi, ce = g
    s = set()
    for i in range(q, hi + 1):
        for jj in range(p, hi + 1):
            s.add((i, jj))
    for i in range(p, hi + 1):
        for jj in range(p, ce + 1):
            s.add((i, jj))
    return s


def check(n, c, t, G, r0):
    last = {}
    for g in range(G):          # sequential order: sweep r0+g after r0+g-1
        r = r0 + g
        j = 0
        while geo(n, c, t, r, j):
            for x in cells(geo(n, c, t, r, j)):
                last[x] = g
            j += 1
    bad = defaultdict(list)
    for x, g in last.items():
        if g != G - 1:
            # which slot's home holds x? slot j such that p0_j <= col < p0_{j+1} roughly
            i, jc = x
            j = max(0, (jc - r0 - (c - t)) // c) if jc >= r0 + (c - t) else 0
            p0 = r0 + (c - t) + j * c
            bad[j].append((i - p0, jc - p0))
    return bad


if __name__ == "__main__":
    n, c, t, G = 600, int(sys.argv[1]) if len(sys.argv) > 1 else 24, int(sys.argv[2]) if len(sys.argv) > 2 else 6, \
        int(sys.argv[3]) if len(sys.argv) > 3 else 3
    r0 = 60
    bad = check(n, c, t, G, r0)
    WT = t + G
    for j in sorted(bad)[:4]:
        pts = bad[j]
        rows = sorted(set(a for a, b in pts)); cols = sorted(set(b for a, b in pts))
        # classify: T-rect columns [0, WT) vs W-rect [WT, c+WT)
        tcols = sorted(set(b for a, b in pts if b < WT)); wrows = sorted(set(a for a, b in pts if b >= WT))
        print(f"slot {j}: {len(pts)} cells; rows {rows[0]}..{rows[-1]}; T-part cols {tcols[:8]}{'...' if len(tcols)>8 else ''}; "
              f"W-part rows {wrows}")
        # verify strips: T-part cols < G-1, W-part rows < G-1 (relative to p0), plus slot-(j-1) region
        outside = [(a, b) for a, b in pts if not ((b < G - 1) or (b >= WT and a < G - 1) or (a < 0))]
        print("   cells outside the strips:", outside[:10], len(outside))


def detail(c, t, G):
    n, r0 = 800, 80
    bad = check(n, c, t, G, r0)
    WT = t + G
    pts = bad[sorted(bad)[2]]
    # region T-home of slot j: rows >= (q0 + WT) - p0 = WT - c, cols [0, WT)
    th = [(a, b) for a, b in pts if b < WT and a >= WT - c]
    # region slot(j-1).W home: rows [-c, WT - c), cols [0, WT)  (top rows of T columns)
    pw = [(a, b) for a, b in pts if b < WT and a < WT - c]
    wh = [(a, b) for a, b in pts if b >= WT]
    print(f"c={c} t={t} G={G}: T-home cells {len(th)} cols {sorted(set(b for a,b in th))} rows {min(a for a,b in th) if th else None}..{max(a for a,b in th) if th else None}")
    print(f"   prev-W cells {len(pw)} rows {sorted(set(a for a,b in pw))} cols {sorted(set(b for a,b in pw))}")
    print(f"   W-home cells {len(wh)} rows {sorted(set(a for a,b in wh))} cols {min(b for a,b in wh) if wh else None}..{max(b for a,b in wh) if wh else None}")


def writer_cells(n, c, t, G, r0, j, ldt):
    """Cells the RELEASE/WRITER warp writes back for slot j (mirror of the kernel)."""
    WT = t + G
    p0 = r0 + (c - t) + j * c
    q0 = p0 - c if j else r0
    trow0 = q0 + WT if j else r0
    out = set()
    for k in range(G - 1):
        for ii in range(ldt):
            i, jc = trow0 + ii, p0 + k
            if i < n and jc < n and jc - i >= -t:
                out.add((i, jc))
    if j == 0:
        for k in range(WT):
            for ii in range(G - 1):
                i, jc = trow0 + ii, p0 + k
                if i < n and jc < n and jc - i >= -t:
                    out.add((i, jc))
    for k in range(c):
        for ii in range(G - 1):
            i, jc = p0 + ii, p0 + WT + k
            if i < n and jc < n and jc - i <= c + t:
                out.add((i, jc))
    return out


def verify(n, c, t, G, r0):
    """every cell last modified by a WG other than the last one is written back"""
    last = {}
    glast = min(G, n) - 1
    for g in range(G):
        j = 0
        while geo(n, c, t, r0 + g, j):
            for x in cells(geo(n, c, t, r0 + g, j)):
                last[x] = g
            j += 1
    J0 = 0
    while geo(n, c, t, r0, J0):
        J0 += 1
    W = set()
    for j in range(J0):
        W |= writer_cells(n, c, t, G, r0, j, c + G + (c + G + 1) % 2)
    missing = [x for x, g in last.items() if g != G - 1 and x not in W]
    extra_glast = [x for x, g in last.items() if g == G - 1 and x in W]
    return missing, extra_glast


if __name__ == "__main__" and len(sys.argv) > 4:
    pass
