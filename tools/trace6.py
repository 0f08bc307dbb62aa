"""Scratch: timeline of the segment-ring kernel (bb_pass_v6.cuh) from a
BB_TRACE_FILE dump.  Slots: 0 WG0 step j start (before its wait), 1 last WG
step j done, 2 producer chunk j issued (after its waits), 3 writer published
step j."""
import sys
import numpy as np

def read(path):
    with open(path, "rb") as f:
        hdr = np.frombuffer(f.read(24), dtype=np.int32)
        ng, ns, c, t, G, grid = [int(x) for x in hdr]
        tr = np.frombuffer(f.read(), dtype=np.uint64).reshape(ng, ns, 16).astype(np.float64)
    return (ng, ns, c, t, G, grid), tr

def summarize(path):
    (ng, ns, c, t, G, grid), tr = read(path)
    print(f"c={c} t={t} G={G} grid={grid} groups traced={ng} steps={ns}")
    st = tr[:, 0, 0]
    ok = st > 0
    idx = np.nonzero(ok)[0]
    lags = np.diff(st[idx])
    mid = slice(len(lags) // 4, 3 * len(lags) // 4)
    print("  group start lag: median %.2f us mean %.2f (per sweep %.2f)" % (
        np.median(lags[mid]) / 1e3, np.mean(lags[mid]) / 1e3, np.median(lags[mid]) / 1e3 / G))
    k = idx[len(idx) // 2]
    print(f"  group {k}: per step (us, relative to WG0 start of step 0)")
    t0 = tr[k, 0, 0]
    for j in list(range(0, 8)) + list(range(ns // 2, ns // 2 + 4)):
        row = tr[k, j]
        prv = tr[k - 1, j] if k > 0 else row * 0
        print("   j=%4d wg0start %9.2f lastdone %9.2f chunk %9.2f pub %9.2f | prev pub j+1 %9.2f prev chunk %9.2f" % (
            j, (row[0] - t0) / 1e3, (row[1] - t0) / 1e3, (row[2] - t0) / 1e3, (row[3] - t0) / 1e3,
            (tr[k - 1, j + 1, 3] - t0) / 1e3 if k > 0 else 0, (prv[2] - t0) / 1e3))
    # step period of WG0 and last WG in the middle of the sweep
    s0 = np.diff(tr[k, 2:ns - 2, 0])
    s1 = np.diff(tr[k, 2:ns - 2, 1])
    a_wait = tr[k, 2:ns - 4, 4] - tr[k, 2:ns - 4, 0]
    a_half = tr[k, 2:ns - 4, 5] - tr[k, 2:ns - 4, 4]
    b_half = tr[k, 2:ns - 4, 6] - tr[k, 2:ns - 4, 5]
    print("  WG0: A wait %.2f us, A half + B wait %.2f us, B half %.2f us (medians)" % (
        np.median(a_wait) / 1e3, np.median(a_half) / 1e3, np.median(b_half) / 1e3))
    g0 = tr[0, 2:ns - 4]
    print("  group 0 WG0: A wait %.2f, A+Bwait %.2f, B %.2f us" % (np.median(g0[:, 4] - g0[:, 0]) / 1e3,
          np.median(g0[:, 5] - g0[:, 4]) / 1e3, np.median(g0[:, 6] - g0[:, 5]) / 1e3))
    cy = tr[k, 2:ns - 4]
    names = ["A: loads+dot+scalars+update (refl_apply)", "A: store row", "A: barrier", "B: ...refl_apply", "B: store col", "B: barrier"]
    pairs = [(8, 9), (9, 10), (10, 11), (12, 13), (13, 14), (14, 15)]
    for nm, (a0, a1) in zip(names, pairs):
        print("  cycles %-42s %7.0f" % (nm, np.median(cy[:, a1] - cy[:, a0])))
    print("  cycles A-post..B-start (incl. B wait) %7.0f" % np.median(cy[:, 12] - cy[:, 11]))
    d1 = tr[k, 2:ns - 6, 7] - tr[k, 3:ns - 5, 6]
    print("  WG1 A(j) start (after wait) - WG0 step j+1 end: median %.2f us" % (np.median(d1) / 1e3))
    print("  WG1 A(j) start - WG0 A(j) start: median %.2f us" % (np.median(tr[k, 2:ns - 6, 7] - tr[k, 2:ns - 6, 4]) / 1e3))
    print("  WG0 step period median %.2f us, last-WG step period %.2f us" % (np.median(s0) / 1e3, np.median(s1) / 1e3))
    print("  last WG done(j) - WG0 start(j): median %.2f us" % (np.median(tr[k, 2:ns - 4, 1] - tr[k, 2:ns - 4, 0]) / 1e3))
    print("  pub(j) - lastdone(j): median %.2f us" % (np.median(tr[k, 2:ns - 4, 3] - tr[k, 2:ns - 4, 1]) / 1e3))
    print("  chunk(j) issue (next group) - pub(j+1) (this group): median %.2f us" % (
        np.median(tr[k + 1, 2:ns - 4, 2] - tr[k, 3:ns - 3, 3]) / 1e3))
    print("  WG0 start(j) (next group) - chunk(j) issue: median %.2f us" % (
        np.median(tr[k + 1, 2:ns - 4, 0] - tr[k + 1, 2:ns - 4, 2]) / 1e3))

if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarize(p)


def dump(path, k=None, j0=None, nj=8):
    (ng, ns, c, t, G, grid), tr = read(path)
    k = k if k is not None else ng // 2
    j0 = j0 if j0 is not None else ns // 2
    t0 = tr[k, j0, 0]
    print("   j   WG0:start  Await-done  Bwait-done  stepend | WG1 Await-done | lastdone  pub")
    for j in range(j0, j0 + nj):
        r = (tr[k, j] - t0) / 1e3
        print("%5d %9.2f %9.2f %9.2f %9.2f | %9.2f | %9.2f %9.2f" % (j, r[0], r[4], r[5], r[6], r[7], r[1], r[3]))


def periods(path):
    (ng, ns, c, t, G, grid), tr = read(path)
    out = []
    for k in [0, 1, 2, 3, 5, 10, 20, 50, 100, 200, 500, 1000, 2000, 3000, 4000]:
        if k >= ng:
            break
        valid = np.nonzero(tr[k, :, 0] > 0)[0]
        if len(valid) < 16:
            continue
        J = valid[-1] + 1
        s0 = tr[k, 2:J - 4, 0]
        per = np.median(np.diff(s0)) / 1e3
        bw = np.median(tr[k, 2:J - 4, 5] - tr[k, 2:J - 4, 4]) / 1e3
        out.append((k, per, bw))
        print("group %5d: WG0 step period %.2f us, A+Bwait %.2f us" % (k, per, bw))
    return out


def crossgroup(path, k=2048, j0=400, nj=200):
    """Where WG0 of group k waits at B(j) (chunk j+1): the previous group's last
    WG finishing step j+2, its writer publishing, our producer issuing, the TMA
    landing -- medians over steps j0 .. j0+nj (absolute times, same clock)."""
    (ng, ns, c, t, G, grid), tr = read(path)
    rows = []
    for j in range(j0, j0 + nj):
        bstart = tr[k, j, 4]        # WG0 A wait done (A half starts)
        bdone = tr[k, j, 5]         # WG0 B wait done
        last = tr[k - 1, j + 2, 1]  # previous group's last WG finished step j+2
        pub = tr[k - 1, j + 2, 3]   # its writer published step j+2 (0 if batched into a later round)
        iss = tr[k, j + 1, 2]       # our producer issued chunk j+1
        if min(bstart, bdone, last, iss) <= 0:
            continue
        rows.append((bdone - bstart, last - bstart, (pub - last) if pub > 0 else np.nan, iss - last, bdone - iss))
    a = np.array(rows) / 1e3
    names = ["B wait (A start -> B wait done)", "prev last done(j+2) - A start", "pub - prev last done",
             "producer issue(j+1) - prev last done", "B wait done - issue (TMA + poll)"]
    print(f"crossgroup k={k} G={G}: {len(rows)} steps")
    for i, nm in enumerate(names):
        print("  %-40s median %7.2f us  mean %7.2f" % (nm, np.nanmedian(a[:, i]), np.nanmean(a[:, i])))


def ring(path, k=2048, j0=300, nj=400):
    """Ring-latency probes (BB_TRACE_RING=1; clock64 of the group's SM, cycles):
    last WG finished step m (13) -> writer saw it (8) -> slot freed after the
    store read it (9) -> producer saw the free slot for chunk m+R (10) -> load
    issued after the previous-group wait (11) -> WG0 past its B wait of step
    m+R-1, i.e. chunk m+R usable (12)."""
    (ng, ns, c, t, G, grid), tr = read(path)
    R = None
    # infer R: the smallest r with producer slot-free(m + r) >= slot freed(m) for most m
    rows = {}
    for r in range(2 * G + 1, 40):
        d = tr[k, j0 + r: j0 + nj + r, 10] - tr[k, j0: j0 + nj, 9]
        if np.median(d) > 0:
            R = r
            break
    print(f"ring k={k} G={G} R~{R}")
    if R is None:
        return
    m = np.arange(j0, j0 + nj)
    s = tr[k]
    parts = [("last WG done -> writer saw", s[m, 8] - s[m, 13]),
             ("writer saw -> slot freed (store read)", s[m, 9] - s[m, 8]),
             ("slot freed -> producer saw (chunk m+R)", s[m + R, 10] - s[m, 9]),
             ("producer saw -> load issued (prev wait)", s[m + R, 11] - s[m + R, 10]),
             ("load issued -> WG0 past B wait (j=m+R-1)", s[m + R - 1, 12] - s[m + R, 11]),
             ("last WG done(m) -> WG0 past B wait(m+R-1)", s[m + R - 1, 12] - s[m, 13])]
    for nm, d in parts:
        print("  %-44s median %8.0f cycles  mean %8.0f" % (nm, np.median(d), np.mean(d)))
