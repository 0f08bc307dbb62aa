"""Scratch: per-phase durations of the unit kernel from BB_TRACE_FILE dumps."""
import os, sys
import numpy as np
def read(path):
    with open(path, "rb") as f:
        hdr = np.frombuffer(f.read(24), dtype=np.int32)
        ng, nu, c, t, G, grid = [int(x) for x in hdr]
        tr = np.frombuffer(f.read(), dtype=np.uint64).reshape(ng, nu, 16).astype(np.float64)
    return (ng, nu, c, t, G, grid), tr
def summarize(path):
    (ng, nu, c, t, G, grid), tr = read(path)
    names = ["A-wait", "V-load", "A-panel", "A-bulk", "WA+pub", "B-wait", "H-load", "B-panel", "B-bulk", "WB+pub"]
    valid = (tr[:, :, 0] > 0) & (tr[:, :, 10] > 0)
    # skip early/late groups: use the middle
    sel = valid.copy(); sel[: ng // 4] = False; sel[3 * ng // 4:] = False
    print(f"c={c} t={t} G={G} grid={grid} groups traced={ng} units={nu}")
    tot = tr[:, :, 10] - tr[:, :, 0]
    print("  unit total (us): median %.2f mean %.2f" % (np.median(tot[sel]) / 1e3, np.mean(tot[sel]) / 1e3))
    for s in range(10):
        dur = tr[:, :, s + 1] - tr[:, :, s]
        print(f"  {names[s]:8s} median {np.median(dur[sel])/1e3:7.2f} us  mean {np.mean(dur[sel])/1e3:7.2f}")
    # group start lag
    st = tr[:, 0, 0]
    ok = st > 0
    lags = np.diff(st[ok])
    print("  group start lag median %.2f us" % (np.median(lags) / 1e3))
    # next-unit gap (end of unit j to start of j+1)
    gap = tr[:, 1:, 0] - tr[:, :-1, 10]
    v2 = valid[:, 1:] & valid[:, :-1] & sel[:, 1:]
    print("  carry gap median %.2f us" % (np.median(gap[v2]) / 1e3))
if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarize(p)


def wa_cycles(path):
    """Cycle breakdown of the A write-back + publish (slots 11-15, clock64 of
    thread 32): own stores issued, all warps' stores issued (barrier), fence,
    release store."""
    (ng, nu, c, t, G, grid), tr = read(path)
    sl = tr[ng // 4: 3 * ng // 4, 2: nu - 2]
    ok = (sl[:, :, 11] > 0) & (sl[:, :, 15] > 0)
    for nm, a0, a1 in (("stores issued (own)", 11, 12), ("barrier (all warps issued)", 12, 13),
                       ("fence.acq_rel.gpu", 13, 14), ("st.release.gpu", 14, 15)):
        d = (sl[:, :, a1] - sl[:, :, a0])[ok]
        print("  WA %-28s median %8.0f cycles  mean %8.0f" % (nm, np.median(d), np.mean(d)))
