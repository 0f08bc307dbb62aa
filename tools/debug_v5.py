"""Scratch: locate differences between the GPU working band after the first
k passes and the oracle's state after the same passes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth, oracle
import paper_2510_12705_b200 as bb

def oracle_after(band, b, tw, npasses):
    o = oracle.Oracle(band, b, tw)
    n = band.shape[0]
    for ps in oracle.passes(n, b, tw)[:npasses]:
        for r in range(n - 1):
            J = oracle.sweep_len(n, ps.c, ps.t, r)
            for j in range(J):
                o.step(ps.c, ps.t, r, j)
    d, e, st = o.extract(store=True)
    o.close()
    return st   # st[i, (j - i) + tw] = A[i, j]

def gpu_after(band, b, tw, npasses, dtype):
    os.environ["BB_DEBUG_PASSES"] = str(npasses)
    n = band.shape[0]
    cfg = bb.Config(tw=tw)
    ws = bb.Workspace(n, b, dtype, 1, cfg=cfg)
    d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=ws)
    torch.cuda.synchronize()
    del os.environ["BB_DEBUG_PASSES"]
    W = ws.band_view()[0].double().cpu().numpy()   # W[j, ku + i - j] = A(i, j)
    return W, ws.stats["ku"]

for (n, b, tw, dtype) in [(1333, 96, 32, "f32"), (400, 96, 32, "f32"), (400, 96, 32, "f64")]:
    band = synth.random_band(n, b, dtype, seed=50)
    for npasses in (1, 2, 3):
        st = oracle_after(band, b, tw, npasses)
        W, ku = gpu_after(band, b, tw, npasses, dtype)
        bad = []
        maxerr = 0.0
        for x in range(n):
            for i in range(max(0, x - b - tw), min(n, x + tw + 1)):
                off = x - i
                g = W[x, ku + i - x]
                o = st[i, off + tw] if -tw <= off <= b + tw else 0.0
                if not np.isfinite(g) or abs(g - o) > (1e-8 if dtype == "f64" else 1e-3) * (1 + abs(o)):
                    bad.append((i, x, g, o))
                elif np.isfinite(g):
                    maxerr = max(maxerr, abs(g - o))
        print(f"n={n} b={b} tw={tw} passes={npasses}: {len(bad)} bad cells, max err ok-cells {maxerr:.2e}", flush=True)
        for (i, x, g, o) in bad[:12]:
            print("   ", i, x, "off", x - i, "gpu", g, "oracle", o)
