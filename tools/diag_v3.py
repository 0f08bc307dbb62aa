"""Debug the multi-sweep kernel: compare against the oracle per case, with v3 on/off."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2510_12705_b200 as bb

def run(n, b, tw, dt, G):
    os.environ["BB_V3_G"] = str(G)
    band = synth.random_band(n, b, dt, seed=1)
    ws = bb.Workspace(n, b, dt, 1, tw=tw)
    t = torch.from_numpy(band).cuda()
    d, e = bb.band_to_bidiag(t, b, workspace=ws); torch.cuda.synchronize()
    W = ws.band_view()[0].double().cpu().numpy(); ku = ws.stats["ku"]
    d0, e0, st = oracle.band_to_bidiag(band, b, tw, store=True)
    d = d.double().cpu().numpy()
    err = np.max(np.abs(np.abs(d) - np.abs(d0)))
    nan = int(np.isnan(d).sum())
    # zeros check: which off-band cells are nonzero
    mask = np.ones_like(W, dtype=bool); mask[:, ku] = False; mask[1:, ku - 1] = False
    nz = np.argwhere((W != 0) & mask)
    return err, nan, nz[:6].tolist(), len(nz)

for (n, b, tw, dt) in [(64, 8, 1, "f64"), (64, 8, 4, "f64"), (1024, 32, 16, "f32"), (1024, 32, 16, "f64"), (300, 24, 4, "f64")]:
    for G in (1, 3):
        err, nan, nz, nnz = run(n, b, tw, dt, G)
        print(f"n={n} b={b} tw={tw} {dt} G={G}: err {err:.3e} nan {nan} nonzero-offband {nnz} {nz}", flush=True)
