"""Matrix-end check: GPU d/e vs oracle for several n (incl. powers of two), kernels v4 / v2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle, paper_2510_12705_b200 as bb
for n, b, dt, tw in [(1024, 128, "f64", 32), (1025, 128, "f64", 32), (1056, 128, "f64", 32), (2048, 128, "f64", 32),
                     (1024, 32, "f64", 31), (1024, 64, "f64", 32), (1024, 128, "f64", 16)]:
    band = synth.random_band(n, b, dt, seed=0)
    d0, e0 = oracle.band_to_bidiag(band, b, tw)
    for G in ("4", "1", "0"):
        os.environ["BB_V4_G"] = G
        d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, tw=tw)
        d = d.double().cpu().numpy(); e = e.double().cpu().numpy()
        bad_d = np.where(np.abs(np.abs(d) - np.abs(d0)) > 1e-8 * max(1, np.abs(d0).max()))[0]
        bad_e = np.where(np.abs(np.abs(e) - np.abs(e0)) > 1e-8 * max(1, np.abs(e0).max()))[0]
        print(n, b, tw, "G", G, "bad d", bad_d[:8], len(bad_d), "bad e", bad_e[:8], len(bad_e),
              "d[-3:]", d[-3:], "oracle", d0[-3:], flush=True)
