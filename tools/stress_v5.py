import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2510_12705_b200 as bb
from tests.gpu_util import gpu_reduce
cases = [("f64", 300, 64, 16), ("f64", 1500, 128, 32), ("f32", 1333, 96, 32), ("f64", 2000, 64, 16)]
for no_unit in (False, True):
    for dtype, n, b, tw in cases:
        band = synth.random_band(n, b, dtype, seed=50)
        cfg = bb.Config(tw=tw, no_unit=no_unit)
        ref = None; diffs = 0; nans = 0
        for it in range(30):
            d, e = gpu_reduce(band, b, cfg=cfg)
            nans += int((~np.isfinite(d)).sum() + (~np.isfinite(e)).sum() > 0)
            if ref is None: ref = (d, e)
            elif not (np.array_equal(ref[0], d) and np.array_equal(ref[1], e)): diffs += 1
        print(f"no_unit={no_unit} {dtype} n={n} b={b} tw={tw}: runs with nan {nans}/30, differing from first {diffs}/29", flush=True)
