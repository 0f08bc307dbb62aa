"""Ad-hoc GPU diagnostics: run a grid of (n, b, dtype, tw, schedule) and print errors vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2510_12705_b200 as bb
from tests.gpu_util import gpu_reduce

cases = [(1024, 32, "f32", 32), (1024, 32, "f32", 16), (1024, 32, "f64", 31), (200, 32, "f32", 31),
         (200, 32, "f64", 31), (200, 8, "f32", 7), (200, 8, "f32", 4), (100, 4, "f32", 3)]
for (n, b, dt, tw) in cases:
    band = synth.random_band(n, b, dt, seed=1)
    for sched in (bb.BB_SCHED_FLAGS, bb.BB_SCHED_CYCLE):
        d, e = gpu_reduce(band, b, cfg=bb.Config(tw=tw, schedule=sched))
        d0, e0 = oracle.band_to_bidiag(band, b, tw)
        nn = int(np.isnan(d).sum() + np.isnan(e).sum())
        err = np.nanmax(np.abs(np.abs(d) - np.abs(d0)))
        first = int(np.argmax(np.isnan(d))) if nn else -1
        print(n, b, dt, tw, sched, "nan", nn, "first", first, "err", err, flush=True)
