import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_2510_12705_b200 as bb
from tests.gpu_util import gpu_reduce
dt = sys.argv[1] if len(sys.argv) > 1 else "f64"
band = synth.random_band(300, 64, dt, seed=60)
for flags in (dict(no_segment=True), dict()):
    d, e = gpu_reduce(band, 64, cfg=bb.Config(tw=32, **flags))
    print(flags, d[:3], flush=True)
