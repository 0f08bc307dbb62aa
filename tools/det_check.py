"""Scratch: run-to-run determinism of a configuration (bitwise)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2510_12705_b200 as bb
from tests.gpu_util import compare
for dt, n, b, tw in (("f32", 2049, 64, 16), ("f64", 2049, 64, 16), ("f32", 2049, 64, 32), ("f32", 1500, 64, 16)):
    band = synth.random_band(n, b, dt, seed=77)
    tb = torch.from_numpy(band).cuda()
    outs = []
    for rep in range(6):
        d, e = bb.band_to_bidiag(tb, b, tw=tw)
        torch.cuda.synchronize()
        outs.append((d.double().cpu().numpy(), e.double().cpu().numpy()))
    same = all(np.array_equal(outs[0][0], o[0]) and np.array_equal(outs[0][1], o[1]) for o in outs)
    errs = compare(band, b, tw, dt, outs[0][0], outs[0][1], svals=False)
    print(dt, n, b, tw, "deterministic" if same else "NONDETERMINISTIC", errs, flush=True)
    for G in ("8", "16"):
        os.environ["BB_V5_G"] = G
        d, e = bb.band_to_bidiag(tb, b, tw=tw); torch.cuda.synchronize()
        print("  G5", G, np.array_equal(d.double().cpu().numpy(), outs[0][0]))
    os.environ.pop("BB_V5_G")
    for flag in (dict(no_unit=True), dict(no_segment=True)):
        d, e = bb.band_to_bidiag(tb, b, cfg=bb.Config(tw=tw, **flag)); torch.cuda.synchronize()
        print("  ", flag, "bitwise vs default:", np.array_equal(d.double().cpu().numpy(), outs[0][0]))
