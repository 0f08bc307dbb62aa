"""Scratch GPU check of the segment-ring kernel (bb_pass_v6.cuh): oracle
comparisons at small n, bitwise equality with the one-sweep-per-CTA kernel,
group-size sweep, headline timings per pass."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2510_12705_b200 as bb
from tests.gpu_util import compare, gpu_reduce
from tools.quick_v5 import time_cfg

def small():
    for dtype, n, b, tw in [("f64", 300, 64, 32), ("f64", 1500, 128, 32), ("f32", 1333, 96, 32), ("f16", 900, 64, 32),
                            ("f64", 1200, 64, 16), ("f32", 777, 40, 16), ("f64", 70, 32, 32), ("f64", 2000, 32, 32)]:
        band = synth.random_band(n, b, dtype, seed=60)
        t0 = time.time()
        d, e = gpu_reduce(band, b, tw=tw)
        d4, e4 = gpu_reduce(band, b, cfg=bb.Config(tw=tw, no_segment=True))
        same = np.array_equal(d, d4) and np.array_equal(e, e4)
        errs = compare(band, b, tw, dtype, d, e, svals=(dtype != "f16"))
        print("small", dtype, n, b, tw, "bitwise-vs-v4", same, errs, "%.2fs" % (time.time() - t0), flush=True)
        for G in ("1", "2", "3"):
            os.environ["BB_V6_G"] = G
            dg, eg = gpu_reduce(band, b, tw=tw)
            del os.environ["BB_V6_G"]
            print("   G", G, np.array_equal(d, dg) and np.array_equal(e, eg), flush=True)

if __name__ == "__main__":
    small()
    from tests.golden_util import load, errors, tol
    for G in (2, 3, 4, 5, 6):
        os.environ["BB_V6_G"] = str(G)
        print("BB_V6_G", G)
        time_cfg(32768, 128, "f64", 32)
        del os.environ["BB_V6_G"]
    d, e = time_cfg(32768, 128, "f64", 32)
    g = load("c4_n32768_b128_f64_s0_m0")
    print("golden f64", {k: v / g["fro"] for k, v in errors(g, d, e).items()}, "tol", tol("f64", 32768), flush=True)
    d, e = time_cfg(32768, 128, "f32", 32)
    g = load("c4_n32768_b128_f32_s0_m0")
    print("golden f32", {k: v / g["fro"] for k, v in errors(g, d, e).items()}, flush=True)
    time_cfg(32768, 128, "f64", 16)
    time_cfg(32768, 128, "f32", 16)
    time_cfg(8192, 64, "f64", 32); time_cfg(8192, 64, "f32", 32); time_cfg(8192, 64, "f16", 32)
    time_cfg(1024, 32, "f64", 32); time_cfg(1024, 32, "f32", 32)
