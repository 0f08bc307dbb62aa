"""Scratch: headline timings per pass (CUDA events on the launching stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_v5 import time_cfg
from tests.golden_util import load, errors, tol
for dt in sys.argv[1:] or ["f64", "f32"]:
    d, e = time_cfg(32768, 128, dt, 32)
    g = load(f"c4_n32768_b128_{dt}_s0_m0")
    err = errors(g, d, e)
    print("golden", dt, {k: v / g["fro"] for k, v in err.items() if k != "fro"}, "tol", tol(dt, 32768), flush=True)
