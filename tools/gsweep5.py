"""Scratch: v5 group-size cap sweep on the headline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_v5 import time_cfg
from tests.golden_util import load, errors
for dt in ("f64", "f32"):
    for G in (32, 16, 8):
        os.environ["BB_V5_G"] = str(G)
        print(dt, "G5cap", G, flush=True)
        d, e = time_cfg(32768, 128, dt, 32, reps=2)
        g = load(f"c4_n32768_b128_{dt}_s0_m0")
        print("   golden", {k: v / g["fro"] for k, v in errors(g, d, e).items() if k != "fro"}, flush=True)
    os.environ.pop("BB_V5_G")
