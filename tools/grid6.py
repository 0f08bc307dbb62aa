"""Scratch: v6 grid-size cap sweep (BB_V6_GRID) on the headline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_v5 import time_cfg
for dt in ("f64", "f32"):
    for grid in (148, 120, 100, 74, 50):
        os.environ["BB_V6_GRID"] = str(grid)
        print(dt, "grid", grid, flush=True)
        time_cfg(32768, 128, dt, 32, reps=1)
