"""Scratch: v6 group-size sweep on the headline (last pass time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_v5 import time_cfg
for dt, Gs in (("f32", (2, 3, 4, 5, 6, 7)), ("f64", (3, 4, 5))):
    for G in Gs:
        os.environ["BB_V6_G"] = str(G)
        print(dt, "G", G, flush=True)
        time_cfg(32768, 128, dt, 32, reps=2)
    os.environ.pop("BB_V6_G")
